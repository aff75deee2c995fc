set -x
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_sharded.py -q -s > gpurun_out/t20.log 2>&1; echo "t20 rc=$?"; tail -3 gpurun_out/t20.log
for c in c4 c1 c2 c3; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err; echo "bench $c rc=$?"
  tail -c 400 gpurun_out/r2_bench_$c.json
done
