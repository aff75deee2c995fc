set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t3.log 2>&1; echo "t3 rc=$?"
tail -15 gpurun_out/t3.log
timeout 900 python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
tail -c 2500 gpurun_out/bench_c3.json; tail -3 gpurun_out/bench_c3.err
