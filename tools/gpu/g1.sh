set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/test_gpu_synth.py tests/test_gpu_configs.py -x -q -s > gpurun_out/t1.log 2>&1; echo "t1 rc=$?"
tail -5 gpurun_out/t1.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t2.log 2>&1; echo "t2 rc=$?"
tail -5 gpurun_out/t2.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_c4.json; tail -5 gpurun_out/bench_c4.err
