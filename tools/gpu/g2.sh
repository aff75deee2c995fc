set -x
python -m pytest tests/test_gpu_synth.py tests/test_gpu_configs.py tests/test_gpu_sharded.py -q -s > gpurun_out/t1.log 2>&1; echo "t1 rc=$?"
tail -15 gpurun_out/t1.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t2.log 2>&1; echo "t2 rc=$?"
tail -15 gpurun_out/t2.log
