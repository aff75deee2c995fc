set -x
timeout 300 python tools/gemm_ncu_probe.py > gpurun_out/gemm_probe3.log 2>&1; cat gpurun_out/gemm_probe3.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t9.log 2>&1; echo "t9 rc=$?"; tail -5 gpurun_out/t9.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4b.json 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_c4b.json').read().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['phases_ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['parity'])"
