set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t18.log 2>&1; echo "t18 rc=$?"; tail -12 gpurun_out/t18.log
grep -E "^c[0-9].*(truncated|randomized|lanczos|krylov) \{" gpurun_out/t18.log | head -20
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4c.json 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_c4c.json').read().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['phases_ms_per_step'], d['roofline']['frac'], d['e2e']['value'], json.dumps(d['parity']), json.dumps(d['e2e']['parity']))"
timeout 600 python tools/eig_time.py 256 512 1024 2048 4096 2>&1 | tail -1
