set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t21.log 2>&1; echo "t21 rc=$?"; tail -4 gpurun_out/t21.log
for c in c4 c2; do
timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pg_$c.json 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_pg_$c.json').read().splitlines()[-1]);print('$c', d['value'], d['e2e']['value'], json.dumps(d['e2e']['pageable']), d['parity']['ok'])"
done
