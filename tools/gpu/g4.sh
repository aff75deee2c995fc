set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t4.log 2>&1; echo "t4 rc=$?"
tail -8 gpurun_out/t4.log
timeout 600 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c3b.json 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_c3b.json').read().splitlines()[-1]);print(d['phases_ms_per_step'], d['ms_per_step'])"
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_probe.py > gpurun_out/san/$tool.log 2>&1; echo "$tool rc=$?"
  tail -4 gpurun_out/san/$tool.log
done
