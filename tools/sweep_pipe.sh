# noise/frame pipeline depth sweep on config 2 (profiling helper)
for p in ${PIPES:-1 4 6 10 14}; do
  timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline --no-dem --no-c3 --no-d100 --pipeline $p > gpurun_out/sp.log 2>&1
  tail -1 gpurun_out/sp.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pipe', $p, round(d['ms_per_step'],3), d['config']['threads'])"
done
