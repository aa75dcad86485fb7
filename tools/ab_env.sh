# A/B an environment switch on the default bench (C2 + d100): bash tools/ab_env.sh VAR "v1 v2"
VAR=$1; VALS=$2
mkdir -p gpurun_out
for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-c3 --no-dem > gpurun_out/env_${VAR}_$v.log 2>&1
  echo "$VAR=$v rc=$?"; python tools/bench_brief.py gpurun_out/env_${VAR}_$v.log | head -2
done
