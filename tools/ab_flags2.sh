# A/B bench flag sets incl. the error-model sampler: bash tools/ab_flags2.sh "flags1" "flags2" ...
mkdir -p gpurun_out
n=0
for f in "$@"; do
  n=$((n+1))
  timeout 600 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-d100 $f > gpurun_out/flags2_$n.log 2>&1
  echo "[$f] rc=$?"; python tools/bench_brief.py gpurun_out/flags2_$n.log | grep "C2\|C3"
done
