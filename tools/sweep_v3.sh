# Layout sweep of the frame pipeline at config 2: (words per tile, groups, threads).
# usage: bash tools/sweep_v3.sh "W G T" "W G T" ...
mkdir -p gpurun_out
B="python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-c3 --no-d100 --no-dem"
for cfg in "$@"; do
  set -- $cfg
  timeout 300 $B --words $1 --groups $2 --threads $3 > gpurun_out/sweep_w$1_g$2_t$3.log 2>&1
  echo "W=$1 G=$2 T=$3 rc=$?"; python tools/bench_brief.py gpurun_out/sweep_w$1_g$2_t$3.log | head -1
done
