# A/B timing of experimental library builds (PFS_LIB=...): short bench each.
# usage: bash tools/ab_libs.sh TAG lib1.so lib2.so ...
TAG=$1; shift
mkdir -p gpurun_out
for lib in "$@"; do
  name=$(basename $lib .so)
  PFS_LIB=$PWD/$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-c3 --no-dem > gpurun_out/${TAG}_${name}.log 2>&1; echo "$name rc=$?"
  python tools/bench_brief.py gpurun_out/${TAG}_${name}.log
done
