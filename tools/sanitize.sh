# compute-sanitizer evidence for barrier elision / shared-memory atomics:
# racecheck, synccheck and memcheck over tools/sanitize_run.py.  usage: bash tools/sanitize.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 600 python tools/sanitize_run.py > gpurun_out/${TAG}_sanitize_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/${TAG}_sanitize_plain.log
for tool in racecheck synccheck memcheck; do
  timeout 2400 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/${TAG}_sanitize_${tool}.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run ok" gpurun_out/${TAG}_sanitize_${tool}.log
done
