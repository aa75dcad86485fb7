# GPU validation pass: gpu tests, smoke, default bench, reference arm, launch list, full captures.
# usage: bash tools/gpu_round.sh TAG   (outputs under gpurun_out/TAG_*)
TAG=${1:-r02}
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/${TAG}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/${TAG}_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/${TAG}_bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-d100 --no-cpu-baseline --no-c3 > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
timeout 300 python tools/profile_run.py --config 2 --shots 262144 --reps 1 > gpurun_out/${TAG}_frame_plain.log 2>&1; echo "frame plain rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:frame_kernel -c 1 -o gpurun_out/${TAG}_frame python tools/profile_run.py --config 2 --shots 262144 --reps 1 > gpurun_out/${TAG}_frame_ncu.log 2>&1; echo "frame ncu rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:noise_kernel -c 1 -o gpurun_out/${TAG}_noise python tools/profile_run.py --config 2 --shots 262144 --reps 1 > gpurun_out/${TAG}_noise_ncu.log 2>&1; echo "noise ncu rc=$?"
ls -la gpurun_out
