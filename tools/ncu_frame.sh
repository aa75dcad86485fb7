# ncu --set full of one frame_kernel launch (2^18 shots of config 2) + per-line summary.
# usage: bash tools/ncu_frame.sh TAG [extra profile_run args]
TAG=${1:-cap}; shift
mkdir -p gpurun_out
timeout 300 python tools/profile_run.py --config 2 --shots 262144 --reps 1 "$@" > gpurun_out/${TAG}_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:frame_kernel -c 1 -f -o gpurun_out/${TAG}_frame python tools/profile_run.py --config 2 --shots 262144 --reps 1 "$@" > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/${TAG}_frame.ncu-rep --page details --csv > gpurun_out/${TAG}_frame_details.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_frame.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_frame_source.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/${TAG}_frame_source.csv 60 > gpurun_out/${TAG}_frame_lines.txt 2>&1
ls -la gpurun_out | tail -8
