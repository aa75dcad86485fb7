# ncu --set full of one kernel launch of tools/profile_run.py.  usage: bash tools/ncu_any.sh TAG KERNEL_REGEX [profile_run args]
TAG=$1; KRE=$2; shift 2
mkdir -p gpurun_out
timeout 600 python tools/profile_run.py --reps 1 "$@" > gpurun_out/${TAG}_plain.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:$KRE -c 1 -f -o gpurun_out/${TAG} python tools/profile_run.py --reps 1 "$@" > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/${TAG}.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
