mkdir -p gpurun_out
timeout 300 python tools/profile_run.py --config 2 --shots 262144 --kernel 4 --reps 1 > gpurun_out/dem_plain.log 2>&1; echo "dem plain rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dem_kernel -c 1 -o gpurun_out/r01s4_dem python tools/profile_run.py --config 2 --shots 262144 --kernel 4 --reps 1 > gpurun_out/dem_ncu.log 2>&1; echo "dem ncu rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:frame_kernel -c 1 -o gpurun_out/r01s4_frame python tools/profile_run.py --config 2 --shots 262144 --reps 1 > gpurun_out/frame_ncu.log 2>&1; echo "frame ncu rc=$?"
ls -la gpurun_out
