# config-2 layout sweep (profiling helper): small groups / fewer warps
mkdir -p gpurun_out
while read -r args; do
  [ -z "$args" ] && continue
  timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline --no-dem --no-c3 --no-d100 $args > gpurun_out/sl.log 2>&1
  tail -1 gpurun_out/sl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$args |', round(d['ms_per_step'],3), 'fk', round(r['frame_kernel_ms'],3), 'nz', round(r['noise_kernel_ms'],3), 'tr', round(r['transpose_kernel_ms'],3), d['config']['W'], d['config']['groups'], d['config']['threads'])" 2>/dev/null || echo "$args | failed: $(tail -1 gpurun_out/sl.log | cut -c1-150)"
done <<'LIST' | tee gpurun_out/sweep_r02.txt
--pipeline 6
--words 8 --groups 2 --threads 256
--words 8 --groups 2 --threads 128
--words 4 --groups 4 --threads 512
--words 4 --groups 4 --threads 256
--words 4 --groups 4 --threads 128
--words 4 --groups 5 --threads 160
--words 4 --groups 5 --threads 320
--words 2 --groups 8 --threads 256
--words 2 --groups 8 --threads 512
LIST
