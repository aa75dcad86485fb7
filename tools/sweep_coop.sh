# cooperative-kernel layout sweep on config 2 (profiling helper)
run() { timeout 200 python bench.py --steps 5 --kernel 1 --no-cpu-baseline --no-e2e --no-d100 "$@" > gpurun_out/sw.log 2>&1; tail -1 gpurun_out/sw.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$*', round(d['ms_per_step'],2), 'fk',round(r['frame_kernel_ms'],2),'nz',round(r.get('noise_kernel_ms',0),2),'tr',round(r['transpose_kernel_ms'],2), d['config']['W'], d['config']['threads'])" 2>&1 | tail -1; }
for a in "$@"; do run $a; done
