"""One-line digest of a bench.py JSON log: python tools/bench_brief.py gpurun_out/x_bench.log"""
import json, sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d = json.loads(l); r = d['roofline']
        print('C2 %.1f M/s step %.2f ms | frame %.2f noise %.2f tr %.2f | frac %.3f' % (
            d['value'] / 1e6, d['ms_per_step'], r['frame_kernel_ms'], r['noise_kernel_ms'], r['transpose_kernel_ms'], r['frac']))
        if 'd100' in d:
            q = d['d100']; rr = q['roofline']
            print('d100 %.3f M/s step %.1f ms | frame %.1f noise %.1f tr %.1f | frac %.3f' % (
                q['value'] / 1e6, q['ms_per_step'], rr['frame_kernel_ms'], rr['noise_kernel_ms'], rr['transpose_kernel_ms'], rr['frac']))
        if 'config3_counts' in d:
            print('C3 frame %.2f G/s dem %.2f G/s' % (d['config3_counts']['frame_sampler']['value'] / 1e9,
                                                     d['config3_counts']['error_model_sampler']['value'] / 1e9))
        if 'e2e' in d: print('e2e %.1f M/s' % (d['e2e']['value'] / 1e6))
        if 'error_model_sampler' in d: print('dem C2 %.1f M/s' % (d['error_model_sampler']['value'] / 1e6))
