#!/usr/bin/env python
"""Benchmark: surface-code detection-event sampling throughput (shots/s).

Workload (BASELINE.json configs[2]): rotated surface code Z-memory, d=25,
25 rounds, p=1e-3 circuit noise, 2^20 shots per GPU per step, detection
events (+ the logical observable) shot-major bit-packed (b8).  One step = one
full pass of the hot path: frame program kernel over all shots (noise sampled
inline) + the shot-major transpose, outputs resident in HBM.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 runs under torchrun, one process per GPU; shots are sharded by global shot
offset (weak scaling: every rank samples its own 2^20 shots), no collective on
the data path; the timing is the max over ranks.  --impl reference times the
reference algorithm on the host cores (the C restatement in oracle/, all
threads) on the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)


METRIC = "surface-code detection-event shots/sec (d=25 & d=100, p=1e-3); frame-update GB/s vs peak"
WORKLOADS = {2: "config2: rotated surface code Z-memory d=25 r=25 p=1e-3",
             4: "config4: rotated surface code Z-memory d=100 r=100 p=1e-3",
             0: "config0: d=3 r=3 p=1e-3", 1: "config1: random Clifford n=64 x200 layers",
             3: "config3: d=5 r=5 p=5e-3"}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--shots", type=int, default=0, help="shots per GPU per step (0 = config)")
    ap.add_argument("--words", type=int, default=0, help="override W (32-shot words per tile)")
    ap.add_argument("--ring", type=int, default=-1)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--kernel", type=int, default=0, help="0 auto / 1 frame sampler, 4 error-model sampler")
    ap.add_argument("--target-hits", type=float, default=0.0)
    ap.add_argument("--fused-hits", type=float, default=0.0)
    ap.add_argument("--groups", type=int, default=0, help="tiles in flight per CTA")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-d100", action="store_true", help="skip the config 4 (d=100) extra line")
    ap.add_argument("--no-dem", action="store_true", help="skip the error-model sampler extra line")
    ap.add_argument("--no-c3", action="store_true", help="skip the config 3 counts extra line")
    ap.add_argument("--presample", type=int, default=0,
                    help="fused noise pre-sampled by noise_kernel (0 auto/on, -1 drawn inline)")
    ap.add_argument("--no-pyref", action="store_true", help="skip timing the Python reference package")
    ap.add_argument("--pipeline", type=int, default=0, help="frame/transpose pipeline sub-chunks (0 auto, 1 off)")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._loop, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for i, n in enumerate(names):
                if len(s) > 5 + i and s[5 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------- helpers
def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def config_text(cfg: int):
    from paper_2103_02202_b200 import generators as gen
    return gen.config_circuit(cfg)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def workload_config(cfg: int, shots: int, world: int) -> dict:
    """The `config` object both arms print (same workload, same keys)."""
    return {"workload": WORKLOADS.get(cfg, f"config{cfg}") + ", detection events + observable, shot-major b8",
            "shots_per_gpu_per_step": shots,
            "parallelism": f"shots sharded x{world} (global shot offsets)"}


# ----------------------------------------------------------------- CPU arms
class PortTimer:
    """The reference algorithm restated in C (oracle/pfs_oracle.c) on the host
    cores: frame simulation of every tile (every coin and noise draw), detector
    XORs, then the shot-major b8 transpose — all host threads.  Setup (circuit
    lowering, oracle build, the RNG layout) is done once, outside the timing."""

    T = 256

    def __init__(self, cfg: int, threads: int):
        from oracle import oracle as O
        from paper_2103_02202_b200.program import flatten

        O.build()
        self.O = O
        self.prog = flatten(config_text(cfg))
        self.threads = threads
        # layout of the draws (chunk length per noise instruction): it fixes the
        # draw order, not the work, so any valid one times the algorithm
        self.chunk_L = np.full(self.prog.num_noise, 512, dtype=np.uint32)

    def run(self, shots: int, seed: int) -> float:
        t0 = time.perf_counter()
        _, ev = self.O.sample(self.prog, shots, self.T, seed=seed, flips=False, nthreads=self.threads,
                              chunk_L=self.chunk_L, vector_shots=128)
        self.O.rows_to_b8(ev, shots, nthreads=self.threads)
        return time.perf_counter() - t0

    def rate(self, seconds: float, seed: int = 1, max_shots: int = 1 << 22):
        """(shots/s, shots, seconds) of one bounded sample of about `seconds`
        (at most `max_shots`: a sample never exceeds the step it stands for)."""
        shots = self.T * self.threads
        dt = self.run(shots, seed)  # calibration (also warms the threads)
        shots = int(min(max(shots / dt * seconds, shots), max_shots))
        shots = max(self.T, (shots // self.T) * self.T)
        dt = self.run(shots, seed + 1)
        return shots / dt, shots, dt


def _pyref_worker(args):
    """One process of the unmodified Python reference (stabsim, pip-installed
    into baseline/_ref): collect_flips + detector_events on its own shots."""
    ref_path, text, shots, seed, batch = args
    sys.path.insert(0, ref_path)
    from stabsim import circuit, frame_sim, io_formats

    c = circuit.parse(text)
    dets = circuit.detector_sets(c)
    t0 = time.perf_counter()
    flips = frame_sim.collect_flips(c, shots, np.random.default_rng(seed), batch)
    io_formats.detector_events(flips, dets)
    return time.perf_counter() - t0


def python_reference_rate(cfg: int, procs: int, batch: int = 8192):
    """the reference package itself on `procs` worker
    processes, one batch each (bounded sample); None when baseline/_ref is
    absent.  Circuits are lowered to the reference dialect."""
    ref_path = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_path, "stabsim")):
        return None
    from paper_2103_02202_b200.circuit import to_reference_dialect

    text = to_reference_dialect(config_text(cfg))
    ctx = multiprocessing.get_context("spawn")
    with ctx.Pool(procs) as pool:
        t0 = time.perf_counter()
        times = pool.map(_pyref_worker, [(ref_path, text, batch, 1000 + i, batch) for i in range(procs)])
        wall = time.perf_counter() - t0
    shots = procs * batch
    return {"value": shots / max(times), "unit": "shots/s", "cores": procs, "kind": "reference",
            "sample": f"{shots} shots of config {cfg}: {procs} processes x collect_flips(batch_size={batch}) + "
                      f"detector_events of the unmodified stabsim package (baseline/_ref), timed inside each "
                      f"worker after parsing; pool wall {wall:.1f}s ({cpu_model()})"}


# ----------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    cores = host_cores()
    pt = PortTimer(args.config, cores)
    shots_cfg = args.shots or __import__("paper_2103_02202_b200.generators", fromlist=["CONFIGS"]).CONFIGS[
        args.config]["shots"]
    per_step_s = max(2.0, min(args.cpu_seconds, 60.0) / max(1, args.steps))
    rates, sample_shots = [], 0
    for i in range(args.warmup + args.steps):
        rate, shots, dt = pt.rate(per_step_s, seed=10 + 2 * i, max_shots=shots_cfg)
        if i >= args.warmup:
            rates.append(rate)
            sample_shots = shots
    value = float(np.median(rates))
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value, "unit": "shots/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * shots_cfg / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded circuit-level noise, Philox)",
        "config": workload_config(args.config, shots_cfg, world),
        "cpu_baseline": {"value": value, "unit": "shots/s", "cores": cores, "kind": "port",
                         "sample": f"per step {sample_shots} of the {shots_cfg} shots (a bounded sample; "
                                   f"ms_per_step is scaled to the full step) of config {args.config}: C "
                                   f"restatement of stabsim frame_sim + detector_events + b8 transpose on "
                                   f"{cores} threads ({cpu_model()})"},
        "e2e": {"value": value, "unit": "shots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_pyref:
        py = python_reference_rate(args.config, min(cores, 8))
        if py is not None:
            line["python_reference"] = py
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- our arm
def native_opts(args):
    return dict(words_per_tile=args.words, ring_in_smem=args.ring, threads=args.threads,
                noise_target_hits=args.target_hits, kernel=args.kernel, groups=args.groups,
                pipeline=args.pipeline, fused_target_hits=args.fused_hits,
                presample_noise=args.presample)


def measure(args, cfg: int, shots: int, steps: int, warmup: int, rank: int, world: int,
            local_rank: int, e2e_steps: int):
    """Time `steps` sampling steps of config `cfg` (device-resident b8 output),
    then the per-kernel durations (CUDA events inside pfs_run), then e2e."""
    import torch

    from paper_2103_02202_b200 import _native as N
    from paper_2103_02202_b200.parallel import rank_offset, reduce_max
    from paper_2103_02202_b200.program import flatten
    from paper_2103_02202_b200.sampler import DetectorSampler, pinned_empty

    dist = world > 1
    if dist:
        import torch.distributed as tdist
    dev = torch.device("cuda", local_rank)
    t0 = time.perf_counter()
    flat = flatten(config_text(cfg))
    kw = native_opts(args)
    ds = DetectorSampler.__new__(DetectorSampler)
    ds.circuit, ds.flat, ds.device = None, flat, local_rank
    ds._seeds = np.random.default_rng(0)
    ds.native = N.NativeProgram(flat, **kw)
    compile_s = time.perf_counter() - t0
    info = ds.info
    T = ds.tile_shots
    nb = (ds.num_columns + 7) // 8
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    pitch = (nb + 31) // 32 * 32  # 32-byte aligned shot rows on device (b8 bytes + zero pad)
    out_full = torch.empty((shots, pitch), dtype=torch.uint8, device=dev)
    out = out_full[:, :nb]
    base_offset = rank_offset(shots, world, rank, T)
    seed = 20260214

    def step(sampler, i):
        sampler.sample(shots, seed=seed + i, out=out, shot_offset=base_offset, stream=sp)

    for i in range(warmup):
        step(ds, i)
    torch.cuda.synchronize()
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches = 0
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for i in range(steps):
            step(ds, warmup + i)
            launches += ds.native.last_launches()
        ev1.record(stream)
        torch.cuda.synchronize()
    elapsed = reduce_max(ev0.elapsed_time(ev1) / 1e3, dev)
    res = {"cfg": cfg, "shots": shots, "steps": steps, "elapsed": elapsed,
           "value": shots * world * steps / elapsed, "clocks": clk.summary(),
           "launches": launches, "info": info, "nb": nb, "compile_s": compile_s}

    # per-kernel durations: CUDA events recorded on the launching stream inside pfs_run
    dt = DetectorSampler.__new__(DetectorSampler)
    dt.circuit, dt.flat, dt.device = None, flat, local_rank
    dt._seeds = np.random.default_rng(0)
    dt.native = N.NativeProgram(flat, timing=True, **kw)
    fr, tr, nz = [], [], []
    for i in range(max(3, min(steps, 10))):
        step(dt, i)
        t = dt.native.last_timing()
        if i:
            fr.append(t[0])
            tr.append(t[1])
            nz.append(t[5])
    res["frame_ms"] = float(np.mean(fr))
    res["transpose_ms"] = float(np.mean(tr))
    res["noise_ms"] = float(np.mean(nz))
    del dt

    if e2e_steps > 0:
        host, _keep = pinned_empty((shots, nb), np.uint8)
        ds.sample(shots, seed=1, out=host, shot_offset=base_offset)
        torch.cuda.synchronize()
        if dist:
            tdist.barrier()
        t0 = time.perf_counter()
        for i in range(e2e_steps):
            ds.sample(shots, seed=seed + i, out=host, shot_offset=base_offset)
        torch.cuda.synchronize()
        e_el = reduce_max(time.perf_counter() - t0, dev)
        res["e2e"] = {"value": shots * world * e2e_steps / e_el, "unit": "shots/s",
                      "h2d_bytes_per_step": 0, "d2h_bytes_per_step": int(shots * nb * world),
                      "steps": e2e_steps,
                      "note": "public API DetectorSampler.sample(out=pinned host ndarray): frame "
                              "kernel + transpose + D2H of the b8 events in a double-buffered "
                              "chunk pipeline; per-step inputs are (seed, shot range) only"}
        del host, _keep
    del out_full, out
    torch.cuda.empty_cache()
    return res


def measure_counts(args, kernel: int, shots: int, steps: int, warmup: int, rank: int, world: int,
                   local_rank: int):
    """Config 3 (BASELINE.json): d=5, 5 rounds, p=5e-3, on-device per-column
    event counts only (no event I/O), `shots` per GPU per step; the per-rank
    u64 counts are summed with one NCCL all-reduce at the end
    — parallel.counts_steps, the helper the gloo test drives."""
    import torch

    from paper_2103_02202_b200.parallel import counts_steps, reduce_max
    from paper_2103_02202_b200.sampler import compile_detector_sampler

    dist = world > 1
    if dist:
        import torch.distributed as tdist
    dev = torch.device("cuda", local_rank)
    ds = compile_detector_sampler(config_text(3), device=local_rank, kernel=kernel)
    T = ds.tile_shots
    counts = torch.zeros(ds.num_columns, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def sample_counts(n, s, off, out):
        ds.sample_counts(n, seed=s, out=out, shot_offset=off, stream=stream.cuda_stream)

    counts_steps(sample_counts, counts, shots, T, 1, 0, warmup, 99)  # warm-up, no reduction
    torch.cuda.synchronize()
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    counts_steps(sample_counts, counts, shots, T, world, rank, steps, 7)
    ev1.record(stream)
    torch.cuda.synchronize()
    elapsed = reduce_max(ev0.elapsed_time(ev1) / 1e3, dev)
    rate = float(counts.sum().item()) / max(1, shots * world)  # mean events per shot (last step, all ranks)
    return {"value": shots * world * steps / elapsed, "unit": "shots/s", "ms_per_step": 1e3 * elapsed / steps,
            "steps": steps, "shots_per_gpu_per_step": shots, "kernel": ds.info["kernel"],
            "mean_events_per_shot_last_step": rate}


def roofline_of(res, smem_peak, hbm):
    info = res["info"]
    bframe_bytes = info["bframe_bits"] / 8.0
    fr = res["frame_ms"]
    achieved = bframe_bytes * res["shots"] / (fr / 1e3) / 1e9
    return {"bound": "smem", "achieved": achieved, "peak": smem_peak, "unit": "GB/s",
            "frac": achieved / smem_peak,
            "traffic": profile_traffic(res["shots"], res["cfg"]),
            "traffic_source": "profiles/frame_kernel_traffic.json (ncu --set full, DRAM bytes per shot "
                              "of the frame kernel)",
            "peak_source": "measured live: pfs_measure_smem_bandwidth (LDS.128/STS.128 CX mix, "
                           "all SMs)",
            "kernel": "frame_kernel (frame table resident in shared memory; fused noise applied from noise_kernel's "
                      "pre-sampled per-warp hit lists)",
            "frame_kernel_ms": fr, "transpose_kernel_ms": res["transpose_ms"],
            "noise_kernel_ms": res["noise_ms"],
            "bytes_per_shot": bframe_bytes,
            "hbm_equiv": {"achieved_gbs": achieved, "peak_gbs": hbm, "frac": achieved / hbm,
                          "note": "frame-update GB/s vs measured HBM copy peak (BASELINE.json "
                                  "metric wording); the frame table never streams through HBM"}}


def run_ours(args, rank, world, local_rank):
    import copy

    import torch

    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200._native import measure_smem_bandwidth

    torch.cuda.set_device(local_rank)
    shots = args.shots or gen.CONFIGS[args.config]["shots"]
    main = measure(args, args.config, shots, args.steps, args.warmup, rank, world, local_rank,
                   0 if args.no_e2e else max(2, args.steps // 4))
    dem = None
    if args.config == 2 and not args.no_dem and args.kernel == 0:
        # the error-model detector sampler (kernel 4) on the same workload
        a2 = copy.copy(args)
        a2.kernel, a2.words, a2.ring, a2.threads, a2.groups = 4, 0, -1, 0, 0
        dem = measure(a2, args.config, shots, max(3, args.steps // 2), args.warmup, rank, world,
                      local_rank, 0)
    c3 = None
    if args.config == 2 and not args.no_c3 and args.kernel == 0:
        c3 = {"workload": WORKLOADS[3] + ", per-column event counts on device (no event I/O), "
                                        "one u64 all-reduce over ranks",
              "frame_sampler": measure_counts(args, 1, 1 << 24, max(3, args.steps // 4), 2, rank, world,
                                              local_rank),
              "error_model_sampler": measure_counts(args, 4, 1 << 24, max(3, args.steps // 4), 2, rank,
                                                    world, local_rank)}
    extra = None
    if args.config == 2 and not args.no_d100:
        s4 = gen.CONFIGS[4]["shots"]
        a4 = copy.copy(args)
        a4.words, a4.groups, a4.threads = 0, 0, 0
        extra = measure(a4, 4, s4, max(3, args.steps // 4), 3, rank, world, local_rank,
                        0 if args.no_e2e else 2)
        if not args.no_dem and args.kernel == 0:
            a5 = copy.copy(args)
            a5.kernel, a5.words, a5.ring, a5.threads, a5.groups = 4, 0, -1, 0, 0
            extra["dem"] = measure(a5, 4, s4, max(3, args.steps // 4), 3, rank, world, local_rank, 0)
    if rank != 0:
        return
    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6469.6))
    smem_peak = measure_smem_bandwidth(local_rank)
    info = main["info"]
    T = info["tile_shots"]
    cfgd = workload_config(args.config, main["shots"], world)
    cfgd.update({"columns": info["num_columns"], "W": info["words_per_tile"], "tile_shots": T,
                 "groups": info["groups"], "ring_in_smem": info["ring_in_smem"], "threads": info["threads"],
                 "device_ops": info["num_ops"], "barriers_per_tile": info["num_barriers"],
                 "fused_noise_instructions": f"{info['fused_noise']}/{info['num_noise']}",
                 "l2": f"outputs {main['shots'] * main['nb'] / 1e9:.2f} GB/step > 126 MB L2 (no flush needed)"})
    line = {
        "metric": METRIC,
        "value": main["value"], "unit": "shots/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * main["elapsed"] / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded circuit-level noise, counter-based Philox)",
        "config": cfgd,
        "roofline": roofline_of(main, smem_peak, hbm),
        "clocks": main["clocks"],
        "gpu_launches": main["launches"],
    }
    if "e2e" in main:
        line["e2e"] = main["e2e"]
    if extra is not None:
        x = {"workload": WORKLOADS[4] + ", detection events + observable, shot-major b8 in HBM",
             "value": extra["value"], "unit": "shots/s", "shots_per_gpu_per_step": extra["shots"],
             "ms_per_step": 1e3 * extra["elapsed"] / extra["steps"], "steps": extra["steps"],
             "host_compile_s": extra["compile_s"],
             "host_reference_sample_s": reference_sample_seconds(config_text(4)),
             "roofline": roofline_of(extra, smem_peak, hbm), "clocks": extra["clocks"],
             "W": extra["info"]["words_per_tile"], "ring_in_smem": extra["info"]["ring_in_smem"],
             "gpu_launches": extra["launches"]}
        if "e2e" in extra:
            x["e2e"] = extra["e2e"]
        if "dem" in extra:
            dm = extra["dem"]
            x["error_model_sampler"] = {
                "value": dm["value"], "unit": "shots/s", "ms_per_step": 1e3 * dm["elapsed"] / dm["steps"],
                "steps": dm["steps"], "kernel_ms": dm["frame_ms"], "transpose_kernel_ms": dm["transpose_ms"],
                "note": "kernel 4 with the column words in global memory (1M columns), then tiles_to_b8"}
        line["d100"] = x
    if dem is not None:
        line["error_model_sampler"] = {
            "workload": "config2 through the error-model detector sampler (kernel 4): every noise hit "
                        "XORs its precomputed detector signature; the same counter-based draws, "
                        "bit-exact with the oracle (tests/test_gpu_parity.py)",
            "value": dem["value"], "unit": "shots/s", "ms_per_step": 1e3 * dem["elapsed"] / dem["steps"],
            "steps": dem["steps"], "kernel_ms": dem["frame_ms"], "gpu_launches": dem["launches"],
            "clocks": dem["clocks"]}
    if c3 is not None:
        line["config3_counts"] = c3
    if not args.no_cpu_baseline:
        cores = host_cores()
        rate, s_shots, dt = PortTimer(args.config, cores).rate(args.cpu_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": "shots/s", "cores": cores, "kind": "port",
                                "sample": f"{s_shots} shots of config {args.config} in {dt:.1f}s on {cores} "
                                          f"threads ({cpu_model()}); C restatement of stabsim frame_sim + "
                                          "detector_events + b8 transpose (same timer as --impl reference)"}
    print(json.dumps(line), flush=True)


def reference_sample_seconds(text) -> float:
    """Host time of the native inverse-tableau reference sample (the step
    before measurement sampling, reported separately per BASELINE.json C4)."""
    from paper_2103_02202_b200 import tableau_sim as T
    t0 = time.perf_counter()
    T.reference_sample(text, np.random.default_rng(1))
    return time.perf_counter() - t0


def profile_traffic(shots=None, cfg=2):
    """DRAM bytes per frame-kernel launch from the committed ncu capture
    (profiles/frame_kernel_traffic.json, per shot x this launch's shots)."""
    p = os.path.join(REPO, "profiles", "frame_kernel_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        d = d if cfg == 2 else d.get(f"config{cfg}")  # top level: config 2; "config4": d=100
        return float(d["dram_bytes_per_shot"]) * shots if (d and shots) else None
    except Exception:
        return None


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as tdist
            tdist.destroy_process_group()


if __name__ == "__main__":
    main()
