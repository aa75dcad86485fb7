"""ctypes binding of libpfs.so (include/pfs.h).

The library is the product: there is no CPU fallback.  If it is missing or no
B200 is visible, calls raise `NativeUnavailable` loudly.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .program import FlatProgram

_PKG = os.path.dirname(os.path.abspath(__file__))
# PFS_PROFILE=1 selects the profiling build (op clock traces, ablations; tools/ only)
# PFS_LIB=<path> loads an experimental build instead (A/B timing in tools/ only)
LIB_PATH = os.environ.get("PFS_LIB") or os.path.join(
    _PKG, "_lib", "libpfs_profile.so" if os.environ.get("PFS_PROFILE") == "1" else "libpfs.so")

MODE_FLIPS, MODE_SAMPLES, MODE_DETECTORS, MODE_COUNTS, MODE_FLIPS_ROWS, MODE_DETECTORS_ROWS = range(6)
E_INVALID, E_CUDA, E_NOMEM, E_NODEVICE = -1, -2, -3, -4


class NativeUnavailable(RuntimeError):
    """libpfs.so is not built or cannot run here (no CPU fallback exists)."""


class Options(ctypes.Structure):
    _fields_ = [("words_per_tile", ctypes.c_int32), ("ring_in_smem", ctypes.c_int32),
                ("threads", ctypes.c_int32), ("ctas_per_sm", ctypes.c_int32),
                ("noise_target_hits", ctypes.c_double), ("timing", ctypes.c_int32),
                ("debug_skip", ctypes.c_int32), ("presample_noise", ctypes.c_int32),
                ("schedule_only", ctypes.c_int32), ("groups", ctypes.c_int32),
                ("kernel", ctypes.c_int32), ("pipeline", ctypes.c_int32),
                ("fused_target_milli", ctypes.c_int32)]


class Info(ctypes.Structure):
    _fields_ = [("num_qubits", ctypes.c_int32), ("words_per_tile", ctypes.c_int32),
                ("tile_shots", ctypes.c_int32), ("threads", ctypes.c_int32),
                ("ring_in_smem", ctypes.c_int32), ("smem_bytes", ctypes.c_int32),
                ("num_measurements", ctypes.c_int64), ("num_columns", ctypes.c_int64),
                ("num_observables", ctypes.c_int64), ("num_ops", ctypes.c_int64),
                ("num_barriers", ctypes.c_int64), ("num_slots", ctypes.c_int64),
                ("num_noise", ctypes.c_int64), ("bframe_bits", ctypes.c_int64),
                ("num_coin_rows", ctypes.c_int64), ("num_noise_rows", ctypes.c_int64),
                ("noise_tab_len", ctypes.c_int64), ("live_coin_rows", ctypes.c_int64),
                ("record_ops", ctypes.c_int64), ("groups", ctypes.c_int64),
                ("kernel", ctypes.c_int64), ("warps_per_cta", ctypes.c_int64),
                ("fused_noise", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


EXPORTS = ("pfs_program_create", "pfs_program_info", "pfs_program_noise_schedule", "pfs_run",
           "pfs_program_last_timing", "pfs_program_last_launches", "pfs_program_destroy",
           "pfs_last_error", "pfs_version", "pfs_measure_smem_bandwidth",
           "pfs_detector_events", "pfs_program_op_clock", "pfs_program_ops", "pfs_program_dump",
           "pfs_reference_sample", "pfs_reference_sample_error", "pfs_write_format")

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is missing: build it with `python -m paper_2103_02202_b200.build`")
    L = ctypes.CDLL(LIB_PATH)
    P, i64, i32, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
    L.pfs_program_create.argtypes = [P, i64, P, i64, P, i64, P, P, i64, i64, i32, i64, i64, i64,
                                     P, ctypes.POINTER(P)]
    L.pfs_program_create.restype = ctypes.c_int
    L.pfs_program_info.argtypes = [P, ctypes.POINTER(Info)]
    L.pfs_program_info.restype = ctypes.c_int
    L.pfs_program_noise_schedule.argtypes = [P, P, i64, P, i64]
    L.pfs_program_noise_schedule.restype = ctypes.c_int
    L.pfs_run.argtypes = [P, ctypes.c_int, u64, u64, i64, ctypes.c_int, P, P, P, i64, P, i64, i64, P]
    L.pfs_run.restype = ctypes.c_int
    L.pfs_program_last_timing.argtypes = [P, ctypes.POINTER(ctypes.c_double), ctypes.c_int]
    L.pfs_program_last_timing.restype = ctypes.c_int
    L.pfs_program_last_launches.argtypes = [P]
    L.pfs_program_last_launches.restype = i64
    L.pfs_program_destroy.argtypes = [P]
    L.pfs_program_destroy.restype = None
    L.pfs_last_error.argtypes = []
    L.pfs_last_error.restype = ctypes.c_char_p
    L.pfs_measure_smem_bandwidth.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    L.pfs_measure_smem_bandwidth.restype = ctypes.c_int
    L.pfs_detector_events.argtypes = [ctypes.c_int, P, i64, i64, i64, P, P, i64, P, i64, i64, P]
    L.pfs_detector_events.restype = ctypes.c_int
    L.pfs_program_op_clock.argtypes = [P, P, i64]
    L.pfs_program_op_clock.restype = ctypes.c_int
    L.pfs_program_ops.argtypes = [P, P, i64]
    L.pfs_program_ops.restype = ctypes.c_int
    L.pfs_program_dump.argtypes = [P, ctypes.c_int, ctypes.c_int, P, i64]
    L.pfs_program_dump.restype = ctypes.c_int64
    L.pfs_write_format.argtypes = [ctypes.c_int, P, i64, i64, i64, ctypes.c_int, P, i64, ctypes.POINTER(i64), P]
    L.pfs_write_format.restype = ctypes.c_int
    L.pfs_reference_sample.argtypes = [P, i64, P, i64, i32, P, i64, P, P, i64, ctypes.POINTER(i64)]
    L.pfs_reference_sample.restype = ctypes.c_int
    L.pfs_reference_sample_error.argtypes = []
    L.pfs_reference_sample_error.restype = ctypes.c_char_p
    L.pfs_version.argtypes = []
    L.pfs_version.restype = ctypes.c_int
    _lib = L
    return L


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().pfs_last_error().decode(errors="replace")
    if rc == E_INVALID:
        raise ValueError(msg)
    if rc == E_NODEVICE:
        raise NativeUnavailable(msg)
    if rc == E_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def _p(a):
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def measure_smem_bandwidth(device: int = 0) -> float:
    v = ctypes.c_double()
    _check(lib().pfs_measure_smem_bandwidth(device, ctypes.byref(v)))
    return float(v.value)


def detector_events_b8(flips_b8: np.ndarray, num_results: int, det_ptr: np.ndarray,
                       det_idx: np.ndarray, device: int = 0) -> np.ndarray:
    """GPU detector_events: b8 flips -> b8 events (pfs_detector_events)."""
    fl = np.ascontiguousarray(flips_b8, dtype=np.uint8)
    S = fl.shape[0]
    D = int(det_ptr.shape[0]) - 1
    out = np.zeros((S, (D + 7) // 8), dtype=np.uint8)
    ptr = np.ascontiguousarray(det_ptr, dtype=np.int64)
    idx = np.ascontiguousarray(det_idx, dtype=np.int64)
    _check(lib().pfs_detector_events(device, _p(fl), S, num_results, fl.shape[1] if fl.ndim == 2 else 0,
                                     _p(ptr), _p(idx) if idx.size else None, D, _p(out), out.nbytes,
                                     out.shape[1], None))
    return out


class NativeProgram:
    """A compiled frame program bound (lazily) to one GPU."""

    def __init__(self, prog: FlatProgram, words_per_tile: int = 0, ring_in_smem: int = -1,
                 threads: int = 0, ctas_per_sm: int = 0, noise_target_hits: float = 0.0,
                 timing: bool = False, debug_skip: int = 0, presample_noise: int = 0,
                 schedule_only: bool = False, groups: int = 0, kernel: int = 0,
                 pipeline: int = 0, fused_target_hits: float = 0.0):
        L = lib()
        self.flat = prog
        self._keep = [np.ascontiguousarray(prog.instrs, dtype=np.int32),
                      np.ascontiguousarray(prog.targets, dtype=np.int32),
                      np.ascontiguousarray(prog.noise_p, dtype=np.float64),
                      np.ascontiguousarray(prog.det_ptr, dtype=np.int64),
                      np.ascontiguousarray(prog.det_idx, dtype=np.int64)]
        ins, tg, p, dp, di = self._keep
        opts = Options(words_per_tile, ring_in_smem, threads, ctas_per_sm, noise_target_hits,
                       1 if timing else 0, debug_skip, presample_noise, 1 if schedule_only else 0,
                       groups, kernel, pipeline, int(round(fused_target_hits * 1000)))
        h = ctypes.c_void_p()
        _check(L.pfs_program_create(_p(ins), ins.shape[0], _p(tg), tg.shape[0], _p(p), p.shape[0],
                                    _p(dp), _p(di), prog.num_columns, prog.num_observables,
                                    prog.num_qubits, prog.num_measurements, prog.num_coin_rows,
                                    prog.num_noise_rows, ctypes.byref(opts), ctypes.byref(h)))
        self._h = h
        inf = Info()
        _check(L.pfs_program_info(h, ctypes.byref(inf)))
        self.info = inf.as_dict()
        self.tile_shots = inf.tile_shots

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.pfs_program_destroy(h)
            self._h = None

    def noise_schedule(self):
        """(params uint32 [num_noise, 12], tables uint64) — the noise RNG schedule:
        per instruction L, cs, ca, nchunks, apps, table offset, table length,
        zone, npat, channel, fused, 0."""
        params = np.zeros((self.flat.num_noise, 12), dtype=np.uint32)
        tab = np.zeros(self.info["noise_tab_len"], dtype=np.uint64)
        _check(lib().pfs_program_noise_schedule(self._h, _p(params) if params.size else None,
                                                params.size, _p(tab) if tab.size else None,
                                                tab.size))
        return params, tab

    def run(self, mode: int, num_shots: int, seed: int, out, out_bytes: int, out_pitch: int = 0,
            shot_offset: int = 0, device: int = 0, ref_bits=None, coins=None, masks=None,
            inject_row_words: int = 0, stream: int = 0):
        _check(lib().pfs_run(self._h, device, seed & 0xFFFFFFFFFFFFFFFF, shot_offset, num_shots,
                             mode, _p(ref_bits), _p(coins), _p(masks), inject_row_words, _p(out),
                             out_bytes, out_pitch, stream or None))

    def last_timing(self) -> list:
        arr = (ctypes.c_double * 6)()
        _check(lib().pfs_program_last_timing(self._h, arr, 6))
        return list(arr)

    def op_clock(self) -> np.ndarray:
        out = np.zeros(self.info["num_ops"] * 12, dtype=np.int64)
        _check(lib().pfs_program_op_clock(self._h, _p(out), out.size))
        return out.reshape(12, self.info["num_ops"])

    def ops(self) -> np.ndarray:
        out = np.zeros((self.info["num_ops"], 2), dtype=np.uint32)
        _check(lib().pfs_program_ops(self._h, _p(out), self.info["num_ops"]))
        return out

    def dump(self, what: int, flavour: int = 0) -> np.ndarray:
        """Raw uint32 table of a compiled flavour (pfs_program_dump; test tooling)."""
        n = int(lib().pfs_program_dump(self._h, flavour, what, None, 0))
        if n < 0:
            raise ValueError(lib().pfs_last_error().decode())
        out = np.zeros(max(n, 1), dtype=np.uint32)
        lib().pfs_program_dump(self._h, flavour, what, _p(out), n)
        return out[:n]

    def last_launches(self) -> int:
        return int(lib().pfs_program_last_launches(self._h))
