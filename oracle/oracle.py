"""ctypes wrapper of the C oracle (oracle/pfs_oracle.c) — TEST INFRASTRUCTURE.

Only tests/, `__graft_entry__.smoke()` and bench.py's CPU-baseline legs may
import this module.  It is the checker, never the thing shipped: the product
(`paper_2103_02202_b200`) has no import path to it, and it uses nothing of the
product's native library (its noise schedule is computed in pfs_oracle.c).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from paper_2103_02202_b200.program import FlatProgram

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libpfs_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or (
            os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(HERE, "pfs_oracle.c"))):
        subprocess.run(["make", "-C", HERE, "-B" if force else "all"], check=True,
                       stdout=subprocess.DEVNULL)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i64, i32, u32, u64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint64
        L.orc_sample.argtypes = [P, i64, P, P, i64, P, i32, i32, i64, P, P, i64, i64, i32, u64, u64,
                                 P, P, i64, P, P, i64, ctypes.c_int]
        L.orc_sample.restype = ctypes.c_int
        L.orc_rows_to_b8.argtypes = [P, i64, i64, i64, P, P, i64, ctypes.c_int]
        L.orc_rows_to_b8.restype = None
        L.orc_philox4x32_10.argtypes = [P, P, P]
        L.orc_philox4x32_10.restype = None
        L.orc_noise_schedule.argtypes = [u32, ctypes.c_int, ctypes.c_double, u32, u32, u32, P, P, ctypes.c_int]
        L.orc_noise_schedule.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def sample(prog: FlatProgram, num_shots: int, tile_shots: int, seed: int = 0,
           tile_offset: int = 0, coins=None, masks=None, flips: bool = True,
           events: bool = True, nthreads: int = 1, chunk_L=None, vector_shots: int = 0):
    """Run the oracle; returns (flip_rows, event_rows), uint32 [rows, words].

    Layout parameters of the counter-based draws: tiles of
    `tile_shots` shots, vectors of `vector_shots` (0 = min(128, T)) and the
    chunk length of every noise instruction, `chunk_L` (uint32 [num_noise]).
    They fix the draw order, not the distribution; the chunk geometry and the
    Binomial tables are computed by the oracle itself.
    """
    L = lib()
    n_tiles = -(-num_shots // tile_shots)
    words = n_tiles * tile_shots // 32
    ins = np.ascontiguousarray(prog.instrs, dtype=np.int32)
    tg = np.ascontiguousarray(prog.targets, dtype=np.int32)
    noise_p = np.ascontiguousarray(prog.noise_p, dtype=np.float64)
    if vector_shots <= 0:
        vector_shots = min(128, tile_shots)
    inject_words = 0
    if coins is not None or masks is not None:
        if coins is None or masks is None:
            raise ValueError("injected mode needs both coin and noise-mask rows")
        coins = _pad_rows(coins, words)
        masks = _pad_rows(masks, words)
        inject_words = words
        chunk_L = np.ones(prog.num_noise, dtype=np.uint32)
    elif chunk_L is None:
        raise ValueError("sampled mode needs the chunk length of every noise instruction")
    cl = np.ascontiguousarray(chunk_L, dtype=np.uint32)
    if cl.shape[0] != prog.num_noise:
        raise ValueError("chunk_L needs one entry per noise instruction")
    fl = np.zeros((prog.num_measurements, words), dtype=np.uint32) if flips else None
    ev = np.zeros((prog.num_columns, words), dtype=np.uint32) if events else None
    rc = L.orc_sample(_ptr(ins), ins.shape[0], _ptr(tg), _ptr(noise_p) if noise_p.size else None,
                      prog.num_noise, _ptr(cl) if cl.size else None, vector_shots,
                      prog.num_qubits, prog.num_measurements, _ptr(prog.det_ptr),
                      _ptr(prog.det_idx), prog.num_columns, num_shots, tile_shots,
                      seed & 0xFFFFFFFFFFFFFFFF, tile_offset, _ptr(coins), _ptr(masks),
                      inject_words, _ptr(fl) if fl is not None and fl.size else None,
                      _ptr(ev) if ev is not None and ev.size else None, words, nthreads)
    if rc != 0:
        raise RuntimeError(f"orc_sample failed ({rc})")
    return fl, ev


def noise_schedule_one(apps: int, channel: int, p: float, L: int, tile_shots: int, vector_shots: int):
    """The oracle's own schedule of one noise instruction: (12 uint32 words
    L, cs, ca, nchunks, apps, 0, len, zone, npat, channel, 0, 0; thresholds)."""
    params = np.zeros(12, dtype=np.uint32)
    tab = np.zeros(256, dtype=np.uint64)
    rc = lib().orc_noise_schedule(apps, channel, float(p), L, tile_shots, vector_shots, _ptr(params),
                                  _ptr(tab), 256)
    if rc != 0:
        raise ValueError(f"orc_noise_schedule failed ({rc})")
    return params, tab[:params[6]].copy()


def _pad_rows(a, words):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    if a.ndim != 2:
        raise ValueError("inject rows must be 2-D [rows, words]")
    if a.shape[1] >= words:
        return np.ascontiguousarray(a[:, :words])
    out = np.zeros((a.shape[0], words), dtype=np.uint32)
    out[:, :a.shape[1]] = a
    return out


def rows_to_b8(rows: np.ndarray, num_shots: int, xor_bits=None, nthreads: int = 1) -> np.ndarray:
    """Row-major bit table -> shot-major b8 (uint8 [shots, ceil(R/8)])."""
    L = lib()
    rows = np.ascontiguousarray(rows, dtype=np.uint32)
    R = rows.shape[0]
    nb = (R + 7) // 8
    out = np.zeros((num_shots, nb), dtype=np.uint8)
    xb = None if xor_bits is None else np.ascontiguousarray(xor_bits, dtype=np.uint8)
    if R and num_shots:
        L.orc_rows_to_b8(_ptr(rows), R, num_shots, rows.shape[1], _ptr(xb), _ptr(out), nb, nthreads)
    return out


def philox(ctr, key):
    L = lib()
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    L.orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(o))
    return o
