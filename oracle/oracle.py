"""ctypes wrapper of the C oracle (oracle/pfs_oracle.c) — TEST INFRASTRUCTURE.

Only tests/, `__graft_entry__.smoke()` and bench.py's CPU-baseline legs may
import this module.  It is the checker, never the thing shipped: the product
(`paper_2103_02202_b200`) has no import path to it.
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
        i64, i32, u64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
        L.orc_sample.argtypes = [P, i64, P, P, P, i32, i64, P, P, i64, i64, i32, u64, u64,
                                 P, P, i64, P, P, i64, ctypes.c_int]
        L.orc_sample.restype = ctypes.c_int
        L.orc_rows_to_b8.argtypes = [P, i64, i64, i64, P, P, i64]
        L.orc_rows_to_b8.restype = None
        L.orc_philox4x32_10.argtypes = [P, P, P]
        L.orc_philox4x32_10.restype = None
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def sample(prog: FlatProgram, num_shots: int, tile_shots: int, seed: int = 0,
           tile_offset: int = 0, coins=None, masks=None, flips: bool = True,
           events: bool = True, nthreads: int = 1, schedule=None):
    """Run the oracle; returns (flip_rows, event_rows), uint32 [rows, words].

    `schedule` = (params, tables) of the noise sampler for this tile size, as
    compiled by the product's host compiler (`NativeProgram.noise_schedule()`):
    the RNG draw order only — the frame semantics are this file's own.
    """
    L = lib()
    n_tiles = -(-num_shots // tile_shots)
    words = n_tiles * tile_shots // 32
    ins = np.ascontiguousarray(prog.instrs, dtype=np.int32)
    tg = np.ascontiguousarray(prog.targets, dtype=np.int32)
    if schedule is None:
        schedule = noise_schedule(prog, tile_shots)
    params = np.ascontiguousarray(schedule[0], dtype=np.uint32)
    tab = np.ascontiguousarray(schedule[1], dtype=np.uint64)
    inject_words = 0
    if coins is not None or masks is not None:
        if coins is None or masks is None:
            raise ValueError("injected mode needs both coin and noise-mask rows")
        coins = _pad_rows(coins, words)
        masks = _pad_rows(masks, words)
        inject_words = words
    fl = np.zeros((prog.num_measurements, words), dtype=np.uint32) if flips else None
    ev = np.zeros((prog.num_columns, words), dtype=np.uint32) if events else None
    rc = L.orc_sample(_ptr(ins), ins.shape[0], _ptr(tg), _ptr(params) if params.size else None,
                      _ptr(tab) if tab.size else None,
                      prog.num_qubits, prog.num_measurements, _ptr(prog.det_ptr),
                      _ptr(prog.det_idx), prog.num_columns, num_shots, tile_shots,
                      seed & 0xFFFFFFFFFFFFFFFF, tile_offset, _ptr(coins), _ptr(masks),
                      inject_words, _ptr(fl) if fl is not None and fl.size else None,
                      _ptr(ev) if ev is not None and ev.size else None, words, nthreads)
    if rc != 0:
        raise RuntimeError(f"orc_sample failed ({rc})")
    return fl, ev


def noise_schedule(prog: FlatProgram, tile_shots: int):
    """Noise RNG schedule for tile size T from the product's host compiler
    (pure host code, no GPU needed)."""
    from paper_2103_02202_b200._native import NativeProgram

    return NativeProgram(prog, words_per_tile=tile_shots // 32, ring_in_smem=0,
                         schedule_only=True).noise_schedule()


def _pad_rows(a, words):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    if a.ndim != 2:
        raise ValueError("inject rows must be 2-D [rows, words]")
    if a.shape[1] >= words:
        return np.ascontiguousarray(a[:, :words])
    out = np.zeros((a.shape[0], words), dtype=np.uint32)
    out[:, :a.shape[1]] = a
    return out


def rows_to_b8(rows: np.ndarray, num_shots: int, xor_bits=None) -> np.ndarray:
    """Row-major bit table -> shot-major b8 (uint8 [shots, ceil(R/8)])."""
    L = lib()
    rows = np.ascontiguousarray(rows, dtype=np.uint32)
    R = rows.shape[0]
    nb = (R + 7) // 8
    out = np.zeros((num_shots, nb), dtype=np.uint8)
    xb = None if xor_bits is None else np.ascontiguousarray(xor_bits, dtype=np.uint8)
    if R and num_shots:
        L.orc_rows_to_b8(_ptr(rows), R, num_shots, rows.shape[1], _ptr(xb), _ptr(out), nb)
    return out


def philox(ctr, key):
    L = lib()
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    L.orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(o))
    return o
