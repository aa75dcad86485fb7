"""Compiled samplers: the user-facing API over libpfs.

Mirrors the paper's `compile_sampler(circuit).sample(n)` /
`compile_detector_sampler(circuit).sample(n)` pattern (
not present in the reference package) on top of the drop-in semantics of
`collect_flips` / `sample_batch` / `detector_events`
(`stabsim/frame_sim.py:208-258`, `stabsim/io_formats.py:208-227`).

Outputs are numpy arrays in the reference's b8 layout (shot-major, LSB-first,
ceil(R/8) bytes per shot — `stabsim/io_formats.py:94-96`), uint64 per-column
counts, or row-major uint32 bit tables.  `out=` accepts a preallocated host
array (pinned memory gives full-speed D2H) or a CUDA tensor (device-resident
output, no copy).
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .circuit import as_circuit
from .program import flatten


def _nbytes(a) -> int:
    """Bytes spanned by a (possibly row-strided) numpy array or torch tensor."""
    if hasattr(a, "data_ptr"):
        es = a.element_size()
        if a.dim() == 2 and a.numel():
            return int(((a.size(0) - 1) * a.stride(0) + a.size(1)) * es)
        return int(a.numel() * es)
    if a.ndim == 2 and a.size:
        return int((a.shape[0] - 1) * a.strides[0] + a.shape[1] * a.itemsize)
    return int(a.nbytes)


def pinned_empty(shape, dtype=np.uint8):
    """Page-locked host array (via torch's pinned allocator) for fast D2H."""
    import torch

    tdt = {np.dtype(np.uint8): torch.uint8, np.dtype(np.uint32): torch.int32,
           np.dtype(np.uint64): torch.int64}[np.dtype(dtype)]
    t = torch.empty(shape, dtype=tdt, pin_memory=True)
    arr = t.numpy().view(dtype)
    return arr, t


class _Compiled:
    def __init__(self, circuit, *, device: int = 0, seed=None, **native_opts):
        self.circuit = as_circuit(circuit)
        self.flat = flatten(self.circuit)
        self.native = N.NativeProgram(self.flat, **native_opts)
        self.device = device
        self._seeds = np.random.default_rng(seed)

    @property
    def tile_shots(self) -> int:
        return self.native.tile_shots

    @property
    def info(self) -> dict:
        return self.native.info

    def _seed(self, seed):
        return int(self._seeds.integers(2 ** 63)) if seed is None else int(seed)

    def _run_b8(self, mode, rows, shots, seed, out, shot_offset, ref=None, coins=None,
                masks=None, stream=0):
        nb = (rows + 7) // 8
        if out is None:
            out = np.empty((shots, nb), dtype=np.uint8)
        pitch = nb
        if isinstance(out, np.ndarray):
            if out.ndim != 2 or out.shape[0] < shots or out.dtype != np.uint8:
                raise ValueError("out must be uint8 [shots, >= ceil(R/8)]")
            pitch = out.strides[0]
        elif hasattr(out, "stride"):
            pitch = out.stride(0) * out.element_size()
        cw = iw = 0
        if coins is not None:
            coins = np.ascontiguousarray(coins, dtype=np.uint32)
            masks = np.ascontiguousarray(masks, dtype=np.uint32)
            iw = coins.shape[1] if coins.ndim == 2 and coins.shape[0] else masks.shape[1]
            cw = iw
        self.native.run(mode, shots, self._seed(seed), out, _nbytes(out), pitch,
                        shot_offset=shot_offset, device=self.device, ref_bits=ref,
                        coins=coins, masks=masks, inject_row_words=cw, stream=stream)
        return out

    def _run_rows(self, mode, rows, shots, seed, out, shot_offset, coins=None, masks=None,
                  stream=0):
        words = (shots + 31) // 32
        if out is None:
            out = np.empty((rows, words), dtype=np.uint32)
        iw = 0
        if coins is not None:
            coins = np.ascontiguousarray(coins, dtype=np.uint32)
            masks = np.ascontiguousarray(masks, dtype=np.uint32)
            iw = coins.shape[1] if coins.ndim == 2 and coins.shape[0] else masks.shape[1]
        self.native.run(mode, shots, self._seed(seed), out, _nbytes(out), 0,
                        shot_offset=shot_offset, device=self.device, coins=coins, masks=masks,
                        inject_row_words=iw, stream=stream)
        return out


class DetectorSampler(_Compiled):
    """Detection-event sampler: columns = detectors, then observables."""

    @property
    def num_detectors(self) -> int:
        return self.flat.num_detectors

    @property
    def num_observables(self) -> int:
        return self.flat.num_observables

    @property
    def num_columns(self) -> int:
        return self.flat.num_columns

    def sample(self, shots: int, *, seed=None, out=None, shot_offset: int = 0, coins=None,
               masks=None, stream: int = 0):
        """Shot-major b8 detection events, uint8 [shots, ceil(columns/8)]."""
        return self._run_b8(N.MODE_DETECTORS, self.num_columns, shots, seed, out, shot_offset,
                            coins=coins, masks=masks, stream=stream)

    def sample_rows(self, shots: int, *, seed=None, out=None, shot_offset: int = 0, coins=None,
                    masks=None, stream: int = 0):
        """Column-major uint32 rows [columns, ceil(shots/32)]."""
        return self._run_rows(N.MODE_DETECTORS_ROWS, self.num_columns, shots, seed, out,
                              shot_offset, coins, masks, stream)

    def sample_counts(self, shots: int, *, seed=None, out=None, shot_offset: int = 0,
                      coins=None, masks=None, stream: int = 0):
        """uint64 [columns] event counts (on-device popcount, no event I/O)."""
        if out is None:
            out = np.zeros(self.num_columns, dtype=np.uint64)
        iw = 0
        if coins is not None:
            coins = np.ascontiguousarray(coins, dtype=np.uint32)
            masks = np.ascontiguousarray(masks, dtype=np.uint32)
            iw = coins.shape[1] if coins.ndim == 2 and coins.shape[0] else masks.shape[1]
        self.native.run(N.MODE_COUNTS, shots, self._seed(seed), out, max(_nbytes(out), 8), 0,
                        shot_offset=shot_offset, device=self.device, coins=coins, masks=masks,
                        inject_row_words=iw, stream=stream)
        return out


class MeasurementSampler(_Compiled):
    """Measurement sampler: flips, or samples = flips XOR a reference sample."""

    def __init__(self, circuit, reference=None, **kw):
        super().__init__(circuit, **kw)
        self.reference = None
        if reference is not None:
            ref = np.asarray(list(reference), dtype=np.uint8).reshape(-1)
            if ref.shape[0] != self.flat.num_measurements:
                raise ValueError(f"reference has {ref.shape[0]} bits, circuit measures "
                                 f"{self.flat.num_measurements}")
            self.reference = np.ascontiguousarray(ref & 1)

    @property
    def num_measurements(self) -> int:
        return self.flat.num_measurements

    def sample(self, shots: int, *, seed=None, out=None, shot_offset: int = 0, coins=None,
               masks=None, stream: int = 0):
        """Shot-major b8 measurement samples (flips XOR the reference sample;
        without one, the native inverse-tableau reference sample is computed
        once, as the paper's compile_sampler does)."""
        if self.reference is None:
            from .tableau_sim import reference_sample
            ref = reference_sample(self.circuit, np.random.default_rng(self._seeds.integers(2 ** 63)))
            self.reference = np.ascontiguousarray(np.asarray(ref, dtype=np.uint8))
        return self._run_b8(N.MODE_SAMPLES, self.num_measurements, shots, seed, out,
                            shot_offset, ref=self.reference, coins=coins, masks=masks,
                            stream=stream)

    def sample_flips(self, shots: int, *, seed=None, out=None, shot_offset: int = 0, coins=None,
                     masks=None, stream: int = 0):
        """Shot-major b8 measurement flips."""
        return self._run_b8(N.MODE_FLIPS, self.num_measurements, shots, seed, out, shot_offset,
                            coins=coins, masks=masks, stream=stream)

    def sample_flip_rows(self, shots: int, *, seed=None, out=None, shot_offset: int = 0,
                         coins=None, masks=None, stream: int = 0):
        return self._run_rows(N.MODE_FLIPS_ROWS, self.num_measurements, shots, seed, out,
                              shot_offset, coins, masks, stream)


def compile_detector_sampler(circuit, **kw) -> DetectorSampler:
    return DetectorSampler(circuit, **kw)


def compile_sampler(circuit, reference=None, **kw) -> MeasurementSampler:
    return MeasurementSampler(circuit, reference=reference, **kw)
