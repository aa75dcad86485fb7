"""Drop-in bulk frame sampling entry points (`stabsim/frame_sim.py:208-258`).

Same names, signatures and error messages as the reference, running on the
B200 through libpfs:

* `collect_flips(circuit, num_shots, rng, batch_size=1024)` -> `SampleTable`
  of measurement flips (frame_sim.py:208-229);
* `sample_batch(circuit, reference, num_shots, rng, batch_size=1024)` ->
  measurement samples = flips XOR reference (frame_sim.py:242-258);
* `sample_detection_events(circuit, num_shots, rng)` -> detection events and
  observables fused on the device (the reference composes collect_flips +
  detector_events, io_formats.py:208-227, "detect mode").

`rng` is a numpy Generator: one 63-bit Philox key is drawn from it per call,
so seeded calls are reproducible; the bit streams differ from numpy's (the
parity contract is statistical for sampled noise).  `batch_size`
is validated like the reference (it padded to 64-bit words and ran batches
sequentially, frame_sim.py:30-33, 217-228); the GPU picks its own shot tiles.
"""

from __future__ import annotations

from collections import OrderedDict

import numpy as np

from .circuit import as_circuit, format_circuit
from .io_formats import SampleTable
from .program import flatten
from .sampler import DetectorSampler, MeasurementSampler

DEFAULT_BATCH = 1024

_CACHE: "OrderedDict[tuple, object]" = OrderedDict()
_CACHE_MAX = 8


def _compiled(kind, circuit, device: int):
    c = as_circuit(circuit)
    key = (kind, format_circuit(c), device)
    obj = _CACHE.get(key)
    if obj is None:
        obj = (DetectorSampler if kind == "det" else MeasurementSampler)(c, device=device)
        _CACHE[key] = obj
        while len(_CACHE) > _CACHE_MAX:
            _CACHE.popitem(last=False)
    else:
        _CACHE.move_to_end(key)
    return obj


def _seed(rng) -> int:
    if rng is None:
        rng = np.random.default_rng()
    if isinstance(rng, (int, np.integer)):
        return int(rng)
    return int(rng.integers(2 ** 63))


def compile_frame_program(circuit):
    """The flat frame program (the reference returns an opcode tuple list,
    frame_sim.py:170-189; here a `FlatProgram` table the native compiler reads)."""
    return flatten(circuit)


def collect_flips(circuit, num_shots: int, rng, batch_size: int = DEFAULT_BATCH,
                  device: int = 0) -> SampleTable:
    """Measurement-flip table for num_shots independent runs (shots-major)."""
    if num_shots < 1:
        raise ValueError("num_shots must be >= 1")
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    s = _compiled("meas", circuit, device)
    b8 = s.sample_flips(num_shots, seed=_seed(rng))
    return SampleTable.from_b8(b8, s.num_measurements)


def sample_batch(circuit, reference, num_shots: int, rng, batch_size: int = DEFAULT_BATCH,
                 device: int = 0) -> SampleTable:
    """Sample the noisy circuit by XORing frame flips against a reference."""
    c = as_circuit(circuit)
    reference = list(reference)
    if len(reference) != c.num_measurements:
        raise ValueError(f"reference has {len(reference)} bits, circuit measures "
                         f"{c.num_measurements}")
    if num_shots < 1:
        raise ValueError("num_shots must be >= 1")
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    s = _compiled("meas", c, device)
    ref = np.asarray(reference, dtype=np.uint8) & 1
    prev = s.reference
    s.reference = np.ascontiguousarray(ref)
    try:
        b8 = s.sample(num_shots, seed=_seed(rng))
    finally:
        s.reference = prev
    return SampleTable.from_b8(b8, s.num_measurements)


def sample_detection_events(circuit, num_shots: int, rng, batch_size: int = DEFAULT_BATCH,
                            device: int = 0) -> SampleTable:
    """Detection events (detectors, then observables) for num_shots shots."""
    if num_shots < 1:
        raise ValueError("num_shots must be >= 1")
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    s = _compiled("det", circuit, device)
    b8 = s.sample(num_shots, seed=_seed(rng))
    return SampleTable.from_b8(b8, s.num_columns)
