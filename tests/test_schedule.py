"""Static verifier of the device program's synchronisation (CPU, no kernel runs).

The frame kernel elides group barriers: a barrier precedes an op only where the
host compiler found a shared frame row or ring slot (pfs_compile.cpp pass 3),
a fused op's noise is applied by the warp that owns the applications
(lower_stream's per-warp operand blocks), and consecutive standalone noise ops
commute through shared-memory atomics.  These tests re-derive every op's
resource set in Python from the raw tables (`pfs_program_dump`) and check the
invariants that make that safe — independent evidence for the barrier
schedule (compute-sanitizer's racecheck is closed on this GPU pool):

* no two ops of one barrier segment touch a common row / slot (noise-noise
  pairs excepted);
* the applications of one op touch pairwise distinct rows and slots;
* every application of a gate op sits in exactly one warp's operand block, in
  the warp's own chunk-aligned range (so pre-sampled hits of a consumer warp
  only ever touch rows that warp updates), padding names dummy rows only.
"""

from __future__ import annotations

import numpy as np
import pytest

from paper_2103_02202_b200 import _native as N
from paper_2103_02202_b200 import generators as gen
from paper_2103_02202_b200.program import flatten
from tests._util import inject_cases, load_inject

K_GATE, K_M, K_R, K_MR, K_NOISE, K_DET, K_OBS, K_SPILL = range(8)
F_BARRIER, F_DUP, F_NOISE = 1, 2, 4
NO_SLOT = 0xFFFFFFFF
COIN_DEAD = 0x80000000
XROW = 0x80000000
DUMMY_ROWS = 4
GATE_AHEAD = 4


def _tables(p, flavour):
    ops = p.dump(0, flavour).reshape(-1, 8)
    return dict(ops=ops, targets=p.dump(1, flavour), det_ptr=p.dump(2, flavour), det_terms=p.dump(3, flavour),
                sops=p.dump(4, flavour).reshape(-1, 12), arena=p.dump(5, flavour),
                fused=p.dump(6, flavour).reshape(-1, 4))


def _arity(kind, code):
    if kind == K_GATE:
        return 2 if code >= 4 else 1
    if kind == K_NOISE:
        return 2 if code == 4 else 1
    return 1


def _resources(t, op):
    """(rows, slots) an op reads or writes; det/obs terms included."""
    kcf, count, off, a = int(op[0]), int(op[1]), int(op[2]), int(op[3])
    kind, code = kcf & 0xFF, (kcf >> 8) & 0xFF
    rows, slots = [], []
    tg = t["targets"]
    if kind in (K_GATE, K_NOISE):
        rows = [int(x) for x in tg[off:off + count * _arity(kind, code)]]
    elif kind in (K_M, K_R, K_MR, K_SPILL):
        pairs = tg[off:off + 2 * count].reshape(-1, 2)
        rows = [int(x) & ~COIN_DEAD for x in pairs[:, 0]]
        slots = [int(x) for x in pairs[:, 1] if int(x) != NO_SLOT]
    elif kind == K_DET:
        for c in range(a, a + count):
            if code:
                terms = t["det_terms"][off + (c - a) * code: off + (c - a + 1) * code]
            else:
                terms = t["det_terms"][t["det_ptr"][c]:t["det_ptr"][c + 1]]
            for x in terms:
                x = int(x)
                (rows if x & XROW else slots).append(x & ~XROW)
    elif kind == K_OBS:
        slots.append(a)
        for x in tg[off:off + count]:
            x = int(x)
            (rows if x & XROW else slots).append(x & ~XROW)
    return rows, slots


def _check_program(p, flavour, n_qubits, warps_per_group, W):
    t = _tables(p, flavour)
    ops, sops = t["ops"], t["sops"]
    assert len(ops) == len(sops)
    seg_rows, seg_slots = {}, {}   # resource -> True when touched only by standalone noise ops
    for i, op in enumerate(ops):
        kcf = int(op[0])
        kind, code, flags = kcf & 0xFF, (kcf >> 8) & 0xFF, kcf >> 16
        rows, slots = _resources(t, op)
        standalone_noise = kind == K_NOISE
        # within one op: distinct rows / slots per application set (detectors only read)
        # (a SPILL only reads its rows: two records homed in one x row go to two slots)
        if kind in (K_GATE, K_M, K_R, K_MR) or (kind == K_NOISE and not (flags & F_DUP)):
            assert len(set(rows)) == len(rows), f"op {i}: applications share a row"
        if kind in (K_M, K_R, K_MR, K_SPILL):
            assert len(set(slots)) == len(slots), f"op {i}: applications share a slot"
        if flags & F_BARRIER:
            seg_rows, seg_slots = {}, {}
        for r in rows:
            if r in seg_rows:
                assert standalone_noise and seg_rows[r], f"op {i} (kind {kind}) shares row {r} with an op of its segment"
        for s in slots:
            assert s not in seg_slots, f"op {i} (kind {kind}) shares slot {s} with an op of its segment"
        for r in set(rows):
            seg_rows[r] = seg_rows.get(r, True) and standalone_noise
        for s in set(slots):
            seg_slots[s] = False
        # stream form: same flags, every application in exactly one warp's block
        so = sops[i]
        assert (int(so[0]) >> 16) & F_BARRIER == flags & F_BARRIER
        if kind == K_GATE:
            ar = _arity(kind, code)
            V = 4 if W >= 4 else W
            PI = 32 // (W // V)
            K, Kc, off = int(so[3]), int(so[10]), int(so[2])
            count = int(op[1])
            apps = t["targets"][int(op[2]): int(op[2]) + count * ar].reshape(-1, ar)
            want = [tuple(int(x) for x in a) for a in apps]
            stride = max(K, GATE_AHEAD) * PI   # a warp's block: at least GATE_AHEAD passes of words
            blk = t["arena"][off: off + warps_per_group * stride].reshape(warps_per_group, stride)
            seen = []
            for w in range(warps_per_group):
                mine = set(want[min(count, w * Kc): min(count, (w + 1) * Kc)])
                for word in blk[w]:
                    r0, r1 = int(word) & 0xFFFF, int(word) >> 16
                    if r0 >= n_qubits:   # padding: dummy rows only
                        assert n_qubits <= r0 < n_qubits + DUMMY_ROWS and (ar == 1 or n_qubits <= r1 < n_qubits + DUMMY_ROWS)
                        continue
                    app = (r0, r1) if ar == 2 else (r0,)
                    assert app in mine, f"op {i}: warp {w} holds an application outside its range"
                    seen.append(app)
            assert sorted(seen) == sorted(want), f"op {i}: operand blocks do not cover the applications once"
            if flags & F_NOISE and int(op[5]) != NO_SLOT and t["fused"].size:
                fi = t["fused"][int(op[5])]
                if int(fi[1]) == 1:   # pre-sampled: the producer's consumer-warp ranges are the blocks' ranges
                    assert int(fi[0]) == Kc
    return len(ops)


LAYOUTS = [dict(), dict(words_per_tile=8, groups=2), dict(words_per_tile=4, groups=4), dict(words_per_tile=1),
           dict(words_per_tile=2, ring_in_smem=0)]


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
def test_barrier_schedule_configs(cfg):
    f = flatten(gen.config_circuit(cfg))
    for lay in LAYOUTS[:3] if cfg == 2 else LAYOUTS:
        p = N.NativeProgram(f, **lay)
        info = p.info
        wpg = info["threads"] // max(1, int(info["groups"])) // 32
        for flavour in (0, 1):
            n = _check_program(p, flavour, f.num_qubits, wpg, info["words_per_tile"])
            assert n > 0


@pytest.mark.parametrize("name", inject_cases())
def test_barrier_schedule_golden_circuits(name):
    """The mixed golden circuits: duplicate targets, `CX 0 1 1 2` splits, MR,
    standalone noise, detectors over old records."""
    text = load_inject(name)[0]
    f = flatten(text)
    for lay in (dict(), dict(words_per_tile=2, groups=2)):
        p = N.NativeProgram(f, **lay)
        info = p.info
        wpg = info["threads"] // max(1, int(info["groups"])) // 32
        for flavour in (0, 1):
            _check_program(p, flavour, f.num_qubits, wpg, info["words_per_tile"])


def test_verifier_catches_a_missing_barrier():
    """Power check: clearing one barrier flag makes the verifier fail."""
    f = flatten(gen.config_circuit(0))
    p = N.NativeProgram(f)

    class Tampered:
        info = p.info

        def dump(self, what, flavour=0):
            a = p.dump(what, flavour).copy()
            if what in (0, 4):
                width = 8 if what == 0 else 12
                ops = a.reshape(-1, width)
                bar = [i for i in range(1, len(ops)) if (int(ops[i, 0]) >> 16) & F_BARRIER]
                ops[bar[len(bar) // 2], 0] &= ~np.uint32(F_BARRIER << 16)
            return a

    wpg = p.info["threads"] // max(1, int(p.info["groups"])) // 32
    with pytest.raises(AssertionError):
        _check_program(Tampered(), 0, f.num_qubits, wpg, p.info["words_per_tile"])
