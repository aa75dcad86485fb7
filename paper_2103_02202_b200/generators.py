"""Circuit generators for the BASELINE.json configs (superset dialect).

The reference's SPEC names `rep_code/random/surface_like` generators in an
absent `bench` module; these are written from the
BASELINE.json config text instead:

* `surface_code_memory(d, rounds, p)` — rotated surface code, Z-basis memory
  (configs 0, 2, 3, 4).  Data qubits at odd (x, y), measure qubits at even
  (x, y) of the (2d+1)^2 grid; weight-2 X plaquettes on the top/bottom
  boundaries, weight-2 Z plaquettes on the left/right.  Each round: R on the
  measure qubits, H on the X-type ones, four CX layers in the N/Z
  hook-avoiding order, H, M.  Noise: DEPOLARIZE1 after each single-qubit gate
  and reset, DEPOLARIZE2 after each CX, X_ERROR before each M.  Detectors
  compare each measure qubit with its previous round (round 0: Z-type only);
  the final data M gives the boundary detectors and the Z-logical observable
  (data row y = 1).
* `random_clifford(n, layers, p, seed)` — config 1.

Qubit numbering is row-major over the grid coordinates (y, then x).
"""

from __future__ import annotations

import numpy as np

# CX offsets (dx, dy) per layer, SURVEY.md Appendix A.
_X_ORDER = ((1, 1), (-1, 1), (1, -1), (-1, -1))
_Z_ORDER = ((1, 1), (1, -1), (-1, 1), (-1, -1))


class SurfaceLayout:
    def __init__(self, d: int):
        if d < 2:
            raise ValueError("distance must be >= 2")
        self.d = d
        side = 2 * d + 1
        data = [(x, y) for y in range(1, 2 * d, 2) for x in range(1, 2 * d, 2)]
        data_set = set(data)
        xm, zm = [], []
        for y in range(0, side, 2):
            for x in range(0, side, 2):
                nbrs = [(x + dx, y + dy) for dx in (-1, 1) for dy in (-1, 1)
                        if (x + dx, y + dy) in data_set]
                is_x = ((x // 2 + y // 2) % 2) == 1
                if len(nbrs) == 4:
                    (xm if is_x else zm).append((x, y))
                elif len(nbrs) == 2:
                    horizontal_edge = y in (0, 2 * d)
                    vertical_edge = x in (0, 2 * d)
                    if is_x and horizontal_edge and not vertical_edge:
                        xm.append((x, y))
                    elif (not is_x) and vertical_edge and not horizontal_edge:
                        zm.append((x, y))
        coords = sorted(data + xm + zm, key=lambda c: (c[1], c[0]))
        self.index = {c: i for i, c in enumerate(coords)}
        self.coords = coords
        self.data = sorted((self.index[c] for c in data))
        self.x_meas = sorted(self.index[c] for c in xm)
        self.z_meas = sorted(self.index[c] for c in zm)
        self.meas = sorted(self.x_meas + self.z_meas)
        self.data_set = data_set

    def support(self, q: int):
        x, y = self.coords[q]
        return sorted(self.index[(x + dx, y + dy)] for dx in (-1, 1) for dy in (-1, 1)
                      if (x + dx, y + dy) in self.data_set)

    def cx_layer(self, layer: int):
        """(control, target) pairs of one CX layer."""
        pairs = []
        for m in self.meas:
            x, y = self.coords[m]
            is_x = m in self._xset
            dx, dy = (_X_ORDER if is_x else _Z_ORDER)[layer]
            c = (x + dx, y + dy)
            if c not in self.data_set:
                continue
            dq = self.index[c]
            pairs.append((m, dq) if is_x else (dq, m))
        return pairs

    @property
    def _xset(self):
        s = getattr(self, "_xs", None)
        if s is None:
            s = self._xs = frozenset(self.x_meas)
        return s


def _fmt_p(p: float) -> str:
    return repr(float(p))


def surface_code_memory(d: int, rounds: int, p: float, use_repeat: bool = True) -> str:
    """Rotated surface-code Z-memory circuit text (superset dialect)."""
    if rounds < 1:
        raise ValueError("rounds must be >= 1")
    lay = SurfaceLayout(d)
    meas = lay.meas
    nm = len(meas)
    xset = set(lay.x_meas)
    ps = _fmt_p(p)
    noisy = p > 0
    mstr = " ".join(map(str, meas))
    xstr = " ".join(map(str, lay.x_meas))

    def round_body(first: bool):
        out = []
        out.append(f"R {mstr}")
        if noisy:
            out.append(f"DEPOLARIZE1({ps}) {mstr}")
        out.append("TICK")
        out.append(f"H {xstr}")
        if noisy:
            out.append(f"DEPOLARIZE1({ps}) {xstr}")
        out.append("TICK")
        for layer in range(4):
            pairs = lay.cx_layer(layer)
            flat = " ".join(f"{a} {b}" for a, b in pairs)
            out.append(f"CX {flat}")
            if noisy:
                out.append(f"DEPOLARIZE2({ps}) {flat}")
            out.append("TICK")
        out.append(f"H {xstr}")
        if noisy:
            out.append(f"DEPOLARIZE1({ps}) {xstr}")
        out.append("TICK")
        if noisy:
            out.append(f"X_ERROR({ps}) {mstr}")
        out.append(f"M {mstr}")
        for i, m in enumerate(meas):
            k = nm - i  # lookback of this round's record of m
            if first:
                if m not in xset:
                    out.append(f"DETECTOR rec[-{k}]")
            else:
                out.append(f"DETECTOR rec[-{k}] rec[-{k + nm}]")
        return out

    lines = round_body(True)
    if rounds > 1:
        body = round_body(False)
        if use_repeat:
            lines.append(f"REPEAT {rounds - 1} {{")
            lines.extend("    " + s for s in body)
            lines.append("}")
        else:
            for _ in range(rounds - 1):
                lines.extend(body)
    data = lay.data
    nd = len(data)
    dstr = " ".join(map(str, data))
    if noisy:
        lines.append(f"X_ERROR({ps}) {dstr}")
    lines.append(f"M {dstr}")
    dpos = {q: i for i, q in enumerate(data)}
    mpos = {q: i for i, q in enumerate(meas)}
    for m in meas:
        if m in xset:
            continue
        recs = [f"rec[-{nd - dpos[q]}]" for q in lay.support(m)]
        recs.append(f"rec[-{nd + nm - mpos[m]}]")
        lines.append("DETECTOR " + " ".join(recs))
    row = [q for q in data if lay.coords[q][1] == 1]
    lines.append("OBSERVABLE_INCLUDE(0) " + " ".join(f"rec[-{nd - dpos[q]}]" for q in row))
    return "\n".join(lines) + "\n"


def random_clifford(n: int = 64, layers: int = 200, p: float = 0.01, seed: int = 0,
                    mr_fraction: float = 0.1) -> str:
    """Config 1: seeded random Clifford circuit with mid-circuit MR.

    Each layer pairs the qubits at random and applies CX or CZ (1/2 each) per
    pair, then one of {H, S, SQRT_X, I} per qubit; then round(0.1 n) random
    qubits get X_ERROR(p) + MR, each MR followed by a detector XOR-ing 3
    distinct records among the most recent 3k; DEPOLARIZE1(p) on every qubit
    closes the layer.
    """
    rng = np.random.default_rng(seed)
    k = max(1, int(round(mr_fraction * n)))
    ps = _fmt_p(p)
    lines = []
    total = 0
    for _ in range(layers):
        perm = rng.permutation(n)
        cx, cz = [], []
        for i in range(0, n - 1, 2):
            a, b = int(perm[i]), int(perm[i + 1])
            (cx if rng.random() < 0.5 else cz).append((a, b))
        if cx:
            lines.append("CX " + " ".join(f"{a} {b}" for a, b in cx))
        if cz:
            lines.append("CZ " + " ".join(f"{a} {b}" for a, b in cz))
        choice = rng.integers(0, 4, size=n)
        for g, name in enumerate(("H", "S", "SQRT_X", "I")):
            qs = np.flatnonzero(choice == g)
            if qs.size:
                lines.append(name + " " + " ".join(map(str, qs.tolist())))
        mq = sorted(rng.choice(n, size=k, replace=False).tolist())
        mstr = " ".join(map(str, mq))
        if p > 0:
            lines.append(f"X_ERROR({ps}) {mstr}")
        lines.append(f"MR {mstr}")
        total += k
        window = min(total, 3 * k)
        for _j in range(k):
            cnt = min(3, window)
            picks = sorted(rng.choice(window, size=cnt, replace=False).tolist())
            lines.append("DETECTOR " + " ".join(f"rec[-{w + 1}]" for w in picks))
        if p > 0:
            lines.append(f"DEPOLARIZE1({ps}) " + " ".join(map(str, range(n))))
        lines.append("TICK")
    return "\n".join(lines) + "\n"


# BASELINE.json configs
CONFIGS = {
    0: dict(kind="surface", d=3, rounds=3, p=1e-3, shots=1024),
    1: dict(kind="random", n=64, layers=200, p=0.01, seed=0, shots=65536),
    2: dict(kind="surface", d=25, rounds=25, p=1e-3, shots=1 << 20),
    3: dict(kind="surface", d=5, rounds=5, p=5e-3, shots=1 << 32, batch=1 << 24),
    4: dict(kind="surface", d=100, rounds=100, p=1e-3, shots=1 << 16),
}


def config_circuit(idx: int) -> str:
    c = CONFIGS[idx]
    if c["kind"] == "surface":
        return surface_code_memory(c["d"], c["rounds"], c["p"])
    return random_clifford(c["n"], c["layers"], c["p"], c["seed"])
