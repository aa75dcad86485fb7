"""Gate registry for the bulk frame sampler.

Only the data the Pauli-frame hot path needs is kept here: the per-gate
frame-update rule (the reference derives it from the gate tableau in
`stabsim/gates.py:70-92` `GateData.frame_plan`), the noise-channel Pauli
patterns (`stabsim/gates.py:98-104, 146-152`), and the collapse flags
(`stabsim/gates.py:40-41, 142-144`).  Tableau / unitary algebra is not on
the frame path and is not rebuilt.

The superset dialect adds TICK, OBSERVABLE_INCLUDE, SQRT_X and SQRT_X_DAG,
which the reference registry lacks (`stabsim/gates.py:107-156`).
"""

from __future__ import annotations

from dataclasses import dataclass, field

UNITARY = "unitary"
COLLAPSING = "collapsing"
NOISE = "noise"
ANNOTATION = "annotation"

# Device frame-rule codes (one per distinct update rule).
RULE_NONE = 0      # Pauli gates / identity: frames unchanged
RULE_SWAPXZ = 1    # H, SQRT_Y, SQRT_Y_DAG:  x <-> z
RULE_ZXORX = 2     # S, S_DAG:               z ^= x
RULE_XXORZ = 3     # SQRT_X, SQRT_X_DAG:     x ^= z
RULE_CX = 4        # x1 ^= x0 ; z0 ^= z1
RULE_CZ = 5        # z0 ^= x1 ; z1 ^= x0
RULE_CY = 6        # x1 ^= x0 ; z0 ^= x1 ^ z1 ; z1 ^= x0
RULE_SWAP = 7      # swap both planes

# Frame plans in the reference's format: (dst_plane, dst_slot, sources),
# sources = ((src_plane, src_slot), ...), all reads of *old* values.  Kept
# so tests can compare against the plan dumped from the reference
# (tests/golden/frame_plans.json, produced by tests/golden/make_golden.py).
_PLANS = {
    RULE_NONE: (),
    RULE_SWAPXZ: ((0, 0, ((1, 0),)), (1, 0, ((0, 0),))),
    RULE_ZXORX: ((1, 0, ((0, 0), (1, 0))),),
    RULE_XXORZ: ((0, 0, ((0, 0), (1, 0))),),
    RULE_CX: ((0, 1, ((0, 0), (0, 1))), (1, 0, ((1, 0), (1, 1)))),
    RULE_CZ: ((1, 0, ((0, 1), (1, 0))), (1, 1, ((0, 0), (1, 1)))),
    RULE_CY: ((0, 1, ((0, 0), (0, 1))), (1, 0, ((0, 1), (1, 0), (1, 1))),
              (1, 1, ((0, 0), (1, 1)))),
    RULE_SWAP: ((0, 0, ((0, 1),)), (0, 1, ((0, 0),)), (1, 0, ((1, 1),)),
                (1, 1, ((1, 0),))),
}

# Algorithmic frame bits touched per shot per application:
# rows read + rows written.
RULE_BITS = {RULE_NONE: 0, RULE_SWAPXZ: 4, RULE_ZXORX: 3, RULE_XXORZ: 3,
             RULE_CX: 6, RULE_CZ: 6, RULE_CY: 7, RULE_SWAP: 8}


def _depolarize2_patterns():
    """15 two-qubit Pauli codes in the reference order (gates.py:98-104)."""
    pats = []
    for code in range(1, 16):
        x = (code & 1) | (((code >> 2) & 1) << 1)
        z = ((code >> 1) & 1) | (((code >> 3) & 1) << 1)
        pats.append((x, z))
    return tuple(pats)


@dataclass(eq=False)
class GateData:
    name: str
    kind: str
    arity: int  # targets per application; 0 = variable (annotations)
    parameter_count: int = 0
    rule: int = RULE_NONE
    noise_patterns: tuple = ()
    records: bool = False
    resets: bool = False
    aliases: tuple = field(default_factory=tuple)

    @property
    def frame_plan(self):
        if self.kind != UNITARY:
            raise ValueError(f"{self.name} has no frame plan")
        return _PLANS[self.rule]

    def __repr__(self):
        return f"GateData({self.name})"


GATES = (
    GateData("I", UNITARY, 1),
    GateData("X", UNITARY, 1),
    GateData("Y", UNITARY, 1),
    GateData("Z", UNITARY, 1),
    GateData("H", UNITARY, 1, rule=RULE_SWAPXZ),
    GateData("S", UNITARY, 1, rule=RULE_ZXORX),
    GateData("S_DAG", UNITARY, 1, rule=RULE_ZXORX),
    GateData("SQRT_Y", UNITARY, 1, rule=RULE_SWAPXZ),
    GateData("SQRT_Y_DAG", UNITARY, 1, rule=RULE_SWAPXZ),
    GateData("SQRT_X", UNITARY, 1, rule=RULE_XXORZ),
    GateData("SQRT_X_DAG", UNITARY, 1, rule=RULE_XXORZ),
    GateData("CNOT", UNITARY, 2, rule=RULE_CX, aliases=("CX",)),
    GateData("CY", UNITARY, 2, rule=RULE_CY),
    GateData("CZ", UNITARY, 2, rule=RULE_CZ),
    GateData("SWAP", UNITARY, 2, rule=RULE_SWAP),
    GateData("M", COLLAPSING, 1, records=True),
    GateData("R", COLLAPSING, 1, resets=True),
    GateData("MR", COLLAPSING, 1, records=True, resets=True),
    GateData("X_ERROR", NOISE, 1, parameter_count=1, noise_patterns=((1, 0),)),
    GateData("Y_ERROR", NOISE, 1, parameter_count=1, noise_patterns=((1, 1),)),
    GateData("Z_ERROR", NOISE, 1, parameter_count=1, noise_patterns=((0, 1),)),
    GateData("DEPOLARIZE1", NOISE, 1, parameter_count=1,
             noise_patterns=((1, 0), (1, 1), (0, 1))),
    GateData("DEPOLARIZE2", NOISE, 2, parameter_count=1,
             noise_patterns=_depolarize2_patterns()),
    GateData("DETECTOR", ANNOTATION, 0),
    # superset dialect (absent from the reference registry)
    GateData("OBSERVABLE_INCLUDE", ANNOTATION, 0, parameter_count=1),
    GateData("TICK", ANNOTATION, 0),
)

GATE_MAP: dict[str, GateData] = {}
for _g in GATES:
    GATE_MAP[_g.name] = _g
    for _a in _g.aliases:
        GATE_MAP[_a] = _g

# Gates the reference itself knows (stabsim/gates.py:107-156); the rest need
# lowering before a circuit can be handed to the reference.
REFERENCE_GATE_NAMES = frozenset(
    ["I", "X", "Y", "Z", "H", "S", "S_DAG", "SQRT_Y", "SQRT_Y_DAG", "CNOT",
     "CX", "CY", "CZ", "SWAP", "M", "R", "MR", "X_ERROR", "Y_ERROR", "Z_ERROR",
     "DEPOLARIZE1", "DEPOLARIZE2", "DETECTOR"])


def get_gate(name: str) -> GateData:
    gate = GATE_MAP.get(name.upper())
    if gate is None:
        raise KeyError(f"unknown gate {name!r}")
    return gate
