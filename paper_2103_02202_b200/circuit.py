"""Circuit text: parsing, canonical printing and flat iteration (superset dialect).

Same grammar and error behaviour as the reference parser
(`stabsim/circuit.py:1-8, 110-211`): one instruction per line, optional
parenthesised parameter, whitespace-separated targets, case-insensitive gate
names, `#` comments, nested `REPEAT N { ... }` blocks, DETECTOR targets
written `rec[-k]`.  Errors are `CircuitParseError` (a `ValueError`) carrying
the 1-based line (`stabsim/circuit.py:18-23`).

Superset additions (needed by the BASELINE configs, absent from the
reference):

* ``TICK`` — layer marker, no targets; a scheduling hint only.
* ``OBSERVABLE_INCLUDE(k) rec[-a] ...`` — accumulates records into logical
  observable ``k``.  Observables are reported after all detectors, in index
  order, exactly as the reference sees them after lowering (a trailing
  DETECTOR per observable).
* ``SQRT_X`` / ``SQRT_X_DAG``.

`Circuit`, `Instruction` and `Repeat` are duck-type compatible with the
reference classes (`stabsim/circuit.py:26-97`); reference `Circuit` objects
are accepted everywhere a circuit is (see `as_circuit`).
"""

from __future__ import annotations

from dataclasses import dataclass

from .gates import ANNOTATION, NOISE, GATE_MAP, REFERENCE_GATE_NAMES, GateData


class CircuitParseError(ValueError):
    """Malformed circuit text; `.line` is the 1-based source line."""

    def __init__(self, message: str, line: int):
        super().__init__(f"line {line}: {message}")
        self.line = line


@dataclass(frozen=True, eq=False)
class Instruction:
    gate: GateData
    param: float | None
    targets: tuple  # qubits, or negative lookbacks for DETECTOR/OBSERVABLE_INCLUDE
    line: int = 0

    def __eq__(self, other):
        if not isinstance(other, Instruction):
            return NotImplemented
        return (self.gate is other.gate and self.param == other.param
                and self.targets == other.targets)

    def __hash__(self):
        return hash((self.gate.name, self.param, self.targets))

    def num_measurements(self) -> int:
        return len(self.targets) if self.gate.records else 0

    def __str__(self):
        name = self.gate.name
        if self.param is not None:
            if self.gate.name == "OBSERVABLE_INCLUDE":
                name += f"({int(self.param)})"
            else:
                name += f"({self.param!r})"
        if self.gate.kind == ANNOTATION:
            body = " ".join(f"rec[{t}]" for t in self.targets)
        else:
            body = " ".join(str(t) for t in self.targets)
        return f"{name} {body}" if body else name


@dataclass(frozen=True)
class Repeat:
    count: int
    body: "Circuit"

    def num_measurements(self) -> int:
        return self.count * self.body.num_measurements


class Circuit:
    """Ordered instructions and nested REPEAT blocks."""

    __slots__ = ("elements", "num_qubits", "num_measurements")

    def __init__(self, elements):
        self.elements = tuple(elements)
        self.num_qubits = _max_qubit(self.elements) + 1
        self.num_measurements = sum(e.num_measurements() for e in self.elements)

    def __eq__(self, other):
        if not isinstance(other, Circuit):
            return NotImplemented
        return self.elements == other.elements

    def __hash__(self):
        return hash(self.elements)

    def __str__(self):
        return format_circuit(self)

    def __repr__(self):
        return (f"Circuit({len(self.elements)} elements, {self.num_qubits} qubits, "
                f"{self.num_measurements} measurements)")

    @property
    def num_detectors(self) -> int:
        return len(detector_sets(self))

    @property
    def num_observables(self) -> int:
        return len(observable_sets(self))


def _max_qubit(elements) -> int:
    best = -1
    for e in elements:
        if isinstance(e, Repeat) or hasattr(e, "body"):
            best = max(best, _max_qubit(e.body.elements))
        elif e.gate.kind != ANNOTATION:
            best = max(best, max(e.targets, default=-1))
    return best


def _is_repeat(e) -> bool:
    return hasattr(e, "body") and hasattr(e, "count")


def iter_flat(circuit):
    """Instructions in execution order with REPEAT expanded
    (`stabsim/circuit.py:100-107`)."""
    for e in circuit.elements:
        if _is_repeat(e):
            for _ in range(e.count):
                yield from iter_flat(e.body)
        else:
            yield e


def _lookback(tok: str):
    t = tok.lower()
    if not (t.startswith("rec[") and t.endswith("]")):
        return None
    inner = t[4:-1]
    # same token shape as the reference's `rec\[(-\d+)\]` (circuit.py:114)
    if len(inner) < 2 or inner[0] != "-" or not inner[1:].isdigit():
        return None
    return int(inner)


def _split_head(line: str):
    """Split 'NAME(param) targets' into (name, param_text|None, rest)."""
    i = 0
    n = len(line)
    if i >= n or not (line[i].isalpha() or line[i] == "_"):
        return None
    while i < n and (line[i].isalnum() or line[i] == "_"):
        i += 1
    name = line[:i]
    j = i
    while j < n and line[j].isspace():
        j += 1
    param = None
    if j < n and line[j] == "(":
        close = line.find(")", j)
        if close < 0:
            return None
        param = line[j + 1:close].strip()
        rest = line[close + 1:]
        if rest and not rest[0].isspace():
            return None
    else:
        rest = line[i:]
        if rest and not rest[0].isspace():
            return None
    return name, param, rest


def _parse_instruction(line: str, line_no: int) -> Instruction:
    head = _split_head(line)
    if head is None:
        raise CircuitParseError(f"unparseable instruction {line!r}", line_no)
    raw_name, param_text, rest = head
    gate = GATE_MAP.get(raw_name.upper())
    if gate is None:
        raise CircuitParseError(f"unknown gate {raw_name!r}", line_no)
    param = None
    if gate.parameter_count == 0:
        if param_text is not None:
            raise CircuitParseError(f"{gate.name} takes no parameter", line_no)
    else:
        if param_text is None:
            raise CircuitParseError(f"{gate.name} needs a parameter", line_no)
        try:
            param = float(param_text)
        except ValueError:
            raise CircuitParseError(f"bad parameter {param_text!r}", line_no) from None
        if gate.kind == NOISE and not 0.0 <= param <= 1.0:
            raise CircuitParseError(
                f"noise parameter must be in [0, 1], got {param}", line_no)
        if gate.name == "OBSERVABLE_INCLUDE" and (param < 0 or param != int(param)):
            raise CircuitParseError(
                f"observable index must be a non-negative integer, got {param_text}",
                line_no)
    tokens = rest.split()
    if gate.kind == ANNOTATION:
        if gate.name == "TICK":
            if tokens:
                raise CircuitParseError("TICK takes no targets", line_no)
            return Instruction(gate, None, (), line_no)
        if not tokens and gate.name == "DETECTOR":
            raise CircuitParseError(f"{gate.name} needs at least one rec[-k] target",
                                    line_no)
        targets = []
        for tok in tokens:
            k = _lookback(tok)
            if k is None:
                raise CircuitParseError(
                    f"bad {gate.name} target {tok!r}, expected rec[-k]", line_no)
            if k >= 0:
                raise CircuitParseError(f"lookback must be negative, got {k}", line_no)
            targets.append(k)
        return Instruction(gate, param, tuple(targets), line_no)
    targets = []
    for tok in tokens:
        if not tok.isdigit():
            raise CircuitParseError(f"bad target {tok!r}, expected a qubit index",
                                    line_no)
        targets.append(int(tok))
    if not targets or len(targets) % gate.arity != 0:
        raise CircuitParseError(
            f"{gate.name} needs a positive multiple of {gate.arity} targets, "
            f"got {len(targets)}", line_no)
    if gate.arity == 2:
        for i in range(0, len(targets), 2):
            if targets[i] == targets[i + 1]:
                raise CircuitParseError(
                    f"{gate.name} targets a qubit pair twice: {targets[i]}", line_no)
    return Instruction(gate, param, tuple(targets), line_no)


def _repeat_count(line: str):
    parts = line.split()
    if len(parts) >= 2 and parts[0].upper() == "REPEAT":
        body = line[len(parts[0]):].strip()
        if body.endswith("{"):
            num = body[:-1].strip()
            if num.isdigit():
                return int(num)
    return None


def parse(text: str, prior_measurements: int = 0) -> Circuit:
    """Parse circuit text (`stabsim/circuit.py:179-211`)."""
    stack = [[]]
    open_counts = []
    lines = text.splitlines()
    for line_no, raw in enumerate(lines, start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if line == "}":
            if len(stack) == 1:
                raise CircuitParseError("unmatched '}'", line_no)
            body = stack.pop()
            stack[-1].append(Repeat(open_counts.pop(), Circuit(body)))
            continue
        count = _repeat_count(line)
        if count is not None:
            if count < 1:
                raise CircuitParseError("REPEAT count must be >= 1", line_no)
            open_counts.append(count)
            stack.append([])
            continue
        stack[-1].append(_parse_instruction(line, line_no))
    if len(stack) != 1:
        raise CircuitParseError("unclosed REPEAT block at end of input", len(lines))
    circuit = Circuit(stack[0])
    _validate_lookbacks(circuit, prior_measurements)
    return circuit


def _validate_lookbacks(circuit, measured_before: int) -> int:
    """Every lookback must resolve at its first execution
    (`stabsim/circuit.py:214-230`)."""
    count = measured_before
    for e in circuit.elements:
        if _is_repeat(e):
            _validate_lookbacks(e.body, count)
            count += e.num_measurements()
        elif e.gate.kind == ANNOTATION:
            for k in e.targets:
                if -k > count:
                    raise CircuitParseError(
                        f"lookback rec[{k}] reaches before the first measurement",
                        e.line)
        else:
            count += e.num_measurements()
    return count


def format_circuit(circuit, indent: int = 0) -> str:
    pad = " " * indent
    out = []
    for e in circuit.elements:
        if _is_repeat(e):
            out.append(f"{pad}REPEAT {e.count} {{")
            out.append(format_circuit(e.body, indent + 4))
            out.append(pad + "}")
        else:
            out.append(pad + str(e))
    return "\n".join(out)


def detector_sets(circuit) -> list:
    """Absolute record indices per DETECTOR, in order
    (`stabsim/circuit.py:247-256`)."""
    sets = []
    count = 0
    for instr in iter_flat(circuit):
        if instr.gate.kind == ANNOTATION:
            if instr.gate.name == "DETECTOR":
                sets.append(tuple(count + k for k in instr.targets))
        else:
            count += instr.num_measurements()
    return sets


def observable_sets(circuit) -> list:
    """Absolute record indices per observable index 0..K-1 (merged includes,
    XOR semantics: an index included twice cancels)."""
    obs: dict[int, dict[int, int]] = {}
    count = 0
    for instr in iter_flat(circuit):
        if instr.gate.kind == ANNOTATION:
            if instr.gate.name == "OBSERVABLE_INCLUDE":
                acc = obs.setdefault(int(instr.param), {})
                for k in instr.targets:
                    m = count + k
                    acc[m] = acc.get(m, 0) ^ 1
        else:
            count += instr.num_measurements()
    if not obs:
        return []
    out = []
    for i in range(max(obs) + 1):
        acc = obs.get(i, {})
        out.append(tuple(sorted(m for m, v in acc.items() if v)))
    return out


def detector_and_observable_sets(circuit) -> list:
    """Output columns of detection-event sampling: detectors, then observables
    (the order the reference sees after SURVEY.md Appendix C lowering)."""
    return detector_sets(circuit) + observable_sets(circuit)


def as_circuit(circuit_or_text) -> Circuit:
    """Accept superset text, our Circuit, or a reference `stabsim` Circuit."""
    if isinstance(circuit_or_text, Circuit):
        return circuit_or_text
    if isinstance(circuit_or_text, str):
        return parse(circuit_or_text)
    if hasattr(circuit_or_text, "elements"):
        # A reference Circuit (or any duck-typed equivalent): re-read through
        # its canonical text form so gate records come from our registry.
        return parse(format_circuit(circuit_or_text))
    raise TypeError(f"cannot interpret {type(circuit_or_text).__name__} as a circuit")


def to_reference_dialect(circuit) -> str:
    """Lower superset text to the reference dialect.

    TICK is dropped; SQRT_X -> H S H and SQRT_X_DAG -> H S_DAG H per target
    (same frame rule x ^= z, same tableau); OBSERVABLE_INCLUDE is removed and each observable becomes one
    trailing DETECTOR whose lookbacks are relative to the end of the circuit.
    """
    circuit = as_circuit(circuit)
    obs = observable_sets(circuit)
    total = circuit.num_measurements

    def lower(c, indent):
        pad = " " * indent
        out = []
        for e in c.elements:
            if _is_repeat(e):
                out.append(f"{pad}REPEAT {e.count} {{")
                out.extend(lower(e.body, indent + 4))
                out.append(pad + "}")
                continue
            name = e.gate.name
            if name in ("TICK", "OBSERVABLE_INCLUDE"):
                continue
            if name in ("SQRT_X", "SQRT_X_DAG"):
                mid = "S" if name == "SQRT_X" else "S_DAG"
                # per target, in order: a repeated target (SQRT_X 2 2) must
                # stay two sequential SQRT_X, which H 2 2 / S 2 2 / H 2 2 is not
                for t in e.targets:
                    out.append(f"{pad}H {t}")
                    out.append(f"{pad}{mid} {t}")
                    out.append(f"{pad}H {t}")
                continue
            assert name in REFERENCE_GATE_NAMES, name
            out.append(pad + str(e))
        return out

    lines = lower(circuit, 0)
    for i, s in enumerate(obs):
        if not s:
            raise ValueError(f"observable {i} includes no records; cannot lower")
        lines.append("DETECTOR " + " ".join(f"rec[{m - total}]" for m in s))
    return "\n".join(lines) + "\n"
