"""Seeded synthetic workloads of BASELINE.json configs C0-C4.

No public suite is involved: circuits are the SURVEY Appendix A grid random
circuits (ABCDCDAB coupler layers, random sqrt(X)/sqrt(Y)/sqrt(W) never
repeated on a qubit, fSim(pi/2, pi/6)), and the micro-benchmarks draw
complex Gaussian operands from ``numpy.random.default_rng``.
"""

from __future__ import annotations

import math
import random
from dataclasses import dataclass

import numpy as np

from .circuit import Circuit, circuit_to_network, open_output_order, parse_circuit
from .labels import Index

ONE_QUBIT = ("x_1_2", "y_1_2", "hz_1_2")
PATTERN = "ABCDCDAB"


def grid_layer(rows: int, cols: int, layer: str) -> list[tuple[int, int]]:
    """Coupler pairs of one layer: A/B horizontal (even/odd column start),
    C/D vertical (even/odd row start)."""
    q = lambda r, c: r * cols + c  # noqa: E731
    pairs = []
    if layer in "AB":
        start = 0 if layer == "A" else 1
        for r in range(rows):
            for c in range(start, cols - 1, 2):
                pairs.append((q(r, c), q(r, c + 1)))
    else:
        start = 0 if layer == "C" else 1
        for r in range(start, rows - 1, 2):
            for c in range(cols):
                pairs.append((q(r, c), q(r + 1, c)))
    return pairs


def grid_circuit_text(rows: int, cols: int, cycles: int, seed: int = 0,
                      theta: float = math.pi / 2, phi: float = math.pi / 6) -> str:
    rng = random.Random(seed)
    n = rows * cols
    last: list[str | None] = [None] * n
    lines = [str(n)]
    for k in range(cycles):
        for qb in range(n):
            g = rng.choice([x for x in ONE_QUBIT if x != last[qb]])
            last[qb] = g
            lines.append(f"{2 * k} {g} {qb}")
        for a, b in grid_layer(rows, cols, PATTERN[k % 8]):
            lines.append(f"{2 * k + 1} fs {a} {b} {theta:.17g} {phi:.17g}")
    return "\n".join(lines) + "\n"


@dataclass
class CircuitWorkload:
    rows: int
    cols: int
    cycles: int
    seed: int
    n_open: int

    @property
    def n_qubits(self) -> int:
        return self.rows * self.cols

    @property
    def open_qubits(self) -> list[int]:
        n = self.n_qubits
        return list(range(n - self.n_open, n))

    def circuit(self) -> Circuit:
        return parse_circuit(grid_circuit_text(self.rows, self.cols, self.cycles, self.seed))

    def network(self, bitstring: str | None = None):
        c = self.circuit()
        bits = bitstring if bitstring is not None else "0" * c.n_qubits
        return circuit_to_network(c, bits, open_qubits=self.open_qubits)

    def output_order(self) -> list[str]:
        return open_output_order(self.circuit(), self.open_qubits)


# BASELINE.json configs
C0 = CircuitWorkload(3, 4, 8, 0, 6)
C3 = CircuitWorkload(6, 6, 14, 0, 6)
C4 = CircuitWorkload(7, 7, 16, 0, 10)
C3_MAX_RANK = 30
C4_MAX_RANK = 32


def gaussian_c64(rng: np.random.Generator, size: int) -> np.ndarray:
    """complex64 with re, im i.i.d. N(0, 1/2)."""
    s = np.sqrt(0.5)
    out = np.empty(size, dtype=np.complex64)
    out.real = rng.standard_normal(size, dtype=np.float32) * s
    out.imag = rng.standard_normal(size, dtype=np.float32) * s
    return out


@dataclass
class PairCase:
    """One single-step micro-benchmark (config C1 a/b/c)."""

    name: str
    a_labels: list[str]
    b_labels: list[str]
    out_labels: list[str]
    seed: int

    def index_lists(self):
        return [Index(l) for l in self.a_labels], [Index(l) for l in self.b_labels], [Index(l) for l in self.out_labels]

    def data(self):
        rng = np.random.default_rng(self.seed)
        a = gaussian_c64(rng, 2 ** len(self.a_labels))
        b = gaussian_c64(rng, 2 ** len(self.b_labels))
        return a, b


def pair_case(name: str, n_free_a: int, n_common: int, n_free_b: int, seed: int) -> PairCase:
    """Shuffled labels: A = free_a + common, B = common + free_b, each shuffled;
    output = a seeded random permutation of free_a ++ free_b."""
    rng = np.random.default_rng(seed)
    fa = [f"a{i}" for i in range(n_free_a)]
    cm = [f"k{i}" for i in range(n_common)]
    fb = [f"b{i}" for i in range(n_free_b)]
    a = fa + cm
    b = cm + fb
    rng.shuffle(a)
    rng.shuffle(b)
    free = [l for l in a if l.startswith("a")] + [l for l in b if l.startswith("b")]
    out = list(free)
    rng.shuffle(out)
    return PairCase(name, a, b, out, seed + 1)


def c1_cases() -> list[PairCase]:
    """C1 a/b/c at BASELINE size: (22,6,4), (12,12,12), (7,20,7)."""
    return [pair_case("C1a", 22, 6, 4, 101), pair_case("C1b", 12, 12, 12, 102),
            pair_case("C1c", 7, 20, 7, 103)]


def small_pair_cases() -> list[PairCase]:
    """Oracle-sized variants with the same structure (golden fixtures)."""
    return [pair_case("C1a-small", 12, 6, 4, 111), pair_case("C1b-small", 7, 7, 7, 112),
            pair_case("C1c-small", 4, 12, 4, 113)]


def haar_unitary(rng: np.random.Generator, n: int) -> np.ndarray:
    z = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2)
    q, r = np.linalg.qr(z)
    d = np.diag(r)
    return q * (d / np.abs(d))


def fsim(theta: float, phi: float) -> np.ndarray:
    u = np.eye(4, dtype=complex)
    u[1, 1] = u[2, 2] = math.cos(theta)
    u[1, 2] = u[2, 1] = -1j * math.sin(theta)
    u[3, 3] = complex(math.cos(phi), -math.sin(phi))
    return u


@dataclass
class ChainCase:
    """Config C2: a rank-``rank`` tensor absorbing ``n_gates`` random gates."""

    rank: int
    n_gates: int
    seed: int

    def build(self):
        """Returns (t_labels, t_data c64, gates) with gates a list of
        (in_a, in_b, out_a, out_b, data c64[16] laid out (out_a,out_b,in_a,in_b))."""
        rng = np.random.default_rng(self.seed)
        t_labels = [f"w{i}" for i in range(self.rank)]
        data = gaussian_c64(rng, 2 ** self.rank)
        wire = list(t_labels)
        gates = []
        for g in range(self.n_gates):
            a, b = (int(x) for x in rng.choice(self.rank, 2, replace=False))
            theta = rng.uniform(0, math.pi / 2)
            phi = rng.uniform(0, math.pi)
            u = np.kron(haar_unitary(rng, 2), haar_unitary(rng, 2)) @ fsim(theta, phi)
            out_a, out_b = f"w{a}_{g + 1}", f"w{b}_{g + 1}"
            gates.append((wire[a], wire[b], out_a, out_b, u.reshape(-1).astype(np.complex64)))
            wire[a], wire[b] = out_a, out_b
        return t_labels, data, gates


C2 = ChainCase(30, 16, 202)
