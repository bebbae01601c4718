"""Netlist generators for the BASELINE.json workloads beyond the reference's
four fixtures.

The reference ships only gen_adder / gen_mux_tree / gen_not_chain / gen_flat
(circuit.py:371-481); the paper synthesised its benchmarks with XLS + Yosys
(PAPER.md:411-426), which is not available.  These generators build the same
arithmetic directly from gates, in the reference's `Circuit` form, so they run
through `evaluate` unchanged and are checked against `simulate_plain`:

* config 2: `gen_adder(8)` (reference) + `gen_multiplier(8)` (8x8 -> 16 bit);
* config 3: `gen_dot_product(n, width)` -- sum_i a_i * b_i (paper: 500 x 16-bit);
* config 4: `gen_fc_layer(n_in, n_out, width)` -- y_o = sum_i w[o][i] * x_i
  (the paper's listing indexes w[j]; we use a full weight matrix);
* config 5: `gen_matmul_sigmoid(n, width)` -- C = A x B, then a bitwise
  piecewise-linear ("hard") sigmoid clamp(C/4 + 1/2) on every output (the
  paper's polynomial sigmoid is replaced).

Products use Baugh-Wooley signed partial products (w^2 AND/NAND gates per
w x w product plus one constant per sum) and every sum is reduced with 3:2
carry-save compression per bit column followed by a single ripple adder --
shallow, wide levels, which is the shape that keeps many gates per level.
"""
from __future__ import annotations

import numpy as np

from .cggi import GateKind
from .circuit import Circuit, Gate, Port

_K = GateKind
_CODE = {k: i for i, k in enumerate(GateKind)}  # scheduler._OPC order
_PAD = {0: (-1, -1, -1), 1: (-1, -1), 2: (-1,), 3: ()}


class NetBuilder:
    """Emits SSA gates; inputs claim the first wire ids."""

    def __init__(self):
        self.inputs: list[Port] = []
        self.outputs: list[Port] = []
        self.gates: list[Gate] = []
        self.nxt = 0
        self._const: dict[int, int] = {}
        # flat copies for the scheduler / plan compiler (scheduler.circuit_arrays)
        self._codes: list[int] = []
        self._ops: list[int] = []

    def add_input(self, name: str, width: int) -> list[int]:
        if self.gates:
            raise RuntimeError("declare inputs before gates")
        wires = list(range(self.nxt, self.nxt + width))
        self.nxt += width
        self.inputs.append(Port(name, tuple(wires)))
        return wires

    def add_output(self, name: str, wires) -> None:
        self.outputs.append(Port(name, tuple(wires)))

    def gate(self, op: GateKind, *ops: int) -> int:
        self.gates.append(Gate(self.nxt, op, tuple(ops)))
        self._codes.append(_CODE[op])
        self._ops.extend(ops + _PAD[len(ops)])
        self.nxt += 1
        return self.nxt - 1

    def const(self, bit: int) -> int:
        if bit not in self._const:
            self._const[bit] = self.gate(_K.CONST1 if bit else _K.CONST0)
        return self._const[bit]

    def build(self) -> Circuit:
        c = Circuit(inputs=tuple(self.inputs), outputs=tuple(self.outputs), gates=tuple(self.gates))
        G = len(self.gates)
        ids = np.fromiter((g.id for g in self.gates), dtype=np.int64, count=G)
        ops = np.asarray(self._ops, dtype=np.int64).reshape(G, 3)
        c.__dict__["_plan_arrays"] = (ids, np.asarray(self._codes, dtype=np.int32), ops,
                                      (ops >= 0).sum(axis=1).astype(np.int32))
        return c

    # -- bit-level blocks ------------------------------------------------------
    def full_add(self, a, b, c):
        t = self.gate(_K.XOR, a, b)
        s = self.gate(_K.XOR, t, c)
        cout = self.gate(_K.OR, self.gate(_K.AND, a, b), self.gate(_K.AND, t, c))
        return s, cout

    def ripple_add(self, a, b, width):
        """(a + b) mod 2^width; a, b little-endian lists, None = 0 bit."""
        out, carry = [], None
        for k in range(width):
            bits = [w for w in ((a[k] if k < len(a) else None), (b[k] if k < len(b) else None),
                                carry) if w is not None]
            if not bits:
                out.append(self.const(0))
                carry = None
            elif len(bits) == 1:
                out.append(bits[0])
                carry = None
            elif len(bits) == 2:
                out.append(self.gate(_K.XOR, *bits))
                carry = self.gate(_K.AND, *bits) if k + 1 < width else None
            else:
                s, carry = self.full_add(*bits)
                out.append(s)
        return out

    def column_sum(self, cols: list[list[int]], constant: int, width: int) -> list[int]:
        """sum over columns (cols[k] = wires of weight 2^k) + constant, mod 2^width:
        3:2 carry-save compression until <= 2 bits per column, then a ripple add."""
        cols = [list(c) for c in cols[:width]] + [[] for _ in range(width - len(cols))]
        constant %= 1 << width
        for k in range(width):
            if (constant >> k) & 1:
                cols[k].append(self.const(1))
        while any(len(c) > 2 for c in cols):
            new: list[list[int]] = [[] for _ in range(width)]
            for k in range(width):
                c = cols[k]
                i = 0
                while len(c) - i >= 3:
                    s, cy = self.full_add(c[i], c[i + 1], c[i + 2])
                    new[k].append(s)
                    if k + 1 < width:
                        new[k + 1].append(cy)
                    i += 3
                new[k].extend(c[i:])
            cols = new
        a = [c[0] if len(c) > 0 else None for c in cols]
        b = [c[1] if len(c) > 1 else None for c in cols]
        return self.ripple_add(a, b, width)

    def signed_product_bits(self, a, b, cols, width):
        """Add the Baugh-Wooley partial products of signed a*b into cols;
        returns the constant term (2^w - 2^(2w-1)) the caller must add once."""
        wa, wb = len(a), len(b)
        assert wa == wb, "equal operand widths"
        w = wa
        for i in range(w - 1):
            for j in range(w - 1):
                if i + j < width:
                    cols[i + j].append(self.gate(_K.AND, a[i], b[j]))
        if 2 * w - 2 < width:
            cols[2 * w - 2].append(self.gate(_K.AND, a[w - 1], b[w - 1]))
        for j in range(w - 1):
            if w - 1 + j < width:
                cols[w - 1 + j].append(self.gate(_K.NAND, a[w - 1], b[j]))
                cols[w - 1 + j].append(self.gate(_K.NAND, a[j], b[w - 1]))
        return (1 << w) - (1 << (2 * w - 1))

    def dot(self, xs, ys, width):
        cols: list[list[int]] = [[] for _ in range(width)]
        const = 0
        for x, y in zip(xs, ys):
            const += self.signed_product_bits(x, y, cols, width)
        return self.column_sum(cols, const, width)

    def mux_vec(self, sel, a, b):
        return [self.gate(_K.MUX, sel, x, y) for x, y in zip(a, b)]


def gen_multiplier(width: int = 8) -> Circuit:
    """Unsigned width x width -> 2*width bit product p = a * b (array of
    width^2 ANDs reduced by carry-save columns)."""
    nb = NetBuilder()
    a = nb.add_input("a", width)
    b = nb.add_input("b", width)
    W = 2 * width
    cols: list[list[int]] = [[] for _ in range(W)]
    for i in range(width):
        for j in range(width):
            cols[i + j].append(nb.gate(_K.AND, a[i], b[j]))
    nb.add_output("p", nb.column_sum(cols, 0, W))
    return nb.build()


def _acc_width(width, terms):
    return 2 * width + max(1, (terms - 1).bit_length())


def gen_dot_product(n: int = 500, width: int = 16, acc_width: int | None = None) -> Circuit:
    """y = sum_{i<n} a_i * b_i over signed width-bit inputs a0.., b0.. (two's
    complement), acc_width-bit result (default 2*width + ceil(log2 n))."""
    A = acc_width or _acc_width(width, n)
    nb = NetBuilder()
    a = [nb.add_input(f"a{i}", width) for i in range(n)]
    b = [nb.add_input(f"b{i}", width) for i in range(n)]
    nb.add_output("y", nb.dot(a, b, A))
    return nb.build()


def gen_fc_layer(n_in: int = 256, n_out: int = 30, width: int = 16,
                 acc_width: int | None = None) -> Circuit:
    """y_o = sum_i w{o}_{i} * x_i (signed), inputs x0.. then w{o}_{i}; outputs y0.."""
    A = acc_width or _acc_width(width, n_in)
    nb = NetBuilder()
    x = [nb.add_input(f"x{i}", width) for i in range(n_in)]
    w = [[nb.add_input(f"w{o}_{i}", width) for i in range(n_in)] for o in range(n_out)]
    for o in range(n_out):
        nb.add_output(f"y{o}", nb.dot(w[o], x, A))
    return nb.build()


def gen_matmul_sigmoid(n: int = 10, width: int = 16, frac: int | None = None,
                       acc_width: int | None = None) -> Circuit:
    """C = A x B (n x n, signed width-bit), then s_ij = hard_sigmoid(C_ij) with
    `frac` fractional output bits.  Inputs a{i}_{k}, b{k}_{j}; outputs s{i}_{j}."""
    A = acc_width or _acc_width(width, n)
    frac = frac or width
    nb = NetBuilder()
    a = [[nb.add_input(f"a{i}_{k}", width) for k in range(n)] for i in range(n)]
    b = [[nb.add_input(f"b{k}_{j}", width) for j in range(n)] for k in range(n)]
    for i in range(n):
        for j in range(n):
            c = nb.dot(a[i], [b[k][j] for k in range(n)], A)
            nb.add_output(f"s{i}_{j}", hard_sigmoid(nb, c, frac))
    return nb.build()


def hard_sigmoid(nb: NetBuilder, c: list[int], frac: int) -> list[int]:
    """clamp(c/4 + 2^(frac-1), 0, 2^frac - 1) for a w-bit two's-complement c
    (c read as fixed point with `frac` fractional bits: clamp(x/4 + 1/2, 0, 1))."""
    w = len(c)
    assert frac <= w - 3
    q = c[2:] + [c[-1]] * 2                                  # arithmetic c >> 2
    half = [None] * (frac - 1) + [nb.const(1)]
    y = nb.ripple_add(q, half, w)                            # no overflow: |c>>2| < 2^(w-3)
    neg = y[-1]
    hi = y[frac:w - 1]
    over = hi[0]
    for bit in hi[1:]:
        over = nb.gate(_K.OR, over, bit)
    big = nb.gate(_K.AND, nb.gate(_K.NOT, neg), over)       # y >= 2^frac
    ones = [nb.const(1)] * frac
    zeros = [nb.const(0)] * frac
    return nb.mux_vec(neg, zeros, nb.mux_vec(big, ones, y[:frac]))


def hard_sigmoid_plain(c: int, w: int, frac: int) -> int:
    """Integer model of hard_sigmoid for a w-bit pattern c."""
    c &= (1 << w) - 1
    cs = c - (1 << w) if c >> (w - 1) else c
    y = (cs >> 2) + (1 << (frac - 1))
    return 0 if y < 0 else min(y, (1 << frac) - 1)


def to_signed(v: int, w: int) -> int:
    v &= (1 << w) - 1
    return v - (1 << w) if v >> (w - 1) else v


def merge_circuits(parts) -> Circuit:
    """Independent circuits side by side in ONE netlist: `parts` is a sequence of
    (prefix, circuit); ports become "<prefix>_<name>", input wires are renumbered in
    declaration order (the text format's rule) and every gate gets a fresh id after
    all inputs.  A level scheduler then runs the circuits' level-k gates together
    (config 2: the adder and the multiplier in one evaluation)."""
    inputs, outputs, gates = [], [], []
    nxt = 0
    maps = []
    for prefix, c in parts:
        m = {}
        for p in c.inputs:
            new = tuple(range(nxt, nxt + p.width))
            nxt += p.width
            m.update(zip(p.wires, new))
            inputs.append(Port(f"{prefix}_{p.name}", new))
        maps.append(m)
    for (prefix, c), m in zip(parts, maps):
        for g in c.gates:
            m[g.id] = nxt
            nxt += 1
            gates.append(Gate(m[g.id], g.opcode, tuple(m[w] for w in g.operands)))
        for p in c.outputs:
            outputs.append(Port(f"{prefix}_{p.name}", tuple(m[w] for w in p.wires)))
    return Circuit(tuple(inputs), tuple(outputs), tuple(gates))
