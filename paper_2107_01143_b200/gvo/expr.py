"""Address-expression trees (drop-in for reference ``gvo.expr``, expr.py:1-425).

The node types, their fields and the exception classes match the
reference so trees, error handling and ``parse(render(t)) == t`` behave the
same.  The trees are host-side descriptors only; every bulk evaluation runs
on the GPU (``evaluate_bulk`` goes through the C ABI), and the hot path never
walks a tree: ``compile_postfix`` lowers each tree once into the bytecode the
device kernels interpret (include/gvo_b200.h, ``gvo_insn``).
"""

from __future__ import annotations

import re
from dataclasses import dataclass
from typing import Iterable, Mapping, Sequence

import numpy as np

INT64_MIN = -(1 << 63)
INT64_MAX = (1 << 63) - 1

COORD_NAMES = ("tidx", "tidy", "tidz", "bidx", "bidy", "bidz")
BLOCKDIM_NAMES = {"BX": 0, "BY": 1, "BZ": 2}
_BINARY = ("+", "-", "*", "//", "%")


class ExprError(ValueError):
    """Invalid expression construction or use (reference expr.py:27)."""


class ExprSyntaxError(ExprError):
    def __init__(self, message: str, position: int):
        super().__init__(f"{message} (at position {position})")
        self.position = position


class AddressOverflowError(ExprError):
    """A subexpression's value bounds leave int64 (reference expr.py:37)."""


def _in_int64(value: int, what: str) -> int:
    if value < INT64_MIN or value > INT64_MAX:
        raise AddressOverflowError(f"{what} {value} outside 64-bit signed range")
    return value


@dataclass(frozen=True)
class IntConstant:
    value: int

    def __post_init__(self):
        _in_int64(self.value, "constant")


@dataclass(frozen=True)
class CoordRef:
    name: str

    def __post_init__(self):
        if self.name not in COORD_NAMES:
            raise ExprError(f"unknown coordinate {self.name!r}")


@dataclass(frozen=True)
class BlockDimRef:
    name: str

    def __post_init__(self):
        if self.name not in BLOCKDIM_NAMES:
            raise ExprError(f"unknown block dimension {self.name!r}")


@dataclass(frozen=True)
class BaseRef:
    field: str


@dataclass(frozen=True)
class BinOp:
    op: str
    left: "AddressExpr"
    right: "AddressExpr"

    def __post_init__(self):
        if self.op not in _BINARY:
            raise ExprError(f"unknown operator {self.op!r}")
        if self.op in ("//", "%"):
            if not isinstance(self.right, IntConstant):
                raise ExprError(f"divisor of {self.op} must be an integer constant")
            if self.right.value <= 0:
                raise ExprError(f"divisor of {self.op} must be positive, got {self.right.value}")


AddressExpr = IntConstant | CoordRef | BlockDimRef | BaseRef | BinOp


def _apply(op: str, a, b):
    if op == "+":
        return a + b
    if op == "-":
        return a - b
    if op == "*":
        return a * b
    if op == "//":
        return a // b
    return a % b


def fold(op: str, left: AddressExpr, right: AddressExpr) -> AddressExpr:
    """BinOp with constant subtrees collapsed (reference expr.py:109-115)."""
    if type(left) is IntConstant and type(right) is IntConstant:
        if op in ("//", "%") and right.value <= 0:
            raise ExprError(f"divisor of {op} must be positive, got {right.value}")
        return IntConstant(_in_int64(_apply(op, left.value, right.value), "constant fold"))
    return BinOp(op, left, right)


def _postorder(expr: AddressExpr):
    """Iterative post-order walk (left subtree, right subtree, node)."""
    stack = [(expr, False)]
    while stack:
        node, seen = stack.pop()
        if type(node) is BinOp and not seen:
            stack.append((node, True))
            stack.append((node.right, False))
            stack.append((node.left, False))
        else:
            yield node


def base_refs(expr: AddressExpr) -> list[str]:
    return [n.field for n in _postorder(expr) if type(n) is BaseRef]


def value_bounds(
    expr: AddressExpr,
    coord_bounds: Mapping[str, tuple[int, int]],
    block_dim: Sequence[int],
    bases: Mapping[str, int],
) -> tuple[int, int]:
    """Exact inclusive interval of every node; AddressOverflowError when a
    BinOp node can leave int64 (reference expr.py:127-168).  Post-order
    evaluation checks nodes in the same order as the reference recursion."""
    vals: list[tuple[int, int]] = []
    for node in _postorder(expr):
        t = type(node)
        if t is IntConstant:
            vals.append((node.value, node.value))
        elif t is CoordRef:
            vals.append(tuple(coord_bounds[node.name]))
        elif t is BlockDimRef:
            v = int(block_dim[BLOCKDIM_NAMES[node.name]])
            vals.append((v, v))
        elif t is BaseRef:
            if node.field not in bases:
                raise ExprError(f"no base substitution for field {node.field!r}")
            v = int(bases[node.field])
            vals.append((v, v))
        else:
            rlo, rhi = vals.pop()
            llo, lhi = vals.pop()
            if node.op == "+":
                lo, hi = llo + rlo, lhi + rhi
            elif node.op == "-":
                lo, hi = llo - rhi, lhi - rlo
            elif node.op == "*":
                c = (llo * rlo, llo * rhi, lhi * rlo, lhi * rhi)
                lo, hi = min(c), max(c)
            elif node.op == "//":
                lo, hi = llo // rlo, lhi // rlo
            else:
                lo, hi = 0, rlo - 1
            _in_int64(lo, "subexpression bound")
            _in_int64(hi, "subexpression bound")
            vals.append((lo, hi))
    return vals[0]


def affine_parts(
    expr: AddressExpr, block_dim: Sequence[int], bases: Mapping[str, int]
) -> tuple[int, dict[str, int]] | None:
    """constant + {coordinate: coefficient}, or None for trees with // or %
    or products of two coordinate-dependent subtrees (reference
    expr.py:171-212; dictionary keys are syntactic, as there)."""
    vals: list = []
    for node in _postorder(expr):
        t = type(node)
        if t is IntConstant:
            vals.append((node.value, {}))
        elif t is CoordRef:
            vals.append((0, {node.name: 1}))
        elif t is BlockDimRef:
            vals.append((int(block_dim[BLOCKDIM_NAMES[node.name]]), {}))
        elif t is BaseRef:
            if node.field not in bases:
                raise ExprError(f"no base substitution for field {node.field!r}")
            vals.append((int(bases[node.field]), {}))
        else:
            r = vals.pop()
            l = vals.pop()
            if node.op in ("//", "%") or l is None or r is None:
                vals.append(None)
                continue
            (lc, ld), (rc, rd) = l, r
            if node.op in ("+", "-"):
                sign = 1 if node.op == "+" else -1
                d = dict(ld)
                for k, v in rd.items():
                    d[k] = d.get(k, 0) + sign * v
                vals.append((lc + sign * rc, d))
            elif not ld:
                vals.append((lc * rc, {k: lc * v for k, v in rd.items()}))
            elif not rd:
                vals.append((lc * rc, {k: rc * v for k, v in ld.items()}))
            else:
                vals.append(None)
    return vals[0]


@dataclass(frozen=True)
class ThreadCoord:
    tidx: int = 0
    tidy: int = 0
    tidz: int = 0
    bidx: int = 0
    bidy: int = 0
    bidz: int = 0

    def get(self, name: str) -> int:
        return getattr(self, name)


def _scalar(expr: AddressExpr, env: Mapping[str, int], block_dim, bases) -> int:
    vals: list[int] = []
    for node in _postorder(expr):
        t = type(node)
        if t is IntConstant:
            vals.append(node.value)
        elif t is CoordRef:
            vals.append(env[node.name])
        elif t is BlockDimRef:
            vals.append(int(block_dim[BLOCKDIM_NAMES[node.name]]))
        elif t is BaseRef:
            vals.append(int(bases[node.field]))
        else:
            r = vals.pop()
            vals.append(_apply(node.op, vals.pop(), r))
    return vals[0]


def evaluate(
    expr: AddressExpr,
    coords: Sequence[ThreadCoord],
    block_dim: Sequence[int],
    bases: Mapping[str, int],
) -> list[int]:
    """Scalar evaluation at a handful of coordinates (reference expr.py:235-264).

    Descriptor-level utility (one address at a time, exact Python ints);
    bulk evaluation goes to the GPU through ``evaluate_bulk``."""
    coords = list(coords)
    if not coords:
        return []
    bounds = {n: (min(c.get(n) for c in coords), max(c.get(n) for c in coords)) for n in COORD_NAMES}
    value_bounds(expr, bounds, block_dim, bases)
    return [_scalar(expr, {n: c.get(n) for n in COORD_NAMES}, block_dim, bases) for c in coords]


def evaluate_bulk(
    expr: AddressExpr,
    env: Mapping[str, np.ndarray],
    block_dim: Sequence[int],
    bases: Mapping[str, int],
) -> np.ndarray:
    """Vectorised evaluation over int64 coordinate arrays (reference
    expr.py:281-304), executed by the device bytecode interpreter."""
    arrays = [np.asarray(env[n], dtype=np.int64) for n in COORD_NAMES]
    if any(a.size == 0 for a in arrays):
        return np.empty(0, dtype=np.int64)
    bounds = {n: (int(a.min()), int(a.max())) for n, a in zip(COORD_NAMES, arrays)}
    value_bounds(expr, bounds, block_dim, bases)
    shape = arrays[0].shape
    coords = np.stack([np.broadcast_to(a, shape).ravel() for a in arrays], axis=1)
    from .. import _native

    return _native.eval_addresses(expr, bases, tuple(int(b) for b in block_dim), coords).reshape(shape)


# ---------------------------------------------------------------------------
# device bytecode (include/gvo_b200.h: gvo_opcode)

OP_CONST, OP_COORD, OP_BDIM, OP_BASE, OP_ADD, OP_SUB, OP_MUL, OP_FLOORDIV, OP_MOD = range(9)
_OPCODE = {"+": OP_ADD, "-": OP_SUB, "*": OP_MUL, "//": OP_FLOORDIV, "%": OP_MOD}


def compile_postfix(expr: AddressExpr, field_index: Mapping[str, int]) -> list[tuple[int, int]]:
    """Post-order (opcode, argument) program of a tree."""
    prog = []
    for node in _postorder(expr):
        t = type(node)
        if t is IntConstant:
            prog.append((OP_CONST, node.value))
        elif t is CoordRef:
            prog.append((OP_COORD, COORD_NAMES.index(node.name)))
        elif t is BlockDimRef:
            prog.append((OP_BDIM, BLOCKDIM_NAMES[node.name]))
        elif t is BaseRef:
            if node.field not in field_index:
                raise ExprError(f"no base substitution for field {node.field!r}")
            prog.append((OP_BASE, field_index[node.field]))
        else:
            prog.append((_OPCODE[node.op], 0))
    return prog


# ---------------------------------------------------------------------------
# text form

_TOKEN = re.compile(r"\s*(?:(?P<int>\d+)|(?P<ident>[A-Za-z_]\w*)|(?P<op>//|[-+*/%()]))")
_LEVEL = {"+": 1, "-": 1, "*": 2, "/": 2, "//": 2, "%": 2}


def _tokens(text: str) -> list[tuple[str, str, int]]:
    out = []
    pos = 0
    n = len(text)
    while pos < n:
        if text[pos].isspace():
            pos += 1
            continue
        m = _TOKEN.match(text, pos)
        if m is None or m.end() == pos:
            raise ExprSyntaxError(f"unexpected character {text[pos]!r}", pos)
        kind = m.lastgroup
        out.append((kind, m.group(kind), m.start(kind)))
        pos = m.end()
    out.append((None, "", n))
    return out


def parse(text: str, fields: Iterable[str] | None = None) -> AddressExpr:
    """Infix text -> tree (reference expr.py:311-407): precedence climbing
    with left associativity, ``/`` meaning floor division, unary minus,
    constant folding at every node, identifiers other than coordinates and
    BX/BY/BZ becoming field bases (restricted to ``fields`` if given)."""
    toks = _tokens(text)
    known = None if fields is None else set(fields)
    i = 0

    def atom() -> AddressExpr:
        nonlocal i
        kind, val, pos = toks[i]
        i += 1
        if kind == "int":
            return IntConstant(int(val))
        if kind == "ident":
            if val in COORD_NAMES:
                return CoordRef(val)
            if val in BLOCKDIM_NAMES:
                return BlockDimRef(val)
            if known is not None and val not in known:
                raise ExprSyntaxError(f"unknown identifier {val!r}", pos)
            return BaseRef(val)
        if kind == "op" and val == "(":
            node = climb(1)
            k2, v2, p2 = toks[i]
            if k2 != "op" or v2 != ")":
                raise ExprSyntaxError(f"expected ')', found {v2!r}" if k2 else "expected ')'", p2)
            i += 1
            return node
        tail = f", found {val!r}" if val else ""
        raise ExprSyntaxError("expected integer, identifier or '('" + tail, pos)

    def unary() -> AddressExpr:
        nonlocal i
        kind, val, _ = toks[i]
        if kind == "op" and val == "-":
            i += 1
            operand = unary()
            if type(operand) is IntConstant:
                return IntConstant(-operand.value)
            return fold("-", IntConstant(0), operand)
        return atom()

    def climb(level: int) -> AddressExpr:
        nonlocal i
        node = unary() if level == 2 else climb(2)
        while True:
            kind, val, _ = toks[i]
            if kind != "op" or _LEVEL.get(val) != level:
                return node
            i += 1
            rhs = unary() if level == 2 else climb(2)
            node = fold("//" if val == "/" else val, node, rhs)

    tree = climb(1)
    kind, val, pos = toks[i]
    if kind is not None:
        raise ExprSyntaxError(f"trailing input {val!r}", pos)
    return tree


def render(expr: AddressExpr) -> str:
    """Minimal-parenthesis infix text such that parse(render(e)) == e."""

    def text(node, outer: int, right_side: bool) -> str:
        t = type(node)
        if t is IntConstant:
            return str(node.value)
        if t is CoordRef or t is BlockDimRef:
            return node.name
        if t is BaseRef:
            return node.field
        lvl = _LEVEL[node.op]
        s = f"{text(node.left, lvl, False)} {node.op} {text(node.right, lvl, True)}"
        return f"({s})" if lvl < outer or (lvl == outer and right_side) else s

    return text(expr, 0, False)
