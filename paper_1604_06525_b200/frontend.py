"""Own plan-time front end: energy text -> "moplan v1" text for the device
solver, without the reference's C++ compiler.

Pipeline (the reference's stages, re-implemented; CPU plan-time work):

  parse      energy language -> statements / expression trees   (parser.hpp)
  lower      vector-valued expressions over a hash-consed scalar DAG, domain
             inference, computed arrays, excludes                (lower.hpp:65-560)
  derive     symbolic partials per unknown access, chain rule through
             cache-mode computed arrays                          (autodiff.hpp)
  transform  implicit bound guards, per-template partials and J p, gathered
             b / m / J^T J p kernels from shifted instances      (transform.hpp:202-262)
  plan       template sets per domain / graph, column layout, evalj lanes,
             computed and exclude kernels                        (plan.hpp:189-375)
  schedule   DAG -> guarded register programs (program.hpp:21-82 format)

The programs are semantically the reference's (same residuals, guards,
partials and gathered sums) but not instruction-for-instruction identical:
the canonical forms, operand orders and register numbering are this module's
own, so results agree with the reference to rounding (tests/test_frontend.py
checks every routine against the reference on the shipped energies through
the C oracle, and the device solver runs the plans unchanged).

Scheduling rule (the reference's guarded evaluation): an output is a sum of
terms; a term that is a product with boolean factors (InBounds, comparisons,
and/or/not) is evaluated inside a block guarded by their conjunction and
contributes through a guarded root, so an instance whose guard is false never
evaluates its (possibly non-finite) value.  select(c, t, 0) is the product
c * t; other selects evaluate both branches (strict, like the reference).
"""
import math
import re
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

from ._lib import MoError

# error codes: 1 + minopt::Err (common.hpp:13-32)
E_SYNTAX, E_UNDECL, E_ARITY, E_NONCONST_OFF, E_MIXED, E_NONCONST_EXP, E_DOMAIN, E_NONBOOL, E_CYCLIC = range(1, 10)
E_SHAPE, E_INDEX, E_GRAPH, E_INTERNAL = 10, 11, 14, 18


def _fail(code, msg):
    raise MoError(code, msg)


# ============================================================== lexer/parser
BUILTINS = {"select", "inbounds", "sqrt", "sin", "cos", "exp", "log", "abs", "atan", "pow", "dot", "vec", "index",
            "eq", "neq", "less", "leq", "greater", "geq", "and", "or", "not", "rotate2d", "rotate3d", "slice",
            "normalize"}
KEYWORDS = {"dim", "param", "unknown", "array", "graph", "computed", "energy", "exclude", "freeze", "cache"}


@dataclass
class Ast:
    kind: str  # num ident slot neg bin chan access call
    text: str = ""
    num: float = 0.0
    op: str = ""
    slot: str = ""
    channel: int = 0
    args: list = field(default_factory=list)
    line: int = 0


def _tokens(src):
    """(kind, text, line) tokens; '#' starts a comment to end of line."""
    out, i, line, n = [], 0, 1, len(src)
    while i < n:
        c = src[i]
        if c == "#":
            while i < n and src[i] != "\n":
                i += 1
            continue
        if c.isspace():
            line += c == "\n"
            i += 1
            continue
        if c.isalpha() or c == "_":
            j = i
            while j < n and (src[j].isalnum() or src[j] == "_"):
                j += 1
            out.append(("id", src[i:j], line))
            i = j
            continue
        if c.isdigit() or (c == "." and i + 1 < n and src[i + 1].isdigit()):
            j = i
            while j < n and (src[j].isdigit() or src[j] == "."):
                j += 1
            if j < n and src[j] in "eE":
                k = j + 1
                if k < n and src[k] in "+-":
                    k += 1
                if k < n and src[k].isdigit():
                    while k < n and src[k].isdigit():
                        k += 1
                    j = k
            try:
                float(src[i:j])
            except ValueError:
                _fail(E_SYNTAX, f"malformed number '{src[i:j]}' at line {line}")
            out.append(("num", src[i:j], line))
            i = j
            continue
        if c not in "()[],:=.+-*/":
            _fail(E_SYNTAX, f"unexpected character '{c}' at line {line}")
        out.append((c, c, line))
        i += 1
    out.append(("end", "", line))
    return out


class _Parser:
    def __init__(self, src):
        self.t = _tokens(src)
        self.i = 0

    def peek(self):
        return self.t[self.i]

    def take(self):
        t = self.t[self.i]
        self.i += 1
        return t

    def expect(self, kind, what):
        t = self.peek()
        if t[0] != kind:
            _fail(E_SYNTAX, f"expected {what} at line {t[2]}")
        return self.take()

    def name(self):
        t = self.expect("id", "name")
        if t[1] in KEYWORDS or t[1] in BUILTINS:
            _fail(E_SYNTAX, f"'{t[1]}' is reserved (line {t[2]})")
        return t[1]

    def program(self):
        stmts = []
        while self.peek()[0] != "end":
            head = self.expect("id", "statement keyword")
            s = {"kind": head[1], "line": head[2]}
            k = head[1]
            if k == "dim":
                s["name"] = self.name()
                n = self.expect("num", "dim extent")
                v = float(n[1])
                if v != int(v) or v < 1:
                    _fail(E_SYNTAX, f"dim extent must be a positive integer at line {n[2]}")
                s["extent"] = int(v)
            elif k == "param":
                s["name"] = self.name()
            elif k in ("unknown", "array"):
                s["name"] = self.name()
                self.expect("[", "'['")
                dims = [self.expect("id", "dim name")[1]]
                while self.peek()[0] == ",":
                    self.take()
                    dims.append(self.expect("id", "dim name")[1])
                self.expect("]", "']'")
                s["dims"], s["channels"] = dims, 1
                if self.peek()[0] == ":":
                    self.take()
                    n = self.expect("num", "channel count")
                    v = float(n[1])
                    if v != int(v) or v < 1:
                        _fail(E_SYNTAX, f"channel count must be a positive integer at line {n[2]}")
                    s["channels"] = int(v)
            elif k == "graph":
                s["name"] = self.name()
                self.expect("(", "'('")
                slots = [self.expect("id", "slot name")[1]]
                while self.peek()[0] == ",":
                    self.take()
                    slots.append(self.expect("id", "slot name")[1])
                self.expect(")", "')'")
                s["slots"] = slots
            elif k == "computed":
                s["name"] = self.name()
                mode = self.expect("id", "freeze|cache")
                if mode[1] not in ("freeze", "cache"):
                    _fail(E_SYNTAX, f"expected 'freeze' or 'cache' at line {mode[2]}")
                s["cache"] = mode[1] == "cache"
                self.expect("=", "'='")
                s["expr"] = self.expr()
            elif k in ("energy", "exclude"):
                s["expr"] = self.expr()
            else:
                _fail(E_SYNTAX, f"unknown statement '{k}' at line {head[2]}")
            stmts.append(s)
        return stmts

    def expr(self):
        lhs = self.term()
        while self.peek()[0] in ("+", "-"):
            op = self.take()
            lhs = Ast("bin", op=op[0], args=[lhs, self.term()], line=op[2])
        return lhs

    def term(self):
        lhs = self.unary()
        while self.peek()[0] in ("*", "/"):
            op = self.take()
            lhs = Ast("bin", op=op[0], args=[lhs, self.unary()], line=op[2])
        return lhs

    def unary(self):
        if self.peek()[0] == "-":
            t = self.take()
            return Ast("neg", args=[self.unary()], line=t[2])
        e = self.primary()
        while self.peek()[0] == "[":
            t = self.take()
            n = self.expect("num", "channel index")
            v = float(n[1])
            if v != int(v) or v < 0:
                _fail(E_SYNTAX, f"channel index must be a non-negative integer at line {n[2]}")
            self.expect("]", "']'")
            e = Ast("chan", channel=int(v), args=[e], line=t[2])
        return e

    def primary(self):
        t = self.peek()
        if t[0] == "num":
            self.take()
            return Ast("num", text=t[1], num=float(t[1]), line=t[2])
        if t[0] == "(":
            self.take()
            e = self.expr()
            self.expect(")", "')'")
            return e
        if t[0] == "id":
            self.take()
            if t[1] in KEYWORDS:
                _fail(E_SYNTAX, f"keyword '{t[1]}' used in expression at line {t[2]}")
            if self.peek()[0] == ".":
                self.take()
                slot = self.expect("id", "slot name")
                return Ast("slot", text=t[1], slot=slot[1], line=t[2])
            if self.peek()[0] == "(":
                self.take()
                node = Ast("call" if t[1] in BUILTINS else "access", text=t[1], line=t[2])
                if self.peek()[0] != ")":
                    node.args.append(self.expr())
                    while self.peek()[0] == ",":
                        self.take()
                        node.args.append(self.expr())
                self.expect(")", "')'")
                return node
            return Ast("ident", text=t[1], line=t[2])
        _fail(E_SYNTAX, f"unexpected token at line {t[2]}")


# ============================================================== scalar DAG
# Node tuple: (kind, a, b, kids) with
#   const: a = value | param: a = index | index: a = axis
#   U / A / C / P (unknown/array/computed/direction access): a = (field, ch), b = acc
#   acc = (graph, o0, o1, o2, slot)
#   sum / prod: kids | pow: a = (num, den), kids = (base,) | un: a = fn | cmp: a = op
#   and / or / not: kids | inb: b = acc | sel: kids = (c, t, f)
RANK = {k: i for i, k in enumerate(["const", "param", "index", "U", "A", "C", "P", "sum", "prod", "pow", "un", "cmp",
                                    "and", "or", "not", "inb", "sel"])}
UN = ["sqrt", "sin", "cos", "exp", "log", "abs", "atan"]
CMP = ["eq", "neq", "less", "leq", "greater", "geq"]
ORIGIN = (False, 0, 0, 0, 0)


def _pow_eval(x, num, den):
    def ipow(v, n):
        if n < 0:
            return 1.0 / ipow(v, -n) if ipow(v, -n) != 0 else math.copysign(math.inf, v) if v != 0 else math.inf
        r = 1.0
        while n > 0:
            if n & 1:
                r *= v
            v *= v
            n >>= 1
        return r
    try:
        if den == 1:
            return ipow(x, num) if -32 <= num <= 32 else math.pow(x, num)
        if den == 2:
            return ipow(math.sqrt(x), num)
        return math.pow(x, num / den)
    except (ValueError, OverflowError, ZeroDivisionError):
        return math.nan


class Dag:
    def __init__(self):
        self.nodes: List[tuple] = []
        self.ids: Dict[tuple, int] = {}
        self.boolean: List[bool] = []
        self.has_u: List[bool] = []

    def _intern(self, n):
        i = self.ids.get(n)
        if i is not None:
            return i
        i = len(self.nodes)
        self.nodes.append(n)
        self.ids[n] = i
        k = n[0]
        if k == "const":
            b = n[1] in (0.0, 1.0)
        elif k in ("cmp", "and", "or", "not", "inb"):
            b = True
        elif k == "prod":
            b = all(self.boolean[c] for c in n[3])
        elif k == "pow":
            b = self.boolean[n[3][0]] and n[1][0] > 0
        elif k == "sel":
            b = self.boolean[n[3][1]] and self.boolean[n[3][2]]
        else:
            b = False
        self.boolean.append(b)
        self.has_u.append(k in ("U", "C") or any(self.has_u[c] for c in n[3]))
        return i

    def kind(self, i):
        return self.nodes[i][0]

    def is_const(self, i, v=None):
        n = self.nodes[i]
        return n[0] == "const" and (v is None or n[1] == v or (isinstance(v, float) and math.isnan(v)
                                                                   and math.isnan(n[1])))

    def cval(self, i):
        return self.nodes[i][1]

    # ---- constructors (light canonical forms)
    def const(self, v):
        v = float(v)
        # (value, sign bit): 0.0 and -0.0 stay distinct nodes; NaN is its own
        # node per construction (like the reference's bit-pattern hash)
        return self._intern(("const", v, math.copysign(1.0, v) < 0, ()))

    def param(self, i):
        return self._intern(("param", i, None, ()))

    def index(self, ax):
        return self._intern(("index", ax, None, ()))

    def access(self, kind, f, ch, acc):
        return self._intern((kind, (f, ch), acc, ()))

    def _order(self, kids):
        return tuple(sorted(kids, key=lambda k: (RANK[self.nodes[k][0]], k)))

    def sum(self, kids):
        flat = []
        for k in kids:
            flat.extend(self.nodes[k][3] if self.kind(k) == "sum" else (k,))
        consts = [self.cval(k) for k in flat if self.kind(k) == "const"]
        rest = [k for k in flat if self.kind(k) != "const"]
        if consts:
            c = math.fsum(consts) if all(math.isfinite(x) for x in consts) else sum(consts)
            if c != 0 or not rest:
                rest.append(self.const(c))
        if not rest:
            return self.const(0)
        if len(rest) == 1:
            return rest[0]
        return self._intern(("sum", None, None, self._order(rest)))

    def product(self, kids):
        flat = []
        for k in kids:
            flat.extend(self.nodes[k][3] if self.kind(k) == "prod" else (k,))
        c = 1.0
        rest = []
        for k in flat:
            if self.kind(k) == "const":
                c *= self.cval(k)
            else:
                rest.append(k)
        if c == 0:
            return self.const(0)
        if not rest:
            return self.const(c)
        if c != 1:
            rest.append(self.const(c))
        if len(rest) == 1:
            return rest[0]
        return self._intern(("prod", None, None, self._order(rest)))

    def pow(self, base, num, den=1):
        g = math.gcd(num, den)
        num, den = num // g, den // g
        if den < 0:
            num, den = -num, -den
        if num == 0:
            return self.const(1)
        if num == 1 and den == 1:
            return base
        if self.is_const(base):
            return self.const(_pow_eval(self.cval(base), num, den))
        return self._intern(("pow", (num, den), None, (base,)))

    def unary(self, fn, a):
        if self.is_const(a):
            x = self.cval(a)
            f = {"sqrt": math.sqrt, "sin": math.sin, "cos": math.cos, "exp": math.exp, "log": math.log,
                 "abs": abs, "atan": math.atan}[fn]
            try:
                return self.const(f(x))
            except (ValueError, OverflowError):
                return self.const(math.nan if fn != "log" or x != 0 else -math.inf)
        return self._intern(("un", fn, None, (a,)))

    def compare(self, op, a, b):
        if self.is_const(a) and self.is_const(b):
            x, y = self.cval(a), self.cval(b)
            r = {"eq": x == y, "neq": x != y, "less": x < y, "leq": x <= y, "greater": x > y, "geq": x >= y}[op]
            return self.const(1 if r else 0)
        return self._intern(("cmp", op, None, (a, b)))

    def logical(self, fn, kids):
        for k in kids:
            if not self.boolean[k]:
                _fail(E_NONBOOL, "logical op on non-boolean operand")
        if fn == "not":
            if len(kids) != 1:
                _fail(E_ARITY, "not() takes one argument")
            a = kids[0]
            if self.is_const(a):
                return self.const(1 if self.cval(a) == 0 else 0)
            if self.kind(a) == "not":
                return self.nodes[a][3][0]
            return self._intern(("not", None, None, (a,)))
        flat = []
        for k in kids:
            flat.extend(self.nodes[k][3] if self.kind(k) == fn else (k,))
        rest = []
        for k in flat:
            if self.is_const(k):
                v = self.cval(k) != 0
                if fn == "and" and not v:
                    return self.const(0)
                if fn == "or" and v:
                    return self.const(1)
                continue
            if k not in rest:
                rest.append(k)
        if not rest:
            return self.const(1 if fn == "and" else 0)
        if len(rest) == 1:
            return rest[0]
        return self._intern((fn, None, None, self._order(rest)))

    def inbounds(self, acc):
        if acc[0]:
            _fail(E_GRAPH, "inbounds() is a stencil construct")
        if acc[1:4] == (0, 0, 0):
            return self.const(1)
        return self._intern(("inb", None, acc, ()))

    def select(self, c, t, f):
        if not self.boolean[c]:
            _fail(E_NONBOOL, "select condition must be boolean")
        if self.is_const(c):
            return t if self.cval(c) != 0 else f
        if t == f:
            return t
        if self.is_const(f, 0.0):  # select(c, t, 0) == c * t, evaluated as a guarded term
            return self.product([c, t])
        return self._intern(("sel", None, None, (c, t, f)))

    def add(self, a, b):
        return self.sum([a, b])

    def mul(self, a, b):
        return self.product([a, b])

    def neg(self, a):
        return self.product([self.const(-1), a])

    def sub(self, a, b):
        return self.sum([a, self.neg(b)])

    def div(self, a, b):
        return self.product([a, self.pow(b, -1)])

    def rebuild(self, n, kids):
        k = n[0]
        if k == "sum":
            return self.sum(kids)
        if k == "prod":
            return self.product(kids)
        if k == "pow":
            return self.pow(kids[0], *n[1])
        if k == "un":
            return self.unary(n[1], kids[0])
        if k == "cmp":
            return self.compare(n[1], kids[0], kids[1])
        if k in ("and", "or", "not"):
            return self.logical(k, list(kids))
        if k == "sel":
            return self.select(*kids)
        _fail(E_INTERNAL, "rebuild of a leaf")


# ============================================================== problem spec
@dataclass
class Field:
    name: str
    dom: Tuple[int, ...]
    channels: int


@dataclass
class Computed:
    name: str
    cache: bool
    dom: Tuple[int, ...]
    value: List[int]
    partials: list = field(default_factory=list)  # (channel, ufield, uchannel, off, expr, store_channel)

    def total_channels(self):
        return len(self.value) + len(self.partials)


@dataclass
class Spec:
    dag: Dag = field(default_factory=Dag)
    dims: List[Tuple[str, int]] = field(default_factory=list)
    params: List[str] = field(default_factory=list)
    unknowns: List[Field] = field(default_factory=list)
    arrays: List[Field] = field(default_factory=list)
    computed: List[Computed] = field(default_factory=list)
    graphs: List[Tuple[str, List[str]]] = field(default_factory=list)
    energies: list = field(default_factory=list)  # (kind 'grid'|'graph', dom or graph, expr)
    excludes: list = field(default_factory=list)  # [dom, pred]

    def shape(self, dom):
        return [self.dims[d][1] for d in dom]

    def extent(self, dom):
        n = 1
        for d in dom:
            n *= self.dims[d][1]
        return n


def _text_to_rat(text):
    m = re.fullmatch(r"(\d*)(?:\.(\d*))?(?:[eE]([+-]?\d+))?", text)
    if not m or not (m.group(1) or m.group(2)):
        return None
    digits = (m.group(1) or "") + (m.group(2) or "")
    net = int(m.group(3) or 0) - len(m.group(2) or "")
    if abs(net) > 18 or len(digits.lstrip("0")) > 17:
        return None
    num = int(digits or "0")
    return (num * 10 ** net, 1) if net >= 0 else (num, 10 ** -net)


class _Lower:
    def __init__(self):
        self.s = Spec()
        self.names = {}

    def declare(self, name, kind, idx, line):
        if name in self.names:
            _fail(E_SYNTAX, f"'{name}' redeclared at line {line}")
        self.names[name] = (kind, idx)

    def run(self, stmts):
        s = self.s
        for st in stmts:
            k = st["kind"]
            if k == "dim":
                self.declare(st["name"], "dim", len(s.dims), st["line"])
                s.dims.append((st["name"], st["extent"]))
            elif k == "param":
                self.declare(st["name"], "param", len(s.params), st["line"])
                s.params.append(st["name"])
            elif k in ("unknown", "array"):
                lst = s.unknowns if k == "unknown" else s.arrays
                self.declare(st["name"], k, len(lst), st["line"])
                lst.append(Field(st["name"], self.domain(st), st["channels"]))
            elif k == "graph":
                self.declare(st["name"], "graph", len(s.graphs), st["line"])
                s.graphs.append((st["name"], st["slots"]))
            elif k == "computed":
                self.computed(st)
            elif k == "energy":
                self.energy(st)
            elif k == "exclude":
                self.exclude(st)
        return s

    def domain(self, st):
        if not 1 <= len(st["dims"]) <= 3:
            _fail(E_SYNTAX, f"fields take 1 to 3 dims (line {st['line']})")
        out = []
        for dn in st["dims"]:
            k = self.names.get(dn)
            if not k or k[0] != "dim":
                _fail(E_UNDECL, f"'{dn}' is not a declared dim (line {st['line']})")
            out.append(k[1])
        return tuple(out)

    # ---- expressions: lists of scalar node ids (vector values)
    def const_int(self, e, code, what):
        if e.kind == "num":
            v = e.num
        elif e.kind == "neg" and e.args[0].kind == "num":
            v = -e.args[0].num
        else:
            _fail(code, f"{what} must be an integer literal at line {e.line}")
        if v != int(v):
            _fail(code, f"{what} must be an integer at line {e.line}")
        return int(v)

    def bcast(self, x, y, e):
        if len(x) == len(y):
            return x, y
        if len(x) == 1:
            return x * len(y), y
        if len(y) == 1:
            return x, y * len(x)
        _fail(E_SHAPE, f"operand widths {len(x)} and {len(y)} do not match at line {e.line}")

    def ex(self, e, cx):
        d = self.s.dag
        k = e.kind
        if k == "num":
            return [d.const(e.num)]
        if k == "ident":
            n = self.names.get(e.text)
            if not n:
                _fail(E_UNDECL, f"'{e.text}' at line {e.line}")
            if n[0] != "param":
                _fail(E_ARITY, f"'{e.text}' must be accessed with (...) at line {e.line}")
            return [d.param(n[1])]
        if k == "slot":
            _fail(E_SYNTAX, f"graph slot reference only valid as an access argument at line {e.line}")
        if k == "neg":
            return [d.neg(c) for c in self.ex(e.args[0], cx)]
        if k == "bin":
            x, y = self.bcast(self.ex(e.args[0], cx), self.ex(e.args[1], cx), e)
            f = {"+": d.add, "-": d.sub, "*": d.mul, "/": d.div}[e.op]
            return [f(a, b) for a, b in zip(x, y)]
        if k == "chan":
            v = self.ex(e.args[0], cx)
            if not 0 <= e.channel < len(v):
                _fail(E_INDEX, f"channel {e.channel} of width-{len(v)} value at line {e.line}")
            return [v[e.channel]]
        if k == "access":
            return self.access(e, cx)
        return self.call(e, cx)

    def access(self, e, cx):
        s, d = self.s, self.s.dag
        n = self.names.get(e.text)
        if not n:
            if cx.get("self") == e.text:
                _fail(E_CYCLIC, f"'{e.text}' refers to itself at line {e.line}")
            _fail(E_UNDECL, f"'{e.text}' at line {e.line}")
        kind, idx = n
        if kind not in ("unknown", "array", "computed"):
            _fail(E_ARITY, f"'{e.text}' is not an accessible field at line {e.line}")
        fld = s.unknowns[idx] if kind == "unknown" else s.arrays[idx] if kind == "array" else s.computed[idx]
        channels = fld.channels if kind != "computed" else len(fld.value)
        if len(e.args) == 1 and e.args[0].kind == "slot":
            sr = e.args[0]
            if not cx["slots"]:
                _fail(E_GRAPH, f"graph slot access is not allowed in this context at line {e.line}")
            g = self.names.get(sr.text)
            if not g or g[0] != "graph":
                _fail(E_UNDECL, f"'{sr.text}' is not a declared graph at line {e.line}")
            if cx["graph"] >= 0 and cx["graph"] != g[1]:
                _fail(E_MIXED, f"energy mixes hyperedges of two graphs at line {e.line}")
            cx["graph"] = g[1]
            slots = s.graphs[g[1]][1]
            if sr.slot not in slots:
                _fail(E_UNDECL, f"graph '{sr.text}' has no slot '{sr.slot}' at line {e.line}")
            if len(fld.dom) != 1:
                _fail(E_GRAPH, f"'{e.text}' must be declared over one dim to be graph-indexed at line {e.line}")
            acc = (True, 0, 0, 0, slots.index(sr.slot))
        else:
            if len(e.args) != len(fld.dom):
                _fail(E_ARITY, f"'{e.text}' takes {len(fld.dom)} offsets, got {len(e.args)} at line {e.line}")
            off = [0, 0, 0]
            for i, a in enumerate(e.args):
                o = self.const_int(a, E_NONCONST_OFF, "stencil offset")
                if not -32768 < o < 32768:
                    _fail(E_NONCONST_OFF, f"offset too large at line {e.line}")
                off[i] = o
            acc = (False, off[0], off[1], off[2], 0)
        tag = {"unknown": "U", "array": "A", "computed": "C"}[kind]
        return [d.access(tag, idx, ch, acc) for ch in range(channels)]

    def call(self, e, cx):
        d, f, a = self.s.dag, e.text, e.args

        def arity(n):
            if len(a) != n:
                _fail(E_ARITY, f"{f}() takes {n} arguments at line {e.line}")

        if f in UN:
            arity(1)
            return [d.unary(f, c) for c in self.ex(a[0], cx)]
        if f == "pow":
            arity(2)
            neg = a[1].kind == "neg"
            lit = a[1].args[0] if neg else a[1]
            q = _text_to_rat(lit.text) if lit.kind == "num" else None
            if q is None:
                _fail(E_NONCONST_EXP, f"pow exponent must be a numeric literal at line {e.line}")
            num, den = (-q[0], q[1]) if neg else q
            return [d.pow(c, num, den) for c in self.ex(a[0], cx)]
        if f == "select":
            arity(3)
            c = self.ex(a[0], cx)
            t, fv = self.bcast(self.ex(a[1], cx), self.ex(a[2], cx), e)
            if len(c) != len(t):
                if len(c) != 1:
                    _fail(E_SHAPE, f"select condition width mismatch at line {e.line}")
                c = c * len(t)
            return [d.select(ci, ti, fi) for ci, ti, fi in zip(c, t, fv)]
        if f == "inbounds":
            if not 1 <= len(a) <= 3:
                _fail(E_ARITY, f"inbounds() takes 1 to 3 offsets at line {e.line}")
            off = [0, 0, 0]
            for i, x in enumerate(a):
                off[i] = self.const_int(x, E_NONCONST_OFF, "inbounds offset")
            return [d.inbounds((False, off[0], off[1], off[2], 0))]
        if f == "index":
            arity(1)
            ax = self.const_int(a[0], E_NONCONST_OFF, "index axis")
            if not 0 <= ax < 3:
                _fail(E_INDEX, f"index axis out of range at line {e.line}")
            return [d.index(ax)]
        if f == "dot":
            arity(2)
            x, y = self.ex(a[0], cx), self.ex(a[1], cx)
            if len(x) != len(y):
                _fail(E_SHAPE, f"dot() width mismatch at line {e.line}")
            return [d.sum([d.mul(p, q) for p, q in zip(x, y)])]
        if f == "vec":
            if not a:
                _fail(E_ARITY, f"vec() needs arguments at line {e.line}")
            out = []
            for x in a:
                out += self.ex(x, cx)
            return out
        if f == "slice":
            arity(3)
            v = self.ex(a[0], cx)
            lo = self.const_int(a[1], E_INDEX, "slice bound")
            hi = self.const_int(a[2], E_INDEX, "slice bound")
            if not (0 <= lo < hi <= len(v)):
                _fail(E_INDEX, f"slice [{lo},{hi}) of width {len(v)} at line {e.line}")
            return v[lo:hi]
        if f == "normalize":
            arity(1)
            v = self.ex(a[0], cx)
            inv = d.pow(d.sum([d.mul(c, c) for c in v]), -1, 2)
            return [d.mul(c, inv) for c in v]
        if f in CMP:
            arity(2)
            x, y = self.bcast(self.ex(a[0], cx), self.ex(a[1], cx), e)
            return [d.compare(f, p, q) for p, q in zip(x, y)]
        if f in ("and", "or"):
            if len(a) < 2:
                _fail(E_ARITY, f"{f}() takes 2+ arguments at line {e.line}")
            vs = [self.ex(x, cx) for x in a]
            width = 1
            for v in vs:
                if len(v) != 1:
                    if width not in (1, len(v)):
                        _fail(E_SHAPE, f"{f}() width mismatch at line {e.line}")
                    width = len(v)
            return [d.logical(f, [v[0] if len(v) == 1 else v[i] for v in vs]) for i in range(width)]
        if f == "not":
            arity(1)
            return [d.logical("not", [c]) for c in self.ex(a[0], cx)]
        if f == "rotate2d":
            arity(2)
            ang = self.ex(a[0], cx)
            if len(ang) != 1:
                _fail(E_SHAPE, f"expected a scalar, got width {len(ang)} at line {e.line}")
            v = self.ex(a[1], cx)
            if len(v) != 2:
                _fail(E_SHAPE, f"rotate2d() expects a width-2 vector at line {e.line}")
            c, sn = d.unary("cos", ang[0]), d.unary("sin", ang[0])
            return [d.sub(d.mul(c, v[0]), d.mul(sn, v[1])), d.add(d.mul(sn, v[0]), d.mul(c, v[1]))]
        if f == "rotate3d":
            arity(2)
            ang, v = self.ex(a[0], cx), self.ex(a[1], cx)
            if len(ang) != 3 or len(v) != 3:
                _fail(E_SHAPE, f"rotate3d() expects width-3 angles and vector at line {e.line}")
            sa, ca = d.unary("sin", ang[0]), d.unary("cos", ang[0])
            sb, cb = d.unary("sin", ang[1]), d.unary("cos", ang[1])
            sc, cc = d.unary("sin", ang[2]), d.unary("cos", ang[2])
            m3 = lambda x, y, z: d.product([x, y, z])  # noqa: E731
            r = [[d.mul(cc, cb), d.sub(m3(cc, sb, sa), d.mul(sc, ca)), d.add(m3(cc, sb, ca), d.mul(sc, sa))],
                 [d.mul(sc, cb), d.add(m3(sc, sb, sa), d.mul(cc, ca)), d.sub(m3(sc, sb, ca), d.mul(cc, sa))],
                 [d.neg(sb), d.mul(cb, sa), d.mul(cb, ca)]]
            return [d.sum([d.mul(r[i][0], v[0]), d.mul(r[i][1], v[1]), d.mul(r[i][2], v[2])]) for i in range(3)]
        _fail(E_INTERNAL, f"unhandled builtin '{f}'")

    # ---- domain inference
    def scan(self, roots):
        s, d = self.s, self.s.dag
        out = {"slot": False, "index": False, "inb": False, "grids": []}
        seen, stack = set(), list(roots)
        while stack:
            i = stack.pop()
            if i in seen:
                continue
            seen.add(i)
            n = d.nodes[i]
            if n[0] in ("U", "A", "C"):
                if n[2][0]:
                    out["slot"] = True
                else:
                    f = n[1][0]
                    dom = (s.unknowns if n[0] == "U" else s.arrays if n[0] == "A" else s.computed)[f].dom
                    if dom not in out["grids"]:
                        out["grids"].append(dom)
            elif n[0] == "index":
                out["index"] = True
            elif n[0] == "inb":
                out["inb"] = True
            stack.extend(n[3])
        return out

    def computed(self, st):
        s, d = self.s, self.s.dag
        cx = {"slots": False, "graph": -1, "self": st["name"]}
        value = self.ex(st["expr"], cx)
        sc = self.scan(value)
        if not sc["grids"]:
            _fail(E_DOMAIN, f"cannot infer the domain of computed '{st['name']}' (line {st['line']})")
        if len(sc["grids"]) != 1:
            _fail(E_DOMAIN, f"computed '{st['name']}' reads fields of different domains (line {st['line']})")
        if sc["inb"]:
            _fail(E_GRAPH, f"inbounds() is not allowed in computed definitions (line {st['line']})")
        idx = len(s.computed)
        self.declare(st["name"], "computed", idx, st["line"])
        ca = Computed(st["name"], st["cache"], sc["grids"][0], value)
        s.computed.append(ca)
        if ca.cache:
            for ch, v in enumerate(value):
                for var in dependent_unknowns(s, v):
                    dv = derivative(s, v, var)
                    if d.is_const(dv, 0.0):
                        continue
                    n = d.nodes[var]
                    ca.partials.append((ch, n[1][0], n[1][1], n[2][1:4], dv, len(value) + len(ca.partials)))

    def energy(self, st):
        s = self.s
        cx = {"slots": True, "graph": -1}
        for root in self.ex(st["expr"], cx):
            sc = self.scan([root])
            if sc["slot"]:
                if sc["grids"]:
                    _fail(E_MIXED, f"energy mixes stencil and hyperedge accesses (line {st['line']})")
                if sc["index"] or sc["inb"]:
                    _fail(E_GRAPH, f"index()/inbounds() are stencil constructs (line {st['line']})")
                s.energies.append(("graph", cx["graph"], root))
            else:
                if not sc["grids"]:
                    _fail(E_DOMAIN, f"cannot infer the domain of an energy with no field accesses (line {st['line']})")
                if len(sc["grids"]) != 1:
                    _fail(E_DOMAIN, f"energy reads fields of different domains (line {st['line']})")
                s.energies.append(("grid", sc["grids"][0], root))

    def exclude(self, st):
        s, d = self.s, self.s.dag
        v = self.ex(st["expr"], {"slots": False, "graph": -1})
        if len(v) != 1:
            _fail(E_SHAPE, f"expected a scalar, got width {len(v)} at line {st['line']}")
        pred = v[0]
        if not d.boolean[pred]:
            _fail(E_NONBOOL, f"exclude predicate must be boolean (line {st['line']})")
        sc = self.scan([pred])
        if sc["grids"]:
            if len(sc["grids"]) != 1:
                _fail(E_DOMAIN, f"exclude predicate reads fields of different domains (line {st['line']})")
            dom = sc["grids"][0]
        else:
            if not s.unknowns:
                _fail(E_DOMAIN, f"exclude with no unknowns declared (line {st['line']})")
            dom = s.unknowns[0].dom
            if any(u.dom != dom for u in s.unknowns):
                _fail(E_DOMAIN, f"cannot infer the exclude domain (line {st['line']})")
        if not any(u.dom == dom for u in s.unknowns):
            _fail(E_DOMAIN, f"exclude domain matches no unknown field (line {st['line']})")
        for r in s.excludes:
            if r[0] == dom:
                r[1] = d.logical("or", [r[1], pred])
                return
        s.excludes.append([dom, pred])


def compile_source(text) -> Spec:
    """Parse and lower energy text (compile_source, lower.hpp:619)."""
    return _Lower().run(_Parser(text).program())


# ============================================================== derivatives
def _acc_key(dag, i):
    n = dag.nodes[i]
    return (n[1][0], n[1][1], n[2][0], n[2][4], n[2][1:4])


def unknown_accesses(spec, expr):
    dag = spec.dag
    found, seen, stack = set(), set(), [expr]
    while stack:
        i = stack.pop()
        if i in seen or not dag.has_u[i]:
            continue
        seen.add(i)
        if dag.kind(i) == "U":
            found.add(i)
        stack.extend(dag.nodes[i][3])
    return sorted(found, key=lambda i: _acc_key(dag, i))


def dependent_unknowns(spec, expr):
    """Syntactic unknown accesses plus the shifted accesses reached through
    cache-mode computed reads (autodiff.hpp:170-204), (field, channel, access)
    ordered."""
    dag = spec.dag
    found, seen, stack = set(), set(), [expr]
    while stack:
        i = stack.pop()
        if i in seen or not dag.has_u[i]:
            continue
        seen.add(i)
        n = dag.nodes[i]
        if n[0] == "U":
            found.add(i)
        if n[0] == "C" and not n[2][0]:
            ca = spec.computed[n[1][0]]
            if ca.cache:
                for (ch, uf, uc, off, _, _) in ca.partials:
                    if ch != n[1][1]:
                        continue
                    acc = (False, n[2][1] + off[0], n[2][2] + off[1], n[2][3] + off[2], 0)
                    found.add(dag.access("U", uf, uc, acc))
        stack.extend(n[3])
    return sorted(found, key=lambda i: _acc_key(dag, i))


def derivative(spec, expr, var, memo=None):
    """d expr / d var for one unknown access var (autodiff.hpp:18-124)."""
    dag = spec.dag
    memo = spec.__dict__.setdefault("_dmemo", {}) if memo is None else memo
    key = (expr, var)
    if key in memo:
        return memo[key]
    n = dag.nodes[expr]
    z = dag.const(0)
    if expr == var:
        d = dag.const(1)
    elif not dag.has_u[expr]:
        d = z
    else:
        k = n[0]
        if k == "U":
            d = z
        elif k == "C":
            v = dag.nodes[var]
            ca = spec.computed[n[1][0]]
            if not ca.cache or v[2][0] or n[2][0]:
                d = z
            else:
                terms = []
                for (ch, uf, uc, off, _, store) in ca.partials:
                    if ch != n[1][1] or uf != v[1][0] or uc != v[1][1]:
                        continue
                    if all(off[a] + n[2][1 + a] == v[2][1 + a] for a in range(3)):
                        terms.append(dag.access("C", n[1][0], store, n[2]))
                d = dag.sum(terms)
        elif k == "sum":
            d = dag.sum([x for x in (derivative(spec, c, var, memo) for c in n[3]) if not dag.is_const(x, 0.0)])
        elif k == "prod":
            terms = []
            for i, c in enumerate(n[3]):
                dc = derivative(spec, c, var, memo)
                if dag.is_const(dc, 0.0):
                    continue
                terms.append(dag.product([dc] + [o for j, o in enumerate(n[3]) if j != i]))
            d = dag.sum(terms)
        elif k == "pow":
            b = n[3][0]
            db = derivative(spec, b, var, memo)
            num, den = n[1]
            d = z if dag.is_const(db, 0.0) else dag.product([dag.const(num / den), dag.pow(b, num - den, den), db])
        elif k == "un":
            b = n[3][0]
            db = derivative(spec, b, var, memo)
            if dag.is_const(db, 0.0):
                d = z
            else:
                fn = n[1]
                if fn == "sqrt":
                    outer = dag.product([dag.const(0.5), dag.pow(b, -1, 2)])
                elif fn == "sin":
                    outer = dag.unary("cos", b)
                elif fn == "cos":
                    outer = dag.neg(dag.unary("sin", b))
                elif fn == "exp":
                    outer = expr
                elif fn == "log":
                    outer = dag.pow(b, -1)
                elif fn == "abs":  # sign(b) = (b > 0) - (b < 0)
                    outer = dag.sub(dag.compare("greater", b, z), dag.compare("less", b, z))
                else:  # atan
                    outer = dag.pow(dag.add(dag.const(1), dag.pow(b, 2)), -1)
                d = dag.mul(outer, db)
        elif k == "sel":
            c, t, f = n[3]
            d = dag.select(c, derivative(spec, t, var, memo), derivative(spec, f, var, memo))
        else:  # const / param / index / array / P / comparisons / logic / InBounds
            d = z
    memo[key] = d
    return d


# ============================================================== transform
def shift(dag, e, s, memo=None):
    """Value at q + s of e evaluated at q (transform.hpp:30-88)."""
    if s == (0, 0, 0):
        return e
    memo = {} if memo is None else memo
    if e in memo:
        return memo[e]
    n = dag.nodes[e]
    k = n[0]
    if k in ("U", "A", "C", "P", "inb"):
        acc = n[2]
        if acc[0]:
            out = e
        else:
            acc = (False, acc[1] + s[0], acc[2] + s[1], acc[3] + s[2], 0)
            out = dag.inbounds(acc) if k == "inb" else dag.access(k, n[1][0], n[1][1], acc)
    elif k == "index":
        out = e if s[n[1]] == 0 else dag.add(e, dag.const(s[n[1]]))
    elif not n[3]:
        out = e
    else:
        kids = [shift(dag, c, s, memo) for c in n[3]]
        out = e if all(a == b for a, b in zip(kids, n[3])) else dag.rebuild(n, kids)
    memo[e] = out
    return out


@dataclass
class Residual:
    kind: str
    dom: tuple = ()
    graph: int = -1
    residual: int = 0
    bound_guard: int = 0
    offsets: list = field(default_factory=list)
    partials: list = field(default_factory=list)  # (field, channel, acc, d)
    jp: int = 0


def _offsets(dag, e):
    out, seen, stack = set(), set(), [e]
    while stack:
        i = stack.pop()
        if i in seen:
            continue
        seen.add(i)
        n = dag.nodes[i]
        if n[0] in ("U", "A", "C") and not n[2][0]:
            out.add(n[2][1:4])
        stack.extend(n[3])
    return sorted(out)


def _guard(dag, offs, w):
    return [g for g in (dag.inbounds((False, v[0] - w[0], v[1] - w[1], v[2] - w[2], 0)) for v in offs)
            if not dag.is_const(g, 1.0)]


def transform(spec):
    """Residual templates and gathered normal-equation kernels
    (transform.hpp:202-262)."""
    dag = spec.dag
    res = []
    for kind, where, expr in spec.energies:
        t = Residual(kind)
        if kind == "grid":
            t.dom = where
            t.offsets = _offsets(dag, expr)
            ibs = _guard(dag, t.offsets, (0, 0, 0))
            t.bound_guard = dag.product(ibs)
            r = dag.product(ibs + [expr])
        else:
            t.graph = where
            t.bound_guard = dag.const(1)
            r = expr
        t.residual = r
        jp = []
        for var in dependent_unknowns(spec, r):
            dv = derivative(spec, r, var)
            if dag.is_const(dv, 0.0):
                continue
            n = dag.nodes[var]
            t.partials.append((n[1][0], n[1][1], n[2], dv))
            jp.append(dag.mul(dv, dag.access("P", n[1][0], n[1][1], n[2])))
        t.jp = dag.sum(jp)
        res.append(t)
    gather = []
    for fi, f in enumerate(spec.unknowns):
        for c in range(f.channels):
            bs, ms, js = [], [], []
            for t in res:
                if t.kind != "grid" or t.dom != f.dom:
                    continue
                for (pf, pc, acc, dv) in t.partials:
                    if pf != fi or pc != c or acc[0]:
                        continue
                    w = acc[1:4]
                    s = (-w[0], -w[1], -w[2])
                    g = _guard(dag, t.offsets, w)
                    memo = {}
                    bs.append(dag.product(g + [shift(dag, dag.mul(t.residual, dv), s, memo)]))
                    ms.append(dag.product(g + [shift(dag, dag.mul(dv, dv), s, memo)]))
                    js.append(dag.product(g + [shift(dag, dag.mul(dv, t.jp), s, memo)]))
            gather.append((fi, c, dag.mul(dag.const(-2), dag.sum(bs)), dag.mul(dag.const(2), dag.sum(ms)),
                           dag.mul(dag.const(2), dag.sum(js))))
    return res, gather


# ============================================================== scheduler
OP = {"imm": 0, "param": 1, "index": 2, "U": 3, "A": 4, "C": 5, "P": 6, "inb": 7, "add": 8, "mul": 9, "pow": 10,
      "un": 11, "cmp": 12, "and": 13, "or": 14, "not": 15, "sel": 16}


class Program:
    def __init__(self):
        self.instrs = []   # (op, sub, dst, a, b, c, gid, field, channel, acc, imm, pnum, pden)
        self.blocks = []   # (gid, begin, end)
        self.guard_regs = [0]
        self.outputs = []  # [(gid, reg), ...]
        self.num_regs = 0

    def text(self, name):
        lines = [f"program {name} {self.num_regs} {len(self.instrs)} {len(self.blocks)} {len(self.guard_regs)} "
                 f"{len(self.outputs)}"]
        for (op, sub, dst, a, b, c, gid, fld, ch, acc, imm, pn, pd) in self.instrs:
            lines.append(f"i {op} {sub} {dst} {a} {b} {c} {gid} {fld} {ch} {int(acc[0])} {acc[1]} {acc[2]} {acc[3]} "
                         f"{acc[4]} {float(imm).hex() if math.isfinite(imm) else _hexf(imm)} {pn} {pd}")
        lines += [f"b {g} {b} {e}" for g, b, e in self.blocks]
        lines += [f"g {r}" for r in self.guard_regs]
        lines += ["o " + " ".join([str(len(o))] + [f"{g} {r}" for g, r in o]) for o in self.outputs]
        return "\n".join(lines) + "\n"


def _hexf(v):
    return "inf" if v > 0 else "-inf" if v < 0 else "nan"


_POW2 = {float(2.0 ** k) for k in range(-60, 61)} | {-float(2.0 ** k) for k in range(-60, 61)}


class _Sched:
    """Guarded register-program emission of a set of output expressions."""

    def __init__(self, dag):
        self.dag = dag
        self.p = Program()
        self.val = {}       # (node, gid) -> register (gid 0: valid everywhere)
        self.gids = {}      # frozenset(cond nodes) -> gid
        self.cur = 0        # gid of the block being appended

    def reg(self):
        r = self.p.num_regs
        self.p.num_regs += 1
        return r

    def emit(self, op, sub=0, a=0, b=0, c=0, fld=0, ch=0, acc=ORIGIN, imm=0.0, pn=1, pd=1, dst=None):
        dst = self.reg() if dst is None else dst
        ins = self.p.instrs
        if not self.p.blocks or self.p.blocks[-1][0] != self.cur:
            self.p.blocks.append([self.cur, len(ins), len(ins)])
        ins.append((OP[op], sub, dst, a, b, c, self.cur, fld, ch, acc, imm, pn, pd))
        self.p.blocks[-1][2] = len(ins)
        return dst

    def value(self, i):
        """Register holding node i, computed in the current block (or earlier
        unconditionally)."""
        for g in (0, self.cur):
            r = self.val.get((i, g))
            if r is not None:
                return r
        dag, n = self.dag, self.dag.nodes[i]
        k = n[0]
        if k == "const":
            r = self.emit("imm", imm=n[1])
        elif k == "param":
            r = self.emit("param", fld=n[1])
        elif k == "index":
            r = self.emit("index", fld=n[1])
        elif k in ("U", "A", "C", "P"):
            r = self.emit(k, fld=n[1][0], ch=n[1][1], acc=n[2])
        elif k == "inb":
            r = self.emit("inb", acc=n[2])
        elif k in ("sum", "prod"):
            kids = [self.value(c) for c in n[3]]
            r = kids[0]
            for x in kids[1:]:
                r = self.emit("add" if k == "sum" else "mul", a=r, b=x)
        elif k == "pow":
            r = self.emit("pow", a=self.value(n[3][0]), pn=n[1][0], pd=n[1][1])
        elif k == "un":
            r = self.emit("un", sub=UN.index(n[1]), a=self.value(n[3][0]))
        elif k == "cmp":
            r = self.emit("cmp", sub=CMP.index(n[1]), a=self.value(n[3][0]), b=self.value(n[3][1]))
        elif k in ("and", "or"):
            kids = [self.value(c) for c in n[3]]
            r = kids[0]
            for x in kids[1:]:
                r = self.emit(k, a=r, b=x)
        elif k == "not":
            r = self.emit("not", a=self.value(n[3][0]))
        else:  # sel: strict (both branches)
            r = self.emit("sel", a=self.value(n[3][0]), b=self.value(n[3][1]), c=self.value(n[3][2]))
        self.val[(i, self.cur)] = r
        return r

    def guard(self, conds):
        """gid of the conjunction of boolean nodes `conds` (computed unguarded:
        reads never fault, out-of-bounds reads are 0)."""
        if not conds:
            return 0
        key = frozenset(conds)
        g = self.gids.get(key)
        if g is not None:
            return g
        save, self.cur = self.cur, 0
        regs = [self.value(c) for c in sorted(conds)]
        r = regs[0]
        for x in regs[1:]:
            r = self.emit("and", a=r, b=x)
        self.cur = save
        g = len(self.p.guard_regs)
        self.p.guard_regs.append(r)
        self.gids[key] = g
        return g

    def terms(self, i, conds=()):
        """Decompose node i into guarded terms [(conds, value node)]."""
        dag, n = self.dag, self.dag.nodes[i]
        if n[0] == "sum":
            out = []
            for c in n[3]:
                out += self.terms(c, conds)
            return out
        if n[0] == "prod":
            bools = [c for c in n[3] if dag.boolean[c] and not dag.is_const(c)]
            rest = [c for c in n[3] if c not in bools]
            if bools and rest:
                return self.terms(dag.product(rest), conds + tuple(bools))
            # a power-of-two factor distributes exactly over a sum
            consts = [c for c in rest if dag.is_const(c)]
            others = [c for c in rest if not dag.is_const(c)]
            if (len(consts) == 1 and len(others) == 1 and dag.kind(others[0]) == "sum"
                    and dag.cval(consts[0]) in _POW2):
                return [(cs, dag.mul(consts[0], v)) for cs, v in self.terms(others[0], conds)]
        if n[0] == "pow" and n[1][1] == 1 and n[1][0] > 0 and dag.kind(n[3][0]) == "prod":
            base = dag.nodes[n[3][0]]
            bools = [c for c in base[3] if dag.boolean[c] and not dag.is_const(c)]
            rest = [c for c in base[3] if c not in bools]
            if bools and rest:  # (g * v)^k == g * v^k for g in {0, 1}
                return self.terms(dag.pow(dag.product(rest), *n[1]), conds + tuple(bools))
        return [(conds, i)]

    def run(self, outputs):
        """Each output accumulates its guarded terms in order into one
        register (acc = acc + v inside the term's block; registers start at
        0), which is exactly run_program's Real(0) + sum of guarded roots
        (program.hpp:159-166) while keeping one value live per output."""
        for e in outputs:
            terms = [(c, v) for c, v in self.terms(e) if not self.dag.is_const(v, 0.0)]
            if len(terms) == 1 and not terms[0][0]:
                self.cur = 0
                self.p.outputs.append([(0, self.value(terms[0][1]))])
                continue
            acc = self.reg() if terms else None
            for conds, v in terms:
                g = self.guard(set(conds))
                self.cur = g
                self.emit("add", a=acc, b=self.value(v), dst=acc)
                self.cur = 0
            self.p.outputs.append([(0, acc)] if terms else [])
        self.p.blocks = [tuple(b) for b in self.p.blocks]
        return self.p


def schedule(dag, outputs) -> Program:
    return _Sched(dag).run(outputs)


# ============================================================== plan
def plan_text(spec: Spec, cfg=None, materialize=0, with_evalj=True) -> str:
    """The "moplan v1" text of a lowered problem (plan.hpp:189-375, the
    export format of integration/minopt_b200_bridge.hpp)."""
    from .solver import SolveConfig
    cfg = cfg or SolveConfig()
    dag = spec.dag
    res, gather = transform(spec)
    out = ["moplan 1"]
    rel = cfg.pcg_rel_tol
    if rel < 0:
        rel = 1e-4 if int(cfg.precision) == 0 else 1e-8
    vals = [int(cfg.method), int(cfg.precision), cfg.nonlinear_iters, cfg.linear_iters, rel, cfg.pcg_abs_tol,
            int(bool(cfg.use_preconditioner)), cfg.lm_radius0, cfg.lm_radius_min, cfg.lm_radius_max, cfg.lm_diag_min,
            cfg.lm_diag_max, cfg.lm_min_decrease, cfg.cost_stop_tol]
    out.append("cfg " + " ".join(float(v).hex() if isinstance(v, float) else str(v) for v in vals))
    if materialize:
        out.append(f"materialize {materialize}")
    dom = lambda d: " ".join([str(len(d))] + [str(x) for x in d])  # noqa: E731
    out.append(f"dims {len(spec.dims)}")
    out += [f"dim {n} {e}" for n, e in spec.dims]
    out.append(f"params {len(spec.params)}")
    out += [f"param {p}" for p in spec.params]
    out.append(f"unknowns {len(spec.unknowns)}")
    out += [f"unknown {u.name} {u.channels} {dom(u.dom)}" for u in spec.unknowns]
    out.append(f"arrays {len(spec.arrays)}")
    out += [f"array {a.name} {a.channels} {dom(a.dom)}" for a in spec.arrays]
    out.append(f"computed {len(spec.computed)}")
    out += [f"computed {c.name} {int(c.cache)} {c.total_channels()} {dom(c.dom)}" for c in spec.computed]
    out.append(f"graphs {len(spec.graphs)}")
    out += [f"graph {n} {len(s)}" for n, s in spec.graphs]
    out.append(f"residuals {len(res)}")
    out += [f"residual grid {dom(t.dom)}" if t.kind == "grid" else f"residual graph {t.graph}" for t in res]
    ubase, col = [], 0
    for u in spec.unknowns:
        ubase.append(col)
        col += spec.extent(u.dom) * u.channels
    out.append("ubase " + " ".join([str(len(ubase))] + [str(u) for u in ubase]))
    out.append(f"num_cols {col}")
    need_jtj = materialize == 0
    has_evalj = with_evalj or materialize != 0

    def prog(name, exprs):
        return schedule(dag, exprs).text(name).rstrip("\n")

    gsets = []
    for ti, t in enumerate(res):
        if t.kind != "grid":
            continue
        for gs in gsets:
            if gs[0] == t.dom:
                gs[1].append(ti)
                break
        else:
            gsets.append((t.dom, [ti]))
    out.append(f"grid_sets {len(gsets)}")
    for d, tmpl in gsets:
        out.append(f"grid_set {dom(d)} {len(tmpl)} " + " ".join(map(str, tmpl)))
        out.append(prog("cost", [dag.sum([dag.pow(res[t].residual, 2) for t in tmpl])]))
        out.append(prog("evalf", [res[t].residual for t in tmpl]))
        if has_evalj:
            jouts, jlines = [], []
            for t in tmpl:
                rt = res[t]
                g_out = len(jouts)
                jouts.append(rt.bound_guard)
                ps = sorted(rt.partials, key=lambda p: (p[0], p[2][1:4], p[1]))
                lanes = []
                for (pf, pc, acc, dv) in ps:
                    lanes.append(f"{len(jouts)} {pf} {pc} {acc[1]} {acc[2]} {acc[3]}")
                    jouts.append(dv)
                origin = 1 if (0, 0, 0) in rt.offsets else 0
                jlines.append(f"jtemplate {t} {g_out} {origin} {len(lanes)}" + "".join(" " + x for x in lanes))
            out.append(f"evalj {len(tmpl)}")
            out += jlines
            out.append(prog("evalj", jouts))
    gat = []
    for (fi, c, b, m, j) in gather:
        d = spec.unknowns[fi].dom
        for gs in gat:
            if gs[0] == d:
                gs[1].append((fi, c, b, m, j))
                break
        else:
            gat.append((d, [(fi, c, b, m, j)]))
    out.append(f"gather_sets {len(gat)}")
    for d, chans in gat:
        out.append(f"gather_set {dom(d)} {len(chans)} " + " ".join(f"{fi} {c}" for fi, c, *_ in chans))
        out.append(prog("bm", [x for (_, _, b, m, _) in chans for x in (b, m)]))
        out.append(prog("jtj", [j for (*_, j) in chans] if need_jtj else []))
    grs = []
    for ti, t in enumerate(res):
        if t.kind != "graph":
            continue
        for gs in grs:
            if gs[0] == t.graph:
                gs[1].append(ti)
                break
        else:
            grs.append((t.graph, [ti]))
    out.append(f"graph_sets {len(grs)}")
    for g, tmpl in grs:
        scats, bm, jtj, jouts, jlines = [], [], [], [], []
        for t in tmpl:
            rt = res[t]
            lanes = []
            for (pf, pc, acc, dv) in rt.partials:
                if not acc[0]:
                    _fail(E_INTERNAL, "graph residual with a stencil unknown access")
                scats.append(f"{acc[4]} {pf} {pc}")
                bm += [dag.mul(dag.const(-2), dag.mul(dv, rt.residual)), dag.mul(dag.const(2), dag.mul(dv, dv))]
                jtj.append(dag.mul(dag.const(2), dag.mul(dv, rt.jp)))
                lanes.append(f"{len(jouts)} {pf} {pc} {acc[4]}")
                jouts.append(dv)
            jlines.append(f"gjtemplate {t} {len(lanes)}" + "".join(" " + x for x in lanes))
        out.append(f"graph_set {g} {len(tmpl)} " + " ".join(map(str, tmpl)) + f" {len(scats)}" +
                   "".join(" " + s for s in scats))
        out.append(prog("cost", [dag.sum([dag.pow(res[t].residual, 2) for t in tmpl])]))
        out.append(prog("evalf", [res[t].residual for t in tmpl]))
        out.append(prog("bm", bm))
        out.append(prog("jtj", jtj if need_jtj else []))
        if has_evalj:
            out.append(f"gevalj {len(tmpl)}")
            out += jlines
            out.append(prog("evalj", jouts))
    out.append(f"computed_kernels {len(spec.computed)}")
    for i, ca in enumerate(spec.computed):
        out.append(f"computed_kernel {i} {dom(ca.dom)}")
        out.append(prog("prog", list(ca.value) + [p[4] for p in ca.partials]))
    out.append(f"exclude_kernels {len(spec.excludes)}")
    for d, pred in spec.excludes:
        out.append(f"exclude_kernel {dom(d)}")
        out.append(prog("prog", [pred]))
    out.append("end")
    return "\n".join(out) + "\n"


def plan_source(text, cfg=None, dims=None, materialize=0) -> str:
    """Energy text -> moplan text (compile_source + plan); `dims` overrides
    declared dim extents by name."""
    spec = compile_source(text)
    if dims:
        spec.dims = [(n, int(dims.get(n, e))) for n, e in spec.dims]
    return plan_text(spec, cfg, materialize)
