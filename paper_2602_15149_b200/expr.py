"""User-expression language: parser (host) and bytecode compiler for the
device evaluator (``csrc/expr_vm.cuh``).

Grammar and semantics follow the reference expression module
(/root/reference/pkg/src/solidsph/expr.py):
  * variables x0 y0 z0 x y z ux uy uz t dt dx (expr.py:46);
  * functions sin cos tan cot sinh cosh tanh coth sqrt log(base 10) ln abs
    (arity 1), pow (2), if (3, lazy) (expr.py:48-56);
  * binary precedence or < and < comparisons < +,- < *,/ < ^ (right
    associative); unary minus sits between * and ^ (expr.py:58-68);
  * ``skip``/``Skip`` is legal only as the whole expression or an if-branch
    (expr.py:264-285);
  * ``<locals>`` are ``name=value;`` constant definitions folded at parse
    time (expr.py:208-232).
ASTs are the same immutable tuples the reference builds, so an ``ExprAst``
from either package can be compiled here.

Instead of walking the AST per particle on the host (the reference's masked
numpy evaluator, expr.py:419-551), ``compile_program`` lowers an AST to a
flat postfix program with conditional jumps; every particle lane runs it on
the device inside the integrator kernel.  Because ``skip`` can only sit in
tail position of an if-chain, it lowers to a terminating opcode.
"""

from __future__ import annotations

import math
import re
from dataclasses import dataclass

import numpy as np


class ExprError(ValueError):
    """Parse or evaluation error; carries the source offset when known."""

    def __init__(self, message, offset=None):
        if offset is not None:
            message = f"{message} (at offset {offset})"
        super().__init__(message)
        self.offset = offset


class _SkipType:
    _one = None

    def __new__(cls):
        if cls._one is None:
            cls._one = super().__new__(cls)
        return cls._one

    def __repr__(self):
        return "skip"


SKIP = _SkipType()

VARIABLES = ("x0", "y0", "z0", "x", "y", "z", "ux", "uy", "uz", "t", "dt", "dx")
ARITY = dict.fromkeys(("sin", "cos", "tan", "cot", "sinh", "cosh", "tanh",
                       "coth", "sqrt", "log", "ln", "abs"), 1)
ARITY.update({"pow": 2, "if": 3})

# binding power of each binary operator; ^ is the only right-associative one
_BP = {"or": 1, "and": 2, "<": 3, ">": 3, "<=": 3, ">=": 3, "==": 3, "!=": 3,
       "+": 4, "-": 4, "*": 5, "/": 5, "^": 6}
_NEG_BP = 5.5

_LEX = re.compile(r"""
    (?P<num>(?:\d+\.\d*|\.\d+|\d+)(?:[eE][+-]?\d+)?)
  | (?P<name>[A-Za-z_]\w*)
  | (?P<op><=|>=|==|!=|[-+*/^<>(),])
  | (?P<ws>\s+)
""", re.VERBOSE | re.ASCII)


def _lex(text):
    out, pos = [], 0
    while pos < len(text):
        m = _LEX.match(text, pos)
        if m is None:
            raise ExprError(f"unexpected character {text[pos]!r}", pos)
        if m.lastgroup != "ws":
            out.append((m.lastgroup, m.group(), pos))
        pos = m.end()
    out.append(("end", "", len(text)))
    return out


@dataclass(frozen=True)
class ExprAst:
    root: tuple
    locals: dict
    source: str

    @property
    def variables(self):
        return frozenset(_walk_vars(self.root))

    @property
    def time_dependent(self):
        """True when the value can change between steps (reference
        expr.py:117-119): anything reading x/y/z, u, t or dt."""
        return bool(self.variables & {"x", "y", "z", "ux", "uy", "uz",
                                      "t", "dt"})


def _walk_vars(node):
    tag = node[0]
    if tag == "var":
        yield node[1]
    elif tag == "un":
        yield from _walk_vars(node[2])
    elif tag == "bin":
        yield from _walk_vars(node[2])
        yield from _walk_vars(node[3])
    elif tag == "call":
        for arg in node[2]:
            yield from _walk_vars(arg)
    elif tag == "if":
        for sub in node[1:]:
            yield from _walk_vars(sub)


class _Pratt:
    def __init__(self, text, consts):
        self.toks = _lex(text)
        self.k = 0
        self.consts = consts

    def _peek(self):
        return self.toks[self.k]

    def _take(self):
        tok = self.toks[self.k]
        self.k += 1
        return tok

    def _need(self, text):
        kind, val, pos = self._peek()
        if val != text:
            shown = val or "end of input"
            raise ExprError(f"expected {text!r}, found {shown!r}", pos)
        return self._take()

    def whole(self):
        tree = self.expr(0)
        kind, val, pos = self._peek()
        if kind != "end":
            raise ExprError(f"unexpected trailing input {val!r}", pos)
        return tree

    def expr(self, floor):
        lhs = self.prefix()
        while True:
            kind, op, _ = self._peek()
            bp = _BP.get(op)
            if kind == "end" or bp is None or bp < floor:
                return lhs
            self._take()
            rhs = self.expr(bp if op == "^" else bp + 1)
            lhs = ("bin", op, lhs, rhs)

    def prefix(self):
        kind, val, pos = self._take()
        if kind == "num":
            return ("num", float(val))
        if val == "-":
            inner = self.expr(_NEG_BP)
            return ("num", -inner[1]) if inner[0] == "num" else ("un", "-", inner)
        if val == "(":
            inner = self.expr(0)
            self._need(")")
            return inner
        if kind == "name":
            if val in ("skip", "Skip"):
                return ("skip",)
            if val in ("and", "or"):
                raise ExprError(f"operator {val!r} missing left operand", pos)
            if self._peek()[1] == "(":
                return self.call(val, pos)
            if val in self.consts:
                return ("num", self.consts[val])
            if val in VARIABLES:
                return ("var", val)
            raise ExprError(f"unknown identifier {val!r}", pos)
        raise ExprError(f"unexpected token {val or 'end of input'!r}", pos)

    def call(self, name, pos):
        want = ARITY.get(name)
        if want is None:
            raise ExprError(f"unknown function {name!r}", pos)
        self._need("(")
        args = [self.expr(0)]
        while self._peek()[1] == ",":
            self._take()
            args.append(self.expr(0))
        self._need(")")
        if len(args) != want:
            raise ExprError(f"function {name!r} takes {want} argument(s), "
                            f"got {len(args)}", pos)
        if name == "if":
            return ("if", *args)
        return ("call", name, tuple(args))


def parse_locals(text, base=None):
    """Fold ``a=1; b=a*2`` into a name -> float map (expr.py:208-232)."""
    consts = dict(base or {})
    for piece in (text or "").split(";"):
        piece = piece.strip()
        if not piece:
            continue
        if "=" not in piece:
            raise ExprError(f"malformed local definition {piece!r}")
        name, _, rhs = piece.partition("=")
        name = name.strip()
        if not re.fullmatch(r"[A-Za-z_][A-Za-z0-9_]*", name):
            raise ExprError(f"invalid local name {name!r}")
        val = eval_node(_Pratt(rhs.strip(), consts).whole(), None)
        if val is SKIP:
            raise ExprError(f"local {name!r} must be a number, not skip")
        consts[name] = val
    return consts


def _skip_legal(node, tail):
    tag = node[0]
    if tag == "skip":
        if not tail:
            raise ExprError(
                "`skip` is only legal as an if branch or the whole expression")
    elif tag == "un":
        _skip_legal(node[2], False)
    elif tag == "bin":
        _skip_legal(node[2], False)
        _skip_legal(node[3], False)
    elif tag == "call":
        for arg in node[2]:
            _skip_legal(arg, False)
    elif tag == "if":
        _skip_legal(node[1], False)
        _skip_legal(node[2], tail)
        _skip_legal(node[3], tail)


def parse(source, locals_src=""):
    """Source (+ optional locals) -> ExprAst (reference expr.py:235-242)."""
    if not source or not source.strip():
        raise ExprError("empty expression")
    consts = parse_locals(locals_src)
    root = _Pratt(source, consts).whole()
    _skip_legal(root, True)
    return ExprAst(root=root, locals=consts, source=source)


# -- scalar evaluation (host; used to fold locals and for single lanes) -----

def _scalar_call(name, a):
    try:
        x = a[0]
        if name == "cot":
            return math.cos(x) / math.sin(x)
        if name == "coth":
            return math.cosh(x) / math.sinh(x)
        if name in ("log", "ln"):
            if x <= 0.0:
                raise ExprError(f"{name} of non-positive value {x!r}")
            return math.log10(x) if name == "log" else math.log(x)
        if name == "sqrt":
            if x < 0.0:
                raise ExprError(f"sqrt of negative value {x!r}")
            return math.sqrt(x)
        if name == "pow":
            return math.pow(x, a[1])
        return {"sin": math.sin, "cos": math.cos, "tan": math.tan,
                "sinh": math.sinh, "cosh": math.cosh, "tanh": math.tanh,
                "abs": abs}[name](x)
    except (ValueError, ZeroDivisionError, OverflowError) as exc:
        raise ExprError(f"domain error in {name}: {exc}") from None


_CMP = {"<": float.__lt__, ">": float.__gt__, "<=": float.__le__,
        ">=": float.__ge__, "==": float.__eq__, "!=": float.__ne__}


def eval_node(node, ctx):
    """Scalar evaluation of one AST node (reference expr.py:307-369)."""
    tag = node[0]
    if tag == "num":
        return node[1]
    if tag == "skip":
        return SKIP
    if tag == "var":
        if ctx is None:
            raise ExprError(f"variable {node[1]!r} not allowed here")
        return float(getattr(ctx, node[1]))
    if tag == "un":
        val = eval_node(node[2], ctx)
        if val is SKIP:
            raise ExprError("skip consumed by unary '-'")
        return -val
    if tag == "if":
        cond = eval_node(node[1], ctx)
        if cond is SKIP:
            raise ExprError("skip consumed by if condition")
        return eval_node(node[2] if cond != 0.0 else node[3], ctx)
    if tag == "call":
        args = [eval_node(a, ctx) for a in node[2]]
        if any(a is SKIP for a in args):
            raise ExprError(f"skip consumed by function {node[1]!r}")
        return _scalar_call(node[1], args)
    op = node[1]
    a = eval_node(node[2], ctx)
    b = eval_node(node[3], ctx)
    if a is SKIP or b is SKIP:
        raise ExprError(f"skip consumed by operator {op!r}")
    a, b = float(a), float(b)
    if op == "+":
        return a + b
    if op == "-":
        return a - b
    if op == "*":
        return a * b
    if op == "/":
        if b == 0.0:
            raise ExprError("division by zero")
        return a / b
    if op == "^":
        try:
            return math.pow(a, b)
        except (ValueError, OverflowError) as exc:
            raise ExprError(f"domain error in '^': {exc}") from None
    if op in _CMP:
        return 1.0 if _CMP[op](a, b) else 0.0
    if op == "and":
        return 1.0 if (a != 0.0 and b != 0.0) else 0.0
    if op == "or":
        return 1.0 if (a != 0.0 or b != 0.0) else 0.0
    raise ExprError(f"unknown operator {op!r}")


@dataclass
class EvalContext:
    x0: float = 0.0
    y0: float = 0.0
    z0: float = 0.0
    x: float = 0.0
    y: float = 0.0
    z: float = 0.0
    ux: float = 0.0
    uy: float = 0.0
    uz: float = 0.0
    t: float = 0.0
    dt: float = 0.0
    dx: float = 0.0


def eval_expr(ast, ctx):
    return eval_node(ast.root, ctx)


# -- bytecode for the device evaluator --------------------------------------
# One instruction = (opcode:int32, operand:int32).  Constants live in a
# per-program float64 pool.  Opcode numbering is shared with
# csrc/expr_vm.cuh (keep in sync; test_expr_compile checks the table).

OP = {
    "END": 0, "CONST": 1, "VAR": 2, "NEG": 3, "JZ": 4, "JMP": 5, "SKIP": 6,
    "ADD": 10, "SUB": 11, "MUL": 12, "DIV": 13, "POW": 14,
    "LT": 15, "GT": 16, "LE": 17, "GE": 18, "EQ": 19, "NE": 20,
    "AND": 21, "OR": 22,
    "SIN": 30, "COS": 31, "TAN": 32, "COT": 33, "SINH": 34, "COSH": 35,
    "TANH": 36, "COTH": 37, "SQRT": 38, "LOG": 39, "LN": 40, "ABS": 41,
    "POWF": 42,
}
_BIN_OP = {"+": "ADD", "-": "SUB", "*": "MUL", "/": "DIV", "^": "POW",
           "<": "LT", ">": "GT", "<=": "LE", ">=": "GE", "==": "EQ",
           "!=": "NE", "and": "AND", "or": "OR"}
VAR_ID = {name: k for k, name in enumerate(VARIABLES)}
# device error codes (ExprError messages the host re-raises)
ERRORS = {1: "division by zero", 2: "log of non-positive value",
          3: "ln of non-positive value", 4: "sqrt of negative value",
          5: "domain error in pow", 6: "domain error in '^'",
          7: "stack overflow in expression program"}
MAX_STACK = 16


@dataclass(frozen=True)
class Program:
    code: np.ndarray      # (m, 2) int32
    consts: np.ndarray    # (c,) float64
    depth: int            # max stack depth
    source: str


def compile_program(ast):
    """Lower an ExprAst (or raw root tuple) to postfix bytecode."""
    root = ast.root if isinstance(ast, ExprAst) else ast
    code, consts = [], []
    depth = [0, 0]   # current, max

    def push(n=1):
        depth[0] += n
        depth[1] = max(depth[1], depth[0])

    def emit(op, arg=0):
        code.append([OP[op], arg])
        return len(code) - 1

    def gen(node):
        tag = node[0]
        if tag == "num":
            consts.append(float(node[1]))
            emit("CONST", len(consts) - 1)
            push()
        elif tag == "var":
            emit("VAR", VAR_ID[node[1]])
            push()
        elif tag == "skip":
            emit("SKIP")
        elif tag == "un":
            gen(node[2])
            emit("NEG")
        elif tag == "bin":
            gen(node[2])
            gen(node[3])
            emit(_BIN_OP[node[1]])
            depth[0] -= 1
        elif tag == "call":
            for arg in node[2]:
                gen(arg)
            emit("POWF" if node[1] == "pow" else node[1].upper())
            depth[0] -= len(node[2]) - 1
        elif tag == "if":
            gen(node[1])
            jz = emit("JZ")
            depth[0] -= 1
            base = depth[0]
            gen(node[2])
            jmp = emit("JMP")
            depth[0] = base
            code[jz][1] = len(code)
            gen(node[3])
            code[jmp][1] = len(code)
        else:
            raise ExprError(f"unknown node {tag!r}")

    gen(root)
    emit("END")
    if depth[1] > MAX_STACK:
        raise ExprError(f"expression too deep for the device evaluator "
                        f"(stack {depth[1]} > {MAX_STACK})")
    src = ast.source if isinstance(ast, ExprAst) else ""
    return Program(code=np.asarray(code, dtype=np.int32).reshape(-1, 2),
                   consts=np.asarray(consts if consts else [0.0],
                                     dtype=np.float64),
                   depth=depth[1], source=src)


def pretty(ast_or_node):
    """Fully parenthesised text that reparses to the same AST."""
    node = ast_or_node.root if isinstance(ast_or_node, ExprAst) else ast_or_node
    tag = node[0]
    if tag == "num":
        return repr(node[1])
    if tag == "var":
        return node[1]
    if tag == "skip":
        return "skip"
    if tag == "un":
        return f"(-{pretty(node[2])})"
    if tag == "bin":
        return f"({pretty(node[2])} {node[1]} {pretty(node[3])})"
    if tag == "call":
        return f"{node[1]}({', '.join(pretty(a) for a in node[2])})"
    if tag == "if":
        return f"if({pretty(node[1])}, {pretty(node[2])}, {pretty(node[3])})"
    raise ExprError(f"unknown node {tag!r}")


# -- static skip patterns ---------------------------------------------------
# A whole-body boundary condition or a restrictphi expression is evaluated on
# every particle every step, but it usually selects a few particles by their
# reference coordinates (``if(x0<=0.0, 0.0, skip)``).  When every ``if`` on
# the way to a ``skip`` tests x0, y0, z0 and constants only, the particles
# where the expression is not skip are fixed: the device evaluates it on
# those alone (simulation.py DeviceBody._setup_bcs) with the same result.

STATIC_VARS = frozenset(("x0", "y0", "z0"))


class _NotStatic(Exception):
    pass


def _has_skip(node):
    tag = node[0]
    if tag == "skip":
        return True
    if tag == "if":
        return _has_skip(node[2]) or _has_skip(node[3])
    return False          # skip is only legal in if branches (_skip_legal)


def skip_static(ast):
    """True when whether ``ast`` evaluates to skip depends on x0, y0, z0
    (and constants) only."""
    def ok(node):
        if not _has_skip(node) or node[0] == "skip":
            return True
        return (frozenset(_walk_vars(node[1])) <= STATIC_VARS and ok(node[2]) and ok(node[3]))
    root = ast.root if isinstance(ast, ExprAst) else ast
    return ok(root)


_VFUN = {"sin": np.sin, "cos": np.cos, "tan": np.tan, "sinh": np.sinh, "cosh": np.cosh,
         "tanh": np.tanh, "abs": np.abs}
_VCMP = {"<": np.less, ">": np.greater, "<=": np.less_equal, ">=": np.greater_equal,
         "==": np.equal, "!=": np.not_equal}


def _veval(node, env):
    """Vectorised value of a skip-free static subexpression; any domain
    error makes the pattern non-static (the device then evaluates it
    everywhere and reports the error as the reference would)."""
    tag = node[0]
    if tag == "num":
        return np.float64(node[1])
    if tag == "var":
        return env[node[1]]
    if tag == "un":
        return -_veval(node[2], env)
    if tag == "if":
        c = _veval(node[1], env)
        return np.where(c != 0.0, _veval(node[2], env), _veval(node[3], env))
    if tag == "call":
        args = [_veval(a, env) for a in node[2]]
        name = node[1]
        with np.errstate(all="ignore"):
            if name in _VFUN:
                r = _VFUN[name](args[0])
            elif name == "sqrt":
                if np.any(args[0] < 0.0):
                    raise _NotStatic
                r = np.sqrt(args[0])
            elif name in ("log", "ln"):
                if np.any(args[0] <= 0.0):
                    raise _NotStatic
                r = np.log10(args[0]) if name == "log" else np.log(args[0])
            elif name == "pow":
                r = np.power(args[0], args[1])
            elif name == "cot":
                r = np.cos(args[0]) / np.sin(args[0])
            elif name == "coth":
                r = np.cosh(args[0]) / np.sinh(args[0])
            else:
                raise _NotStatic
        if not np.all(np.isfinite(r)):
            raise _NotStatic
        return r
    op = node[1]
    a, b = _veval(node[2], env), _veval(node[3], env)
    if op in _VCMP:
        return _VCMP[op](a, b).astype(np.float64)
    if op == "and":
        return ((a != 0.0) & (b != 0.0)).astype(np.float64)
    if op == "or":
        return ((a != 0.0) | (b != 0.0)).astype(np.float64)
    with np.errstate(all="ignore"):
        if op == "+":
            r = a + b
        elif op == "-":
            r = a - b
        elif op == "*":
            r = a * b
        elif op == "/":
            if np.any(b == 0.0):
                raise _NotStatic
            r = a / b
        elif op == "^":
            r = np.power(a, b)
        else:
            raise _NotStatic
    if not np.all(np.isfinite(r)):
        raise _NotStatic
    return r


def nonskip_mask(ast, X0):
    """Boolean (n,) mask of the particles (reference positions X0, (n, 3))
    where ``ast`` is not skip, or None when its skip pattern is not static."""
    if not skip_static(ast):
        return None
    X0 = np.asarray(X0, dtype=np.float64)
    env = {"x0": X0[:, 0], "y0": X0[:, 1], "z0": X0[:, 2]}
    n = X0.shape[0]

    def walk(node, sel):
        # sel: particles reaching this node; returns the non-skip subset
        if node[0] == "skip":
            return np.zeros(n, dtype=bool)
        if not _has_skip(node):
            return sel
        c = _veval(node[1], env)
        c = np.broadcast_to(c, (n,)) != 0.0
        return walk(node[2], sel & c) | walk(node[3], sel & ~c)

    root = ast.root if isinstance(ast, ExprAst) else ast
    try:
        return walk(root, np.ones(n, dtype=bool))
    except _NotStatic:
        return None


# -- skip patterns static after a time threshold ----------------------------
# ``if(x0<=0.0, 0.0, if(t<=0.0, v, skip))`` (an initial condition) selects
# every particle at t = 0 and the clamped end afterwards: its skip pattern is
# static once t exceeds the constants t is compared with.

_T_FLIP = {"<": ">", ">": "<", "<=": ">=", ">=": "<="}


def _t_compare(node):
    """(op, c) for ``t op c`` (``c op t`` mirrored), else None."""
    if node[0] != "bin" or node[1] not in _T_FLIP:
        return None
    a, b = node[2], node[3]
    if a[0] == "var" and a[1] == "t" and b[0] == "num":
        return node[1], float(b[1])
    if b[0] == "var" and b[1] == "t" and a[0] == "num":
        return _T_FLIP[node[1]], float(a[1])
    return None


def skip_static_after(ast):
    """Threshold T such that whether ``ast`` is skip depends on x0, y0, z0
    only for t > T (-inf when it never depends on t), or None."""
    T = [-math.inf]

    def ok(node):
        if not _has_skip(node) or node[0] == "skip":
            return True
        cond = node[1]
        tc = _t_compare(cond)
        if tc is not None:
            T[0] = max(T[0], tc[1])
        elif not frozenset(_walk_vars(cond)) <= STATIC_VARS:
            return False
        return ok(node[2]) and ok(node[3])

    root = ast.root if isinstance(ast, ExprAst) else ast
    return T[0] if ok(root) else None


def nonskip_mask_after(ast, X0):
    """(T, mask): for t > T, ``ast`` is not skip exactly on ``mask`` (n,);
    None when its skip pattern depends on more than x0, y0, z0 and t
    thresholds."""
    T = skip_static_after(ast)
    if T is None:
        return None
    X0 = np.asarray(X0, dtype=np.float64)
    env = {"x0": X0[:, 0], "y0": X0[:, 1], "z0": X0[:, 2]}
    n = X0.shape[0]

    def walk(node, sel):
        if node[0] == "skip":
            return np.zeros(n, dtype=bool)
        if not _has_skip(node):
            return sel
        tc = _t_compare(node[1])
        if tc is not None:      # t > T >= c: the comparison's late-time value
            late = tc[0] in (">", ">=")
            return walk(node[2] if late else node[3], sel)
        c = np.broadcast_to(_veval(node[1], env), (n,)) != 0.0
        return walk(node[2], sel & c) | walk(node[3], sel & ~c)

    root = ast.root if isinstance(ast, ExprAst) else ast
    try:
        return T, walk(root, np.ones(n, dtype=bool))
    except _NotStatic:
        return None


def _literal(node):
    """The value of a literal number (or its negation), else None."""
    if node[0] == "num":
        return float(node[1])
    if node[0] == "un" and node[2][0] == "num":
        return -float(node[2][1])
    return None


def late_constant(ast, X0):
    """The one value ``ast`` takes wherever it is not skip for t > T
    (nonskip_mask_after's T) when every branch reached there is the same
    literal number -- ``if(x0<=0.0, 0.0, if(t<=0.0, v, skip))`` is 0.0 on
    the clamped end after t = 0 -- else None.  The device then stores the
    constant instead of running the expression: the VM would push the same
    double, so the result is bit-identical."""
    T = skip_static_after(ast)
    if T is None:
        return None
    X0 = np.asarray(X0, dtype=np.float64)
    env = {"x0": X0[:, 0], "y0": X0[:, 1], "z0": X0[:, 2]}
    n = X0.shape[0]
    vals = {}

    def walk(node, sel):
        if node[0] == "skip" or not sel.any():
            return
        if not _has_skip(node):
            v = _literal(node)
            if v is None:
                raise _NotStatic
            vals[np.float64(v).tobytes()] = v     # by bit pattern: 0.0 and -0.0 differ
            return
        tc = _t_compare(node[1])
        if tc is not None:
            late = tc[0] in (">", ">=")
            walk(node[2] if late else node[3], sel)
            return
        c = np.broadcast_to(_veval(node[1], env), (n,)) != 0.0
        walk(node[2], sel & c)
        walk(node[3], sel & ~c)

    root = ast.root if isinstance(ast, ExprAst) else ast
    try:
        walk(root, np.ones(n, dtype=bool))
    except _NotStatic:
        return None
    return next(iter(vals.values())) if len(vals) == 1 else None


# -- skip guards ---------------------------------------------------------------
# ``if(z<1.0e-12, 0.0, if(t<=0.0, Vinit, skip))`` (a wall) depends on the
# current z, so no particle set is fixed -- but after t = 0 it is skip wherever
# the single comparison z < 1e-12 is false.  The step tests that comparison
# inline and runs the expression only where it holds.

_GUARD_OPS = {"<": 0, ">": 1, "<=": 2, ">=": 3}
_GUARD_VARS = ("x0", "y0", "z0", "x", "y", "z", "ux", "uy", "uz")


def skip_guard_after(ast):
    """(T, var index, op code, const): for t > T, ``ast`` is skip wherever
    ``var op const`` is false (expr.VARIABLES index; op 0 <, 1 >, 2 <=, 3 >=).
    None when its late-time skip pattern is not one such comparison."""
    T = [-math.inf]

    def late(node):
        """The node with t-comparisons on skip paths resolved for t -> inf."""
        while node[0] == "if" and _has_skip(node):
            tc = _t_compare(node[1])
            if tc is None:
                return node
            T[0] = max(T[0], tc[1])
            node = node[2] if tc[0] in (">", ">=") else node[3]
        return node

    node = late(ast.root if isinstance(ast, ExprAst) else ast)
    if node[0] != "if" or not _has_skip(node):
        return None
    cond, a, b = node[1], late(node[2]), late(node[3])
    if cond[0] != "bin" or cond[1] not in _GUARD_OPS:
        return None
    lhs, rhs, op = cond[2], cond[3], cond[1]
    if lhs[0] == "num" and rhs[0] == "var":
        lhs, rhs, op = rhs, lhs, _T_FLIP[op]
    if lhs[0] != "var" or lhs[1] not in _GUARD_VARS or rhs[0] != "num":
        return None
    if b[0] == "skip" and not _has_skip(a):          # if(guard, value, skip)
        return T[0], VARIABLES.index(lhs[1]), _GUARD_OPS[op], float(rhs[1])
    return None
