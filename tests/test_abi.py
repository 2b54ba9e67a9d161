"""CPU-side checks of the C ABI and the host logic (no GPU calls)."""
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden

HEADER = os.path.join(ROOT, "include", "tlsph.h")


def _header_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const\s+char\s*\*)\s*(tl_\w+)\s*\(", txt, re.M)))


def test_library_loads_and_exports_header_symbols():
    from paper_2602_15149_b200 import _lib
    L = _lib.load_library()
    declared = _header_functions()
    assert set(declared) == set(_lib.EXPORTED)
    for name in declared:
        assert hasattr(L, name), name


def test_struct_layouts_match_ctypes():
    import ctypes
    from paper_2602_15149_b200 import _lib
    L = _lib.load_library()
    for k, st in enumerate(_lib.STRUCTS):
        assert L.tl_struct_size(k) == ctypes.sizeof(st), st.__name__


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2602_15149_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace(
                    "oracle_", ""), f


def test_no_gpu_means_loud_failure(monkeypatch):
    import torch
    from paper_2602_15149_b200 import _lib
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(_lib.NativeLibraryError):
        _lib.lib()


# -- expression compiler: run the bytecode with a tiny host interpreter and
#    compare with the golden masked evaluation of the reference -------------

def _run(prog, vars_):
    from paper_2602_15149_b200 import expr as ex
    inv = {v: k for k, v in ex.OP.items()}
    st = []
    pc = 0
    code = prog.code
    while pc < len(code):
        op, arg = inv[int(code[pc, 0])], int(code[pc, 1])
        pc += 1
        if op == "END":
            return st[-1], False
        if op == "CONST":
            st.append(float(prog.consts[arg]))
        elif op == "VAR":
            st.append(float(vars_[arg]))
        elif op == "NEG":
            st[-1] = -st[-1]
        elif op == "JZ":
            if st.pop() == 0.0:
                pc = arg
        elif op == "JMP":
            pc = arg
        elif op == "SKIP":
            return 0.0, True
        elif op in ("SIN", "COS", "TAN", "SINH", "COSH", "TANH", "SQRT", "ABS"):
            st[-1] = getattr(np, op.lower() if op != "ABS" else "abs")(st[-1])
        elif op == "COT":
            st[-1] = np.cos(st[-1]) / np.sin(st[-1])
        elif op == "COTH":
            a = min(max(st[-1], -700.0), 700.0)
            st[-1] = np.cosh(a) / np.sinh(a)
        elif op == "LOG":
            st[-1] = np.log10(st[-1])
        elif op == "LN":
            st[-1] = np.log(st[-1])
        else:
            b = st.pop()
            a = st[-1]
            st[-1] = {"ADD": lambda: a + b, "SUB": lambda: a - b, "MUL": lambda: a * b,
                      "DIV": lambda: a / b, "POW": lambda: math.pow(a, b),
                      "POWF": lambda: math.pow(a, b), "LT": lambda: float(a < b),
                      "GT": lambda: float(a > b), "LE": lambda: float(a <= b),
                      "GE": lambda: float(a >= b), "EQ": lambda: float(a == b),
                      "NE": lambda: float(a != b),
                      "AND": lambda: float(a != 0.0 and b != 0.0),
                      "OR": lambda: float(a != 0.0 or b != 0.0)}[op]()
    return st[-1], False


def test_bytecode_matches_reference_masked_eval():
    from paper_2602_15149_b200 import expr as ex
    G = golden("expr")
    srcs = bytes(G["sources"]).decode().split("\n")
    names = ex.VARIABLES
    n = G["x0"].shape[0]
    for k, line in enumerate(srcs):
        src, loc = line.split("\t")
        prog = ex.compile_program(ex.parse(src, loc))
        assert prog.depth <= ex.MAX_STACK
        ref_v, ref_s = G[f"e{k}.vals"], G[f"e{k}.skip"]
        for i in range(0, n, 7):
            vars_ = [float(G[nm][i]) if G[nm].ndim else float(G[nm]) for nm in names]
            val, skip = _run(prog, vars_)
            assert skip == bool(ref_s[i]), (src, i)
            if not skip:
                assert val == pytest.approx(ref_v[i], rel=1e-14, abs=1e-300), (src, i)


def test_parse_errors_and_skip_rules():
    from paper_2602_15149_b200 import expr as ex
    for bad, msg in [("", "empty"), ("1 +", "unexpected token"), ("foo", "unknown identifier"),
                     ("sin(1, 2)", "takes 1"), ("1 + skip", "skip"), ("and 1", "missing left"),
                     ("(1", "expected '\\)'"), ("1 $", "unexpected character")]:
        with pytest.raises(ex.ExprError, match=msg):
            ex.parse(bad)
    assert ex.parse("if(x0 > 1, skip, 2)").root[0] == "if"
    assert ex.parse("-2^2").root == ("num", -4.0) or ex.eval_expr(ex.parse("-2^2"), None) == -4.0
    assert ex.eval_expr(ex.parse("2^3^2"), None) == 512.0
    assert ex.parse("a*b", "a=2; b=a+1").root == ("bin", "*", ("num", 2.0), ("num", 3.0))
    assert not ex.parse("x0*2").time_dependent and ex.parse("t*2").time_dependent


def test_case_roundtrip():
    from paper_2602_15149_b200 import cases
    cfg = cases.make_case("kalthoff2d", dp_scale=2, mapfac=1, build_adjacency=False)
    d = cases.case_to_dict(cfg)
    back = cases.case_from_dict(d)
    assert np.array_equal(back.bodies[0].state.X, cfg.bodies[0].state.X)
    assert back.bodies[0].material == cfg.bodies[0].material
    for a, b in zip(back.bodies[0].bcs, cfg.bodies[0].bcs):
        assert a.kind == b.kind and a.const == b.const and a.expr == b.expr
        assert (a.target is None and b.target is None) or np.array_equal(a.target, b.target)


def test_workload_sizes():
    """BASELINE configs at their stated particle counts;
    C4 and C5 are counted from the lattice rule without materialising."""
    from paper_2602_15149_b200 import cases
    c1 = cases.make_case("C1", build_adjacency=False)
    assert c1.bodies[0].n == 3800
    # C4: round(99.5/0.1836) x round(10/0.1836) x round(99.5/0.1836)
    dpb = 1e-3 * 0.918 / 5
    assert (round(99.5e-3 / dpb) * round(10e-3 / dpb) * round(99.5e-3 / dpb)) == 15863256


def test_output_hooks_install_and_reject_host_bodies():
    """output.install routes a reference-style module's OutputManager to the
    device reductions; host (non-device) bodies are refused, not computed
    on the CPU."""
    import types
    from paper_2602_15149_b200 import output
    mod = types.SimpleNamespace(compute_energies=None, measure_row=None)
    output.install(mod)
    assert mod.compute_energies is output.compute_energies
    assert mod.measure_row is output.measure_row
    body = types.SimpleNamespace(state=types.SimpleNamespace())
    with pytest.raises(TypeError):
        output.compute_energies(body)


def test_fourpoint3d_spec_matches_reference_case():
    """cases.py's transcription of fourpoint3d.xml (the paper's benchmark
    body, bench.py workload P1) reproduces the case the reference's loader
    built for the golden run: lattice, material, notch, BCs, expressions."""
    from paper_2602_15149_b200 import cases
    G = golden("run_fourpoint3d")
    g = cases.case_from_dict(G)
    c = cases.make_case("fourpoint3d", dp_scale=6, build_adjacency=False)
    bg, bc = g.bodies[0], c.bodies[0]
    assert np.array_equal(bg.state.X, bc.state.X)
    assert (bg.h, bg.dp_body, bg.restrictphi_expr, bg.nbsrange, bg.fracture) == \
        (bc.h, bc.dp_body, bc.restrictphi_expr, bc.nbsrange, bc.fracture)
    assert vars(bg.material) == vars(bc.material)
    assert (g.cfl, g.time_out, g.time_max, int(g.kernel), g.dp) == \
        (c.cfl, c.time_out, c.time_max, int(c.kernel), c.dp)
    assert [(b.kind, b.expr, b.const) for b in bg.bcs] == [(b.kind, b.expr, b.const) for b in bc.bcs]
    for k in g.expressions:
        assert g.expressions[k].source.strip() == c.expressions[k].source.strip()
        assert g.expressions[k].locals == c.expressions[k].locals
    assert np.array_equal(np.asarray(bg.notches[0].points), np.asarray(bc.notches[0].points))


def test_static_skip_patterns_of_shipped_expressions():
    """expr.skip_static / nonskip_mask on the shipped cases' expressions."""
    from paper_2602_15149_b200 import cases, expr as ex
    X = np.array([[-1e-3, 0, 0], [0.0, 0, 0], [0.05, 0, 0], [0.1, 0, 0.0]])
    col = cases.make_case("column3d", dp_scale=8, build_adjacency=False)
    assert ex.nonskip_mask(col.expressions[2], X).tolist() == [True, True, False, False]
    assert ex.nonskip_mask(col.expressions[1], X).tolist() == [False, False, False, True]
    tay = cases.make_case("taylor3d", dp_scale=8, build_adjacency=False)
    assert not ex.skip_static(tay.expressions[1])       # tests the current z
    assert ex.nonskip_mask(tay.expressions[1], X) is None
    fp = cases.make_case("fourpoint3d", dp_scale=8, build_adjacency=False)
    Xb = fp.bodies[0].state.X
    m = ex.nonskip_mask(fp.expressions[1], Xb)
    ref = np.array([ex.eval_expr(fp.expressions[1], ex.EvalContext(x0=p[0], y0=p[1], z0=p[2]))
                    is not ex.SKIP for p in Xb])
    assert np.array_equal(m, ref) and 0 < m.sum() < m.size
    assert ex.nonskip_mask(ex.parse("if(x0/(x0-x0)>0,1,skip)"), X) is None   # domain error


def test_skip_patterns_static_after_a_time():
    """expr.nonskip_mask_after: beam2d's initial-condition BC selects every
    particle at t <= 0 and only the clamped end (x0 <= 0) afterwards."""
    from paper_2602_15149_b200 import cases, expr as ex
    b = cases.make_case("beam2d", dp_scale=8, build_adjacency=False)
    X = np.array([[-1e-3, 0, 0], [0.0, 0, 0], [0.05, 0, 0.0]])
    T, m = ex.nonskip_mask_after(b.expressions[1], X)
    assert T == 0.0 and m.tolist() == [True, True, False]
    assert ex.nonskip_mask_after(b.expressions[2], X)[0] == -np.inf
    assert ex.nonskip_mask_after(ex.parse("if(t>2e-6, skip, if(x0>0.01, 1.0, skip))"),
                                 X)[1].tolist() == [False, False, False]
    assert ex.nonskip_mask_after(ex.parse("if(z<1.0e-12,0.0,if(t<=0.0,1.0,skip))"), X) is None


def test_late_constants():
    """expr.late_constant: the literal an expression takes wherever it is not
    skip after its threshold (beam2d: 0.0 on the clamped end after t = 0)."""
    from paper_2602_15149_b200 import cases, expr as ex
    b = cases.make_case("beam2d", dp_scale=8, build_adjacency=False)
    X = np.array([[-1e-3, 0, 0], [0.0, 0, 0], [0.05, 0, 0.0]])
    for k in (1, 2):
        v = ex.late_constant(b.expressions[k], X)
        assert v == 0.0 and np.signbit(v) == False  # noqa: E712
    assert ex.late_constant(ex.parse("if(x0<=0,-2.5,skip)"), X) == -2.5
    assert ex.late_constant(ex.parse("if(x0<=0,1.0,if(x0>0.04,2.0,skip))"), X) is None
    assert ex.late_constant(ex.parse("if(x0<=0,1.0,if(x0>0.06,2.0,skip))"), X) == 1.0
    assert ex.late_constant(ex.parse("if(x0<=0,t,skip)"), X) is None
    assert ex.late_constant(ex.parse("if(x0<=0,0.0,if(x0>0.04,-0.0,skip))"), X) is None
    assert ex.late_constant(ex.parse("if(z<1.0e-12,0.0,if(t<=0.0,1.0,skip))"), X) is None


def test_skip_guards():
    """expr.skip_guard_after: the late-time skip pattern as one comparison."""
    from paper_2602_15149_b200 import expr as ex
    assert ex.skip_guard_after(ex.parse("if(z<1.0e-12,0.0,if(t<=0.0,Vinit,skip))",
                                        "Vinit=-227;")) == (0.0, 5, 0, 1e-12)
    assert ex.skip_guard_after(ex.parse("if(1.0>ux,3.0,skip)")) == (-np.inf, 6, 0, 1.0)
    assert ex.skip_guard_after(ex.parse("if(z<0.0, skip, 1.0)")) is None
    assert ex.skip_guard_after(ex.parse("if(x*x<1.0, 1.0, skip)")) is None
