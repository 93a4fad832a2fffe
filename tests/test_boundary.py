"""The drop-in boundary, checked without a GPU: the C-ABI library loads and
exports every entry point include/stkb200.h declares; the matcher routes the
reference's kernel forms; the device bytecode evaluates (on a CPU emulation
of its stack machine) to exactly the oracle's results; plans mirror
planning.py."""

from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, build_case, golden_cases, load_golden
from paper_2309_04671_b200 import _lib as L
from paper_2309_04671_b200 import corpus
from paper_2309_04671_b200.front import node_kind
from paper_2309_04671_b200.matcher import coef_index, compile_expr, map_box, match_map
from paper_2309_04671_b200 import PlanError, plan_gpu


def _maps(stmts):
    for s in stmts:
        if type(s).__name__ == "BoundMap":
            yield s
        elif type(s).__name__ == "BoundFor":
            yield from _maps(s.body)


def header_symbols():
    text = (ROOT / "include" / "stkb200.h").read_text()
    return sorted(set(re.findall(r"\b(stkb_[a-z_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(L.EXPORTS)


@pytest.mark.parametrize("cc,std,lang", [("gcc", "-std=c99", "c"), ("g++", "-std=c++11", "c++")])
def test_header_is_plain_c(cc, std, lang):
    """include/stkb200.h is a plain C header (extern "C" for C++): it compiles on its own."""
    import shutil
    import subprocess

    if shutil.which(cc) is None:
        pytest.skip(f"needs {cc}")
    r = subprocess.run([cc, std, "-Wall", "-Wextra", "-Werror", "-fsyntax-only", "-x", lang,
                        str(ROOT / "include" / "stkb200.h")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_library_loads_and_exports_every_symbol():
    if not L.LIB_PATH.exists():
        pytest.skip("libstkb200.so not built (run __graft_entry__.build())")
    lib = L.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.stkb_abi_version() == 1


def test_library_rejects_bad_descriptors_without_gpu():
    if not L.LIB_PATH.exists():
        pytest.skip("libstkb200.so not built")
    import ctypes

    lib = L.load()
    d = L.DomainDesc()
    d.dtype = 7
    h = ctypes.c_void_p()
    assert lib.stkb_domain_create(ctypes.byref(d), ctypes.byref(h)) == L.STKB_ERR_ARG
    assert b"dtype" in lib.stkb_last_error()


@pytest.mark.parametrize("builder,kind", [("star3d4r", "star"), ("star3d1r", "star"), ("star3d2r", "star"),
                                          ("star3d3r", "star"), ("star3d4r_norm", "star"), ("jacobi7", "star"),
                                          ("wave", "wave"), ("j3d27pt", "box"), ("box3d2r", "box"),
                                          ("box3d1r", "box"), ("box3d3r", "box"), ("box3d4r", "box"), ("star2d4r", "star"),
                                          ("j2d5pt", "star"), ("box2d1r", "box"), ("box2d4r", "box"),
                                          ("j2d9pt_gol", "box")])
def test_matcher_routes(builder, kind):
    shape = (16, 16) if corpus.KERNELS.get(builder) and corpus.KERNELS[builder].dims == 2 else (16, 16, 16)
    bound, _ = corpus.config_target(builder, shape, 1)
    plan = match_map(next(_maps(bound.stmts)))
    assert plan.kind == kind, plan.reason


def test_star_coefficients_land_in_abi_slots():
    bound, _ = corpus.config_target("star3d4r", (16, 16, 16), 1)
    plan = match_map(next(_maps(bound.stmts)))
    for off, c in corpus.coefficients(corpus.KERNELS["star3d4r"]):
        assert plan.coef[coef_index(off, 4)] == c
    assert plan.divisor == 0.0 and plan.radius == 4


def test_normalised_star_keeps_divisor():
    bound, _ = corpus.config_target("star3d4r_norm", (16, 16, 16), 1)
    plan = match_map(next(_maps(bound.stmts)))
    total = round(sum(c for _, c in corpus.coefficients(corpus.KERNELS["star3d4r"])), 5)
    assert plan.divisor == total


def test_wave_form_extracted():
    bound, _ = corpus.config_target("wave", (16, 16, 16), 1)
    p = match_map(next(_maps(bound.stmts)))
    assert (p.src, p.dst, p.prev, p.vel) == ("u", "up", "up", "kap")
    assert p.wave_a == 2.0 and p.wave_b == -1.0
    assert p.coef[0] == pytest.approx(3 * corpus.LAP8[0])
    assert p.coef[coef_index((0, 0, 4), 4)] == pytest.approx(corpus.LAP8[4])


def test_in_place_jacobi_goes_exact():
    import dataclasses

    bound, _ = corpus.config_target("star3d1r", (8, 8, 8), 1)
    m = next(_maps(bound.stmts))
    k = m.kernel
    kk = dataclasses.replace(k, locals=(), updates=(dataclasses.replace(k.updates[0], dest="u"),))
    p = match_map(dataclasses.replace(m, kernel=kk, scalar_args=()))
    assert p.kind == "expr" and "in-place" in p.reason


def emulate_bytecode(plan, state, bmap):
    """CPU model of expr_kernel's stack machine, row-vectorised in float64."""
    code = plan.code
    box = plan.box if plan.box else None
    grids = [state[g] for g in plan.args]
    snaps = [g.data.astype(np.float64) for g in grids]
    o = grids[0].order
    nd = len(grids[0].shape)
    bounds = box
    ext = tuple(hi - lo for lo, hi in bounds)
    st, loc = [], {}
    for op, a, b, c, d in code:
        off = (b, c, d)[:nd]
        if op == L.OP_CONST:
            st.append(np.full(ext, plan.consts[a]))
        elif op == L.OP_READ:
            st.append(snaps[a][tuple(slice(o + lo + q, o + hi + q) for (lo, hi), q in zip(bounds, off))])
        elif op == L.OP_LOCAL:
            st.append(loc[a])
        elif op == L.OP_NEG:
            st.append(-st.pop())
        elif op == L.OP_SETLOCAL:
            loc[a] = st.pop()
        elif op == L.OP_STORE:
            g = grids[a]
            g.data[tuple(slice(o + lo + q, o + hi + q) for (lo, hi), q in zip(bounds, off))] = st.pop().astype(g.data.dtype)
        else:
            y, x = st.pop(), st.pop()
            st.append(x + y if op == L.OP_ADD else x - y if op == L.OP_SUB else x * y if op == L.OP_MUL else x / y)
    assert not st


@pytest.mark.parametrize("case", golden_cases())
def test_device_bytecode_semantics_bitwise(case):
    meta, _, _, ins, outs = load_golden(case)
    bound = build_case(meta)
    state = {n: b.copy() for n, b in ins.items()}

    def run(stmts):
        for s in stmts:
            k = type(s).__name__
            if k == "BoundSwap":
                state[s.first], state[s.second] = state[s.second], state[s.first]
            elif k == "BoundFor":
                for _ in range(s.count):
                    run(s.body)
            else:
                plan = compile_expr(s)
                plan.box = map_box(s)
                emulate_bytecode(plan, state, s)

    run(bound.stmts)
    for n, ref in outs.items():
        assert np.array_equal(state[n].data, ref.data), n


def test_plans_come_from_the_reference_planner():
    """The plan token is the reference's own GpuPlan (planning.py:104-202), not a copy;
    B200's compute capability "10.0" passes its asyncMemcpy gate."""
    import paper_2309_04671_b200 as pkg

    bound, _ = corpus.config_target("star3d4r", (16, 16, 16), 1)
    info = next(_maps(bound.stmts)).info
    assert pkg.plan_gpu is pkg.front.module("planning").plan_gpu
    assert pkg.GridBuffer is pkg.front.module("grids").GridBuffer
    p = plan_gpu(info, {"template": "unroll", "computeCapability": "10.0", "asyncMemcpy": True})
    assert isinstance(p, pkg.front.module("planning").GpuPlan) and p.template == "unroll"
    with pytest.raises(PlanError, match="unknown GPU template"):
        plan_gpu(info, {"template": "tma"})


def test_dead_inputs_detected():
    from paper_2309_04671_b200.backend import dead_on_entry, halo_is_zero
    from paper_2309_04671_b200 import GridBuffer

    for builder, expect in (("star3d4r", {"v"}), ("wave", set()), ("j3d27pt", {"v"}), ("star2d4r", {"v"})):
        shape = (16, 16) if builder.startswith("star2d") else (16, 16, 16)
        bound, decls = corpus.config_target(builder, shape, 3)
        assert dead_on_entry(bound.stmts, list(decls), {}) == expect, builder
    bound, decls = corpus.config_target("star3d4r", (16, 16, 16), "n")
    assert dead_on_entry(bound.stmts, list(decls), {}) == set()  # unknown loop bound: conservative
    assert dead_on_entry(bound.stmts, list(decls), {"n": 0}) == set()  # the body never runs
    g = GridBuffer.zeros((4, 5, 6), 2)
    g.interior[...] = 1.0
    assert halo_is_zero(g)
    g.data[0, 3, 3] = 1.0
    assert not halo_is_zero(g)
    g.data[0, 3, 3] = -0.0  # equal to 0.0 numerically, not bit for bit: must be uploaded
    assert not halo_is_zero(g)
    g.data[0, 3, 3] = 0.0
    assert halo_is_zero(g)


def emulate_xstar(plan, state):
    """CPU model of star_exact.cuh's evaluation order, in float64 with one rounding:
    centre, d0-negative (m = R..1), d1-negative, d2-negative, d2-positive (m = 1..R),
    d1-positive, d0-positive, then the division."""
    src, dst = state[plan.src], state[plan.dst]
    R, o = plan.radius, src.order
    u = src.data.astype(np.float64)
    box = plan.box
    n = tuple(hi - lo for lo, hi in box)

    def tap(off):
        return u[tuple(slice(o + lo + q, o + lo + q + e) for (lo, _), q, e in zip(box, off, n))]

    def c(off):
        return plan.coef[coef_index(off, R)]

    def axis_off(ax, m):
        v = [0, 0, 0]
        v[ax] = m
        return tuple(v)

    acc = c((0, 0, 0)) * tap((0, 0, 0))
    order = ([axis_off(0, -m) for m in range(R, 0, -1)] + [axis_off(1, -m) for m in range(R, 0, -1)] +
             [axis_off(2, -m) for m in range(R, 0, -1)] + [axis_off(2, m) for m in range(1, R + 1)] +
             [axis_off(1, m) for m in range(1, R + 1)] + [axis_off(0, m) for m in range(1, R + 1)])
    for off in order:
        acc = acc + c(off) * tap(off)
    if plan.divisor:
        acc = acc / plan.divisor
    dst.data[tuple(slice(dst.order + lo, dst.order + hi) for lo, hi in box)] = acc.astype(dst.data.dtype)


@pytest.mark.parametrize("case", ["star3d1r_12", "star3d2r_12", "star3d3r_10x12x14", "star3d4r_16", "star3d4r_f64",
                                  "star3d4r_norm_16", "jacobi7_16", "star3d4r_w2_cross", "star3d4r_w3_slab7"])
def test_exact_star_kernel_order_bitwise(case):
    """precision='exact' routes the corpus stars (and c2's Jacobi-7, the normalised stars)
    to the exact streaming kernel; its evaluation order, modelled here, reproduces the
    reference's outputs bit for bit."""
    meta, _, _, ins, outs = load_golden(case)
    bound = build_case(meta)
    state = {n: b.copy() for n, b in ins.items()}

    def run(stmts):
        for s in stmts:
            k = type(s).__name__
            if k == "BoundSwap":
                state[s.first], state[s.second] = state[s.second], state[s.first]
            elif k == "BoundFor":
                for _ in range(s.count):
                    run(s.body)
            else:
                plan = match_map(s, exact=True)
                assert plan.kind == "xstar", plan.reason
                emulate_xstar(plan, state)

    run(bound.stmts)
    for n, ref in outs.items():
        assert np.array_equal(state[n].data, ref.data), n


def test_exact_star_refuses_other_orders():
    """Any other term order, a missing tap or a local goes to the bytecode kernel."""
    import dataclasses

    bound, _ = corpus.config_target("star3d1r", (8, 8, 8), 1)
    m = next(_maps(bound.stmts))
    assert match_map(m, exact=True).kind == "xstar"
    e = m.kernel.updates[0].expr  # ((... + t5) + t6): swap the last two terms
    swapped = dataclasses.replace(e, left=dataclasses.replace(e.left, right=e.right), right=e.left.right)
    k2 = dataclasses.replace(m.kernel, updates=(dataclasses.replace(m.kernel.updates[0], expr=swapped),))
    p = match_map(dataclasses.replace(m, kernel=k2), exact=True)
    assert p.kind == "expr" and "corpus order" in p.reason
    short = dataclasses.replace(m.kernel, updates=(dataclasses.replace(m.kernel.updates[0], expr=e.left),))
    assert match_map(dataclasses.replace(m, kernel=short), exact=True).kind == "expr"
    wave, _ = corpus.config_target("wave", (8, 8, 8), 1)
    assert match_map(next(_maps(wave.stmts)), exact=True).kind == "xwave"


def emulate_xwave(plan, state):
    """CPU model of wave_exact_kernel's evaluation (star_exact.cuh): per ring m the six taps
    d0-, d0+, d1-, d1+, d2-, d2+ summed left to right, the laplacian chain, then
    (A*u - p) + k*lap, in float64 with one rounding."""
    src, dst, prev, vel = state[plan.src], state[plan.dst], state[plan.prev], state[plan.vel]
    R, o = plan.radius, src.order
    box = plan.box
    n = tuple(hi - lo for lo, hi in box)

    def at(g, off):
        d = g.data.astype(np.float64)
        return d[tuple(slice(g.order + lo + q, g.order + lo + q + e) for (lo, _), q, e in zip(box, off, n))]

    u0 = at(src, (0, 0, 0))
    lap = plan.coef[0] * u0
    for m in range(1, R + 1):
        s = at(src, (-m, 0, 0)) + at(src, (m, 0, 0))
        for off in ((0, -m, 0), (0, m, 0), (0, 0, -m), (0, 0, m)):
            s = s + at(src, off)
        lap = lap + plan.coef[m] * s
    out = (plan.wave_a * u0 - at(prev, (0, 0, 0))) + at(vel, (0, 0, 0)) * lap
    dst.data[tuple(slice(dst.order + lo, dst.order + hi) for lo, hi in box)] = out.astype(dst.data.dtype)


@pytest.mark.parametrize("case", ["wave_16", "wave_f64_12"])
def test_exact_wave_kernel_order_bitwise(case):
    """precision='exact' routes the c3 acoustic wave to the exact wave kernel; its evaluation
    order, modelled here, reproduces the reference's outputs bit for bit."""
    meta, _, _, ins, outs = load_golden(case)
    bound = build_case(meta)
    state = {n: b.copy() for n, b in ins.items()}
    for s in bound.stmts[0].body * bound.stmts[0].count:
        if type(s).__name__ == "BoundSwap":
            state[s.first], state[s.second] = state[s.second], state[s.first]
        else:
            plan = match_map(s, exact=True)
            assert plan.kind == "xwave", plan.reason
            emulate_xwave(plan, state)
    for n, ref in outs.items():
        assert np.array_equal(state[n].data, ref.data), n


def emulate_xbox(plan, state):
    """CPU model of box_exact_kernel's evaluation (box_exact.cu), in float64 with one rounding:
    the centre, then the d0 = -R .. 0 layers as output q starts (planes resident in the ring),
    then each later plane's layer as it arrives — every layer row by row (d1), tap by tap
    (d2) — then the division."""
    src, dst = state[plan.src], state[plan.dst]
    R, o = plan.radius, src.order
    box = plan.box
    n = tuple(hi - lo for lo, hi in box)
    u = src.data.astype(np.float64)
    w = 2 * R + 1

    def tap(off):
        return u[tuple(slice(o + lo + q, o + lo + q + e) for (lo, _), q, e in zip(box, off, n))]

    def c(dz, dy, dx):
        return plan.coef[((dz + R) * w + (dy + R)) * w + (dx + R)]

    acc = c(0, 0, 0) * tap((0, 0, 0))
    for dz in range(-R, R + 1):
        for dy in range(-R, R + 1):
            for dx in range(-R, R + 1):
                if (dz, dy, dx) != (0, 0, 0):
                    acc = acc + c(dz, dy, dx) * tap((dz, dy, dx))
    if plan.divisor:
        acc = acc / plan.divisor
    dst.data[tuple(slice(dst.order + lo, dst.order + hi) for lo, hi in box)] = acc.astype(dst.data.dtype)


@pytest.mark.parametrize("case", ["box3d2r_10", "j3d27pt_12"])
def test_exact_box_kernel_order_bitwise(case):
    """precision='exact' routes the corpus boxes (R <= 2) and j3d27pt to the exact box kernel;
    its evaluation order, modelled here, reproduces the reference's outputs bit for bit."""
    meta, _, _, ins, outs = load_golden(case)
    bound = build_case(meta)
    state = {n: b.copy() for n, b in ins.items()}
    for s in bound.stmts[0].body * bound.stmts[0].count:
        if type(s).__name__ == "BoundSwap":
            state[s.first], state[s.second] = state[s.second], state[s.first]
        else:
            plan = match_map(s, exact=True)
            assert plan.kind == "xbox", plan.reason
            emulate_xbox(plan, state)
    for n, ref in outs.items():
        assert np.array_equal(state[n].data, ref.data), n


def test_exact_box_routes():
    """The full cube (square in 2-D) in corpus order goes to XBOX (2-D stars to XSTAR); a
    reordered or incomplete cube goes to the bytecode kernel."""
    import dataclasses

    for name, kind in (("box3d1r", "xbox"), ("box3d2r", "xbox"), ("j3d27pt", "xbox"), ("box3d3r", "xbox"),
                       ("box3d4r", "xbox"), ("box2d4r", "xbox"), ("j2d9pt_gol", "xbox"), ("star2d4r", "xstar"),
                       ("j2d5pt", "xstar")):
        bound, _ = corpus.config_target(name, (12, 12, 12) if "3d" in name else (12, 12), 1)
        assert match_map(next(_maps(bound.stmts)), exact=True).kind == kind, name
    bound, _ = corpus.config_target("box3d1r", (8, 8, 8), 1)
    m = next(_maps(bound.stmts))
    e = m.kernel.updates[0].expr
    swapped = dataclasses.replace(e, left=dataclasses.replace(e.left, right=e.right), right=e.left.right)
    k2 = dataclasses.replace(m.kernel, updates=(dataclasses.replace(m.kernel.updates[0], expr=swapped),))
    p = match_map(dataclasses.replace(m, kernel=k2), exact=True)
    assert p.kind == "expr" and "full box in corpus order" in p.reason
    short = dataclasses.replace(m.kernel, updates=(dataclasses.replace(m.kernel.updates[0], expr=e.left),))
    assert match_map(dataclasses.replace(m, kernel=short), exact=True).kind == "expr"


@pytest.mark.parametrize("name,shape", [("box3d1r", (8, 8, 8)), ("box3d4r", (10, 10, 10)), ("box2d4r", (16, 16)),
                                        ("j2d9pt_gol", (12, 12)), ("star2d4r", (12, 12))])
def test_exact_descriptors(name, shape):
    """The C-ABI descriptor of an exact box / 2-D map: kind, radius and the coefficient table in
    the header's layout (box_coef for <= 125 values, box_coef_ext beyond; 2-D stars use the
    STAR slots of the grid's own two axes), the divisor passed through."""
    from paper_2309_04671_b200 import _lib as L
    from paper_2309_04671_b200.backend import map_desc_for

    bound, _ = corpus.config_target(name, shape, 1)
    m = next(_maps(bound.stmts))
    plan = match_map(m, exact=True)
    d = map_desc_for(plan, {"u": 0, "v": 1}, 0)
    r = plan.radius
    if plan.kind == "xbox":
        assert d.kind == L.STKB_MAP_XBOX and d.radius == r
        n = (2 * r + 1) ** len(shape)
        assert len(plan.coef) == n
        got = [d.box_coef_ext[i] for i in range(n)] if n > 125 else [d.box_coef[i] for i in range(n)]
        assert got == plan.coef and all(c != 0.0 for c in got)  # every corpus tap is non-zero
        centre = plan.coef[n // 2]
        text = m.kernel.updates[0].expr
        while node_kind(text) == "Binary" and text.op in "+/":
            text = text.left
        assert centre == float(text.left.value)  # the first term is the centre's
    else:
        assert d.kind == L.STKB_MAP_XSTAR and d.radius == r
        assert [d.coef[i] for i in range(4 * r + 1)] == plan.coef[:4 * r + 1]  # axes 0, 1 of the 2-D grid
        assert all(c == 0.0 for c in plan.coef[4 * r + 1:])
    assert d.divisor == plan.divisor
