"""The reference's C-ABI, served by libstkb200.so: ``void run_<target>(T *g..., int64_t iter)``.

The reference's only C entry point is the one its C emitters generate
(codegen/serial.py:126-208): caller-owned, padded, C-order host buffers in
target-parameter order, then the scalars (``int64_t`` for ``i32``, ``double``
otherwise), mutated in place, every buffer landing its final contents under its
own name; no status code.  Its acceptance criterion 10
(tests/test_acceptance.py:325-343) compiles such an artifact with a plain
``cc -O2 -fPIC -shared`` and calls the entry through ctypes.

:func:`emit` generates a C translation unit with exactly that entry for a bound
target whose statements are maps, swaps and ``for`` loops over maps and swaps (loop
counts literal or a scalar parameter).  The generated function builds a device
domain from static descriptors (the matched maps, as ``stkb_map_desc`` initialisers),
uploads the buffers, runs the statements (CUDA-graph replay per loop), downloads
every buffer and frees the domain.  It loads libstkb200.so with ``dlopen`` by
absolute path, so the criterion-10 compile line needs no extra flags; any failure
prints ``stkb_last_error()`` and aborts (the reference ABI has no error channel).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional

from . import _lib as L
from . import front
from .backend import ExecutionError, map_desc_for
from .front import stmt_kind
from .matcher import MatchError, match_map

INCLUDE = Path(__file__).resolve().parent.parent / "include" / "stkb200.h"


@dataclass
class ShimArtifact:
    """Shaped like the reference's codegen artifact (``files``, ``entry``)."""

    files: list = field(default_factory=list)  # [(file name, C source)]
    entry: str = ""


def _c_double(x: float) -> str:
    return repr(float(x)) if x == x and abs(x) != float("inf") else ("NAN" if x != x else ("INFINITY" if x > 0 else "-INFINITY"))


def _map_init(d: L.MapDesc, i: int, decls: list) -> str:
    """C initialiser of one stkb_map_desc (arrays it points to are emitted into ``decls``)."""
    f = []
    for name in ("kind", "radius", "src", "dst", "prev", "vel", "precision", "tag"):
        f.append(f".{name} = {getattr(d, name)}")
    f.append(".coef = {" + ", ".join(_c_double(c) for c in d.coef) + "}")
    for name in ("divisor", "wave_a", "wave_b"):
        f.append(f".{name} = {_c_double(getattr(d, name))}")
    f.append(".lo = {" + ", ".join(str(v) for v in d.lo) + "}")
    f.append(".hi = {" + ", ".join(str(v) for v in d.hi) + "}")
    if d.kind == L.STKB_MAP_EXPR:
        code = [d.code[k] for k in range(5 * d.n_code)]
        consts = [d.consts[k] for k in range(max(1, d.n_consts))]
        decls.append(f"static const int32_t code_{i}[] = {{{', '.join(map(str, code))}}};")
        decls.append(f"static const double consts_{i}[] = {{{', '.join(_c_double(c) for c in consts)}}};")
        f.append(f".n_args = {d.n_args}")
        f.append(".args = {" + ", ".join(str(d.args[k]) for k in range(L.EXPR_MAX_ARGS)) + "}")
        f.append(f".n_code = {d.n_code}, .code = code_{i}, .n_consts = {d.n_consts}, .consts = consts_{i}")
    if d.kind in (L.STKB_MAP_BOX, L.STKB_MAP_XBOX):
        if d.box_coef_ext:
            n = (2 * d.radius + 1) ** 3
            decls.append(f"static const double cube_{i}[] = {{{', '.join(_c_double(d.box_coef_ext[k]) for k in range(n))}}};")
            f.append(f".box_coef_ext = cube_{i}")
        else:
            f.append(".box_coef = {" + ", ".join(_c_double(c) for c in d.box_coef) + "}")
    return "{" + ", ".join(f) + "}"


def emit(unit, target: Optional[str] = None, precision: str = "exact", scheme: Optional[str] = None,
         lib_path: Optional[str] = None) -> ShimArtifact:
    """A criterion-10-compatible C artifact running ``unit``'s target on the B200."""
    if precision not in ("fast", "exact"):
        raise ExecutionError(f"unknown precision '{precision}' (fast | exact)")
    analysis = front.module("analysis")
    if hasattr(unit, "grids") and hasattr(unit, "targets"):
        bound = analysis.bind_target(unit, target, None, scheme, freeze_loop_bounds=False)
        decls_by_name = {g.name: g for g in unit.grids}
    else:
        raise ExecutionError("shim.emit needs the reference SourceUnit (grid declarations)")
    params = [g for _, g in bound.grid_params]
    if len(set(params)) != len(params):
        raise ExecutionError("a grid bound to two target parameters cannot take a buffer per parameter")
    grids = [decls_by_name[g] for g in params]
    dt0 = grids[0]
    for g in grids:
        if (g.dtype, len(g.shape)) != (dt0.dtype, len(dt0.shape)):
            raise ExecutionError("the device domain needs one dtype and rank for every grid of the target")
    index = {g: i for i, g in enumerate(params)}
    ctype = "float" if dt0.dtype == "f32" else "double"
    nd = len(dt0.shape)
    shape = [max(g.shape[d] for g in grids) for d in range(nd)]
    order = max(g.order for g in grids)
    scalars = [(p, t) for p, t in _target_params(unit, bound) if t != "grid"]

    decls: list = []
    maps: list = []
    steps: list = []  # C statements of the run

    def program(stmts) -> list:
        out = []
        for s in stmts:
            k = stmt_kind(s)
            if k == "BoundSwap":
                out.append(f"    CHECK(p_add_swap(dom, {index[s.first]}, {index[s.second]}));")
            elif k == "BoundMap":
                if s.scalar_args:
                    raise ExecutionError(f"kernel '{s.kernel.name}' takes scalar arguments: not served by the shim")
                try:
                    plan = match_map(s, exact=precision == "exact" or s.info.dims == 1)
                except MatchError as why:
                    raise ExecutionError(f"kernel '{s.kernel.name}': {why}") from None
                d = map_desc_for(plan, index, len(maps))
                maps.append(_map_init(d, len(maps), decls))
                out.append(f"    CHECK(p_add_map(dom, &MAPS[{len(maps) - 1}]));")
            else:
                raise ExecutionError(f"unsupported statement {k} inside a loop body")
        return out

    for s in bound.stmts:
        k = stmt_kind(s)
        steps.append("    CHECK(p_reset(dom));")
        if k == "BoundFor":
            body = program(s.body)
            count = s.count if isinstance(s.count, int) else None
            if count is None:
                names = [p for p, _ in scalars]
                if s.count not in names:
                    raise ExecutionError(f"loop bound '{s.count}' is not a scalar parameter")
                count = f"(int64_t)({s.count})"
            steps += body + [f"    CHECK(p_run(dom, {count}));"]
        else:
            steps += program((s,)) + ["    CHECK(p_run(dom, 1));"]

    entry = f"run_{bound.name}"
    lib = lib_path or str(Path(L.__file__).resolve().parent / "libstkb200.so")
    args = [f"{ctype} *g{i}" for i in range(len(params))]
    args += [f"int64_t {p}" if t == "i32" else f"double {p}" for p, t in scalars]
    uploads = "\n".join(
        f"    {{ const int64_t s[3] = {{{', '.join(str(e) for e in g.shape)}}}; "
        f"CHECK(p_upload(dom, {i}, g{i}, s, {g.order}, 0)); }}" for i, g in enumerate(grids))
    downloads = "\n".join(
        f"    {{ const int64_t s[3] = {{{', '.join(str(e) for e in g.shape)}}}; "
        f"CHECK(p_download(dom, {i}, g{i}, s, {g.order}, 0)); }}" for i, g in enumerate(grids))
    # swaps move buffers between names; every name's final contents land in its own buffer
    # argument (serial.py:191-204): the download reads the buffer each name is bound to
    src = f"""/* generated by paper_2309_04671_b200.shim: target {bound.name}, precision {precision}
 * The reference C-ABI (codegen/serial.py:126-208) served by libstkb200.so on a B200. */
#include <dlfcn.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include "{INCLUDE}"

static const char *LIB = "{lib}";
{chr(10).join(decls)}
static const stkb_map_desc MAPS[] = {{
    {(',' + chr(10) + '    ').join(maps) if maps else '{0}'}
}};

static void *h;
#define SYM(T, n) ((T)sym(#n))
static void *sym(const char *n) {{
    void *f = dlsym(h, n);
    if (!f) {{ fprintf(stderr, "{entry}: %s missing in %s\\n", n, LIB); abort(); }}
    return f;
}}
static const char *(*p_err)(void);
#define CHECK(x) do {{ if ((x) != 0) {{ fprintf(stderr, "{entry}: %s: %s\\n", #x, p_err()); abort(); }} }} while (0)

void {entry}({', '.join(args)}) {{
    if (!h) {{
        h = dlopen(LIB, RTLD_NOW | RTLD_GLOBAL);
        if (!h) {{ fprintf(stderr, "{entry}: %s\\n", dlerror()); abort(); }}
    }}
    p_err = SYM(const char *(*)(void), stkb_last_error);
    int (*p_create)(const stkb_domain_desc *, stkb_domain **) = SYM(int (*)(const stkb_domain_desc *, stkb_domain **), stkb_domain_create);
    int (*p_destroy)(stkb_domain *) = SYM(int (*)(stkb_domain *), stkb_domain_destroy);
    int (*p_reset)(stkb_domain *) = SYM(int (*)(stkb_domain *), stkb_program_reset);
    int (*p_add_map)(stkb_domain *, const stkb_map_desc *) = SYM(int (*)(stkb_domain *, const stkb_map_desc *), stkb_program_add_map);
    int (*p_add_swap)(stkb_domain *, int32_t, int32_t) = SYM(int (*)(stkb_domain *, int32_t, int32_t), stkb_program_add_swap);
    int (*p_run)(stkb_domain *, int64_t) = SYM(int (*)(stkb_domain *, int64_t), stkb_run);
    int (*p_sync)(stkb_domain *) = SYM(int (*)(stkb_domain *), stkb_sync);
    int (*p_upload)(stkb_domain *, int32_t, const void *, const int64_t *, int32_t, int32_t) =
        SYM(int (*)(stkb_domain *, int32_t, const void *, const int64_t *, int32_t, int32_t), stkb_upload_grid);
    int (*p_download)(stkb_domain *, int32_t, void *, const int64_t *, int32_t, int32_t) =
        SYM(int (*)(stkb_domain *, int32_t, void *, const int64_t *, int32_t, int32_t), stkb_download_grid);
    stkb_domain_desc desc = {{{L.STKB_F32 if dt0.dtype == "f32" else L.STKB_F64}, {nd}, {{{', '.join(str(e) for e in shape + [0] * (3 - nd))}}}, {order}, {len(params)}, 0, 0}};
    const char *dev = getenv("LOCAL_RANK");
    if (dev) desc.device = atoi(dev);
    stkb_domain *dom = NULL;
    CHECK(p_create(&desc, &dom));
{uploads}
{chr(10).join(steps)}
{downloads}
    CHECK(p_sync(dom));
    CHECK(p_destroy(dom));
}}
"""
    return ShimArtifact(files=[(f"{bound.name}_stkb200.c", src)], entry=entry)


def _target_params(unit, bound) -> list:
    t = next(t for t in unit.targets if t.name == bound.name)
    return list(t.params)


def build(artifact: ShimArtifact, out_dir, cc: str = "cc") -> Path:
    """Compile like the reference's criterion-10 harness (``cc -O2 -fPIC -shared``)."""
    import subprocess

    out_dir = Path(out_dir)
    name, text = artifact.files[0]
    src = out_dir / name
    src.write_text(text)
    so = out_dir / (src.stem + ".so")
    subprocess.run([cc, "-O2", "-fPIC", "-shared", str(src), "-o", str(so)], check=True, capture_output=True)
    ctypes.CDLL(str(so))  # loads (dlopen of libstkb200.so happens at the first call)
    return so
