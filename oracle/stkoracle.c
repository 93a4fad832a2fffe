/*
 * stkoracle.c — compiled CPU oracle for one map invocation. TEST
 * INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline; never linked into the product.
 *
 * Restates the reference oracle's arithmetic (pkg/src/stencilkit/executor.py
 * :1-10, _MapContext :56-138): every grid argument that is written by the map
 * and also read is snapshotted first (:66-69), each point's expression is
 * evaluated in float64 in parse order — one IEEE operation per tree node —
 * and rounded once on store (:108-124).  Evaluation is row-vectorised: the
 * bytecode (oracle.py:bytecode, same opcodes as include/stkb200.h) runs over
 * whole d2 rows, so interpretation is amortised and the per-element work is
 * the same sequence of double ops the reference performs.  Build with
 * -ffp-contract=off so no a*b+c is fused.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { CONST = 1, READ, LOCAL, ADD, SUB, MUL, DIV, NEG, SETLOCAL, STORE };
#define MAXS 32
#define MAXL 16
#define MAXA 8

typedef struct {
    int64_t z, y, x;    /* padded extents */
    int64_t oz, o;      /* halo of d0 (0 for lifted 2-D) and of the others */
    int64_t sz, sy;     /* strides */
} geom;

static inline int64_t at(const geom *g, int64_t z, int64_t y, int64_t x) {
    return (z + g->oz) * g->sz + (y + g->o) * g->sy + (x + g->o);
}

int stko_run_map(int dtype, int ndim, const int64_t *shape, int order, int n_args, void **grids,
                 const int32_t *code, int n_code, const double *consts, const int64_t *lo_in,
                 const int64_t *hi_in, int nthreads) {
    if (n_args < 1 || n_args > MAXA || (ndim != 2 && ndim != 3)) return 1;
    geom g;
    int64_t lo[3], hi[3];
    if (ndim == 3) {
        g.z = shape[0] + 2 * order; g.y = shape[1] + 2 * order; g.x = shape[2] + 2 * order;
        g.oz = order;
        for (int d = 0; d < 3; ++d) { lo[d] = lo_in[d]; hi[d] = hi_in[d]; }
    } else {
        g.z = 1; g.y = shape[0] + 2 * order; g.x = shape[1] + 2 * order;
        g.oz = 0;
        lo[0] = 0; hi[0] = 1; lo[1] = lo_in[0]; hi[1] = hi_in[0]; lo[2] = lo_in[1]; hi[2] = hi_in[1];
    }
    g.o = order;
    g.sy = g.x;
    g.sz = g.x * g.y;
    const size_t esz = dtype == 1 ? 4 : 8;
    const size_t total = (size_t)(g.z * g.y * g.x);
    const int64_t n = hi[2] - lo[2];
    if (n <= 0 || hi[1] <= lo[1] || hi[0] <= lo[0]) return 0;

    /* lift 2-D offsets: (d0, d1) -> (0, d0, d1) */
    int32_t *prog = (int32_t *)malloc(sizeof(int32_t) * 5 * (size_t)n_code);
    memcpy(prog, code, sizeof(int32_t) * 5 * (size_t)n_code);
    if (ndim == 2)
        for (int pc = 0; pc < n_code; ++pc)
            if (prog[5 * pc] == READ || prog[5 * pc] == STORE) {
                prog[5 * pc + 4] = prog[5 * pc + 3];
                prog[5 * pc + 3] = prog[5 * pc + 2];
                prog[5 * pc + 2] = 0;
            }

    /* snapshots of grids both written and read (aliases share one) */
    int written[MAXA] = {0}, read[MAXA] = {0};
    for (int pc = 0; pc < n_code; ++pc) {
        if (prog[5 * pc] == READ) read[prog[5 * pc + 1]] = 1;
        if (prog[5 * pc] == STORE) written[prog[5 * pc + 1]] = 1;
    }
    const void *rd[MAXA];
    void *snap[MAXA] = {0};
    for (int i = 0; i < n_args; ++i) {
        int w = 0, r = 0;
        for (int j = 0; j < n_args; ++j)
            if (grids[j] == grids[i]) { w |= written[j]; r |= read[j]; }
        rd[i] = grids[i];
        if (w && r) {
            for (int j = 0; j < i; ++j)
                if (grids[j] == grids[i] && snap[j]) { rd[i] = snap[j]; break; }
            if (rd[i] == grids[i]) {
                snap[i] = malloc(total * esz);
                memcpy(snap[i], grids[i], total * esz);
                rd[i] = snap[i];
            }
        }
    }

    const int64_t rows1 = hi[1] - lo[1];
    const int64_t nrows = (hi[0] - lo[0]) * rows1;
    int bad = 0;
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1) reduction(| : bad)
    {
        double *st = (double *)malloc(sizeof(double) * (size_t)n * MAXS);
        double *loc = (double *)malloc(sizeof(double) * (size_t)n * MAXL);
#pragma omp for schedule(static)
        for (int64_t r = 0; r < nrows; ++r) {
            const int64_t z = lo[0] + r / rows1, y = lo[1] + r % rows1;
            int sp = 0;
            for (int pc = 0; pc < n_code && !bad; ++pc) {
                const int32_t *in = prog + 5 * pc;
                double *top = st + (size_t)sp * n;
                double *a = st + (size_t)(sp - 2) * n, *b = st + (size_t)(sp - 1) * n;
                switch (in[0]) {
                    case CONST: { const double c = consts[in[1]]; for (int64_t i = 0; i < n; ++i) top[i] = c; ++sp; break; }
                    case READ: {
                        const int64_t off = at(&g, z + in[2], y + in[3], lo[2] + in[4]);
                        if (dtype == 1) { const float *s = (const float *)rd[in[1]] + off; for (int64_t i = 0; i < n; ++i) top[i] = (double)s[i]; }
                        else { const double *s = (const double *)rd[in[1]] + off; for (int64_t i = 0; i < n; ++i) top[i] = s[i]; }
                        ++sp; break;
                    }
                    case LOCAL: memcpy(top, loc + (size_t)in[1] * n, sizeof(double) * n); ++sp; break;
                    case ADD: for (int64_t i = 0; i < n; ++i) a[i] = a[i] + b[i]; --sp; break;
                    case SUB: for (int64_t i = 0; i < n; ++i) a[i] = a[i] - b[i]; --sp; break;
                    case MUL: for (int64_t i = 0; i < n; ++i) a[i] = a[i] * b[i]; --sp; break;
                    case DIV: for (int64_t i = 0; i < n; ++i) a[i] = a[i] / b[i]; --sp; break;
                    case NEG: for (int64_t i = 0; i < n; ++i) b[i] = -b[i]; break;
                    case SETLOCAL: memcpy(loc + (size_t)in[1] * n, b, sizeof(double) * n); --sp; break;
                    case STORE: {
                        const int64_t off = at(&g, z + in[2], y + in[3], lo[2] + in[4]);
                        if (dtype == 1) { float *d = (float *)grids[in[1]] + off; for (int64_t i = 0; i < n; ++i) d[i] = (float)b[i]; }
                        else { double *d = (double *)grids[in[1]] + off; for (int64_t i = 0; i < n; ++i) d[i] = b[i]; }
                        --sp; break;
                    }
                    default: bad = 1;
                }
                if (sp < 0 || sp > MAXS) bad = 1;
            }
        }
        free(st);
        free(loc);
    }
    for (int i = 0; i < n_args; ++i) free(snap[i]);
    free(prog);
    return bad ? 2 : 0;
}
