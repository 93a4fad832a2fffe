/*
 * stkb200.h — C-ABI of the B200 star-stencil backend (libstkb200.so).
 *
 * This is the drop-in boundary for the reference's GPU execution path.
 * Reference interfaces it replaces (paths under the reference package
 * pkg/src/stencilkit/):
 *
 *   - executor.py:491-557  run_tile_plan(unit, GpuPlan, grids) GPU branch, which
 *     emulates the emitted CUDA in numpy (the Python drop-in sits above this ABI,
 *     see paper_2309_04671_b200/backend.py::run_gpu);
 *   - codegen/serial.py:126-208  emit_entry: the only C-ABI the reference has,
 *     `void run_<target>(T *g0, T *g1, ..., int64_t iter)` over caller-owned,
 *     padded, C-order host buffers, mutated in place, final contents landed under
 *     each grid's own name (copy-back, serial.py:191-204);
 *   - codegen/gpu.py:450-466  _host_stub: the emitted CUDA's host side, which is
 *     a comment only (no cudaMalloc / memcpy / stream / graph).
 *
 * Every entry point returns int (STKB_OK = 0); on failure stkb_last_error()
 * returns a thread-local message.  Host buffers belong to the caller; device
 * buffers, streams, CUDA graphs and tensor maps belong to the domain.  Calls on
 * one domain must be serialised by the caller (one domain per host thread), as
 * the reference's single-threaded driver does.
 */
#ifndef STKB200_H
#define STKB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STKB_ABI_VERSION 1

/* status codes */
#define STKB_OK 0
#define STKB_ERR_ARG 1         /* bad argument (maps to ExecutionError/PlanError) */
#define STKB_ERR_CUDA 2        /* CUDA runtime/driver failure */
#define STKB_ERR_UNSUPPORTED 3 /* form/radius/dtype not provided by a tuned kernel */
#define STKB_ERR_STATE 4       /* call out of order */

/* element types: identical to the STG1 dtype codes, grids.py:13-14 */
#define STKB_F32 1
#define STKB_F64 2

/* map kinds */
#define STKB_MAP_STAR 1 /* dst = (sum_k c_k * src[o_k]) [/ divisor], star offsets, radius <= 4 */
#define STKB_MAP_WAVE 2 /* dst = a*src[0] + b*prev[0] + vel[0] * (sum_k c_k * src[o_k]) */
#define STKB_MAP_BOX 4  /* dst = (sum over the dense (2R+1)^3 cube c[dz][dy][dx] * src[o]) [/ divisor],
                           R <= 2: box, j3d27pt-style and "other" shapes inside the cube */
#define STKB_MAP_EXPR 3 /* any kernel: bytecode evaluated in float64, parse order,
                           one rounding per store (bit-identical to run_target,
                           executor.py:267-286) */
#define STKB_MAP_XSTAR 5 /* exact star: dst = ((c0*src[0] + c_1*src[o_1]) + ... ) [/ divisor] in
                            float64 with the terms in the corpus order (centre, then the star
                            offsets sorted), one rounding per store: bit-identical to run_target
                            at streaming speed; 3-D, radius 1..4, coef layout as STAR */
#define STKB_MAP_XWAVE 6 /* exact acoustic wave: dst = (wave_a*src[0] - prev[0]) + vel[0] * (coef[0]*src[0]
                            + coef[1]*S_1 + ... + coef[R]*S_R), S_m = the six +-m axis taps of src summed
                            d0-, d0+, d1-, d1+, d2-, d2+; float64 in that order, one rounding per store
                            (the c3 program as run_target evaluates it); 3-D, radius 1..4 */

#define STKB_MAP_XBOX 7  /* exact dense box: dst = ((c0*src[0] + c_1*src[o_1]) + ... ) [/ divisor] over every
                            offset of the (2R+1)^3 cube, centre first and the rest sorted (d0, d1, d2):
                            the corpus box / j3d27pt form, float64 in that order, one rounding per
                            store (bit-identical to run_target); 3-D, radius 1..2, box_coef layout */

/* step-program execution precision for STAR/WAVE maps */
#define STKB_PREC_FAST 0 /* accumulate in the grid dtype with FMA (tolerance-checked) */

/* EXPR bytecode opcodes (5 int32 words per instruction: op, a, b, c, d) */
#define STKB_OP_CONST 1    /* push consts[a] */
#define STKB_OP_READ 2     /* push (double) grid_arg[a][p + (b, c, d)] */
#define STKB_OP_LOCAL 3    /* push locals[a] */
#define STKB_OP_ADD 4
#define STKB_OP_SUB 5
#define STKB_OP_MUL 6
#define STKB_OP_DIV 7
#define STKB_OP_NEG 8
#define STKB_OP_SETLOCAL 9 /* locals[a] = pop */
#define STKB_OP_STORE 10   /* grid_arg[a][p + (b, c, d)] = (T) pop */
#define STKB_EXPR_MAX_ARGS 8
#define STKB_EXPR_MAX_LOCALS 16
#define STKB_EXPR_MAX_STACK 32

typedef struct stkb_domain stkb_domain;

/* One domain = n_grids named grids sharing dtype and one device geometry: the
 * largest interior extents and halo order of the target's grids (GridBuffer,
 * grids.py:20-64; the grids of one target may differ in order and shape,
 * parser.py:681-691 — see stkb_upload_grid).  Device layout is pitched: a row of
 * the contiguous dim d2 starts on a 128-byte boundary and the first interior
 * element of each row sits at `lead` elements (128 bytes) into the row.  1-D grids
 * are one row of one plane, 2-D grids one plane (EXPR maps only for 1-D). */
typedef struct {
    int32_t dtype;    /* STKB_F32 | STKB_F64 */
    int32_t ndim;     /* 1, 2 or 3 */
    int64_t shape[3]; /* interior extents (d0 streaming/slab axis, d1, d2 contiguous) */
    int32_t order;    /* halo width on every side, >= every kernel radius */
    int32_t n_grids;  /* number of named grids (names are 0..n_grids-1) */
    int32_t device;   /* CUDA device ordinal */
    int32_t flags;    /* reserved, 0 */
} stkb_domain_desc;

typedef struct {
    int32_t kind;      /* STKB_MAP_* */
    int32_t radius;    /* STAR/WAVE: star radius 1..4; BOX: 1..2 */
    int32_t src;       /* STAR/WAVE: name read at the star offsets */
    int32_t dst;       /* STAR/WAVE: name written at offset 0 */
    int32_t prev;      /* WAVE: name read at offset 0 (may equal dst: in-place) */
    int32_t vel;       /* WAVE: name read at offset 0 (velocity / kappa) */
    int32_t precision; /* STKB_PREC_FAST */
    int32_t tag;       /* caller's map id, reported by stkb_nonfinite */
    /* STAR/WAVE coefficients: coef[0] = centre; axis a (0=d0,1=d1,2=d2), distance
     * m in 1..radius: coef[1 + a*2*radius + 2*(m-1) + 0] for offset -m,
     *                 coef[1 + a*2*radius + 2*(m-1) + 1] for offset +m. */
    double coef[25];
    double divisor; /* STAR: 0 = none, else the sum is divided by it */
    double wave_a;  /* WAVE */
    double wave_b;  /* WAVE */
    int64_t lo[3];  /* output region box, interior coordinates, half open */
    int64_t hi[3];
    /* EXPR only */
    int32_t n_args;                        /* kernel grid params */
    int32_t args[STKB_EXPR_MAX_ARGS];      /* name bound to each grid param */
    int32_t n_code;                        /* instructions (5 words each) */
    const int32_t *code;
    int32_t n_consts;
    const double *consts;
    /* BOX and XBOX: box_coef[((dz+R)*(2R+1) + (dy+R))*(2R+1) + (dx+R)] (3-D, R <= 2) or
     * box_coef[(dy+R)*(2R+1) + (dx+R)] (2-D, R <= 4) */
    double box_coef[125];
    /* BOX, 3-D, R = 3..4: the (2R+1)^3 coefficients in the same order (copied at add_map) */
    const double *box_coef_ext;
} stkb_map_desc;

/* library */
int stkb_abi_version(void);
const char *stkb_last_error(void);
int stkb_device_count(int32_t *count);

/* domain lifetime and layout */
int stkb_domain_create(const stkb_domain_desc *desc, stkb_domain **out);
int stkb_domain_destroy(stkb_domain *dom);
int stkb_layout(const stkb_domain *dom, int64_t *pitch_elems, int64_t *plane_elems,
                int64_t *lead_elems, int64_t *buffer_elems);
/* Raw device pointer of the buffer bound to `name`.  Handing it out marks that buffer
 * "written from outside" (halo flag and fused-sweep scratch are re-derived at the next
 * stkb_run*).  Writes through a pointer kept across runs must be followed by
 * stkb_mark_dirty(name) (or a fresh stkb_device_ptr) before the next stkb_run*, or the
 * kernels may read a stale "halo is zero" flag. */
int stkb_device_ptr(stkb_domain *dom, int32_t name, void **dptr);
int stkb_mark_dirty(stkb_domain *dom, int32_t name);
int stkb_set_stream(stkb_domain *dom, void *cuda_stream); /* NULL = domain's own */
int stkb_zero(stkb_domain *dom, int32_t name);            /* whole buffer (halo, padding) = 0, async */

/* host <-> device, GridBuffer.data layout (C-order, padded, unpitched) */
int stkb_upload(stkb_domain *dom, int32_t name, const void *host_padded);
int stkb_download(stkb_domain *dom, int32_t name, void *host_padded);
int stkb_upload_async(stkb_domain *dom, int32_t name, const void *host_padded);
int stkb_download_async(stkb_domain *dom, int32_t name, void *host_padded);
/* The same for a grid with its own layout: host_padded is C-order with
 * (shape[d] + 2*order) elements per axis (the domain's ndim axes); shape[d] <= the
 * domain's extents and order <= the domain's order.  Its interior origin is the
 * domain's; after an upload every device cell outside its padded box is +0.0.
 * sync != 0 waits for the copy. */
int stkb_upload_grid(stkb_domain *dom, int32_t name, const void *host_padded, const int64_t *shape,
                     int32_t order, int32_t sync);
int stkb_download_grid(stkb_domain *dom, int32_t name, void *host_padded, const int64_t *shape,
                       int32_t order, int32_t sync);

/* step program: a sequence of maps and swaps replayed `steps` times */
int stkb_program_reset(stkb_domain *dom);
int stkb_program_add_map(stkb_domain *dom, const stkb_map_desc *map);
int stkb_program_add_swap(stkb_domain *dom, int32_t a, int32_t b);
int stkb_run(stkb_domain *dom, int64_t steps); /* CUDA-graph replay, async */
int stkb_run_once(stkb_domain *dom);             /* one step, direct launches (ncu-friendly) */
int stkb_sync(stkb_domain *dom);
int stkb_elapsed_ms(stkb_domain *dom, double *ms); /* device time of the last stkb_run */
int stkb_launches(stkb_domain *dom, int64_t *count); /* kernels launched by the last stkb_run */
/* how the last stkb_run executed: 0 = one launch per map and step (CUDA graphs), 1 = fused
 * two-step sweeps (stkb_set_fused_steps), 2 = multi-step launches (stkb_set_multi_steps) */
int stkb_run_mode(const stkb_domain *dom, int32_t *mode);
int stkb_binding(const stkb_domain *dom, int32_t name, int32_t *buffer);
int stkb_nonfinite(stkb_domain *dom, int32_t tag, int32_t *flag); /* sticky; clears it */

/* Fine-grained control for the multi-GPU z-slab driver: launch program map
 * `map_index` restricted to interior d0 planes [lo0, hi0) on the domain's
 * current stream; apply a name swap now; address a contiguous run of d0
 * planes (interior index z0, may be negative for halo planes) of the buffer a
 * name is bound to, for halo exchange over NCCL / peer memory. */
int stkb_launch_map(stkb_domain *dom, int32_t map_index, int64_t lo0, int64_t hi0);
/* One launch over several disjoint d0 ranges; the first n_signal ranges are
 * scheduled first and every stored item of them adds 1 to the map's signal
 * counter (*signal_items = how much this launch adds once they are all stored).
 * The counter only grows (it is never reset, so a waiter can never see a stale
 * value): the caller keeps the running sum and stkb_stream_wait_signal makes
 * `stream` (e.g. the halo-exchange stream) wait, without occupying an SM,
 * until the counter reaches it (cyclic >= comparison). */
int stkb_launch_map_ranges(stkb_domain *dom, int32_t map_index, int32_t n_ranges, const int64_t *lo0,
                           const int64_t *hi0, int32_t n_signal, int32_t *signal_items);
int stkb_stream_wait_signal(stkb_domain *dom, void *stream, int32_t map_index, int32_t value);
/* Zero map `map_index`'s signal counter on `stream` (NULL = the domain's): a caller that resets
 * it before every launch waits for that launch's own signal_items, so the same wait value
 * repeats every step and the step can be captured into a CUDA graph and replayed. */
int stkb_reset_signal(stkb_domain *dom, int32_t map_index, void *stream);
int stkb_set_max_ctas(stkb_domain *dom, int32_t ctas); /* 0 = one CTA per SM (leave SMs for NCCL) */

/* Two time steps per d0 sweep (temporal blocking, on by default): when the step
 * program is the Jacobi ping-pong `v = S(u); swap(u, v)` of a fast 3-D STAR map of
 * radius <= 2 (executor.py:267-286 semantics), stkb_run of n >= 4 steps runs
 * (n - 2) / 2 fused sweeps u(t+2) = S(S(u(t))) — v(t+1) stays in registers — and
 * the last 2..3 steps singly, so every grid ends with exactly the single-step
 * kernel's values (bit for bit; the fused sweep keeps each step's FMA order).  It
 * allocates one scratch grid; u's name rotates between its buffer and the scratch
 * (stkb_binding may then report buffer index n_grids).  Such a run also launches one
 * small check kernel (are v's frozen values next to the region all zero? then the
 * sweeps need not stage them): stkb_launches counts it.  enable = 0 turns it off. */
int stkb_set_fused_steps(stkb_domain *dom, int32_t enable);

/* Several time steps per launch for small grids (on by default): when the step program
 * is the Jacobi ping-pong `v = S(u); swap(u, v)` of a fast 3-D STAR map and the grid has
 * at most max_points interior points (0 keeps the current limit, 2^25 by default),
 * stkb_run launches up to 64 steps at a time; a grid barrier inside the kernel separates
 * the steps (a cooperative launch: all CTAs resident).  Every grid ends bit-identical to
 * single steps.  enable = 0 turns it off. */
int stkb_set_multi_steps(stkb_domain *dom, int32_t enable, int64_t max_points);

/* Let `device` read and write `peer`'s memory (cudaDeviceEnablePeerAccess; already
 * enabled is fine).  Used to wire in-process slab domains on different GPUs
 * (slabs.connect_local, the peer-pull probe); IPC-opened memory does not need it. */
int stkb_enable_peer(int32_t device, int32_t peer);

/* Bring the per-buffer halo flags up to date after outside writes (normally done by the
 * next uncaptured launch): call before capturing launches into a CUDA graph so the captured
 * kernels can read zero halos through interior-only tensor maps. */
int stkb_prepare(stkb_domain *dom);

/* Fused halo exchange over NVLink peer memory (z-slab neighbours, one process
 * per GPU).  Each rank exports its buffers and its 2-slot flag array with CUDA
 * IPC handles (64 bytes), opens its neighbours' with stkb_ipc_open and
 * registers them with stkb_set_peer (side 0 = lower neighbour, rank-1; side 1 =
 * upper, rank+1; buffer i of the neighbour pairs with my buffer i).
 * stkb_launch_map_pull runs a streaming map over its whole box; its TMA
 * producer reads the src planes beyond the slab (q < 0, q >= n0) straight from
 * the neighbours' buffers over NVLink instead of from this slab's halo — the
 * halo exchange IS the kernel's own loads, no copy and no extra kernel.  Ranks
 * count their pulling launches; launch c is bracketed by stkb_peer_wait(c-1)
 * (both neighbours finished launch c-1: the planes I read are final) and
 * stkb_peer_signal(c) (a fenced stream write into each neighbour's flag, so a
 * neighbour's launch c+1 cannot overwrite planes my launch c still reads) —
 * stream memory operations only: no kernel ever waits on another.  A flag word
 * encodes "launch v done" as the bits {v mod 3, (v-1) mod 3}, so the values repeat
 * every three launches and a captured CUDA graph of the step can be replayed;
 * callers must keep the launch count identical on every rank (one counted launch
 * per map per step).  stkb_peer_fetch_halo copies the neighbours' boundary planes into this
 * slab's halo planes (after the last step, to return consistent slabs). */
int stkb_launch_map_pull(stkb_domain *dom, int32_t map_index);
int stkb_peer_fetch_halo(stkb_domain *dom, void *stream, int32_t planes);
int stkb_buffer_ipc_handle(stkb_domain *dom, int32_t buffer, void *handle64);
int stkb_flags_ipc_handle(stkb_domain *dom, void *handle64);
int stkb_buffer_ptr(stkb_domain *dom, int32_t buffer, void **dptr);
int stkb_flags_ptr(stkb_domain *dom, void **dptr);
int stkb_ipc_open(int32_t device, const void *handle64, void **dptr);
int stkb_ipc_close(int32_t device, void *dptr);
int stkb_set_peer(stkb_domain *dom, int32_t side, int32_t n_bufs, void *const *bufs, void *flags, int64_t peer_n0);
int stkb_peer_signal(stkb_domain *dom, void *stream, int32_t value);
int stkb_peer_wait(stkb_domain *dom, void *stream, int32_t value);
int stkb_apply_swap(stkb_domain *dom, int32_t a, int32_t b);
int stkb_plane_span(stkb_domain *dom, int32_t name, int64_t z0, int64_t nplanes, void **dptr,
                    int64_t *bytes);

/* Compatibility entry with the reference C-ABI's semantics (serial.py:126-208):
 * upload every grid, run the program `iters` times, download every grid under
 * its final name, synchronously.  host[i] is GridBuffer.data of name i. */
int stkb_run_target(stkb_domain *dom, void *const *host, int64_t iters);

/* device-side comparison (grids.py:163-174): max |a-b|, sum (a-b)^2, argmax,
 * max |a| over the interior of two names (a is the reference side). */
int stkb_compare(stkb_domain *dom, int32_t a, int32_t b, double *max_err, double *sum_sq,
                 int64_t *worst_flat, double *scale);

#ifdef __cplusplus
}
#endif
#endif /* STKB200_H */
