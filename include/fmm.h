/*
 * fmm.h -- C-ABI of the B200-native 3D Laplace FMM hot path (libfmm.so).
 *
 * The path (BASELINE.json north_star): Morton keys and radix sort,
 * level-by-level octree with tight cell boxes, P2M/M2M upward pass, dual tree traversal
 * emitting M2L and P2P lists, the M2L and P2P kernels, L2L/L2P downward pass.
 * Paper: §II-A (the six operators and their data flow)
 * §II-B (Morton keys, tight bounding boxes, MAC), §II-C (local tree,
 * post-order P2M/M2M, dual tree traversal, pre-order L2L/L2P), Table I PAPER.md:153-169.
 * Rules R1-R20 and readings: DESIGN.md §2.
 *
 * Types: plain C only (no CUDA, no torch types).  `stream` is a cudaStream_t passed as
 * void* (NULL = the legacy default stream).  Device pointers are CUDA device addresses.
 *
 * Errors: every call returns an fmm_status; nothing is thrown across the ABI.  A
 * per-context message is available from fmm_last_error() until the next call on that
 * context.  CUDA failures map to FMM_ERR_CUDA.
 *
 * Threading: a context is used by one host thread at a time.
 */
#ifndef FMM_H
#define FMM_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct fmm_ctx fmm_ctx; /* opaque, library-owned */

typedef enum {
    FMM_OK = 0,
    FMM_ERR_ARG = 1,       /* bad argument: n<0 or n>n_max, p outside 1..16, theta outside (0,1),
                              ncrit<1, NULL pointer, precision mismatch */
    FMM_ERR_STATE = 2,     /* call order violated (evaluate before build, pos/n changed since build) */
    FMM_ERR_NONFINITE = 3, /* a position is NaN or Inf */
    FMM_ERR_OOM = 4,       /* device allocation failed */
    FMM_ERR_CUDA = 5,      /* a CUDA runtime error; see fmm_last_error */
    FMM_ERR_NCCL = 6       /* reserved for the multi-GPU layer */
} fmm_status;

typedef enum { FMM_F32 = 0, FMM_F64 = 1 } fmm_prec;

typedef struct {
    int64_t n;                /* particles of the last build */
    int64_t ncell;            /* cells, canonical BFS (level, key) order (R6) */
    int64_t nleaf;
    int64_t depth;            /* deepest level (root = 0) */
    int64_t n_m2l;            /* M2L cell pairs (R9) */
    int64_t n_p2p;            /* P2P leaf pairs (R9) */
    int64_t p2p_interactions; /* sum over P2P pairs of |A| * |B| */
} fmm_counts;

/* fmm_create: allocate a context for up to n_max particles.
 *   p      expansion order P, 1..16 (coefficients |alpha| <= P-1; "order of
 *          multipole/local expansion"; R11)
 *   theta  MAC parameter in (0,1): cell pair accepted for M2L iff (R_A+R_B) < theta*d (R8)
 *   ncrit  maximum particles per leaf, >= 1 (R6)
 *   prec   FMM_F64: every step in fp64.  FMM_F32: fp32 inputs/outputs, P2P and M2L
 *          arithmetic in fp32, keys/geometry/MAC and the P2M/M2M/L2L/L2P expansions in
 *          fp64 (R19; BASELINE.json configs[1] "fp32 (fp64 accumulation of expansions)")
 *   device CUDA device ordinal the context lives on.
 * Ownership: *out is owned by the caller and released by fmm_destroy. */
fmm_status fmm_create(int64_t n_max, int p, double theta, int ncrit, int prec, int device, fmm_ctx** out);
fmm_status fmm_destroy(fmm_ctx* ctx);
const char* fmm_last_error(const fmm_ctx* ctx);

/* fmm_build: tree structure from positions only (R2-R10): bounds and root cube, 63-bit
 * Morton keys, stable radix sort, level-by-level octree, tight geometry, dual tree
 * traversal, canonical M2L/P2P lists.
 *   pos  device, [n][3] row-major, float (F32) or double (F64), 16-B aligned.
 * Synchronises `stream` (it reads per-level counts back to the host).  n == 0 is an
 * FMM_OK no-op (R20).  The positions must stay unchanged until fmm_evaluate. */
fmm_status fmm_build(fmm_ctx* ctx, const void* pos, int64_t n, void* stream);

/* fmm_evaluate: potentials and gradients for the last build (R12-R18).
 *   pos  the same device pointer passed to the last fmm_build (else FMM_ERR_STATE)
 *   q    device [n] charges;  phi device [n];  grad device [n][3] (grad = +grad(phi), R1)
 * Outputs are in the caller's original particle order.  Asynchronous on `stream`. */
fmm_status fmm_evaluate(fmm_ctx* ctx, const void* pos, const void* q, void* phi, void* grad, void* stream);

/* fmm_solve_host: build + evaluate on HOST buffers (pos[n][3], q[n] in; phi[n],
 * grad[n][3] out), host<->device copies included; synchronous.  Pinned host memory is
 * recommended for copy speed but not required. */
fmm_status fmm_solve_host(fmm_ctx* ctx, const void* pos_h, const void* q_h, int64_t n, void* phi_h,
                          void* grad_h, void* stream);

/* ---- introspection (parity tests); destinations are HOST buffers ---------------- */
fmm_status fmm_get_counts(const fmm_ctx* ctx, fmm_counts* out);
/* sorted keys [n] and permutation [n] (perm[k] = original index of the k-th sorted body) */
fmm_status fmm_copy_sorted(const fmm_ctx* ctx, uint64_t* keys, uint32_t* perm);
/* SoA cell arrays [ncell] (any may be NULL): key = level-l prefix key >> 3(21-l) of the
 * member keys; leaves have child_begin = child_count = 0; root parent = -1;
 * bmin/bmax/center [ncell][3], radius [ncell] in fp64 (R7). */
fmm_status fmm_copy_cells(const fmm_ctx* ctx, int32_t* level, uint64_t* key, uint32_t* body_begin,
                          uint32_t* body_count, uint32_t* child_begin, uint32_t* child_count, int32_t* parent,
                          double* bmin, double* bmax, double* center, double* radius);
/* canonical lists: m2l [n_m2l][2], p2p [n_p2p][2] as (target, source) ascending (R10) */
fmm_status fmm_copy_lists(const fmm_ctx* ctx, uint32_t* m2l, uint32_t* p2p);
/* fp64 expansions [ncell][ncoef] after fmm_evaluate (R11 order); either may be NULL */
fmm_status fmm_copy_expansions(const fmm_ctx* ctx, double* M, double* L);

/* ---- timing (bench): per-phase device time from CUDA events recorded on the stream
 * each phase runs on.  enable != 0 turns recording on (small overhead).
 * fmm_phase_times fills up to `cap` entries of ms accumulated since the last reset and
 * returns the number of phases through *n; names via fmm_phase_name. */
fmm_status fmm_set_timing(fmm_ctx* ctx, int enable);
fmm_status fmm_phase_times(fmm_ctx* ctx, double* ms, int cap, int* n, int reset);
const char* fmm_phase_name(int phase);
/* number of kernel launches issued by the library since the last reset (bench claim) */
int64_t fmm_launch_count(fmm_ctx* ctx, int reset);

int fmm_version(void);

#ifdef __cplusplus
}
#endif
#endif
