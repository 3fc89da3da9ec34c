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
    FMM_ERR_NCCL = 6       /* an NCCL call of the multi-GPU driver failed (or libnccl is missing) */
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

/* The two halves of fmm_build, for the multi-GPU path, where remote LET
 * cells are grafted between the tree and the traversal:
 * fmm_build_tree: R2-R7 only (keys, sort, tree, geometry); synchronises `stream`.  Discards
 *   grafted LETs and lists of an earlier build.
 * fmm_dtt: dual tree traversal (R8-R10, §II-C).  remote == 0: from (root,
 *   root), replacing earlier lists; remote != 0: from (root, r) for the root r of every LET
 *   grafted by fmm_let_graft, appended to the lists of the last fmm_dtt.  Synchronises.
 *   FMM_ERR_STATE if the traversal needs children of a remote cell that were not exported.
 *   The traversal is organised by target cell (default): each target's lists come out
 *   grouped, in a deterministic order (by traversal generation; R10 fixes the set, and
 *   fmm_copy_lists returns the canonical ascending order); FMM_DTT=bfs selects the
 *   breadth-first traversal whose lists fmm_lists sorts into ascending order.
 * fmm_lists: finishes the lists (CSR by target): the local ones followed, per target, by the
 *   sources found in each remote traversal (graft order), and the P2P source runs.
 * fmm_build(pos, n) == fmm_build_tree + fmm_dtt(0) + fmm_lists. */
fmm_status fmm_build_tree(fmm_ctx* ctx, const void* pos, int64_t n, void* stream);
/* fmm_set_root_bounds: later builds take the R2 root cube from these bounds (HOST [6]: lo xyz,
 *   hi xyz) instead of the particles' own min/max -- for a Morton-range partition, the global
 *   box, so every rank's local tree is a subtree of one global octree (HOT, PAPER.md:83-92;
 *   DESIGN.md §2 reading 9).  NULL restores the default.  A build whose particles lie outside
 *   the bounds returns FMM_ERR_ARG. */
fmm_status fmm_set_root_bounds(fmm_ctx* ctx, const double* bounds);
fmm_status fmm_dtt(fmm_ctx* ctx, int remote, void* stream);
fmm_status fmm_lists(fmm_ctx* ctx, void* stream);

/* The two halves of fmm_evaluate:
 * fmm_upward: gathers q (device [n]) into the sorted bodies and runs P2M/M2M (R12, R13)
 *   over the local tree; pos must be the pointer of the last build.
 * fmm_interact: M2L (R14) and P2P (R17) over the lists -- including grafted LET sources,
 *   whose data must have arrived by fmm_let_unpack -- then L2L/L2P (R15, R16) and the
 *   output scatter (R18).  phi [n], grad [n][3] device, caller order.  Asynchronous.
 * fmm_evaluate(pos, q, phi, grad) == fmm_upward + fmm_interact. */
fmm_status fmm_upward(fmm_ctx* ctx, const void* pos, const void* q, void* stream);
fmm_status fmm_interact(fmm_ctx* ctx, void* phi, void* grad, void* stream);

/* fmm_evaluate: potentials and gradients for the last build (R12-R18).
 *   pos  the same device pointer passed to the last fmm_build (else FMM_ERR_STATE)
 *   q    device [n] charges;  phi device [n];  grad device [n][3] (grad = +grad(phi), R1)
 * Outputs are in the caller's original particle order.  Asynchronous on `stream`. */
fmm_status fmm_evaluate(fmm_ctx* ctx, const void* pos, const void* q, void* phi, void* grad, void* stream);

/* fmm_solve: fmm_build followed by fmm_evaluate on the same device buffers, in one call, so
 * the library can overlap independent passes: P2M/M2M (R12, R13; they need the tree and q
 * only) run on the library's aux stream while the dual tree traversal and the list grouping
 * (R9, R10) run on `stream`; L2L/L2P run on the aux stream while P2P runs on `stream`.  The
 * results are identical to fmm_build + fmm_evaluate.  pos device [n][3], q device [n],
 * phi device [n], grad device [n][3] (prec type, caller order); n as in fmm_build.
 * Synchronises `stream` once (the build's host round trips); the evaluation is enqueued
 * asynchronously and joined back into `stream`.  Errors as fmm_build / fmm_evaluate. */
fmm_status fmm_solve(fmm_ctx* ctx, const void* pos, const void* q, int64_t n, void* phi, void* grad, void* stream);

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

/* ---- debug stage entry points: the hot kernels on a CALLER-SUPPLIED tree and
 * interaction list, so each stage can be checked against an independent implementation (the
 * parity tests feed the oracle's tree and lists).  Every pointer in the view is DEVICE memory;
 * cells are indexed 0..ncell-1 in the caller's order; bodies are in the caller's (sorted) order,
 * cell c owning bodies [body_begin[c], body_begin[c] + body_count[c]).
 *   n, ncell          bodies and cells (n <= the context's n_max)
 *   pos, q            [n][3], [n] in the context precision (P2P)
 *   body_begin, body_count, child_count   u32 [ncell] (P2P; leaves = child_count 0, their body
 *                     ranges disjoint)
 *   center            fp64 [ncell][3] expansion centres (M2L)
 *   level             int32 [ncell] tree level of each cell (M2L; sets the power-of-two operand
 *                     scale rho = 2^(E - level), 2^E >= 2 root_half_width; exact)
 *   M                 fp64 [ncell][ncoef] multipoles, R11 order (M2L)
 *   root_half_width   the root cube's half-width h (M2L)
 * Pair lists are DEVICE u32 [n_pairs][2] (target, source) cell pairs in ascending order (R10);
 * FMM_ERR_ARG if out of order or naming a cell >= ncell.  Both calls synchronise `stream` and
 * leave the context without a build (fmm_evaluate then returns FMM_ERR_STATE).
 * fmm_debug_p2p: phi [n], grad [n][3] (device, context precision, the view's body order) = the
 *   near field of R17 over the P2P pairs (§II-A "P2P"); bodies of leaves without
 *   pairs get 0.
 * fmm_debug_m2l: L (device fp64 [ncell][ncoef], overwritten) = sum over the M2L pairs (A <- B)
 *   of R14 ("M2L"); cells without pairs get 0. */
typedef struct {
    int64_t n, ncell;
    const void* pos;
    const void* q;
    const uint32_t* body_begin;
    const uint32_t* body_count;
    const uint32_t* child_count;
    const double* center;
    const int32_t* level;
    const double* M;
    double root_half_width;
} fmm_tree_view;
fmm_status fmm_debug_p2p(fmm_ctx* ctx, const fmm_tree_view* view, const uint32_t* p2p, int64_t n_pairs, void* phi,
                         void* grad, void* stream);
fmm_status fmm_debug_m2l(fmm_ctx* ctx, const fmm_tree_view* view, const uint32_t* m2l, int64_t n_pairs, double* L,
                         void* stream);

/* fmm_debug_check: memory checking without compute-sanitizer.  In a context created with the
 * environment variable FMM_GUARD=1 every device buffer has a 4 KiB guard zone after its usable
 * bytes; this call synchronises the device and verifies every live guard zone of the context's
 * device: FMM_ERR_STATE (and *nbad > 0, HOST, may be NULL) if any was overwritten.  FMM_POISON=1
 * fills fresh allocations with 0xFF bytes (NaN / huge values) so reads of unwritten memory
 * surface in the results. */
fmm_status fmm_debug_check(fmm_ctx* ctx, int64_t* nbad);

/* ---- multi-GPU: Morton-range partition (§II-B,
 * Eq. (1)).  The collectives between these calls are the caller's (the
 * Python layer uses torch.distributed over NCCL); every step on the data runs here.
 * fmm_bounds: exact fp64 min/max of pos (device [n][3], ctx precision) into out (HOST [6]:
 *   lo xyz, hi xyz; +inf/-inf when n == 0).  Synchronises.  FMM_ERR_NONFINITE on NaN/Inf.
 * fmm_part_keys: 63-bit Morton keys (R3, R4) of pos under the root cube (R2) of the given
 *   GLOBAL bounds (HOST [6], the all-reduce of every rank's fmm_bounds); keys device [n].
 * fmm_part_histogram: hist (device [2^bits] fp64, overwritten): every key whose top
 *   prefix_bits bits equal prefix adds w[i] (device [n] fp32, NULL = 1) at the bin of its
 *   next `bits` bits; prefix_bits = 0 takes every key.  1 <= bits <= 24, prefix_bits + bits
 *   <= 63.  The caller all-reduces it and refines the splitters bin by bin.
 * fmm_part_pack: destination rank of particle i = number of splitters (HOST [nranks-1]
 *   ascending keys) <= key[i]; writes the particles grouped by destination, stable within a
 *   group, to out_pos [n][3] / out_q [n] (device, ctx precision) with global ids
 *   out_gid [n] = gid_base + i (device int64), and counts (HOST [nranks]) per destination.
 *   Synchronises.  1 <= nranks <= 256. */
fmm_status fmm_bounds(fmm_ctx* ctx, const void* pos, int64_t n, double* out, void* stream);
fmm_status fmm_part_keys(fmm_ctx* ctx, const void* pos, int64_t n, const double* bounds, uint64_t* keys, void* stream);
fmm_status fmm_part_histogram(fmm_ctx* ctx, const uint64_t* keys, const float* w, int64_t n, uint64_t prefix,
                              int prefix_bits, int bits, double* hist, void* stream);
fmm_status fmm_part_pack(fmm_ctx* ctx, const void* pos, const void* q, const uint64_t* keys, int64_t n,
                         const uint64_t* splitters, int nranks, int64_t gid_base, void* out_pos, void* out_q,
                         int64_t* out_gid, int64_t* counts, void* stream);

/* ORB multisection: particles carry a group id (device
 * int32 [n], the rank range they will be split into); coordinates are the R3 21-bit
 * quantised coordinates recovered from keys (fmm_part_keys).
 * fmm_orb_histogram: hist (device [ngroups][2^bits] fp64, overwritten) += w (NULL = 1) of every
 *   particle of group g with axis[g] >= 0 whose coordinate along axis[g] (0 x, 1 y, 2 z) has
 *   its top prefix_bits bits equal to prefix[g], at the bin of its next `bits` bits
 *   (HOST arrays axis, prefix [ngroups]; 1 <= bits <= 16, prefix_bits + bits <= 21).
 * fmm_orb_split: particles of group g with axis[g] >= 0 and coordinate >= cut[g] move to
 *   group right[g] (HOST arrays [ngroups]).
 * fmm_part_pack_dest: as fmm_part_pack with the destination rank given per particle
 *   (dest, device int32 [n], values < nranks).  All three synchronise. */
fmm_status fmm_orb_histogram(fmm_ctx* ctx, const uint64_t* keys, const float* w, const int32_t* group, int64_t n,
                             int ngroups, const int32_t* axis, const uint32_t* prefix, int prefix_bits, int bits,
                             double* hist, void* stream);
fmm_status fmm_orb_split(fmm_ctx* ctx, const uint64_t* keys, int32_t* group, int64_t n, int ngroups,
                         const int32_t* axis, const uint32_t* cut, const int32_t* right, void* stream);
fmm_status fmm_part_pack_dest(fmm_ctx* ctx, const void* pos, const void* q, const int32_t* dest, int64_t n,
                              int nranks, int64_t gid_base, void* out_pos, void* out_q, int64_t* out_gid,
                              int64_t* counts, void* stream);

/* ---- multi-GPU: local essential tree (§II-C).
 * Sender-initiated: every rank publishes a cover of its local tree, every sender exports to
 * each receiver the part of its tree the receiver's traversal can need (let.cu states the
 * rule), the receiver grafts the parts after its local cells and traverses them.
 * fmm_let_cover: the cover of this rank's tree into cover (HOST [FMM_LET_MAX_COVER][8]:
 *   kind (0 summary, 1 guard), radius, box lo xyz, box hi xyz) and its entry count.
 *   Needs fmm_build_tree.  Synchronises.
 * fmm_let_plan: which cells and bodies go to `peer` (any id >= 0 the caller chooses) given
 *   that peer's cover; returns the byte sizes of its structure and data messages.  Needs
 *   fmm_build_tree.  Synchronises.
 * fmm_let_pack_struct: writes the structure message for `peer` (geometry, child/body
 *   counts, sender cell ids, body positions) to dst (device, struct_bytes, 16-B aligned).
 * fmm_let_pack_data: writes the data message (fp64 multipoles, body charges) to dst
 *   (device, data_bytes); needs fmm_upward.
 * fmm_let_graft: appends the npeers received structure messages (device pointers src[k] of
 *   bytes[k] bytes, HOST arrays) after the local cells, bodies and the LETs grafted earlier
 *   in this build (fragments may arrive one by one: PAPER.md:129-149, the per-message `when`);
 *   then fmm_dtt(remote = 1), which traverses the LETs grafted since its last call, and
 *   fmm_lists once all have arrived.  Synchronises.
 * fmm_let_unpack: writes npeers received data messages into grafted LETs first ..
 *   first + npeers - 1 (graft order); call after fmm_upward, before fmm_interact.
 * fmm_let_remote: grafted LET k: first cell index, cell and body counts, and (HOST [ncell],
 *   may be NULL) the sender's cell index of each grafted cell (parity tests). */
#define FMM_LET_MAX_COVER 73
#define FMM_LET_ABSENT 0xFFFFFFFFu
fmm_status fmm_let_cover(fmm_ctx* ctx, double* cover, int* ncover, void* stream);
fmm_status fmm_let_plan(fmm_ctx* ctx, int peer, const double* cover, int ncover, int64_t* struct_bytes,
                        int64_t* data_bytes, void* stream);
fmm_status fmm_let_pack_struct(fmm_ctx* ctx, int peer, void* dst, void* stream);
fmm_status fmm_let_pack_data(fmm_ctx* ctx, int peer, void* dst, void* stream);
fmm_status fmm_let_graft(fmm_ctx* ctx, int npeers, const void* const* src, const int64_t* bytes, void* stream);
fmm_status fmm_let_unpack(fmm_ctx* ctx, int first, int npeers, const void* const* src, const int64_t* bytes,
                          void* stream);
fmm_status fmm_let_remote(const fmm_ctx* ctx, int k, int64_t* base, int64_t* ncell, int64_t* nbody, uint32_t* orig);

/* fmm_work: Eq. (1) weights of the last build for the next partition,
 *   w[i] = l_i + alpha * r_i into w (device [n] fp32, caller order), where l_i / r_i count the
 *   work of particle i's interaction lists with local / grafted-LET sources: 1 per P2P source
 *   body of its leaf, c_m2l / |C| per M2L pair of its leaf or any ancestor C (c_m2l = cost of
 *   one M2L pair in P2P interactions).  lr_sums (HOST [2], may be NULL): sum of l and of r;
 *   synchronises when given.  Needs fmm_lists. */
fmm_status fmm_work(fmm_ctx* ctx, double c_m2l, float alpha, float* w, double* lr_sums, void* stream);

/* ---- multi-GPU driver (SURVEY §8(b) fmm_create_dist / fmm_set_weights, §8(e), §8(f) f1, f3, f4).
 * One context per rank; the LIBRARY owns the communicator, the partition arithmetic and every
 * exchange of a distributed step (dist.cu states the step with its PAPER.md passages).
 * Transports: NCCL (one rank per process or thread; libnccl is dlopen'ed -- the copy the process
 * already loaded, e.g. torch's, else libnccl.so.2 -- so this library has no link-time NCCL
 * dependency; failures return FMM_ERR_NCCL), or an in-process group of K ranks, one host thread
 * per rank, for several GPUs of one process or K ranks sharing one GPU in the parity tests
 * (host barriers swap device pointers and events; no kernel ever waits for another rank's).
 * fmm_group_create / destroy: the in-process group (destroy after every member context).
 * fmm_dist_unique_id: a fresh 128-byte ncclUniqueId (rank 0 makes it, the caller broadcasts it).
 * fmm_create_dist: as fmm_create, plus nranks, rank, and EXACTLY ONE of nccl_unique_id (HOST
 *   128 B) / group; partitioner FMM_PART_MORTON (Morton-curve ranges weighted by Eq. (1),
 *   north_star) or FMM_PART_ORB (multisection).  n_local_max bounds the
 *   particles a rank may own after the partition (FMM_ERR_ARG from fmm_dist_solve otherwise).
 *   Every rank must call the same sequence of fmm_dist_* calls.
 * fmm_set_weights: partition weights (DEVICE fp32 [n], caller order; NULL clears) for the next
 *   fmm_dist_solve with the same n; default 1 (Eq. (1) at the first step).
 * fmm_dist_set_alpha: Eq. (1) w = l + alpha r for the weights this rank computes;
 *   c_m2l > 0 overrides the cost of one M2L pair in P2P interactions (default: the kernel's
 *   FP32 lane-op ratio).  fmm_dist_tune_alpha: golden-section search of log alpha over [lo, hi]
 *   by the measured step runtime ("optimized over the time steps"); lo = hi = 0 stops
 *   it (alpha stays at the best probe).
 * fmm_dist_solve: ONE distributed step on this rank's particles pos [n][3], q [n] (DEVICE, context
 *   precision; their global ids are gid_base + i): partition (weights: with reuse_weights the
 *   Eq. (1) weights this context computed in its previous step if n is unchanged, else those of
 *   fmm_set_weights, else 1), particle exchange, local tree, LET exchange overlapped with the
 *   traversal, interactions, results back.  phi [n], grad [n][3] (DEVICE) in the caller's order.
 *   Synchronises `stream`; every stream the step used is joined into it before return.
 * fmm_dist_get_stats: the last step's bounds, alpha, byte counts, local size, work sums.
 * fmm_dist_local: the last step's local particles' global ids (HOST int64 [n_local], may be NULL)
 *   and the peers whose LETs were grafted, in graft order (HOST int32 [nranks], -1 padded).
 *   fmm_get_counts / fmm_copy_* / fmm_let_remote on the same context describe the local tree.
 * fmm_dist_weights: the Eq. (1) weights of the last step for the caller's particles (HOST fp32 [n]).
 * fmm_dist_orb_boxes: ORB boxes of the last step (HOST int32 [nranks][6], quantised lo xyz, hi xyz).
 * fmm_dist_timeline: with fmm_set_timing on, per span of the last step (names by
 *   fmm_dist_timeline_name) its start and end in ms after the step began (CUDA events on the
 *   stream the span ran on; -1 if the span did not run); ms HOST [cap][2]. */
typedef struct fmm_group fmm_group;
typedef struct {
    double bounds[6];
    double alpha, c_m2l;
    int64_t n_local;
    int32_t npeers;
    int32_t tuner_probes;
    int64_t let_struct_bytes, let_data_bytes, part_bytes;
    double work_local, work_remote;
    int32_t tuner_converged, pad;
    double tuner_best;
} fmm_dist_stats;
#define FMM_PART_MORTON 0
#define FMM_PART_ORB 1
fmm_status fmm_group_create(int nranks, fmm_group** out);
fmm_status fmm_group_destroy(fmm_group* group);
fmm_status fmm_dist_unique_id(void* out);
fmm_status fmm_create_dist(int64_t n_local_max, int p, double theta, int ncrit, int prec, int device, int nranks,
                           int rank, const void* nccl_unique_id, fmm_group* group, int partitioner, fmm_ctx** out);
fmm_status fmm_set_weights(fmm_ctx* ctx, const float* w, int64_t n);
fmm_status fmm_dist_set_alpha(fmm_ctx* ctx, double alpha, double c_m2l);
fmm_status fmm_dist_tune_alpha(fmm_ctx* ctx, double lo, double hi, double tol);
fmm_status fmm_dist_solve(fmm_ctx* ctx, const void* pos, const void* q, int64_t n, int64_t gid_base,
                          int reuse_weights, void* phi, void* grad, void* stream);
fmm_status fmm_dist_get_stats(const fmm_ctx* ctx, fmm_dist_stats* out);
fmm_status fmm_dist_local(const fmm_ctx* ctx, int64_t* gid, int32_t* peers);
fmm_status fmm_dist_weights(const fmm_ctx* ctx, float* w);
fmm_status fmm_dist_orb_boxes(const fmm_ctx* ctx, int32_t* boxes);
fmm_status fmm_dist_timeline(const fmm_ctx* ctx, double* ms, int cap, int* n);
const char* fmm_dist_timeline_name(int i);

/* ---- the driver's host logic, callable without a device (CPU tests of the partition rules):
 * fmm_splitters: the K-1 Morton splitters (rank j takes keys >= splitter j) by histogram
 *   refinement ("each bit of the key is examined at each step"): `bits` key bits per
 *   round until the bin holding the j/K weight quantile carries <= tol/K of the total.  fn returns
 *   the GLOBAL weights of the keys under each of nprefix prefixes (top prefix_bits bits) binned by
 *   their next `bits` bits, into hist [nprefix][2^bits]; nonzero return = failure.
 * fmm_orb_plan: ORB multisection through the two callbacks (histogram of the
 *   quantised coordinate along axis[g] for every group g with axis[g] >= 0, and the split of the
 *   groups at cut[g] into right[g]); boxes HOST int32 [nranks][6].
 * fmm_alpha_tuner_*: the golden-section alpha search fmm_dist_tune_alpha runs (next() before a
 *   step's weights, report(runtime) after the step). */
typedef int (*fmm_hist_fn)(void* user, const uint64_t* prefixes, int nprefix, int prefix_bits, int bits, double* hist);
typedef int (*fmm_orb_hist_fn)(void* user, const int32_t* axis, const uint32_t* prefix, int prefix_bits, int bits,
                               double* hist);
typedef int (*fmm_orb_split_fn)(void* user, const int32_t* axis, const uint32_t* cut, const int32_t* right);
fmm_status fmm_splitters(int nranks, int bits, double tol, fmm_hist_fn fn, void* user, uint64_t* splitters);
fmm_status fmm_orb_plan(int nranks, int bits, fmm_orb_hist_fn hist, fmm_orb_split_fn split, void* user,
                        int32_t* boxes);
typedef struct fmm_alpha_tuner fmm_alpha_tuner;
fmm_status fmm_alpha_tuner_create(double lo, double hi, double tol, fmm_alpha_tuner** out);
double fmm_alpha_tuner_next(const fmm_alpha_tuner* t);
fmm_status fmm_alpha_tuner_report(fmm_alpha_tuner* t, double runtime);
fmm_status fmm_alpha_tuner_state(const fmm_alpha_tuner* t, int* converged, double* best, int* nhist, double* hist,
                                 int cap);
fmm_status fmm_alpha_tuner_destroy(fmm_alpha_tuner* t);

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
