// common.cuh -- internal definitions shared by the libfmm translation units.
// Product code: never includes or links anything under oracle/ (DESIGN.md §3).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <array>
#include <string>
#include <utility>
#include <vector>

#include "../../include/fmm.h"

#define FMM_MAXP 16
#define FMM_MAXLEVEL 21
#define P2P_BIG_LEAF 128u   // leaves with at least this many bodies take the 4-pairs-per-thread P2P
#define P2P_TINY_LEAF 16u   // leaves with at most this many bodies take the warp-per-leaf P2P

// ---- coefficient indexing (R11: degree n, then alpha_x descending, then alpha_y descending)
__host__ __device__ __forceinline__ int ncoef_of(int P) { return P * (P + 1) * (P + 2) / 6; }
// index of multi-index (a,b,c): ncoef(n) + m(m+1)/2 + c with n = a+b+c, m = b+c
__host__ __device__ __forceinline__ int cidx(int a, int b, int c) {
    int n = a + b + c, m = b + c;
    return ncoef_of(n) + m * (m + 1) / 2 + c;
}

// inverse of cidx: coefficient index -> (a,b,c)
__host__ __device__ __forceinline__ void decode_cidx(int k, int& a, int& b, int& c) {
    int n = 0;
    while (ncoef_of(n + 1) <= k) ++n;
    int r = k - ncoef_of(n);
    int m = 0;
    while ((m + 1) * (m + 2) / 2 <= r) ++m;
    c = r - m * (m + 1) / 2;
    b = m - c;
    a = n - m;
}

// fill a block-shared exponent table (uchar4: a, b, c, degree) for ncoef entries
__device__ __forceinline__ void fill_ex_table(uchar4* ex, int ncoef) {
    for (int k = threadIdx.x; k < ncoef; k += blockDim.x) {
        int a, b, c;
        decode_cidx(k, a, b, c);
        ex[k] = make_uchar4((unsigned char)a, (unsigned char)b, (unsigned char)c, (unsigned char)(a + b + c));
    }
}

// ---- phases for event timing
enum Phase {
    PH_BOUNDS = 0, PH_SORT, PH_TREE, PH_GEOM, PH_DTT, PH_LISTS,
    PH_UP, PH_M2L, PH_P2P, PH_DOWN, PH_COPY, PH_M2L_KERNEL, PH_P2P_KERNEL, PH_COUNT
};

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

// per-peer LET export plan (let.cu): opened / exported flags, compacted cell and body offsets
struct LetPeer {
    DevBuf opened, eflag, eidx, bflag, boff;
    int64_t ncell = 0, nbody = 0;
    bool planned = false;
};
// one grafted remote LET: cells [base, base + ncell), bodies [bbase, bbase + nbody)
struct LetRemote {
    int64_t base, ncell, bbase, nbody;
    int depth;   // deepest level of the sender's tree (bounds the traversal's level count)
};

// CSR lists written by the target-ordered traversal (tct.cu)
struct TcLists {
    DevBuf* off_m;
    DevBuf* src_m;
    DevBuf* off_p;
    DevBuf* src_p;
    int64_t* n_m;
    int64_t* n_p;
    int64_t* est_m;   // capacity estimates for the next run
    int64_t* est_p;
};
// one remote (LET) traversal's lists, concatenated after the local ones by tct_concat
struct TcPart {
    DevBuf off_m, src_m, off_p, src_p;
    int64_t n_m = 0, n_p = 0, est_m = 0, est_p = 0;
};

struct DistState;   // dist.cu: multi-GPU driver state of a context made by fmm_create_dist
void dist_destroy(DistState* d);

struct TimedEvent {
    int phase;
    cudaEvent_t a, b;
};

struct fmm_ctx {
    // configuration
    int64_t n_max = 0;
    int P = 4, ncoef = 20;
    double theta = 0.5;
    int ncrit = 32;
    int prec = FMM_F64;
    bool use_fast_m2l = true;
    bool use_fast_p2p = true;   // fp32 grouped P2P (FMM_P2P_GENERIC=1 disables)
    int p2p_variant = 0;
    int p2p_mutual = 0;         // mutual P2P (p2p_mutual.cu): 0 off, 1 on, 2 auto (mean leaf >= P2P_BIG_LEAF)
    bool mut_ready = false;     // this build's mirror indices / reaction slots are prepared
    DevBuf mut_mir, mut_w, mut_so, mut_slot;
    int m2l_variant = 0;        // fp32 register M2L: 0 mirror-paired f32x2, 1 scalar (FMM_M2L_VARIANT)
    int p2p_np = 2;             // CTA P2P: target pairs per thread (FMM_P2P_NP = 1, 2, 4)        // 0: CTA per leaf over source runs, 1: warp per leaf (FMM_P2P_VARIANT)
    // split multi-GPU interactions (dist.cu): operand layout capacity, first cell to prepare, skip
    // the reduced -> full L expansion, and the remote lists' offsets for the expansion's "no list"
    int64_t m2l_cap = 0, m2l_prep_c0 = 0;
    bool m2l_no_expand = false;
    bool m2l_span_fixed = false;   // m2l_pass keeps m2l_deep as set by the caller (no span reduction)
    const uint64_t* m2l_off2 = nullptr;
    int* m2l_sexp = nullptr;     // per-cell scale exponents of the last register-kernel operand preparation
    bool m2l_deep = false;       // m2l_pass: tree spans > 14 levels, fp32 mode uses the fp64 kernel
    int m2l_part = 0;            // m2l_pass: 0 all, 1 operand preparation only, 2 without it (fmm_solve split)
    int list_sort = 0;           // list grouping: 0 counting scatter + per-segment sorts, 1 one radix sort of the packed pairs (FMM_LIST_SORT)
    bool canonical_m2l = true;   // sort M2L sources within each target on the device (FMM_CANONICAL_M2L=0: skip)
    // aux-stream overlap of the latency-bound passes (FMM_OVERLAP=0: everything on the caller's
    // stream): L2L/L2P run concurrently with P2P; in fmm_solve P2M/M2M also run concurrently with
    // the traversal and list grouping
    bool overlap = true;
    int device = 0;
    int num_sms = 148;
    std::string err;

    // aux stream and the events that order it against the caller's stream
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_up = nullptr, ev_done = nullptr;
    cudaStream_t hp = nullptr;   // high-priority stream for fmm_solve's critical path (FMM_PRIO=0: none)

    // timing
    bool timing = false;
    std::vector<TimedEvent> pending;
    std::vector<cudaEvent_t> event_pool;
    double phase_ms[PH_COUNT] = {0};
    int64_t launches = 0;

    // build state
    const void* built_pos = nullptr;
    int64_t n = 0;
    bool built = false;        // lists ready (fmm_lists)
    bool tree_built = false;   // keys, tree and geometry ready (fmm_build_tree)
    bool evaluated = false;

    // root cube (device): [0..2] lo, [3..5] hi, [6..8] origin, [9] scale, [10] h
    DevBuf root, root_given;
    bool has_root_bounds = false;   // fmm_set_root_bounds: R2 from these bounds, not the particles'
    double root_bounds[6] = {0, 0, 0, 0, 0, 0};
    // sort buffers
    DevBuf key_a, key_b, idx_a, idx_b, sort_counts, scan_tmp, red_tmp;
    uint64_t* d_keys = nullptr;   // sorted keys (points into key_a or key_b)
    uint32_t* d_perm = nullptr;   // perm (points into idx_a or idx_b)
    DevBuf iperm;                 // inverse of d_perm (gather_bodies_q), for the output merge
    DevBuf body;                  // sorted (x,y,z,q): float4 (F32) or double4-like (F64)

    // cells (SoA, BFS order)
    int64_t ncell = 0, nleaf = 0, depth = 0, cell_cap = 0;
    std::vector<int64_t> level_begin;  // host: first cell of each level, size depth+2
    DevBuf c_key, c_level, c_bb, c_bc, c_cb, c_cc, c_parent, c_bmin, c_bmax, c_cr;  // c_cr: double4 (cx,cy,cz,R)
    DevBuf split_tmp, split_cnt;       // per-level temporaries
    DevBuf tree_lb;                    // sync-free build: level starts + overflow flag (device)
    bool tree_fast = true;             // levels from the previous build's sizes (FMM_TREE_FAST=0: off)
    int sort_staged = -1;              // onesweep pass: -1 staged above one wave of tiles, 0 direct, 1 staged
    int64_t tree_prev_depth = -1, tree_prev_ncell = 0, tree_prev_maxw = 0;
    DevBuf leaf_ids;                   // u32 list of leaf cells

    // lists (CSR by target, canonical order): m2l_off[ncell+1] (u64), m2l_src[n_m2l] (u32); p2p likewise.
    // lst_m2l / lst_p2p are the unsorted packed (target<<32|source) append buffers of the DTT.
    int64_t n_m2l = 0, n_p2p = 0, p2p_inter = 0;
    DevBuf fr_a, fr_b, lst_m2l, lst_p2p, lst_tmp, m2l_src, p2p_src, m2l_off, p2p_off, cnt_tmp, cnt_tmp2, dcount;
    DevBuf dtt_lvl;                                          // per-level frontier sizes (dtt.cu fast path)
    // target-ordered traversal (tct.cu): per-level counts/scans, level_begin, pass-down sets
    // (ping-pong CSR), global split lists of overflowed targets
    DevBuf tc_cnt, tc_voff, tc_lb, tc_d[2], tc_doff[2], tc_glob, tc_slab, tc_bsum;
    std::vector<std::array<uint32_t, 3>> tc_max;   // per-level max list lengths of the last build
    std::vector<unsigned> tc_novf;                  // per-level overflowed targets of the last local build
    bool tc_force_skip = false;                     // tests: skip the overflow kernels at every level (FMM_TCT_SKIP=1)
    std::vector<std::array<uint64_t, 3>> tc_tot;   // per-level list totals of the last build
    DevBuf tc_rec;                                  // per-level device records (bases, totals, maxima)
    std::vector<TcPart> tc_rem;                     // remote traversal parts (buffers reused)
    int tc_nrem = 0;                                // parts written since the last fmm_lists
    DevBuf tc_mixflag;                              // per target: an M2L source beyond levels l-1..l+1
    int64_t tc_mix_ncell = -1;                      // cells the flags describe (-1: none; tct_lists)
    int tc_scap = 0;                                // shared split-list capacity override (FMM_TCT_CAP, tests)
    bool tc_tight = false;                          // fast mode treats outputs as 16 entries (FMM_TCT_TIGHT, tests)
    DevBuf tc_cat_off, tc_cat_src;                  // concatenation output (swapped with the lists)
    bool tc_single = true;      // single pass into slots sized from tc_max (FMM_TCT_SINGLE=0: count + emit)
    int64_t tc_est_m2l = 0, tc_est_p2p = 0;
    bool lists_csr = false;     // lists came from tct (CSR only; no packed pair list)
    int dtt_mode = 0;           // 0: target-ordered traversal (tct.cu), 1: breadth-first (FMM_DTT=bfs)
    int64_t dtt_est_front = 0, dtt_est_m2l = 0, dtt_est_p2p = 0;   // buffer sizes learnt from the last build
    // P2P source runs: runs[n_runs] = {start body, flat offset}; run_off[ncell+1] (+1 spare), then rtot[ncell]
    int64_t n_runs = 0;
    DevBuf runs, run_off, run_tmp, run_pre, run_len64, dcount2, tcnt, cnt64, big_off, seg_lists;
    DevBuf leaf_cls;                    // leaves by P2P size class c at [c nleaf, (c+1) nleaf): tiny, mid, big
    int64_t n_leaf_cls[3] = {0, 0, 0};

    // expansions
    DevBuf M, L, Mr, Lr, fold_tab;
    DevBuf m2l_mix;               // per-target "list mixes levels" flags + level bounds (m2l_fast.cu)
    int fold_P = -1;              // P of the fold table in fold_tab (m2l_fast.cu)
    int64_t fold_nt = 0;   // fp64 [ncell][ncoef]; Mr: packed reduced multipoles for the M2L kernel; Lr: reduced L
    DevBuf near_phi, near_grad;  // P2P partials in sorted order (prec type)
    DevBuf far;                  // L2P far field in sorted order, double4 (phi, grad) (overlap mode)
    bool upward_done = false;

    // multi-GPU (let.cu, part.cu): remote LET cells live at [ncell, ncell + nrem) of every
    // cell array the traversal and the M2L/P2P kernels read, remote bodies at [n, n + nrem_body)
    int64_t nrem = 0, nrem_body = 0;
    std::vector<LetPeer> let_peers;
    std::vector<LetRemote> let_remote;
    size_t let_traversed = 0;   // grafted LETs already seeded into the traversal
    DevBuf let_tmp, let_cov, c_orig, part_tmp, orb_tmp;
    DevBuf h_stage;              // device staging for fmm_solve_host
    // dist.cu: the partition's keys were sorted by the driver (key_a / idx_a hold the sorted keys
    // and permutation of this build's positions): build_keys only derives the root cube and gathers
    bool presorted = false;
    bool guard = false, poison = false;   // FMM_GUARD / FMM_POISON (capi.cu buf_ensure, fmm_debug_check)
    DistState* dist = nullptr;   // fmm_create_dist contexts only
};

// ---- error helpers
#define FMM_CUDA_TRY(ctx, expr)                                                          \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess) {                                                         \
            (ctx)->err = std::string(#expr) + ": " + cudaGetErrorString(_e);             \
            return _e == cudaErrorMemoryAllocation ? FMM_ERR_OOM : FMM_ERR_CUDA;         \
        }                                                                                \
    } while (0)

#define FMM_TRY(expr)                   \
    do {                                \
        fmm_status _s = (expr);         \
        if (_s != FMM_OK) return _s;    \
    } while (0)

// grow a device buffer to at least `bytes` (contents discarded unless keep)
// makes `dev` current for the scope of an ABI call and restores the caller's device after it
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

fmm_status buf_ensure(fmm_ctx* ctx, DevBuf& b, size_t bytes, bool keep = false, cudaStream_t s = 0);
void buf_free(DevBuf& b);

template <typename T>
__host__ __forceinline__ T* P_(DevBuf& b) { return reinterpret_cast<T*>(b.p); }

// sorted body record in fp64 mode (32-B aligned for vector loads)
struct __align__(32) dbody { double x, y, z, w; };  // w = charge

template <typename Real> struct BodyT;
template <> struct BodyT<float> { using type = float4; };
template <> struct BodyT<double> { using type = dbody; };

// timing helpers (no-ops when timing is off)
struct PhaseScope {
    fmm_ctx* ctx; int phase; cudaStream_t s; cudaEvent_t a = nullptr;
    PhaseScope(fmm_ctx* c, int ph, cudaStream_t st);
    ~PhaseScope();
};

// launch accounting
#define FMM_LAUNCH(ctx) ((ctx)->launches++)

// function attributes are per device: set once per (call site, device)
#define FMM_FUNC_ATTR_ONCE(ctx, attr, value, ...)                                                   \
    do {                                                                                           \
        static unsigned long long done_mask_ = 0ull;                                               \
        const unsigned long long bit_ = 1ull << ((ctx)->device & 63);                              \
        if (!(done_mask_ & bit_)) {                                                                \
            FMM_CUDA_TRY(ctx, cudaFuncSetAttribute(__VA_ARGS__, attr, value));                     \
            done_mask_ |= bit_;                                                                    \
        }                                                                                          \
    } while (0)

// Lanes whose BITS-bit digit d equals this lane's, among the lanes in `valid` (a ballot-based
// multi-split: one vote per digit bit).  Same result as __match_any_sync restricted to `valid`;
// MATCH.ANY measured far slower on sm_100 (top stall of the list and sort kernels).
template <int BITS>
__device__ __forceinline__ unsigned match_digit(uint32_t d, unsigned valid) {
    unsigned m = valid;
#pragma unroll
    for (int b = 0; b < BITS; ++b) {
        const bool bit = (d >> b) & 1u;
        const unsigned v = __ballot_sync(0xffffffffu, bit);
        m &= bit ? v : ~v;
    }
    return m;
}

// ---- entry points of the translation units (all enqueue on the given stream)
// scan.cu
fmm_status scan_exclusive_u32(fmm_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t n, uint32_t* total_dev,
                              cudaStream_t s);
fmm_status scan_exclusive_u64(fmm_ctx* ctx, const uint64_t* in, uint64_t* out, int64_t n, uint64_t* total_dev,
                              cudaStream_t s);
// sort.cu: stable LSD radix sort of (key, val) over the 8-bit digits of [bit_lo, bit_hi) that
// `vary` touches (0: find the varying digits on the device, one host read); result pointers returned
fmm_status radix_sort_pairs(fmm_ctx* ctx, uint64_t* k0, uint64_t* k1, uint32_t* v0, uint32_t* v1, int64_t n,
                            int bit_lo, int bit_hi, uint64_t** kout, uint32_t** vout, cudaStream_t s,
                            uint64_t vary = 0);
fmm_status radix_sort_keys(fmm_ctx* ctx, uint64_t* k0, uint64_t* k1, int64_t n, int bit_lo, int bit_hi,
                           uint64_t** kout, cudaStream_t s, uint64_t vary = 0);
// keys.cu
fmm_status build_keys(fmm_ctx* ctx, const void* pos, int64_t n, cudaStream_t s);
fmm_status gather_bodies_q(fmm_ctx* ctx, const void* q, cudaStream_t s);
// tree.cu
fmm_status build_tree(fmm_ctx* ctx, cudaStream_t s);
// dtt.cu: traversal from the given seed pairs (target << 32 | source), appended to the
// unsorted lists when append; lists_pass groups them into canonical CSR lists + P2P runs
// max_depth_src: deepest source tree among the seeds (-1 unknown: synchronous levels for append)
fmm_status dtt_pass(fmm_ctx* ctx, const uint64_t* seeds, int nseeds, bool append, cudaStream_t s,
                    int max_depth_src = -1);
fmm_status lists_pass(fmm_ctx* ctx, cudaStream_t s);
// tct.cu: target-ordered traversal writing the CSR lists directly: the local traversal, a
// remote one from the given grafted LET roots (one more part), and the per-target concatenation
// of the local lists with the remote parts
fmm_status tct_lists(fmm_ctx* ctx, cudaStream_t s);
fmm_status tct_remote(fmm_ctx* ctx, const std::vector<uint32_t>& roots, cudaStream_t s);
fmm_status tct_concat(fmm_ctx* ctx, cudaStream_t s);
// dtt.cu: P2P interaction count and source runs of the CSR lists (synchronises s)
fmm_status lists_finish(fmm_ctx* ctx, cudaStream_t s);
fmm_status p2p_mutual_prep(fmm_ctx* ctx, cudaStream_t s);
fmm_status p2p_mutual(fmm_ctx* ctx, cudaStream_t s);
fmm_status build_lists(fmm_ctx* ctx, cudaStream_t s);
// let.cu
fmm_status let_cover(fmm_ctx* ctx, double* cover, int* ncover, cudaStream_t s);
fmm_status let_plan(fmm_ctx* ctx, int peer, const double* cover, int ncover, int64_t* sbytes, int64_t* dbytes,
                    cudaStream_t s);
fmm_status let_pack(fmm_ctx* ctx, int peer, int part, void* dst, cudaStream_t s);
fmm_status let_graft(fmm_ctx* ctx, int npeers, const void* const* src, const int64_t* bytes, cudaStream_t s);
fmm_status let_unpack(fmm_ctx* ctx, int first, int npeers, const void* const* src, const int64_t* bytes,
                      cudaStream_t s);
// upward.cu / downward.cu / m2l.cu / p2p.cu
fmm_status upward_pass(fmm_ctx* ctx, cudaStream_t s);
fmm_status m2l_pass(fmm_ctx* ctx, cudaStream_t s);
fmm_status m2l_fast(fmm_ctx* ctx, cudaStream_t s);
bool m2l_fast_available(int P, int prec);
fmm_status m2l_expand(fmm_ctx* ctx, const uint64_t* off2, cudaStream_t s);
fmm_status p2p_pass(fmm_ctx* ctx, cudaStream_t s);
fmm_status downward_pass(fmm_ctx* ctx, void* phi, void* grad, cudaStream_t s);
// L2L + L2P writing the far field to ctx->far (sorted order); merge_nearfar adds P2P and un-permutes
fmm_status downward_far(fmm_ctx* ctx, cudaStream_t s);
fmm_status merge_nearfar(fmm_ctx* ctx, void* phi, void* grad, cudaStream_t s);
