// tree.cu -- level-by-level octree build on the sorted keys (a4) and tight geometry (a5).
//
// R6 (§II-C local octree; PAPER.md:189 N_crit "maximum number of particles
// per leaf cell"): the root holds all particles; a cell at level l is internal iff
// count > ncrit and l < 21; its children are its non-empty octants in ascending digit
// order; cells are stored in (level, key) order, children contiguous.
// Build: one pass per level.  Thread per cell binary-searches the 7 digit boundaries
// inside its key range (keys are sorted and share the cell prefix), a scan allocates the
// children, a second kernel writes them.  The host reads one count per level.
//
// R7 (§II-B "squeezes the bounding box of each cell to tightly fit the
// particles"): exact fp64 min/max (leaves from bodies, internal cells from children,
// bottom-up: min/max is exact, so this equals the per-member definition), centre
// (bmin+bmax)*0.5, R = 0.5*sqrt((dx*dx + dy*dy) + dz*dz) with _rn intrinsics (no FMA).
#include "common.cuh"

namespace {

__global__ void k_init_root(int64_t n, uint64_t* key, int32_t* level, uint32_t* bb, uint32_t* bc, uint32_t* cb,
                            uint32_t* cc, int32_t* parent) {
    key[0] = 0; level[0] = 0; bb[0] = 0; bc[0] = (uint32_t)n; cb[0] = 0; cc[0] = 0; parent[0] = -1;
}

__device__ __forceinline__ uint32_t lower_bound_digit(const uint64_t* __restrict__ keys, uint32_t lo, uint32_t hi,
                                                      int shift, uint32_t d) {
    // first index in [lo,hi) whose digit >= d
    while (lo < hi) {
        uint32_t mid = lo + ((hi - lo) >> 1);
        if (((uint32_t)(keys[mid] >> shift) & 7u) < d) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void k_split_count(const uint64_t* __restrict__ keys, int64_t cbeg, int64_t nl, int level, int ncrit,
                              const uint32_t* __restrict__ bb, const uint32_t* __restrict__ bc,
                              uint32_t* __restrict__ bounds /* [nl][8] */, uint32_t* __restrict__ cnt) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nl) return;
    uint32_t b = bb[cbeg + i], c = bc[cbeg + i];
    uint32_t nc = 0;
    if (c > (uint32_t)ncrit && level < FMM_MAXLEVEL) {
        int shift = 3 * (FMM_MAXLEVEL - level - 1);
        uint32_t e = b + c;
        uint32_t prev = b;
        bounds[i * 8 + 0] = b;
        for (uint32_t d = 1; d < 8; ++d) {
            uint32_t p = lower_bound_digit(keys, prev, e, shift, d);
            bounds[i * 8 + d] = p;
            nc += (p > prev);
            prev = p;
        }
        nc += (e > prev);
    }
    cnt[i] = nc;
}

// Warp per cell: the 7 digit boundaries are found together by 32-ary searches (each round
// every boundary's interval shrinks 32x; the 7 probes of a round are independent loads), so
// the dependent-load chain of a 2^20-body cell is ~4 rounds instead of 7 x 20 binary steps.
__device__ __forceinline__ void split_count_cell(const uint64_t* __restrict__ keys, int64_t cbeg, int64_t i, int level,
                                                 int ncrit, const uint32_t* __restrict__ bb,
                                                 const uint32_t* __restrict__ bc, uint32_t* __restrict__ bounds,
                                                 uint32_t* __restrict__ cnt);

__global__ void k_split_count_warp(const uint64_t* __restrict__ keys, int64_t cbeg, int64_t nl, int level, int ncrit,
                                   const uint32_t* __restrict__ bb, const uint32_t* __restrict__ bc,
                                   uint32_t* __restrict__ bounds /* [nl][8] */, uint32_t* __restrict__ cnt) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= nl) return;
    split_count_cell(keys, cbeg, i, level, ncrit, bb, bc, bounds, cnt);
}

// the same with the level's cells read from the device (sync-free build): lb = level starts
__global__ void k_split_count_dev(const uint64_t* __restrict__ keys, const int64_t* __restrict__ lb, int level, int ncrit,
                                  const uint32_t* __restrict__ bb, const uint32_t* __restrict__ bc,
                                  uint32_t* __restrict__ bounds, uint32_t* __restrict__ cnt,
                                  const unsigned* __restrict__ flag, int64_t max_nl) {
    if (*reinterpret_cast<const volatile unsigned*>(flag)) return;
    const int64_t cbeg = lb[level], nl = lb[level + 1] - cbeg;
    if (nl > max_nl) return;   // wider than planned: k_split_scan_emit flags it
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nl; i += nw)
        split_count_cell(keys, cbeg, i, level, ncrit, bb, bc, bounds, cnt);
}

__device__ __forceinline__ void split_count_cell(const uint64_t* __restrict__ keys, int64_t cbeg, int64_t i, int level,
                                                 int ncrit, const uint32_t* __restrict__ bb,
                                                 const uint32_t* __restrict__ bc, uint32_t* __restrict__ bounds,
                                                 uint32_t* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const uint32_t b = bb[cbeg + i], c = bc[cbeg + i];
    if (!(c > (uint32_t)ncrit && level < FMM_MAXLEVEL)) {
        if (lane == 0) cnt[i] = 0;
        return;
    }
    const int shift = 3 * (FMM_MAXLEVEL - level - 1);
    const uint32_t e = b + c;
    // first index in [lo_d, hi_d] whose digit >= d (hi_d = e: none)
    uint32_t lo[8], hi[8];
#pragma unroll
    for (int d = 1; d < 8; ++d) lo[d] = b, hi[d] = e;
    bool busy = true;
    while (busy) {
        uint32_t q[8];
        uint32_t dig[8];
#pragma unroll
        for (int d = 1; d < 8; ++d) {
            q[d] = lo[d] + (uint32_t)(((uint64_t)(hi[d] - lo[d]) * (uint32_t)lane) >> 5);
            dig[d] = lo[d] < hi[d] ? ((uint32_t)(__ldg(keys + q[d]) >> shift) & 7u) : 8u;
        }
        busy = false;
#pragma unroll
        for (int d = 1; d < 8; ++d) {
            if (lo[d] < hi[d]) {   // warp-uniform
                const unsigned ge = __ballot_sync(0xffffffffu, dig[d] >= (uint32_t)d);
                const int t = __popc(~ge);   // samples below d (monotone: a prefix of the lanes)
                if (t == 0) {
                    hi[d] = lo[d];
                } else {
                    const uint32_t qa = __shfl_sync(0xffffffffu, q[d], t - 1);
                    const uint32_t qb = t < 32 ? __shfl_sync(0xffffffffu, q[d], t & 31) : hi[d];
                    lo[d] = qa + 1;
                    hi[d] = qb;
                }
                busy |= lo[d] < hi[d];
            }
        }
    }
    if (lane == 0) {
        uint32_t nc = 0, prev = b;
        bounds[i * 8 + 0] = b;
#pragma unroll
        for (int d = 1; d < 8; ++d) {
            const uint32_t p = lo[d];
            bounds[i * 8 + d] = p;
            nc += (p > prev);
            prev = p;
        }
        nc += (e > prev);
        cnt[i] = nc;
    }
}

__global__ void k_split_emit(const uint64_t* __restrict__ keys, int64_t cbeg, int64_t nl, int level, int64_t nbeg,
                             const uint32_t* __restrict__ bounds, const uint32_t* __restrict__ cnt,
                             const uint32_t* __restrict__ off, uint64_t* key, int32_t* lev, uint32_t* bb,
                             uint32_t* bc, uint32_t* cb, uint32_t* cc, int32_t* parent) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nl) return;
    uint32_t nc = cnt[i];
    int64_t me = cbeg + i;
    if (nc == 0) return;  // leaf: child fields were zeroed at creation
    uint32_t first = (uint32_t)(nbeg + off[i]);
    cb[me] = first;
    cc[me] = nc;
    uint64_t pk = key[me];
    uint32_t e = bb[me] + bc[me];
    uint32_t k = first;
    for (uint32_t d = 0; d < 8; ++d) {
        uint32_t lo = bounds[i * 8 + d];
        uint32_t hi = d < 7 ? bounds[i * 8 + d + 1] : e;
        if (hi > lo) {
            key[k] = (pk << 3) | d;
            lev[k] = level + 1;
            bb[k] = lo;
            bc[k] = hi - lo;
            cb[k] = 0;
            cc[k] = 0;
            parent[k] = (int32_t)me;
            ++k;
        }
    }
}

// Sync-free build: per level the child counts are scanned by tiles (block sums), one block
// scans the block sums (the level's total -> lb[level + 2]), and the children are written in
// (level, key) order as k_split_emit does.  Sizes come from lb (device); a level wider than
// planned or children over the cell capacity set the flag (the build is then redone with host
// round trips).
constexpr int SE_THREADS = 256, SE_ITEMS = 8, SE_TILE = SE_THREADS * SE_ITEMS;
__device__ __forceinline__ uint32_t se_block_excl(uint32_t v, uint32_t* s_w, uint32_t* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    uint32_t pre = 0, tot = 0;
    for (int i = 0; i < SE_THREADS / 32; ++i) {
        if (i < w) pre += s_w[i];
        tot += s_w[i];
    }
    *total = tot;
    return pre + x - v;
}

__global__ void __launch_bounds__(SE_THREADS) k_split_scan_tiles(const int64_t* __restrict__ lb, int level,
                                                                const uint32_t* __restrict__ cnt,
                                                                uint32_t* __restrict__ off, uint32_t* __restrict__ bsum,
                                                                int64_t max_nl, const unsigned* __restrict__ flag) {
    __shared__ uint32_t s_w[SE_THREADS / 32];
    if (*reinterpret_cast<const volatile unsigned*>(flag)) return;
    const int64_t nl = lb[level + 1] - lb[level];
    if (nl > max_nl || (int64_t)blockIdx.x * SE_TILE >= nl) return;
    const int64_t base = (int64_t)blockIdx.x * SE_TILE + (int64_t)threadIdx.x * SE_ITEMS;
    uint32_t v[SE_ITEMS], sum = 0;
#pragma unroll
    for (int k = 0; k < SE_ITEMS; ++k) {
        v[k] = base + k < nl ? cnt[base + k] : 0u;
        sum += v[k];
    }
    uint32_t tot;
    uint32_t run = se_block_excl(sum, s_w, &tot);
#pragma unroll
    for (int k = 0; k < SE_ITEMS; ++k) {
        if (base + k < nl) off[base + k] = run;
        run += v[k];
    }
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SE_THREADS) k_split_scan_top(int64_t* __restrict__ lb, int level,
                                                              uint32_t* __restrict__ bsum, int64_t max_nl, int64_t cap,
                                                              unsigned* __restrict__ flag) {
    __shared__ uint32_t s_w[SE_THREADS / 32];
    const int64_t nbeg = lb[level + 1], nl = nbeg - lb[level];
    if (*reinterpret_cast<volatile unsigned*>(flag) || nl > max_nl) {
        if (threadIdx.x == 0) {
            if (nl > max_nl) atomicOr(flag, 1u);
            lb[level + 2] = nbeg;
        }
        return;
    }
    const int64_t nb = (nl + SE_TILE - 1) / SE_TILE;
    uint32_t carry = 0;
    for (int64_t c0 = 0; c0 < nb; c0 += SE_THREADS) {
        const int64_t i = c0 + threadIdx.x;
        const uint32_t v = i < nb ? bsum[i] : 0u;
        uint32_t t;
        const uint32_t e = se_block_excl(v, s_w, &t);
        if (i < nb) bsum[i] = carry + e;
        carry += t;
    }
    if (threadIdx.x == 0) {
        if (nbeg + (int64_t)carry > cap) atomicOr(flag, 1u);   // children would overflow the cell arrays
        lb[level + 2] = nbeg + carry;
    }
}

__global__ void k_split_emit_dev(const int64_t* __restrict__ lb, int level, const uint32_t* __restrict__ bounds,
                                 const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ off,
                                 const uint32_t* __restrict__ bsum, uint64_t* key, int32_t* lev, uint32_t* bb,
                                 uint32_t* bc, uint32_t* cb, uint32_t* cc, int32_t* parent,
                                 const unsigned* __restrict__ flag) {
    if (*reinterpret_cast<const volatile unsigned*>(flag)) return;
    const int64_t cbeg = lb[level], nbeg = lb[level + 1], nl = nbeg - cbeg;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += stride) {
        const uint32_t nch = cnt[i];
        if (nch == 0) continue;
        const int64_t me = cbeg + i;
        const uint32_t first = (uint32_t)(nbeg + bsum[i / SE_TILE] + off[i]);
        cb[me] = first;
        cc[me] = nch;
        const uint64_t pk = key[me];
        const uint32_t e = bb[me] + bc[me];
        uint32_t kk = first;
        for (uint32_t d = 0; d < 8; ++d) {
            const uint32_t lo = bounds[i * 8 + d];
            const uint32_t hi = d < 7 ? bounds[i * 8 + d + 1] : e;
            if (hi > lo) {
                key[kk] = (pk << 3) | d;
                lev[kk] = level + 1;
                bb[kk] = lo;
                bc[kk] = hi - lo;
                cb[kk] = 0;
                cc[kk] = 0;
                parent[kk] = (int32_t)me;
                ++kk;
            }
        }
    }
}

template <typename Body>
__global__ void k_leaf_bounds(const Body* __restrict__ body, int64_t cbeg, int64_t cend,
                              const uint32_t* __restrict__ bb, const uint32_t* __restrict__ bc,
                              const uint32_t* __restrict__ cc, double* __restrict__ bmin, double* __restrict__ bmax) {
    const int lane = threadIdx.x & 31;
    int64_t c = cbeg + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (c >= cend || cc[c] != 0) return;
    uint32_t b = bb[c], n = bc[c];
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (uint32_t j = lane; j < n; j += 32) {
        Body p = body[b + j];
        double x = (double)p.x, y = (double)p.y, z = (double)p.z;
        lo[0] = fmin(lo[0], x); hi[0] = fmax(hi[0], x);
        lo[1] = fmin(lo[1], y); hi[1] = fmax(hi[1], y);
        lo[2] = fmin(lo[2], z); hi[2] = fmax(hi[2], z);
    }
#pragma unroll
    for (int s = 16; s; s >>= 1)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], s));
            hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], s));
        }
    if (lane < 3) {
        bmin[3 * c + lane] = lo[lane];
        bmax[3 * c + lane] = hi[lane];
    }
}

__global__ void k_internal_bounds(int64_t cbeg, int64_t cend, const uint32_t* __restrict__ cb,
                                  const uint32_t* __restrict__ cc, double* __restrict__ bmin,
                                  double* __restrict__ bmax) {
    int64_t c = cbeg + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cend) return;
    uint32_t k0 = cb[c], nk = cc[c];
    if (nk == 0) return;
    double lo[3], hi[3];
    for (int d = 0; d < 3; ++d) { lo[d] = bmin[3 * (int64_t)k0 + d]; hi[d] = bmax[3 * (int64_t)k0 + d]; }
    for (uint32_t k = 1; k < nk; ++k)
        for (int d = 0; d < 3; ++d) {
            lo[d] = fmin(lo[d], bmin[3 * (int64_t)(k0 + k) + d]);
            hi[d] = fmax(hi[d], bmax[3 * (int64_t)(k0 + k) + d]);
        }
    for (int d = 0; d < 3; ++d) { bmin[3 * c + d] = lo[d]; bmax[3 * c + d] = hi[d]; }
}

__global__ void k_center_radius(int64_t ncell, const double* __restrict__ bmin, const double* __restrict__ bmax,
                                double4* __restrict__ cr) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncell) return;
    double ctr[3], dd[3];
    for (int d = 0; d < 3; ++d) {
        double lo = bmin[3 * c + d], hi = bmax[3 * c + d];
        ctr[d] = __dmul_rn(__dadd_rn(lo, hi), 0.5);
        dd[d] = __dsub_rn(hi, lo);
    }
    double s = __dadd_rn(__dadd_rn(__dmul_rn(dd[0], dd[0]), __dmul_rn(dd[1], dd[1])), __dmul_rn(dd[2], dd[2]));
    cr[c] = make_double4(ctr[0], ctr[1], ctr[2], __dmul_rn(0.5, __dsqrt_rn(s)));
}

__global__ void k_leaf_flags(int64_t ncell, const uint32_t* __restrict__ cc, uint32_t* __restrict__ flag) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < ncell) flag[c] = cc[c] == 0;
}

__global__ void k_leaf_compact(int64_t ncell, const uint32_t* __restrict__ cc, const uint32_t* __restrict__ off,
                               uint32_t* __restrict__ leaf_ids) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < ncell && cc[c] == 0) leaf_ids[off[c]] = (uint32_t)c;
}

fmm_status ensure_cells(fmm_ctx* ctx, int64_t need, cudaStream_t s) {
    if (need <= ctx->cell_cap) return FMM_OK;
    int64_t cap = std::max<int64_t>(need, ctx->cell_cap + ctx->cell_cap / 2);
    cap = std::max<int64_t>(cap, 1024);
    FMM_TRY(buf_ensure(ctx, ctx->c_key, cap * 8, true, s));
    FMM_TRY(buf_ensure(ctx, ctx->c_level, cap * 4, true, s));
    FMM_TRY(buf_ensure(ctx, ctx->c_bb, cap * 4, true, s));
    FMM_TRY(buf_ensure(ctx, ctx->c_bc, cap * 4, true, s));
    FMM_TRY(buf_ensure(ctx, ctx->c_cb, cap * 4, true, s));
    FMM_TRY(buf_ensure(ctx, ctx->c_cc, cap * 4, true, s));
    FMM_TRY(buf_ensure(ctx, ctx->c_parent, cap * 4, true, s));
    ctx->cell_cap = cap;
    return FMM_OK;
}

template <typename Body>
fmm_status geometry(fmm_ctx* ctx, cudaStream_t s) {
    PhaseScope ps(ctx, PH_GEOM, s);
    const int64_t nc = ctx->ncell;
    FMM_TRY(buf_ensure(ctx, ctx->c_bmin, nc * 24));
    FMM_TRY(buf_ensure(ctx, ctx->c_bmax, nc * 24));
    FMM_TRY(buf_ensure(ctx, ctx->c_cr, nc * 32));
    const Body* body = P_<Body>(ctx->body);
    double* bmin = P_<double>(ctx->c_bmin);
    double* bmax = P_<double>(ctx->c_bmax);
    // leaves: every cell of every level may be a leaf
    k_leaf_bounds<Body><<<(unsigned)((nc * 32 + 255) / 256), 256, 0, s>>>(body, 0, nc, P_<uint32_t>(ctx->c_bb),
                                                                           P_<uint32_t>(ctx->c_bc),
                                                                           P_<uint32_t>(ctx->c_cc), bmin, bmax);
    FMM_LAUNCH(ctx);
    for (int64_t l = ctx->depth - 1; l >= 0; --l) {
        int64_t b = ctx->level_begin[l], e = ctx->level_begin[l + 1];
        k_internal_bounds<<<(unsigned)((e - b + 127) / 128), 128, 0, s>>>(b, e, P_<uint32_t>(ctx->c_cb),
                                                                          P_<uint32_t>(ctx->c_cc), bmin, bmax);
        FMM_LAUNCH(ctx);
    }
    k_center_radius<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(nc, bmin, bmax, P_<double4>(ctx->c_cr));
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}
}  // namespace

fmm_status build_levels_fast(fmm_ctx* ctx, cudaStream_t s, bool& built);
fmm_status build_levels_sync(fmm_ctx* ctx, cudaStream_t s);

fmm_status build_tree(fmm_ctx* ctx, cudaStream_t s) {
    {
        PhaseScope ps(ctx, PH_TREE, s);
        bool built = false;
        if (ctx->tree_fast && ctx->tree_prev_depth >= 0) {
            FMM_TRY(build_levels_fast(ctx, s, built));
        }
        if (!built) FMM_TRY(build_levels_sync(ctx, s));
        ctx->tree_prev_depth = ctx->depth;
        ctx->tree_prev_ncell = ctx->ncell;
        int64_t mw = 1;
        for (size_t l = 0; l + 1 < ctx->level_begin.size(); ++l)
            mw = std::max(mw, ctx->level_begin[l + 1] - ctx->level_begin[l]);
        ctx->tree_prev_maxw = mw;
        // leaf list (ascending cell index)
        const int64_t nc = ctx->ncell;
        FMM_TRY(buf_ensure(ctx, ctx->split_cnt, (size_t)(2 * nc + 4) * 4));
        FMM_TRY(buf_ensure(ctx, ctx->leaf_ids, (size_t)nc * 4));
        uint32_t* flag = P_<uint32_t>(ctx->split_cnt);
        uint32_t* off = flag + nc;
        uint32_t* d_total = off + nc;
        k_leaf_flags<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(nc, P_<uint32_t>(ctx->c_cc), flag);
        FMM_LAUNCH(ctx);
        FMM_TRY(scan_exclusive_u32(ctx, flag, off, nc, d_total, s));
        k_leaf_compact<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(nc, P_<uint32_t>(ctx->c_cc), off,
                                                                    P_<uint32_t>(ctx->leaf_ids));
        FMM_LAUNCH(ctx);
        uint32_t nleaf = 0;
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&nleaf, d_total, 4, cudaMemcpyDeviceToHost, s));
        FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        ctx->nleaf = nleaf;
    }
    if (ctx->prec == FMM_F32) return geometry<float4>(ctx, s);
    return geometry<dbody>(ctx, s);
}

// levels with the previous build's sizes: every level launched back to back (count, then one
// block scanning and emitting), sizes read on the device, one host round trip at the end; a
// capacity or width overflow, or a tree deeper than planned, leaves built = false
fmm_status build_levels_fast(fmm_ctx* ctx, cudaStream_t s, bool& built) {
    built = false;
    const int64_t n = ctx->n;
    const int L = (int)std::min<int64_t>(ctx->tree_prev_depth + 2, FMM_MAXLEVEL + 1);   // levels to launch
    const int64_t max_nl = ctx->tree_prev_maxw + ctx->tree_prev_maxw / 4 + 1024;
    const int64_t cap = std::max<int64_t>(ctx->tree_prev_ncell + ctx->tree_prev_ncell / 4 + 1024, 1024);
    FMM_TRY(ensure_cells(ctx, cap, s));
    FMM_TRY(buf_ensure(ctx, ctx->split_tmp, (size_t)max_nl * 8 * 4 + 64));
    FMM_TRY(buf_ensure(ctx, ctx->split_cnt, (size_t)(2 * max_nl + 4 + max_nl / SE_TILE + 1) * 4));
    FMM_TRY(buf_ensure(ctx, ctx->tree_lb, (size_t)(FMM_MAXLEVEL + 4) * 8 + 16));
    int64_t* lb = P_<int64_t>(ctx->tree_lb);
    unsigned* flag = reinterpret_cast<unsigned*>(lb + FMM_MAXLEVEL + 4);
    const int64_t lb0[2] = {0, 1};
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->tree_lb.p, 0, (size_t)(FMM_MAXLEVEL + 4) * 8 + 16, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(lb, lb0, sizeof(lb0), cudaMemcpyHostToDevice, s));
    k_init_root<<<1, 1, 0, s>>>(n, P_<uint64_t>(ctx->c_key), P_<int32_t>(ctx->c_level), P_<uint32_t>(ctx->c_bb),
                                P_<uint32_t>(ctx->c_bc), P_<uint32_t>(ctx->c_cb), P_<uint32_t>(ctx->c_cc),
                                P_<int32_t>(ctx->c_parent));
    FMM_LAUNCH(ctx);
    uint32_t* bounds = P_<uint32_t>(ctx->split_tmp);
    uint32_t* cnt = P_<uint32_t>(ctx->split_cnt);
    uint32_t* off = cnt + max_nl;
    uint32_t* bsum = off + max_nl;   // (split_cnt holds 2 max_nl + 4 + max_nl / SE_TILE + 1 words)
    // grids for the widest level planned; the upper levels' blocks find nothing and exit
    const unsigned gc = (unsigned)std::min<int64_t>((max_nl * 32 + 255) / 256, (int64_t)ctx->num_sms * 16);
    const unsigned gt = (unsigned)((max_nl + SE_TILE - 1) / SE_TILE);
    const unsigned ge = (unsigned)std::min<int64_t>((max_nl + 255) / 256, (int64_t)ctx->num_sms * 8);
    for (int level = 0; level < L; ++level) {
        k_split_count_dev<<<gc, 256, 0, s>>>(ctx->d_keys, lb, level, ctx->ncrit, P_<uint32_t>(ctx->c_bb),
                                             P_<uint32_t>(ctx->c_bc), bounds, cnt, flag, max_nl);
        k_split_scan_tiles<<<gt, SE_THREADS, 0, s>>>(lb, level, cnt, off, bsum, max_nl, flag);
        k_split_scan_top<<<1, SE_THREADS, 0, s>>>(lb, level, bsum, max_nl, ctx->cell_cap, flag);
        k_split_emit_dev<<<ge, 256, 0, s>>>(lb, level, bounds, cnt, off, bsum, P_<uint64_t>(ctx->c_key),
                                            P_<int32_t>(ctx->c_level), P_<uint32_t>(ctx->c_bb), P_<uint32_t>(ctx->c_bc),
                                            P_<uint32_t>(ctx->c_cb), P_<uint32_t>(ctx->c_cc), P_<int32_t>(ctx->c_parent),
                                            flag);
        ctx->launches += 4;
    }
    std::vector<int64_t> h(L + 2);
    unsigned hflag = 0;
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(h.data(), lb, (size_t)(L + 2) * 8, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&hflag, flag, 4, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    if (hflag) return FMM_OK;
    // depth = first level whose cells had no children (lb[l + 2] == lb[l + 1])
    int d = -1;
    for (int l = 0; l < L; ++l)
        if (h[l + 2] == h[l + 1]) {
            d = l;
            break;
        }
    if (d < 0) return FMM_OK;   // still growing at the last launched level: deeper than planned
    ctx->level_begin.assign(h.begin(), h.begin() + d + 2);
    ctx->depth = d;
    ctx->ncell = ctx->level_begin.back();
    built = true;
    return FMM_OK;
}

// levels with a host round trip each (first build, or the fast path failed)
fmm_status build_levels_sync(fmm_ctx* ctx, cudaStream_t s) {
    const int64_t n = ctx->n;
    {
        FMM_TRY(ensure_cells(ctx, std::max<int64_t>(1024, 2 * n / std::max(ctx->ncrit, 1) + 64), s));
        k_init_root<<<1, 1, 0, s>>>(n, P_<uint64_t>(ctx->c_key), P_<int32_t>(ctx->c_level), P_<uint32_t>(ctx->c_bb),
                                    P_<uint32_t>(ctx->c_bc), P_<uint32_t>(ctx->c_cb), P_<uint32_t>(ctx->c_cc),
                                    P_<int32_t>(ctx->c_parent));
        FMM_LAUNCH(ctx);
        ctx->level_begin.assign({0, 1});
        uint32_t* d_total = nullptr;
        for (int level = 0; level < FMM_MAXLEVEL; ++level) {
            int64_t cbeg = ctx->level_begin[level], nl = ctx->level_begin[level + 1] - cbeg;
            FMM_TRY(buf_ensure(ctx, ctx->split_tmp, (size_t)nl * 8 * 4 + 64));
            FMM_TRY(buf_ensure(ctx, ctx->split_cnt, (size_t)(2 * nl + 4) * 4));
            uint32_t* bounds = P_<uint32_t>(ctx->split_tmp);
            uint32_t* cnt = P_<uint32_t>(ctx->split_cnt);
            uint32_t* off = cnt + nl;
            d_total = off + nl;
            unsigned g = (unsigned)((nl + 127) / 128);
            k_split_count_warp<<<(unsigned)((nl * 32 + 255) / 256), 256, 0, s>>>(
                ctx->d_keys, cbeg, nl, level, ctx->ncrit, P_<uint32_t>(ctx->c_bb), P_<uint32_t>(ctx->c_bc), bounds, cnt);
            FMM_LAUNCH(ctx);
            FMM_TRY(scan_exclusive_u32(ctx, cnt, off, nl, d_total, s));
            uint32_t total = 0;
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&total, d_total, 4, cudaMemcpyDeviceToHost, s));
            FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
            if (total == 0) break;
            int64_t nbeg = ctx->level_begin[level + 1];
            FMM_TRY(ensure_cells(ctx, nbeg + total, s));
            k_split_emit<<<g, 128, 0, s>>>(ctx->d_keys, cbeg, nl, level, nbeg, bounds, cnt, off,
                                           P_<uint64_t>(ctx->c_key), P_<int32_t>(ctx->c_level), P_<uint32_t>(ctx->c_bb),
                                           P_<uint32_t>(ctx->c_bc), P_<uint32_t>(ctx->c_cb), P_<uint32_t>(ctx->c_cc),
                                           P_<int32_t>(ctx->c_parent));
            FMM_LAUNCH(ctx);
            FMM_CUDA_TRY(ctx, cudaGetLastError());
            ctx->level_begin.push_back(nbeg + total);
        }
        ctx->depth = (int64_t)ctx->level_begin.size() - 2;
        ctx->ncell = ctx->level_begin.back();
    }
    return FMM_OK;
}
