// tct.cu -- the dual tree traversal (a8, R8-R10) organised by TARGET cell, emitting the CSR
// M2L and P2P lists directly (no unsorted pair list, no grouping, no segment sorts).
//
// R9 visits pair (A, B) iff (A, B) = (root, root), or (parent(A), B) is visited and splits A,
// or (A, parent(B)) is visited and splits B.  So, for a target T, its visited sources are
//   * the sources its parent passed down: D(parent(T)) = { B : (parent(T), B) visited, splits A }
//     (the root's: { root }), and
//   * the children of every source B whose pair (T, B) splits B,
// and every visited (T, B) is classified by the same R8/R9 test as the breadth-first
// traversal (dtt.cu): MAC -> M2L, both leaves -> P2P, split A -> D(T), split B -> B's children.
// Targets are processed level by level (a warp per target); the pass-down sets D of one level
// feed the next.  Each level runs twice: a counting pass (list lengths per target, scanned into
// the CSR offsets) and an emitting pass that writes the entries at those offsets.
//
// Order inside a target's list (deterministic; R10 fixes the set, fmm_copy_lists sorts for the
// canonical order): by source level; within a level, first the sources inherited from the
// parent (in the parent's order), then the children of the split sources (ascending).  The
// split-B sources of a level wait in a per-warp shared-memory list; a target whose list
// outgrows it (Plummer: shallow halo leaves next to the core) is redone by a second kernel
// with per-warp lists in global memory sized for a whole tree level.
#include <array>

#include "common.cuh"

namespace {

constexpr int TC_WARPS = 4;
constexpr int TC_CAP = 512;    // split-B sources per target and level held in shared memory
constexpr int TC_GWARPS_MAX = 1024;   // warps of the global-memory kernel (overflowed targets), at most

struct Cells {
    const double4* __restrict__ cr;
    const uint32_t* __restrict__ cb;
    const uint32_t* __restrict__ cc;
};

// outcome of (T, s): 0 M2L, 1 P2P, 2 split T (s passed down), 3 split s (its children visited)
// the child count is loaded with the centre, before the MAC test needs neither (one round trip;
// a plain load is sunk into the non-MAC branch by the compiler, a second round trip for ~80% of
// the candidates)
__device__ __forceinline__ uint32_t ld_early_u32(const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

__device__ __forceinline__ int tc_classify(const double4 T, uint32_t nT, const Cells& v, uint32_t s, double theta) {
    const uint32_t nB = ld_early_u32(v.cc + s);
    const double4 B = v.cr[s];
    const double dx = __dsub_rn(T.x, B.x), dy = __dsub_rn(T.y, B.y), dz = __dsub_rn(T.z, B.z);
    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    if (__dadd_rn(T.w, B.w) < __dmul_rn(theta, __dsqrt_rn(d2))) return 0;
    if (nT == 0 && nB == 0) return 1;
    if (nB == 0 || (nT != 0 && T.w >= B.w)) return 2;
    return 3;
}

__global__ void k_widen_u32_tc(const uint32_t* __restrict__ in, int64_t n, uint64_t* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = in[i];
}

struct TcOut {   // per-target output cursors (warp-uniform)
    uint32_t m, p, d;
};

// MODE 0: count; 1: write at offM/offP/offD + cursor; 2 (single pass): write into per-target slab
// slots of capM/capP/capD entries (srcM/srcP/dsrc = slabs) and count -- a target whose lists
// outgrow a slot is recorded like a split-list overflow.  GLOB = false: targets [tb, te), split
// lists in shared memory, a target that overflows them is recorded (ovf flag + list) and
// skipped by MODE 1; GLOB = true: the recorded targets, split lists in global memory (gcap).
template <int MODE, bool GLOB>
__global__ void __launch_bounds__(TC_WARPS * 32, 8) k_tct_level(
    int64_t tb, int64_t te, const int32_t* __restrict__ parent, int64_t pb, const uint64_t* __restrict__ doff_prev,
    const uint32_t* __restrict__ dsrc_prev, Cells v, const uint32_t* __restrict__ seeds, int nseeds, double theta,
    uint32_t* __restrict__ cnt_m, uint32_t* __restrict__ cnt_p, uint32_t* __restrict__ cnt_d,
    const uint64_t* __restrict__ offM, const uint64_t* __restrict__ offP, const uint64_t* __restrict__ offD,
    uint32_t* __restrict__ srcM, uint32_t* __restrict__ srcP, uint32_t* __restrict__ dsrc,
    uint8_t* __restrict__ ovf, uint32_t* __restrict__ ovf_list, unsigned* __restrict__ n_ovf,
    uint32_t* __restrict__ gscratch, int64_t gcap, uint32_t capM, uint32_t capP, uint32_t capD,
    unsigned* __restrict__ err, int S, uint64_t lenM = ~0ull, uint64_t lenP = ~0ull, uint64_t lenD = ~0ull,
    uint32_t* __restrict__ mixflag = nullptr, int64_t band_lo = 0, int64_t band_hi = 0, bool ovf_redo = false) {
    constexpr bool EMIT = MODE != 0, COUNT = MODE != 1, SLAB = MODE == 2;
    // an earlier level outgrew the buffers sized from the previous build: the traversal is
    // redone, so stop here instead of reading incomplete pass-down sets
    if (*reinterpret_cast<volatile unsigned*>(err) & 2u) return;
    __shared__ uint32_t s_sb[GLOB ? 1 : TC_WARPS][2][GLOB ? 1 : TC_CAP];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t nwarps = (int64_t)gridDim.x * TC_WARPS;
    const int64_t gw = (int64_t)blockIdx.x * TC_WARPS + w;
    uint32_t* list0;
    uint32_t* list1;
    int64_t cap;
    if (GLOB) {
        list0 = gscratch + (size_t)gw * 2 * gcap;
        list1 = list0 + gcap;
        cap = gcap;
    } else {
        list0 = s_sb[w][0];
        list1 = s_sb[w][GLOB ? 0 : 1];
        cap = min((int64_t)TC_CAP, gcap);   // gcap: shared-list cap (tests force overflows with it)
    }
    // work items are (target, slice) pairs, slice k of S taking the k-th part of the target's
    // pass-down set (and everything it generates): more warps for the wide upper levels
    const int64_t nitems = GLOB ? (int64_t)*n_ovf : (te - tb) * S;
    for (int64_t it = gw; it < nitems; it += nwarps) {
        const int64_t vi = GLOB ? (int64_t)ovf_list[it] : it;   // virtual target index
        const int64_t t = tb + vi / S;
        const int64_t slice = vi % S;
        if (!GLOB && MODE == 1 && ovf[vi]) continue;   // done by the global-memory kernel
        const double4 T = v.cr[t];
        const uint32_t nT = v.cc[t];
        uint64_t x0 = 0, x1 = (uint64_t)nseeds;   // root targets: the seed sources
        if (doff_prev) {
            const int64_t pi = (int64_t)parent[t] - pb;
            x0 = doff_prev[pi];
            x1 = doff_prev[pi + 1];
        }
        {
            const uint64_t len = x1 - x0;
            x1 = x0 + len * (uint64_t)(slice + 1) / (uint64_t)S;
            x0 = x0 + len * (uint64_t)slice / (uint64_t)S;
        }
        uint64_t oM = 0, oP = 0, oD = 0;
        if (MODE == 1 && (offM[vi] + cnt_m[vi] > lenM || offP[vi] + cnt_p[vi] > lenP ||
                          offD[vi] + cnt_d[vi] > lenD)) {   // outputs sized from the previous build
            if (lane == 0) atomicOr(err, 2u);
            continue;
        }
        if (SLAB) {
            oM = (uint64_t)vi * capM;
            oP = (uint64_t)vi * capP;
            oD = (uint64_t)vi * capD;
        } else if (EMIT) {
            oM = offM[vi];
            oP = offP[vi];
            oD = offD[vi];
        }
        TcOut o{0u, 0u, 0u};
        bool over = false;
        // an M2L source outside the levels l-1 .. l+1 (cells [band_lo, band_hi)): the target needs
        // the M2L kernel with operand scaling (m2l_fast.cu; noted here instead of a list re-scan)
        bool mix = false;
        const uint32_t blo = (uint32_t)band_lo, bw = (uint32_t)(band_hi - band_lo);
        int cur = 0;
        uint32_t ncur = 0;
        uint64_t xp = x0;
        // emit the outcome of this lane's pair; `act` = lanes holding a pair, in emission order
        auto put = [&](int oc, uint32_t s, bool act, uint32_t* nxt, uint32_t& nnext) {
            const unsigned bm = __ballot_sync(0xffffffffu, act && oc == 0);
            const unsigned bp = __ballot_sync(0xffffffffu, act && oc == 1);
            const unsigned bd = __ballot_sync(0xffffffffu, act && oc == 2);
            const unsigned bs = __ballot_sync(0xffffffffu, act && oc == 3);
            // one select chain and one (generic) store instead of four divergent branches: the
            // lanes of a round usually hold every outcome, and SIMT ran all four paths
            const unsigned mine = oc == 0 ? bm : oc == 1 ? bp : oc == 2 ? bd : bs;
            const uint32_t k = (oc == 0 ? o.m : oc == 1 ? o.p : oc == 2 ? o.d : nnext) + __popc(mine & lt);
            uint32_t* const dst = oc == 0 ? srcM + oM : oc == 1 ? srcP + oP : oc == 2 ? dsrc + oD : nxt;
            const uint64_t lim = oc == 3 ? (uint64_t)cap : !EMIT ? 0ull : !SLAB ? ~0ull
                                 : (uint64_t)(oc == 0 ? capM : oc == 1 ? capP : capD);
            if (act && k < lim) dst[k] = s;
            if (COUNT && mixflag) mix |= act && oc == 0 && s - blo >= bw;   // outside [blo, blo + bw)
            o.m += __popc(bm);
            o.p += __popc(bp);
            o.d += __popc(bd);
            nnext += __popc(bs);
        };
        // generation 0: the sources the parent passed down (the root: the seeds), in order
        for (int gen = 0; gen == 0 || ncur > 0; ++gen) {
            uint32_t* nxt = cur ? list0 : list1;
            uint32_t nnext = 0;
            if (gen == 0 && xp < x1) {
                // the next round's source ids are loaded before this round is classified
                const uint32_t* ids = doff_prev ? dsrc_prev : seeds;
                uint32_t s_next = xp + lane < x1 ? ids[xp + lane] : 0u;
                for (; xp < x1; xp += 32) {
                    const uint64_t i = xp + (uint64_t)lane;
                    const bool act = i < x1;
                    const uint32_t s = s_next;
                    if (i + 32 < x1) s_next = ids[i + 32];
                    const int oc = act ? tc_classify(T, nT, v, s, theta) : -1;
                    put(oc, s, act, nxt, nnext);
                }
            }
            // generation g >= 1: the children of the sources generation g-1 split, in (source,
            // child) order, flattened over the lanes: a round of 32 split sources is expanded into its
            // children (prefix sum of the child counts), and each lane classifies one child per
            // step -- every step issues 32 independent cell loads
            const uint32_t* sb = cur ? list1 : list0;
            for (uint32_t base = 0; base < ncur; base += 32) {
                const bool has = base + lane < ncur;
                const uint32_t B = has ? sb[base + lane] : 0u;
                uint32_t c0 = has ? v.cb[B] : 0u, nc = has ? v.cc[B] : 0u;
                if (c0 == FMM_LET_ABSENT) {   // a grafted LET cell whose children were not exported:
                    atomicOr(err, 1u);        // the traversal fails (FMM_ERR_STATE); the root stands in
                    c0 = 0u;                  // for the missing child so that every listed source
                    nc = 1u;                  // owns >= 1 position (the owner arithmetic below)
                }
                uint32_t incl = nc;   // inclusive scan of the child counts
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
                    if (lane >= d) incl += y;
                }
                const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
                const uint32_t excl = incl - nc;   // first flattened position of this lane's source
                for (uint32_t f0 = 0; f0 < total; f0 += 32) {
                    const uint32_t f = f0 + lane;
                    const bool act = f < total;
                    // owner lane of position f: every listed source (a prefix of the lanes) owns
                    // >= 1 position, so it is k0 (the owner of f0: the last source starting at or
                    // before it) plus the number of sources starting in (f0, f] -- one ballot and
                    // one OR-reduction of start bits instead of a 5-step binary search of shuffles
                    const int k0 = 31 - __clz(__ballot_sync(0xffffffffu, has && excl <= f0));
                    const uint32_t rel = excl - f0;
                    const unsigned starts = __reduce_or_sync(0xffffffffu, has && excl > f0 && rel < 32u ? 1u << rel : 0u);
                    const int own = (k0 + __popc(starts & ((2u << lane) - 2u))) & 31;
                    const uint32_t own_excl = __shfl_sync(0xffffffffu, excl, own);
                    const uint32_t own_c0 = __shfl_sync(0xffffffffu, c0, own);
                    const uint32_t sc = own_c0 + (f - own_excl);
                    const int oc = act ? tc_classify(T, nT, v, sc, theta) : -1;
                    put(oc, sc, act, nxt, nnext);
                }
            }
            if (nnext > cap) {   // (global lists hold a whole level: cannot happen there)
                over = true;
                break;
            }
            __syncwarp();
            cur ^= 1;
            ncur = nnext;
        }
        if (SLAB) over |= o.m > capM || o.p > capP || o.d > capD;
        if (COUNT && mixflag && __any_sync(0xffffffffu, mix) && lane == 0) atomicOr(mixflag + t, 1u);
        if (COUNT && lane == 0) {
            if (over && !GLOB) {
                // no overflow kernel follows this level (the previous build had none here): the
                // traversal stops and is redone with them (tct_lists)
                if (ovf_redo) atomicOr(err, 2u);
                ovf[vi] = 1;
                ovf_list[atomicAdd(n_ovf, 1u)] = (uint32_t)vi;
            }
            cnt_m[vi] = o.m;
            cnt_p[vi] = o.p;
            cnt_d[vi] = o.d;
        }
        __syncwarp();
    }
}

// Per-level offsets of the three lists in three launches: tile scans (+ maxima), a one-block
// scan of the tile sums (level totals to tot[3] for the host), then base + offsets written
// straight to the CSR arrays: om/op = m2l_off/p2p_off + tb (base = entries of the previous
// levels), od = the pass-down offsets (nt + 1 entries).
constexpr int S3_THREADS = 256, S3_ITEMS = 4, S3_TILE = S3_THREADS * S3_ITEMS;

__device__ __forceinline__ unsigned long long s3_block_excl(unsigned long long v, unsigned long long* s_w,
                                                            unsigned long long* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    __syncthreads();
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    unsigned long long pre = 0, tot = 0;
    for (int i = 0; i < S3_THREADS / 32; ++i) {
        if (i < w) pre += s_w[i];
        tot += s_w[i];
    }
    *total = tot;
    return pre + x - v;
}

__global__ void __launch_bounds__(S3_THREADS) k_scan3_tiles(const uint32_t* __restrict__ c0, const uint32_t* __restrict__ c1,
                                                           const uint32_t* __restrict__ c2, int64_t n,
                                                           uint64_t* __restrict__ o0, uint64_t* __restrict__ o1,
                                                           uint64_t* __restrict__ o2, uint64_t* __restrict__ bsum,
                                                           int64_t nb, unsigned* __restrict__ mx) {
    __shared__ unsigned long long s_w[S3_THREADS / 32];
    const uint32_t* in[3] = {c0, c1, c2};
    uint64_t* out[3] = {o0, o1, o2};
    const int64_t base = (int64_t)blockIdx.x * S3_TILE + (int64_t)threadIdx.x * S3_ITEMS;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        uint32_t v[S3_ITEMS];
        unsigned long long sum = 0;
        unsigned m = 0;
#pragma unroll
        for (int k = 0; k < S3_ITEMS; ++k) {
            v[k] = base + k < n ? in[a][base + k] : 0u;
            sum += v[k];
            m = max(m, v[k]);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((threadIdx.x & 31) == 0 && m) atomicMax(&mx[a], m);
        unsigned long long tot;
        unsigned long long run = s3_block_excl(sum, s_w, &tot);
#pragma unroll
        for (int k = 0; k < S3_ITEMS; ++k) {
            if (base + k < n) out[a][base + k] = run;
            run += v[k];
        }
        if (threadIdx.x == 0) bsum[(int64_t)a * nb + blockIdx.x] = tot;
    }
}

// one block: exclusive scan of the tile sums of each list in place; totals to tot[a]
__global__ void __launch_bounds__(S3_THREADS) k_scan3_top(uint64_t* __restrict__ bsum, int64_t nb,
                                                         unsigned long long* __restrict__ tot,
                                                         const uint64_t* __restrict__ base_in,
                                                         uint64_t* __restrict__ base_out) {
    __shared__ unsigned long long s_w[S3_THREADS / 32];
    for (int a = 0; a < 3; ++a) {
        uint64_t* b = bsum + (int64_t)a * nb;
        unsigned long long carry = 0;
        for (int64_t c0 = 0; c0 < nb; c0 += S3_THREADS) {
            const int64_t i = c0 + threadIdx.x;
            const unsigned long long v = i < nb ? b[i] : 0ull;
            unsigned long long t;
            const unsigned long long e = s3_block_excl(v, s_w, &t);
            if (i < nb) b[i] = carry + e;
            carry += t;
        }
        if (threadIdx.x == 0) {
            tot[a] = carry;
            if (a < 2) base_out[a] = base_in[a] + carry;   // entries up to the end of this level
        }
    }
}

// adds the tile bases; the first slice of every target also lands in the targets' CSR offsets
// (om/op: m2l_off/p2p_off + tb; od: the level's pass-down offsets, nt + 1 entries)
__global__ void k_scan3_add(int64_t n, uint64_t* __restrict__ o0, uint64_t* __restrict__ o1, uint64_t* __restrict__ o2,
                            const uint64_t* __restrict__ bsum, int64_t nb, const uint64_t* __restrict__ base,
                            const unsigned long long* __restrict__ tot, int S, int64_t nt, uint64_t* __restrict__ om,
                            uint64_t* __restrict__ op, uint64_t* __restrict__ od) {
    const uint64_t base0 = base[0], base1 = base[1];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int64_t b = i / S3_TILE;
        const uint64_t v0 = o0[i] + base0 + bsum[b], v1 = o1[i] + base1 + bsum[nb + b], v2 = o2[i] + bsum[2 * nb + b];
        o0[i] = v0;
        o1[i] = v1;
        o2[i] = v2;
        if (i % S == 0) {
            const int64_t t = i / S;
            om[t] = v0;
            op[t] = v1;
            od[t] = v2;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        o0[n] = base0 + tot[0];
        o1[n] = base1 + tot[1];
        o2[n] = tot[2];
        od[nt] = tot[2];
    }
}

// single pass: slab slots -> CSR positions (warp per target; overflowed targets are written
// by the global-memory kernel instead)
__global__ void k_slab_gather(int64_t nt, const uint8_t* __restrict__ ovf, const uint32_t* __restrict__ cm,
                              const uint32_t* __restrict__ cp, const uint32_t* __restrict__ cd,
                              const uint64_t* __restrict__ om, const uint64_t* __restrict__ op,
                              const uint64_t* __restrict__ od, const uint32_t* __restrict__ slabM,
                              const uint32_t* __restrict__ slabP, const uint32_t* __restrict__ slabD, uint32_t capM,
                              uint32_t capP, uint32_t capD, uint32_t* __restrict__ srcM, uint32_t* __restrict__ srcP,
                              uint32_t* __restrict__ dsrc, uint64_t lenM, uint64_t lenP, uint64_t lenD,
                              unsigned* __restrict__ err) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (*reinterpret_cast<volatile unsigned*>(err) & 2u) return;   // being redone (see k_tct_level)
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nt; i += nw) {
        if (ovf[i]) continue;
        if (om[i] + cm[i] > lenM || op[i] + cp[i] > lenP || od[i] + cd[i] > lenD) {   // outputs sized from
            if (lane == 0) atomicOr(err, 2u);                                           // the previous build
            continue;
        }
        for (uint32_t k = lane; k < cm[i]; k += 32) srcM[om[i] + k] = slabM[(uint64_t)i * capM + k];
        for (uint32_t k = lane; k < cp[i]; k += 32) srcP[op[i] + k] = slabP[(uint64_t)i * capP + k];
        for (uint32_t k = lane; k < cd[i]; k += 32) dsrc[od[i] + k] = slabD[(uint64_t)i * capD + k];
    }
}

// per-level maxima of the three counts (slot sizes of the next build's single pass)
__global__ void k_max3(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, const uint32_t* __restrict__ c,
                       int64_t n, unsigned* __restrict__ mx) {
    unsigned ma = 0, mb = 0, mc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        ma = max(ma, a[i]);
        mb = max(mb, b[i]);
        mc = max(mc, c[i]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        ma = max(ma, __shfl_xor_sync(0xffffffffu, ma, o));
        mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
        mc = max(mc, __shfl_xor_sync(0xffffffffu, mc, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&mx[0], ma);
        atomicMax(&mx[1], mb);
        atomicMax(&mx[2], mc);
    }
}


}  // namespace

// One target-ordered traversal of the local target tree from the given seed sources at the root
// (local: the root itself; remote: the roots of grafted LETs) into the CSR lists `o`.
fmm_status tct_run(fmm_ctx* ctx, cudaStream_t s, const std::vector<uint32_t>& seeds, TcLists& o, bool single,
                   std::vector<std::array<uint32_t, 3>>& tc_max, std::vector<std::array<uint64_t, 3>>& tc_tot,
                   bool allow_fast, uint32_t* mixflag = nullptr, std::vector<unsigned>* novf_hist = nullptr) {
    const int64_t nc = ctx->ncell;
    const int nlev = (int)ctx->depth + 1;
    const Cells v{P_<double4>(ctx->c_cr), P_<uint32_t>(ctx->c_cb), P_<uint32_t>(ctx->c_cc)};
    int64_t maxw = 1;
    for (int l = 0; l < nlev; ++l) maxw = std::max(maxw, ctx->level_begin[l + 1] - ctx->level_begin[l]);
    // slices per target: levels with fewer targets than ~32 warps per SM split each target's
    // pass-down set over up to 32 warps
    const int64_t want = (int64_t)ctx->num_sms * 32;
    std::vector<int> S(nlev, 1);
    int64_t maxv = maxw;   // (target, slice) items of the widest level
    for (int l = 0; l < nlev; ++l) {
        const int64_t nt = ctx->level_begin[l + 1] - ctx->level_begin[l];
        S[l] = (int)std::min<int64_t>(32, std::max<int64_t>(1, want / std::max<int64_t>(nt, 1)));
        maxv = std::max(maxv, nt * S[l]);
    }
    FMM_TRY(buf_ensure(ctx, *o.off_m, (size_t)(nc + 1) * 8));
    FMM_TRY(buf_ensure(ctx, *o.off_p, (size_t)(nc + 1) * 8));
    // per-level scratch over (target, slice) items: counts (3 x u32), overflow flags (u8) and
    // list (u32), item offsets (3 x u64)
    FMM_TRY(buf_ensure(ctx, ctx->tc_cnt, (size_t)maxv * 12 + (size_t)maxv * 5 + 256));
    FMM_TRY(buf_ensure(ctx, ctx->tc_voff, (size_t)(maxv + 1) * 8 * 3 + 64));
    uint64_t* vm = P_<uint64_t>(ctx->tc_voff);
    uint64_t* vp = vm + (maxv + 1);
    uint64_t* vd = vp + (maxv + 1);
    FMM_TRY(buf_ensure(ctx, ctx->tc_lb, seeds.size() * 4 + 64));
    FMM_TRY(buf_ensure(ctx, ctx->dcount2, 128));
    uint32_t* cm = P_<uint32_t>(ctx->tc_cnt);
    uint32_t* cp = cm + maxv;
    uint32_t* cd = cp + maxv;
    uint32_t* ovf_list = cd + maxv;
    uint8_t* ovf = reinterpret_cast<uint8_t*>(ovf_list + maxv);
    uint32_t* d_seeds = P_<uint32_t>(ctx->tc_lb);
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(d_seeds, seeds.data(), seeds.size() * 4, cudaMemcpyHostToDevice, s));
    const int nseeds = (int)seeds.size();
    const int64_t scap = ctx->tc_scap > 0 ? ctx->tc_scap : TC_CAP;   // shared split-list capacity
    // per-level device records, zeroed once: bases (entries before each level) [nlev+1][2],
    // totals [nlev][3], overflow counts [nlev], maxima [nlev][3], error flags
    const size_t rec_bytes = (size_t)(nlev + 1) * 16 + (size_t)nlev * 24 + (size_t)nlev * 4 + (size_t)nlev * 12 + 64;
    FMM_TRY(buf_ensure(ctx, ctx->tc_rec, rec_bytes));
    uint64_t* d_base = P_<uint64_t>(ctx->tc_rec);
    unsigned long long* d_tot = reinterpret_cast<unsigned long long*>(d_base + 2 * (nlev + 1));
    unsigned* d_novf = reinterpret_cast<unsigned*>(d_tot + 3 * nlev);
    unsigned* d_mx = d_novf + nlev;
    unsigned* d_err = d_mx + 3 * nlev;
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->tc_rec.p, 0, rec_bytes, s));
    const int grid_max = ctx->num_sms * 8;
    const int32_t* par = P_<int32_t>(ctx->c_parent);
    FMM_TRY(buf_ensure(ctx, ctx->tc_bsum, (size_t)((maxv + S3_TILE - 1) / S3_TILE) * 3 * 8 + 64));
    uint64_t* bsum = P_<uint64_t>(ctx->tc_bsum);
    // overflow kernel: two level-sized split lists per warp, as many warps as 1 GB allows
    const int gwarps = (int)std::max<int64_t>(TC_WARPS, std::min<int64_t>(TC_GWARPS_MAX,
                                                                   ((int64_t)1 << 30) / (2 * maxw * 4)) / TC_WARPS * TC_WARPS);
    FMM_TRY(buf_ensure(ctx, ctx->tc_glob, (size_t)gwarps * 2 * maxw * 4));
    FMM_TRY(buf_ensure(ctx, ctx->tc_doff[0], (size_t)(maxw + 1) * 8));
    FMM_TRY(buf_ensure(ctx, ctx->tc_doff[1], (size_t)(maxw + 1) * 8));
    // slot sizes per level from the previous build's maxima (single pass); with the previous
    // build's per-level totals too, every buffer is sized up front and the levels run without
    // host round trips (fast), a capacity overflow being detected at the end (then: redone)
    auto slot = [](uint32_t m) { return (m + m / 4 + 32 + 31) & ~31u; };
    std::vector<char> use_slab(nlev, 0);
    size_t slab_bytes = 64;
    for (int l = 0; l < nlev && single && (int)tc_max.size() == nlev; ++l) {
        const int64_t nv = (ctx->level_begin[l + 1] - ctx->level_begin[l]) * S[l];
        const size_t b = (size_t)nv * (slot(tc_max[l][0]) + slot(tc_max[l][1]) + slot(tc_max[l][2])) * 4;
        use_slab[l] = b <= ((size_t)16 << 30);
        if (use_slab[l]) slab_bytes = std::max(slab_bytes, b + 64);
    }
    FMM_TRY(buf_ensure(ctx, ctx->tc_slab, slab_bytes));
    bool fast = allow_fast && single && (int)tc_max.size() == nlev && (int)tc_tot.size() == nlev;
    uint64_t maxd = 1;
    for (int l = 0; l < nlev && fast; ++l) {
        fast = fast && use_slab[l];
        maxd = std::max<uint64_t>(maxd, tc_tot[l][2]);
    }
    maxd += maxd / 8 + 1024;
    FMM_TRY(buf_ensure(ctx, *o.src_m, (size_t)std::max<int64_t>(*o.est_m, 1024) * 4));
    FMM_TRY(buf_ensure(ctx, *o.src_p, (size_t)std::max<int64_t>(*o.est_p, 1024) * 4));
    if (fast) {
        FMM_TRY(buf_ensure(ctx, ctx->tc_d[0], (size_t)maxd * 4));
        FMM_TRY(buf_ensure(ctx, ctx->tc_d[1], (size_t)maxd * 4));
    }
    uint64_t baseM = 0, baseP = 0;   // host copies (synchronous levels only)
    DevBuf* dprev = &ctx->tc_d[0];
    DevBuf* dcur = &ctx->tc_d[1];
    const uint64_t* doff_prev = nullptr;
    int64_t pb = 0;
    const int64_t gcap = maxw;   // a split list never exceeds one tree level
    for (int l = 0; l < nlev; ++l) {
        const int64_t tb = ctx->level_begin[l], te = ctx->level_begin[l + 1], nt = te - tb;
        const int Sl = S[l];
        const int64_t nv = nt * Sl;
        const unsigned g = (unsigned)std::min<int64_t>((nv + TC_WARPS - 1) / TC_WARPS, grid_max);
        const uint32_t* dsrc_prev = doff_prev ? P_<uint32_t>(*dprev) : nullptr;
        const bool slab = use_slab[l];
        uint32_t capM = 0, capP = 0, capD = 0;
        if (slab) {
            capM = slot(tc_max[l][0]);
            capP = slot(tc_max[l][1]);
            capD = slot(tc_max[l][2]);
        }
        uint32_t* slabM = P_<uint32_t>(ctx->tc_slab);
        uint32_t* slabP = slabM + (size_t)nv * capM;
        uint32_t* slabD = slabP + (size_t)nv * capP;
        unsigned* n_ovf = d_novf + l;
        unsigned* mx = d_mx + 3 * l;
        // the two overflow-kernel launches find nothing to do at a level where the previous build
        // had no overflowed target (~4 us each at c2): skipped then, and an overflow that does
        // appear stops the traversal for a redo with them (ovf_redo)
        const bool skip_glob = fast && novf_hist &&
                               (ctx->tc_force_skip || (l < (int)novf_hist->size() && (*novf_hist)[l] == 0));
        // sources of this level's targets that need no operand scaling: levels l-1 .. l+1
        const int64_t band_lo = ctx->level_begin[std::max(l - 1, 0)];
        const int64_t band_hi = ctx->level_begin[std::min(l + 2, nlev)];
        FMM_CUDA_TRY(ctx, cudaMemsetAsync(ovf, 0, (size_t)nv, s));
        if (slab)
            k_tct_level<2, false><<<g, TC_WARPS * 32, 0, s>>>(tb, te, par, pb, doff_prev, dsrc_prev, v, d_seeds, nseeds,
                                                              ctx->theta, cm, cp, cd, nullptr, nullptr, nullptr, slabM,
                                                              slabP, slabD, ovf, ovf_list, n_ovf, nullptr, scap, capM,
                                                              capP, capD, d_err, Sl, ~0ull, ~0ull, ~0ull, mixflag,
                                                              band_lo, band_hi, skip_glob);
        else
            k_tct_level<0, false><<<g, TC_WARPS * 32, 0, s>>>(tb, te, par, pb, doff_prev, dsrc_prev, v, d_seeds, nseeds,
                                                              ctx->theta, cm, cp, cd, nullptr, nullptr, nullptr,
                                                              nullptr, nullptr, nullptr, ovf, ovf_list, n_ovf, nullptr,
                                                              scap, 0, 0, 0, d_err, Sl, ~0ull, ~0ull, ~0ull, mixflag,
                                                              band_lo, band_hi, skip_glob);
        FMM_LAUNCH(ctx);
        // overflowed targets (count read on the device: a no-op launch when there are none)
        if (!skip_glob) {
            k_tct_level<0, true><<<gwarps / TC_WARPS, TC_WARPS * 32, 0, s>>>(
                tb, te, par, pb, doff_prev, dsrc_prev, v, d_seeds, nseeds, ctx->theta, cm, cp, cd, nullptr, nullptr,
                nullptr, nullptr, nullptr, nullptr, ovf, ovf_list, n_ovf, P_<uint32_t>(ctx->tc_glob), gcap, 0, 0, 0, d_err,
                Sl, ~0ull, ~0ull, ~0ull, mixflag, band_lo, band_hi);
            FMM_LAUNCH(ctx);
        }
        // offsets written straight into m2l_off / p2p_off (+ the entries of earlier levels, a
        // device value) and the pass-down CSR of this level
        uint64_t* om = P_<uint64_t>(*o.off_m) + tb;
        uint64_t* op = P_<uint64_t>(*o.off_p) + tb;
        uint64_t* od = P_<uint64_t>(ctx->tc_doff[l & 1]);
        // offsets per (target, slice) item (M2L/P2P absolute, pass-down level-local), then the
        // targets' CSR offsets (their first slice)
        const int64_t nb = (nv + S3_TILE - 1) / S3_TILE;
        k_scan3_tiles<<<(unsigned)nb, S3_THREADS, 0, s>>>(cm, cp, cd, nv, vm, vp, vd, bsum, nb, mx);
        FMM_LAUNCH(ctx);
        k_scan3_top<<<1, S3_THREADS, 0, s>>>(bsum, nb, d_tot + 3 * l, d_base + 2 * l, d_base + 2 * (l + 1));
        FMM_LAUNCH(ctx);
        const unsigned gw = (unsigned)std::min<int64_t>((nv + 255) / 256, grid_max);
        k_scan3_add<<<gw, 256, 0, s>>>(nv, vm, vp, vd, bsum, nb, d_base + 2 * l, d_tot + 3 * l, Sl, nt, om, op, od);
        FMM_LAUNCH(ctx);
        if (!fast) {   // sizes now: grow the outputs (keeping the earlier levels' entries)
            uint64_t tot[3];
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync(tot, d_tot + 3 * l, 24, cudaMemcpyDeviceToHost, s));
            FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
            const uint64_t needM = baseM + tot[0], needP = baseP + tot[1];
            if (needM * 4 > o.src_m->bytes) FMM_TRY(buf_ensure(ctx, *o.src_m, (size_t)(needM + needM / 4) * 4, true, s));
            if (needP * 4 > o.src_p->bytes) FMM_TRY(buf_ensure(ctx, *o.src_p, (size_t)(needP + needP / 4) * 4, true, s));
            FMM_TRY(buf_ensure(ctx, *dcur, (size_t)std::max<uint64_t>(tot[2], 1) * 4));
            baseM = needM;
            baseP = needP;
        }
        uint64_t lenM = o.src_m->bytes / 4, lenP = o.src_p->bytes / 4, lenD = dcur->bytes / 4;
        if (fast && ctx->tc_tight) lenM = lenP = lenD = 16;   // tests: force the capacity-overflow redo
        if (slab) {
            k_slab_gather<<<(unsigned)std::min<int64_t>((nv + 7) / 8, grid_max), 256, 0, s>>>(
                nv, ovf, cm, cp, cd, vm, vp, vd, slabM, slabP, slabD, capM, capP, capD, P_<uint32_t>(*o.src_m),
                P_<uint32_t>(*o.src_p), P_<uint32_t>(*dcur), lenM, lenP, lenD, d_err);
        } else {
            k_tct_level<1, false><<<g, TC_WARPS * 32, 0, s>>>(tb, te, par, pb, doff_prev, dsrc_prev, v, d_seeds, nseeds,
                                                              ctx->theta, cm, cp, cd, vm, vp, vd,
                                                              P_<uint32_t>(*o.src_m), P_<uint32_t>(*o.src_p),
                                                              P_<uint32_t>(*dcur), ovf, ovf_list, n_ovf, nullptr, scap,
                                                              0, 0, 0, d_err, Sl, lenM, lenP, lenD);
        }
        FMM_LAUNCH(ctx);
        if (!skip_glob) {
            k_tct_level<1, true><<<gwarps / TC_WARPS, TC_WARPS * 32, 0, s>>>(
                tb, te, par, pb, doff_prev, dsrc_prev, v, d_seeds, nseeds, ctx->theta, cm, cp, cd, vm, vp, vd,
                P_<uint32_t>(*o.src_m), P_<uint32_t>(*o.src_p), P_<uint32_t>(*dcur), ovf, ovf_list, n_ovf,
                P_<uint32_t>(ctx->tc_glob), gcap, 0, 0, 0, d_err, Sl, lenM, lenP, lenD);
            FMM_LAUNCH(ctx);
        }
        // this level's pass-down offsets (od, nt + 1 entries) are the next level's input
        doff_prev = od;
        pb = tb;
        std::swap(dprev, dcur);
    }
    // the list ends (device bases after the last level), the records for the next build
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(P_<uint64_t>(*o.off_m) + nc, d_base + 2 * nlev, 8, cudaMemcpyDeviceToDevice, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(P_<uint64_t>(*o.off_p) + nc, d_base + 2 * nlev + 1, 8, cudaMemcpyDeviceToDevice, s));
    std::vector<uint64_t> hbase(2 * (nlev + 1)), htot(3 * (size_t)nlev);
    std::vector<unsigned> hmx(3 * (size_t)nlev);
    unsigned herr = 0;
    std::vector<unsigned> hnovf(nlev);
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(hnovf.data(), d_novf, hnovf.size() * 4, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(hbase.data(), d_base, hbase.size() * 8, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(htot.data(), d_tot, htot.size() * 8, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(hmx.data(), d_mx, hmx.size() * 4, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&herr, d_err, 4, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    if (herr & 1u) {
        ctx->err = "dual tree traversal needed children of a remote LET cell that were not exported";
        return FMM_ERR_STATE;
    }
    std::vector<std::array<uint32_t, 3>> maxc(nlev);
    std::vector<std::array<uint64_t, 3>> totc(nlev);
    for (int l = 0; l < nlev; ++l)
        for (int a = 0; a < 3; ++a) {
            maxc[l][a] = hmx[3 * l + a];
            totc[l][a] = htot[3 * l + a];
        }
    tc_max = maxc;
    tc_tot = totc;
    if (novf_hist) *novf_hist = hnovf;   // (a stopped traversal's counts: the redo rewrites them)
    const uint64_t endM = hbase[2 * nlev], endP = hbase[2 * nlev + 1];
    *o.est_m = (int64_t)(endM + endM / 8 + 1024);
    *o.est_p = (int64_t)(endP + endP / 8 + 1024);
    if (herr & 2u) return FMM_ERR_OOM;   // outputs sized from the previous build were too small: redo
    *o.n_m = (int64_t)endM;
    *o.n_p = (int64_t)endP;
    return FMM_OK;
}

// local traversal: the root is the only seed; the lists land in the context's CSR arrays
// (also flags, per target, an M2L source more than one level away: ctx->tc_mixflag, read by the
// M2L pass instead of re-scanning the list)
fmm_status tct_lists(fmm_ctx* ctx, cudaStream_t s) {
    TcLists o{&ctx->m2l_off, &ctx->m2l_src, &ctx->p2p_off, &ctx->p2p_src, &ctx->n_m2l, &ctx->n_p2p,
              &ctx->tc_est_m2l, &ctx->tc_est_p2p};
    const std::vector<uint32_t> seeds{0u};
    ctx->tc_mix_ncell = -1;
    FMM_TRY(buf_ensure(ctx, ctx->tc_mixflag, (size_t)std::max<int64_t>(ctx->ncell, 1) * 4));
    uint32_t* mixflag = P_<uint32_t>(ctx->tc_mixflag);
    // (a redo after a short capacity guess revisits the same pairs: the flags are an OR)
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(mixflag, 0, (size_t)ctx->ncell * 4, s));
    fmm_status st = tct_run(ctx, s, seeds, o, ctx->tc_single, ctx->tc_max, ctx->tc_tot, true, mixflag, &ctx->tc_novf);
    if (st == FMM_ERR_OOM && ctx->err.empty())   // a capacity guess was short: sizes are known now
        st = tct_run(ctx, s, seeds, o, ctx->tc_single, ctx->tc_max, ctx->tc_tot, false, mixflag, &ctx->tc_novf);
    if (st == FMM_OK) ctx->tc_mix_ncell = ctx->ncell;
    return st;
}

// remote traversal of the LET roots grafted since the last one: one more CSR part
fmm_status tct_remote(fmm_ctx* ctx, const std::vector<uint32_t>& roots, cudaStream_t s) {
    if ((int)ctx->tc_rem.size() <= ctx->tc_nrem) ctx->tc_rem.emplace_back();   // buffers kept for reuse
    TcPart& pt = ctx->tc_rem[ctx->tc_nrem++];
    TcLists o{&pt.off_m, &pt.src_m, &pt.off_p, &pt.src_p, &pt.n_m, &pt.n_p, &pt.est_m, &pt.est_p};
    std::vector<std::array<uint32_t, 3>> none;   // count + emit passes (no slot history)
    std::vector<std::array<uint64_t, 3>> none_t;
    return tct_run(ctx, s, roots, o, false, none, none_t, false);
}

namespace {
constexpr int CAT_MAX = 8;   // CSR parts concatenated per pass
struct CatParts {
    const uint64_t* off[CAT_MAX];
    const uint32_t* src[CAT_MAX];
    int n;
};

__global__ void k_cat_count(int64_t nc, CatParts pa, uint32_t* __restrict__ cnt) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nc; t += stride) {
        uint64_t c = 0;
        for (int k = 0; k < pa.n; ++k) c += pa.off[k][t + 1] - pa.off[k][t];
        cnt[t] = (uint32_t)c;
    }
}

__global__ void k_cat_copy(int64_t nc, CatParts pa, const uint64_t* __restrict__ off, uint32_t* __restrict__ src) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < nc; t += nw) {
        uint64_t o = off[t];
        for (int k = 0; k < pa.n; ++k) {
            const uint64_t b = pa.off[k][t], e = pa.off[k][t + 1];
            for (uint64_t p = b + lane; p < e; p += 32) src[o + (p - b)] = pa.src[k][p];
            o += e - b;
        }
    }
}
}  // namespace

// lists of the local traversal followed, per target, by each remote part in graft order
fmm_status tct_concat(fmm_ctx* ctx, cudaStream_t s) {
    const int64_t nc = ctx->ncell;
    struct L {
        DevBuf* off;
        DevBuf* src;
        int64_t* n;
        bool m2l;
    } lists[2] = {{&ctx->m2l_off, &ctx->m2l_src, &ctx->n_m2l, true}, {&ctx->p2p_off, &ctx->p2p_src, &ctx->n_p2p, false}};
    FMM_TRY(buf_ensure(ctx, ctx->tc_cnt, (size_t)(nc + 1) * 12 + 256));
    uint32_t* cnt = P_<uint32_t>(ctx->tc_cnt);
    FMM_TRY(buf_ensure(ctx, ctx->cnt64, (size_t)(nc + 1) * 8));
    uint64_t* c64 = P_<uint64_t>(ctx->cnt64);
    const unsigned g = (unsigned)std::min<int64_t>((nc + 255) / 256, (int64_t)ctx->num_sms * 8);
    const unsigned gw = (unsigned)std::min<int64_t>((nc + 7) / 8, (int64_t)ctx->num_sms * 8);
    size_t done = 0;
    const size_t nparts = (size_t)ctx->tc_nrem;
    while (done < nparts) {
        const size_t take = std::min<size_t>(CAT_MAX - 1, nparts - done);
        for (auto& li : lists) {
            CatParts pa{};
            pa.off[0] = P_<uint64_t>(*li.off);
            pa.src[0] = P_<uint32_t>(*li.src);
            int64_t total = *li.n;
            for (size_t k = 0; k < take; ++k) {
                TcPart& pt = ctx->tc_rem[done + k];
                pa.off[k + 1] = P_<uint64_t>(li.m2l ? pt.off_m : pt.off_p);
                pa.src[k + 1] = P_<uint32_t>(li.m2l ? pt.src_m : pt.src_p);
                total += li.m2l ? pt.n_m : pt.n_p;
            }
            pa.n = (int)take + 1;
            k_cat_count<<<g, 256, 0, s>>>(nc, pa, cnt);
            FMM_LAUNCH(ctx);
            DevBuf& noff = ctx->tc_cat_off;
            DevBuf& nsrc = ctx->tc_cat_src;
            FMM_TRY(buf_ensure(ctx, noff, (size_t)(nc + 1) * 8));
            FMM_TRY(buf_ensure(ctx, nsrc, (size_t)std::max<int64_t>(total, 1) * 4));
            k_widen_u32_tc<<<g, 256, 0, s>>>(cnt, nc, c64);
            FMM_LAUNCH(ctx);
            FMM_TRY(scan_exclusive_u64(ctx, c64, P_<uint64_t>(noff), nc, P_<uint64_t>(noff) + nc, s));
            k_cat_copy<<<gw, 256, 0, s>>>(nc, pa, P_<uint64_t>(noff), P_<uint32_t>(nsrc));
            FMM_LAUNCH(ctx);
            std::swap(*li.off, noff);
            std::swap(*li.src, nsrc);
            *li.n = total;
        }
        done += take;
    }
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    ctx->tc_nrem = 0;
    return FMM_OK;
}
