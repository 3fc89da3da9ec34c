// dtt.cu -- breadth-first dual tree traversal producing explicit M2L and P2P lists (a8), used
// with FMM_DTT=bfs; the default traversal is target-ordered (tct.cu).  The P2P source runs
// (build_runs) and the list finishing below serve both.
//
// PAPER.md:151 §II-C: "the M2L and P2P kernels are processed ... by using the dual tree
// traversal [Dehnen]"; north_star asks for the traversal to emit explicit lists.
// R8 MAC: accept (A <- B) iff (R_A + R_B) < theta * sqrt((dx*dx + dy*dy) + dz*dz) over
//         the tight-box centres; fp64 with _rn intrinsics so it is bit-exact with the oracle.
// R9 from (root, root): MAC -> M2L; both leaves -> P2P; else split A if B is a leaf or
//         (A internal and R_A >= R_B), else split B.  The rule is a pure function of the
//         pair, so this breadth-first frontier emits the same SETS as the oracle's recursion.
// R10 canonical order: ascending (target, source).  Lists are stored as CSR by target:
//         off[ncell+1] (u64) and src[n] (u32), sources ascending within a target.
//
// Frontier step = ONE kernel: classify each pair, append M2L/P2P pairs and children with
// warp-aggregated atomics (buffers pre-sized: a pair emits at most one list entry or 8
// children), and histogram the list entries per target.  The host reads three counters.
// Grouping without a global sort: scan the per-target counts (CSR offsets) and scatter each
// unsorted pair's source into its target segment (atomic cursor).  P2P segments are then
// sorted in shared memory (bitonic, u32) -- canonical order; M2L segments only when
// FMM_CANONICAL_M2L=1 (otherwise fmm_copy_lists orders each segment on the host).
// Segments longer than the shared-memory sort are gathered and radix-sorted as packed
// (target, source) keys.
// P2P source runs (build_runs) merge Morton-contiguous source leaves for the P2P kernel.
#include "common.cuh"

namespace {

struct CellView {
    const double4* __restrict__ cr;
    const uint32_t* __restrict__ cb;
    const uint32_t* __restrict__ cc;
};

// outcome: 0 = M2L, 1 = P2P, 2 = split A, 3 = split B; nchild = children emitted
__device__ __forceinline__ int classify(const CellView& v, uint32_t a, uint32_t b, double theta, uint32_t& nchild) {
    const double4 A = v.cr[a], B = v.cr[b];
    const double dx = __dsub_rn(A.x, B.x), dy = __dsub_rn(A.y, B.y), dz = __dsub_rn(A.z, B.z);
    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    nchild = 0;
    if (__dadd_rn(A.w, B.w) < __dmul_rn(theta, __dsqrt_rn(d2))) return 0;
    const uint32_t ca = v.cc[a], cbn = v.cc[b];
    if (ca == 0 && cbn == 0) return 1;
    if (cbn == 0 || (ca != 0 && A.w >= B.w)) {
        nchild = ca;
        return 2;
    }
    nchild = cbn;
    return 3;
}

__device__ __forceinline__ unsigned long long warp_append(unsigned long long* counter, uint32_t cnt) {
    // exclusive warp scan of cnt, one atomic per warp; returns this lane's base
    const int lane = threadIdx.x & 31;
    uint32_t x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, x, 31);
    unsigned long long base = 0;
    if (lane == 31 && total) base = atomicAdd(counter, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 31);
    return base + (x - cnt);
}

__device__ __forceinline__ unsigned long long ballot_append(unsigned long long* counter, bool pred) {
    const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
    const unsigned m = __ballot_sync(0xffffffffu, pred);
    unsigned long long base = 0;
    if ((threadIdx.x & 31) == 0 && m) base = atomicAdd(counter, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    return base + __popc(m & lt);
}

// One block = 1024 consecutive frontier pairs (4 consecutive per thread, one 32-B load).  Each thread packs
// its (m2l, p2p, children) counts into one u64, a block-wide exclusive scan gives every
// thread its output offsets, and one thread reserves the block's space with 3 atomics.
constexpr int DT_THREADS = 256;
constexpr int DT_ITEMS = 4;

// cnt[0], cnt[1]: M2L / P2P list cursors; next_count: next-frontier cursor; cnt[3]: flags
// (1: absent LET children, 2: next frontier over cap_next, 4: a list over its capacity).  With
// nf_dev the frontier size is read on the device (levels launched back to back, no host sync).
__global__ void __launch_bounds__(DT_THREADS) k_dtt_step(const uint64_t* __restrict__ fr, int64_t nf_host,
                                                         const unsigned long long* __restrict__ nf_dev, CellView v,
                                                         double theta, unsigned long long* __restrict__ cnt,
                                                         unsigned long long* __restrict__ next_count,
                                                         uint64_t* __restrict__ m2l, uint64_t* __restrict__ p2p,
                                                         uint64_t* __restrict__ next, uint64_t cap_next,
                                                         uint64_t cap_m2l, uint64_t cap_p2p, int children_only) {
    __shared__ unsigned long long s_warp[DT_THREADS / 32];
    __shared__ unsigned long long s_base[3];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int64_t nf = nf_host;
    if (nf_dev) {
        // back-to-back levels: after an overflow in an earlier level the frontier in memory is
        // incomplete -- every later level is a no-op and the host re-runs synchronously
        if (*reinterpret_cast<volatile unsigned long long*>(&cnt[3]) & 6ull) return;
        nf = (int64_t)min(*nf_dev, (unsigned long long)cap_next);
    }
    // thread tid owns frontier entries i0 .. i0+3 of a tile: the outputs (block scan in thread
    // order) keep the frontier order, so the children of a split source stay adjacent downstream.
    // The next tile's entries are loaded while this tile is classified (ncu: the frontier load
    // was the top long-scoreboard stall).
    auto load_tile = [&](int64_t tile, uint64_t (&pr)[DT_ITEMS]) {
        const int64_t i0 = tile + (int64_t)tid * DT_ITEMS;
        if (i0 + DT_ITEMS <= nf) {
            const ulonglong2 u0 = *reinterpret_cast<const ulonglong2*>(fr + i0);
            const ulonglong2 u1 = *reinterpret_cast<const ulonglong2*>(fr + i0 + 2);
            pr[0] = u0.x; pr[1] = u0.y; pr[2] = u1.x; pr[3] = u1.y;
        } else {
#pragma unroll
            for (int k = 0; k < DT_ITEMS; ++k) pr[k] = i0 + k < nf ? fr[i0 + k] : 0ull;
        }
    };
    const int64_t tstride = (int64_t)gridDim.x * DT_THREADS * DT_ITEMS;
    uint64_t nxt[DT_ITEMS];
    if ((int64_t)blockIdx.x * DT_THREADS * DT_ITEMS < nf) load_tile((int64_t)blockIdx.x * DT_THREADS * DT_ITEMS, nxt);
    for (int64_t tile = (int64_t)blockIdx.x * DT_THREADS * DT_ITEMS; tile < nf; tile += tstride) {
        uint32_t a[DT_ITEMS], b[DT_ITEMS], nch[DT_ITEMS];
        int o[DT_ITEMS];
        unsigned long long packed = 0;   // m2l | p2p << 16 | children << 32
        const int64_t i0 = tile + (int64_t)tid * DT_ITEMS;
#pragma unroll
        for (int k = 0; k < DT_ITEMS; ++k) {
            o[k] = -1; nch[k] = 0;
            a[k] = (uint32_t)(nxt[k] >> 32);
            b[k] = (uint32_t)nxt[k];
        }
        if (tile + tstride < nf) load_tile(tile + tstride, nxt);
#pragma unroll
        for (int k = 0; k < DT_ITEMS; ++k) {
            const int64_t i = i0 + k;
            if (i < nf) o[k] = classify(v, a[k], b[k], theta, nch[k]);
            packed += (unsigned long long)(o[k] == 0) | ((unsigned long long)(o[k] == 1) << 16) |
                      ((unsigned long long)nch[k] << 32);
        }
        // block exclusive scan of the packed counts (fields never overflow: <= 1024, <= 1024, <= 8192)
        unsigned long long x = packed;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) s_warp[wid] = x;
        __syncthreads();
        if (wid == 0) {
            unsigned long long w = lane < DT_THREADS / 32 ? s_warp[lane] : 0ull;
#pragma unroll
            for (int d = 1; d < DT_THREADS / 32; d <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, w, d);
                if (lane >= d) w += y;
            }
            if (lane < DT_THREADS / 32) s_warp[lane] = w;
            if (lane == DT_THREADS / 32 - 1) {
                s_base[0] = children_only ? 0ull : atomicAdd(&cnt[0], w & 0xFFFFull);
                s_base[1] = children_only ? 0ull : atomicAdd(&cnt[1], (w >> 16) & 0xFFFFull);
                s_base[2] = atomicAdd(next_count, w >> 32);
            }
        }
        __syncthreads();
        const unsigned long long ex = (wid ? s_warp[wid - 1] : 0ull) + x - packed;
        unsigned long long pm = s_base[0] + (ex & 0xFFFFull);
        unsigned long long pp = s_base[1] + ((ex >> 16) & 0xFFFFull);
        unsigned long long pc = s_base[2] + (ex >> 32);
#pragma unroll
        for (int k = 0; k < DT_ITEMS; ++k) {
            const uint64_t pr = ((uint64_t)a[k] << 32) | b[k];
            if (nch[k] && pc + nch[k] > cap_next) {
                // next frontier larger than its buffer: the host grows it to the exact size
                // (the cursor still advances) and re-runs the step for the children only
                atomicOr(&cnt[3], 2ull);
                pc += nch[k];
            } else if (o[k] == 0) {
                if (!children_only) {
                    if (pm < cap_m2l) m2l[pm] = pr;
                    else atomicOr(&cnt[3], 4ull);
                    ++pm;
                }
            } else if (o[k] == 1) {
                if (!children_only) {
                    if (pp < cap_p2p) p2p[pp] = pr;
                    else atomicOr(&cnt[3], 4ull);
                    ++pp;
                }
            } else if (o[k] == 2) {
                const uint32_t k0 = v.cb[a[k]];
                for (uint32_t c = 0; c < nch[k]; ++c) next[pc + c] = ((uint64_t)(k0 + c) << 32) | b[k];
                pc += nch[k];
            } else if (o[k] == 3) {
                const uint32_t k0 = v.cb[b[k]];
                // a grafted LET cell whose children were not exported (let.cu): the cover was
                // insufficient; flag it instead of reading past the LET
                if (k0 == FMM_LET_ABSENT) atomicOr(&cnt[3], 1ull);
                for (uint32_t c = 0; c < nch[k]; ++c)
                    next[pc + c] = ((uint64_t)a[k] << 32) | (k0 == FMM_LET_ABSENT ? b[k] : k0 + c);
                pc += nch[k];
            }
        }
        __syncthreads();   // s_warp / s_base reuse
    }
}


__global__ void k_widen_u32(const uint32_t* __restrict__ in, int64_t n, uint64_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[i];
}

// Runs of equal targets in adjacent lanes (the valid lanes are a prefix of the warp): the run's
// first lane (head) and its length.  Replaces __match_any_sync (ncu: MATCH.ANY was the top
// stall of the count and scatter kernels); the traversal keeps a split source's children adjacent.
__device__ __forceinline__ void lane_runs(uint32_t t, bool ok, int& head, int& len) {
    const int lane = threadIdx.x & 31;
    const uint32_t prev = __shfl_up_sync(0xffffffffu, t, 1);
    const unsigned valid = __ballot_sync(0xffffffffu, ok);
    const unsigned heads = __ballot_sync(0xffffffffu, ok && (lane == 0 || prev != t));
    const unsigned upto = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
    head = 31 - __clz(heads & upto);
    const unsigned above = heads & ~(head == 31 ? 0xffffffffu : ((2u << head) - 1u));
    const int end = above ? __ffs(above) - 1 : __popc(valid);
    len = end - head;
}

// per-target counts of an unsorted (target, source) list: one atomic per run of equal targets
__global__ void k_count_targets(const uint64_t* __restrict__ lst, int64_t n, uint32_t* __restrict__ tcnt) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
        const int64_t i = i0 + threadIdx.x;
        const bool ok = i < n;
        const uint32_t t = ok ? (uint32_t)(lst[i] >> 32) : 0xffffffffu;
        int head, len;
        lane_runs(t, ok, head, len);
        if (ok && (int)(threadIdx.x & 31) == head) atomicAdd(&tcnt[t], (uint32_t)len);
    }
}

// counting-sort scatter of unsorted (target, source) pairs into per-target segments; the
// traversal emits the pairs of one target in runs (children of a split source are adjacent),
// so lanes of a warp with the same target share one atomic (__match_any_sync)
__global__ void k_scatter_src(const uint64_t* __restrict__ lst, int64_t n, const uint64_t* __restrict__ off,
                              uint32_t* __restrict__ cursor, uint32_t* __restrict__ src) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
        const int64_t i = i0 + threadIdx.x;
        const bool ok = i < n;
        const uint64_t pr = ok ? lst[i] : ~0ull;
        const uint32_t t = (uint32_t)(pr >> 32);
        int head, len;
        lane_runs(t, ok, head, len);
        const int lane = threadIdx.x & 31;
        uint32_t base = 0;
        if (ok && lane == head) base = atomicAdd(&cursor[t], (uint32_t)len);
        base = __shfl_sync(0xffffffffu, base, head);
        if (ok) src[off[t] + base + (uint32_t)(lane - head)] = (uint32_t)pr;
    }
}

constexpr int SEG_THREADS = 256;
constexpr int SEG_MAX = 4096;

// ascending sort of each target segment in shared memory (bitonic over the next power of two)
__global__ void __launch_bounds__(SEG_THREADS) k_segsort(const uint64_t* __restrict__ off, const uint32_t* __restrict__ tl,
                                                         int64_t nt, uint32_t* __restrict__ src) {
    __shared__ uint32_t s[SEG_MAX];
    for (int64_t ti = blockIdx.x; ti < nt; ti += gridDim.x) {
        const uint32_t t = tl[ti];
        const uint64_t b = off[t];
        const int n = (int)(off[t + 1] - b);
        int m = 1;
        while (m < n) m <<= 1;
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += SEG_THREADS) s[i] = i < n ? src[b + i] : 0xFFFFFFFFu;
        __syncthreads();
        for (int k = 2; k <= m; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < m; i += SEG_THREADS) {
                    const int l = i ^ j;
                    if (l > i) {
                        const uint32_t x = s[i], y = s[l];
                        const bool up = (i & k) == 0;
                        if ((x > y) == up) {
                            s[i] = y;
                            s[l] = x;
                        }
                    }
                }
                __syncthreads();
            }
        for (int i = threadIdx.x; i < n; i += SEG_THREADS) src[b + i] = s[i];
    }
}

// Warp-per-segment bitonic sort in registers: K elements per lane (lane-major: element
// e = lane*K + r), padded with 0xFFFFFFFF to the next power of two >= n (<= 32K).  Stages with
// partner distance j >= K exchange through __shfl_xor_sync, stages with j < K stay in the
// lane with compile-time register indices.
template <int K>
__device__ __forceinline__ void warp_bitonic(uint32_t (&v)[K], int np, int lane) {
    for (int k = 2; k <= np; k <<= 1) {
        for (int j = k >> 1; j >= K; j >>= 1) {
            const int pl = j / K;
            const bool lower = (lane & pl) == 0;
#pragma unroll
            for (int r = 0; r < K; ++r) {
                const uint32_t p = __shfl_xor_sync(0xffffffffu, v[r], pl);
                const bool up = (((lane * K) + r) & k) == 0;
                const uint32_t lo = min(v[r], p), hi = max(v[r], p);
                v[r] = (lower == up) ? lo : hi;
            }
        }
#pragma unroll
        for (int jj = K / 2; jj >= 1; jj >>= 1) {
            if (jj < k) {
#pragma unroll
                for (int r = 0; r < K; ++r) {
                    if ((r & jj) == 0) {
                        const int r2 = r | jj;
                        const bool up = (((lane * K) + r) & k) == 0;
                        const uint32_t lo = min(v[r], v[r2]), hi = max(v[r], v[r2]);
                        v[r] = up ? lo : hi;
                        v[r2] = up ? hi : lo;
                    }
                }
            }
        }
    }
}

template <int K>
__global__ void __launch_bounds__(128) k_segsort_warp(const uint64_t* __restrict__ off, const uint32_t* __restrict__ tl,
                                                      int64_t nt, uint32_t* __restrict__ src) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t ti = warp; ti < nt; ti += nw) {
        const uint32_t t = tl[ti];
        const uint64_t b = off[t];
        const int n = (int)(off[t + 1] - b);
        int np = 1;
        while (np < n) np <<= 1;
        uint32_t v[K];
#pragma unroll
        for (int r = 0; r < K; ++r) {
            const int e = lane * K + r;
            v[r] = e < n ? src[b + e] : 0xFFFFFFFFu;
        }
        warp_bitonic<K>(v, np, lane);
#pragma unroll
        for (int r = 0; r < K; ++r) {
            const int e = lane * K + r;
            if (e < n) src[b + e] = v[r];
        }
    }
}

// Warp-per-segment stable LSD radix sort in shared memory for up to MAXN keys: BITS-bit
// digits; ranking row by row (32 keys) with a ballot multi-split and a per-warp running
// histogram, exclusive scan of the bins, scatter to the other buffer.  ~25 instr/key/pass.
// <1024, 8>: 11 KB of shared memory per warp (20 warps/SM); <2048, 10>: 24 KB.
constexpr int WR_WARPS = 4;

template <int MAXN, int BITS>
constexpr size_t wradix_smem() { return (size_t)WR_WARPS * (2 * MAXN + MAXN / 2 + (1 << BITS)) * 4; }

template <int MAXN, int BITS>
__global__ void __launch_bounds__(WR_WARPS * 32) k_segsort_wradix(const uint64_t* __restrict__ off,
                                                                  const uint32_t* __restrict__ tl, int64_t nt,
                                                                  uint32_t* __restrict__ src, int nbits) {
    constexpr int BINS = 1 << BITS;
    extern __shared__ uint32_t wr_smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t* A = wr_smem + (size_t)w * (2 * MAXN + MAXN / 2 + BINS);
    uint32_t* B = A + MAXN;
    uint16_t* pos = reinterpret_cast<uint16_t*>(B + MAXN);
    uint32_t* hist = B + MAXN + MAXN / 2;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t warp = (int64_t)blockIdx.x * WR_WARPS + w;
    const int64_t nw = (int64_t)gridDim.x * WR_WARPS;
    for (int64_t ti = warp; ti < nt; ti += nw) {
        const uint32_t t = tl[ti];
        const uint64_t b0 = off[t];
        const int n = (int)(off[t + 1] - b0);
        for (int i = lane; i < n; i += 32) A[i] = src[b0 + i];
        uint32_t* in = A;
        uint32_t* out = B;
        for (int shift = 0; shift < nbits; shift += BITS) {
            for (int i = lane; i < BINS; i += 32) hist[i] = 0;
            __syncwarp();
            for (int r = 0; r < n; r += 32) {
                const int i = r + lane;
                const bool ok = i < n;
                const uint32_t d = ok ? (in[i] >> shift) & (BINS - 1) : 0u;
                const unsigned peers = match_digit<BITS>(d, __ballot_sync(0xffffffffu, ok));
                uint32_t before = 0;
                if (ok) before = hist[d];
                __syncwarp();
                if (ok) {
                    pos[i] = (uint16_t)(before + __popc(peers & lt));
                    if ((peers & lt) == 0) hist[d] = before + __popc(peers);
                }
                __syncwarp();
            }
            // exclusive scan of the bins (BINS / 32 per lane)
            constexpr int PER = BINS / 32;
            uint32_t loc = 0;
#pragma unroll
            for (int k = 0; k < PER; ++k) loc += hist[lane * PER + k];
            uint32_t x = loc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            uint32_t run = x - loc;
            __syncwarp();
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const uint32_t c = hist[lane * PER + k];
                hist[lane * PER + k] = run;
                run += c;
            }
            __syncwarp();
            for (int i = lane; i < n; i += 32) {
                const uint32_t v = in[i];
                out[hist[(v >> shift) & (BINS - 1)] + pos[i]] = v;
            }
            __syncwarp();
            uint32_t* tmp = in;
            in = out;
            out = tmp;
        }
        for (int i = lane; i < n; i += 32) src[b0 + i] = in[i];
        __syncwarp();
    }
}

// segment size classes for the sorts: 0: 2..256 (warp bitonic), 1: 257..1024 (radix<1024,8>),
// 2: 1025..2048 (radix<2048,10>), 3: 2049..SEG_MAX (CTA bitonic), 4: longer (global radix)
constexpr int NSEGCLS = 5;
__device__ __forceinline__ int seg_class(uint64_t n) {
    return n <= 1 ? -1 : n <= 256 ? 0 : n <= 1024 ? 1 : n <= 2048 ? 2 : n <= (uint64_t)SEG_MAX ? 3 : 4;
}

__global__ void k_seg_classify(const uint64_t* __restrict__ off, int64_t nc, uint32_t* __restrict__ lists,
                               unsigned* __restrict__ counts) {
    const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
    for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x; t0 < nc; t0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = t0 + threadIdx.x;
        const int c = t < nc ? seg_class(off[t + 1] - off[t]) : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, c);
        unsigned base = 0;
        if (c >= 0 && (peers & lt) == 0) base = atomicAdd(&counts[c], (unsigned)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, __ffs(peers) - 1);
        if (c >= 0) lists[(size_t)c * nc + base + __popc(peers & lt)] = (uint32_t)t;
    }
}

__global__ void k_max_u32(const uint32_t* __restrict__ in, int64_t n, unsigned* __restrict__ out) {
    unsigned m = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, in[i]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// fallback for very long segments: sorted packed keys -> src
__global__ void k_unpack_src(const uint64_t* __restrict__ lst, int64_t n, uint32_t* __restrict__ src) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) src[i] = (uint32_t)lst[i];
}

// segments longer than SEG_MAX: gather them as packed (target, source) keys, radix-sort that
// (small) array, write the sources back in place
__global__ void k_big_flags(const uint64_t* __restrict__ off, int64_t ncell, uint64_t* __restrict__ sz) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < ncell) {
        const uint64_t n = off[t + 1] - off[t];
        sz[t] = n > (uint64_t)SEG_MAX ? n : 0ull;
    }
}

__global__ void k_big_gather(const uint64_t* __restrict__ off, const uint64_t* __restrict__ boff, int64_t ncell,
                             const uint32_t* __restrict__ src, uint64_t* __restrict__ tmp) {
    for (int64_t t = blockIdx.x; t < ncell; t += gridDim.x) {
        const uint64_t n = off[t + 1] - off[t];
        if (n <= (uint64_t)SEG_MAX) continue;
        for (uint64_t i = threadIdx.x; i < n; i += blockDim.x)
            tmp[boff[t] + i] = ((uint64_t)t << 32) | src[off[t] + i];
    }
}

__global__ void k_big_scatter(const uint64_t* __restrict__ off, const uint64_t* __restrict__ boff, int64_t ncell,
                              const uint64_t* __restrict__ tmp, uint32_t* __restrict__ src) {
    for (int64_t t = blockIdx.x; t < ncell; t += gridDim.x) {
        const uint64_t n = off[t + 1] - off[t];
        if (n <= (uint64_t)SEG_MAX) continue;
        for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) src[off[t] + i] = (uint32_t)tmp[boff[t] + i];
    }
}

// sorted packed (target << 32 | source) list -> CSR: src[i] = low word; off[t] = first entry of
// target t (filled for every target between two consecutive distinct targets), off[nc] = n
__global__ void k_list_csr(const uint64_t* __restrict__ lst, int64_t n, int64_t nc, uint64_t* __restrict__ off,
                           uint32_t* __restrict__ src) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t x = lst[i];
        const int64_t t = (int64_t)(x >> 32);
        src[i] = (uint32_t)x;
        const int64_t tp = i == 0 ? -1 : (int64_t)(lst[i - 1] >> 32);
        for (int64_t u = tp + 1; u <= t; ++u) off[u] = (uint64_t)i;
        if (i == n - 1)
            for (int64_t u = t + 1; u <= nc; ++u) off[u] = (uint64_t)n;
    }
}

// canonical R10 order by one stable radix sort of the packed (target, source) words over the
// digits that can vary (source bits [0, nb_src), target bits [32, 32 + nb_tgt)), then CSR.
// FMM_LIST_SORT=1 only: at c2 the four onesweep passes over the 2.7e7 M2L words (~120 Gkeys/s
// per pass) cost 2x the counting scatter + per-segment sorts of canonicalise (measured round 1)
fmm_status canonicalise_sorted(fmm_ctx* ctx, DevBuf& lst, int64_t n, DevBuf& off, DevBuf& src, cudaStream_t s) {
    const int64_t nc = ctx->ncell;
    FMM_TRY(buf_ensure(ctx, off, (size_t)(nc + 1) * 8));
    FMM_TRY(buf_ensure(ctx, src, (size_t)std::max<int64_t>(n, 1) * 4));
    if (n == 0) {
        FMM_CUDA_TRY(ctx, cudaMemsetAsync(off.p, 0, (size_t)(nc + 1) * 8, s));
        return FMM_OK;
    }
    int nbs = 1, nbt = 1;
    while (((int64_t)1 << nbs) < nc + ctx->nrem) ++nbs;
    while (((int64_t)1 << nbt) < nc) ++nbt;
    const uint64_t vary = (((uint64_t)1 << nbs) - 1) | ((((uint64_t)1 << nbt) - 1) << 32);
    FMM_TRY(buf_ensure(ctx, ctx->lst_tmp, (size_t)n * 8));
    uint64_t* sorted = nullptr;
    FMM_TRY(radix_sort_keys(ctx, P_<uint64_t>(lst), P_<uint64_t>(ctx->lst_tmp), n, 0, 64, &sorted, s, vary));
    const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 16);
    k_list_csr<<<g, 256, 0, s>>>(sorted, n, nc, P_<uint64_t>(off), P_<uint32_t>(src));
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}

// unsorted packed list (n pairs) + per-target counts -> CSR off/src, canonical order
fmm_status canonicalise(fmm_ctx* ctx, DevBuf& lst, int64_t n, uint32_t* tcnt, DevBuf& off, DevBuf& src,
                        bool sort_segments, cudaStream_t s) {
    const int64_t nc = ctx->ncell;
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(tcnt, 0, (size_t)nc * 4, s));
    if (n > 0) {
        k_count_targets<<<(unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 16), 256, 0, s>>>(
            P_<uint64_t>(lst), n, tcnt);
        FMM_LAUNCH(ctx);
    }
    FMM_TRY(buf_ensure(ctx, off, (size_t)(nc + 1) * 8));
    FMM_TRY(buf_ensure(ctx, src, (size_t)std::max<int64_t>(n, 1) * 4));
    FMM_TRY(buf_ensure(ctx, ctx->cnt64, (size_t)(nc + 1) * 8));
    uint64_t* c64 = P_<uint64_t>(ctx->cnt64);
    k_widen_u32<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(tcnt, nc, c64);
    FMM_LAUNCH(ctx);
    FMM_TRY(scan_exclusive_u64(ctx, c64, P_<uint64_t>(off), nc, P_<uint64_t>(off) + nc, s));
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(tcnt, 0, (size_t)nc * 4, s));   // reuse as cursors
    const int g = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 16);
    k_scatter_src<<<std::max(g, 1), 256, 0, s>>>(P_<uint64_t>(lst), n, P_<uint64_t>(off), tcnt, P_<uint32_t>(src));
    FMM_LAUNCH(ctx);
    if (sort_segments) {
        // segments grouped by size class (one list of targets per class), each class sorted by
        // the kernel that fits it; only the classes that occur are launched
        FMM_TRY(buf_ensure(ctx, ctx->seg_lists, (size_t)NSEGCLS * nc * 4 + 64));
        uint32_t* lists = P_<uint32_t>(ctx->seg_lists);
        unsigned* d_ccnt = P_<unsigned>(ctx->dcount2) + 8;
        FMM_CUDA_TRY(ctx, cudaMemsetAsync(d_ccnt, 0, NSEGCLS * 4, s));
        k_seg_classify<<<(unsigned)std::min<int64_t>((nc + 255) / 256, (int64_t)ctx->num_sms * 8), 256, 0, s>>>(
            P_<uint64_t>(off), nc, lists, d_ccnt);
        FMM_LAUNCH(ctx);
        unsigned cc[NSEGCLS];
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(cc, d_ccnt, sizeof(cc), cudaMemcpyDeviceToHost, s));
        FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        int nbits = 1;
        while (((int64_t)1 << nbits) < nc + ctx->nrem) ++nbits;
        auto gwarps = [&](unsigned cnt, int wpb) {
            return (unsigned)std::max<int64_t>(std::min<int64_t>(((int64_t)cnt + wpb - 1) / wpb, (int64_t)ctx->num_sms * 32), 1);
        };
        if (cc[0]) {
            k_segsort_warp<8><<<gwarps(cc[0], 4), 128, 0, s>>>(P_<uint64_t>(off), lists, cc[0], P_<uint32_t>(src));
            FMM_LAUNCH(ctx);
        }
        if (cc[1]) {
            constexpr size_t sm = wradix_smem<1024, 8>();
            FMM_FUNC_ATTR_ONCE(ctx, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm, k_segsort_wradix<1024, 8>);
            k_segsort_wradix<1024, 8><<<gwarps(cc[1], WR_WARPS), WR_WARPS * 32, sm, s>>>(
                P_<uint64_t>(off), lists + (size_t)nc, cc[1], P_<uint32_t>(src), nbits);
            FMM_LAUNCH(ctx);
        }
        if (cc[2]) {
            constexpr size_t sm = wradix_smem<2048, 10>();
            FMM_FUNC_ATTR_ONCE(ctx, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm, k_segsort_wradix<2048, 10>);
            k_segsort_wradix<2048, 10><<<gwarps(cc[2], WR_WARPS), WR_WARPS * 32, sm, s>>>(
                P_<uint64_t>(off), lists + 2 * (size_t)nc, cc[2], P_<uint32_t>(src), nbits);
            FMM_LAUNCH(ctx);
        }
        if (cc[3]) {
            k_segsort<<<(unsigned)std::min<int64_t>(cc[3], (int64_t)ctx->num_sms * 16), SEG_THREADS, 0, s>>>(
                P_<uint64_t>(off), lists + 3 * (size_t)nc, cc[3], P_<uint32_t>(src));
            FMM_LAUNCH(ctx);
        }
        const unsigned mx = cc[4] ? (unsigned)SEG_MAX + 1 : 0u;
        if (mx > (unsigned)SEG_MAX) {
            // c64 (count widening buffer, nc+1 entries) is free again: reuse it for the sizes
            uint64_t* bsz = c64;
            FMM_TRY(buf_ensure(ctx, ctx->big_off, (size_t)(nc + 1) * 8));
            uint64_t* boff = P_<uint64_t>(ctx->big_off);
            k_big_flags<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(P_<uint64_t>(off), nc, bsz);
            FMM_LAUNCH(ctx);
            FMM_TRY(scan_exclusive_u64(ctx, bsz, boff, nc, boff + nc, s));
            uint64_t nbig = 0;
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&nbig, boff + nc, 8, cudaMemcpyDeviceToHost, s));
            FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
            FMM_TRY(buf_ensure(ctx, ctx->lst_tmp, (size_t)nbig * 16 + 16));
            uint64_t* t0 = P_<uint64_t>(ctx->lst_tmp);
            uint64_t* t1 = t0 + nbig;
            const unsigned gb = (unsigned)std::min<int64_t>(nc, (int64_t)ctx->num_sms * 8);
            k_big_gather<<<gb, 256, 0, s>>>(P_<uint64_t>(off), boff, nc, P_<uint32_t>(src), t0);
            FMM_LAUNCH(ctx);
            int nb = 0;
            while (((int64_t)1 << nb) < nc + ctx->nrem) ++nb;
            uint64_t* sorted = nullptr;
            FMM_TRY(radix_sort_keys(ctx, t0, t1, (int64_t)nbig, 0, 32 + nb, &sorted, s));
            k_big_scatter<<<gb, 256, 0, s>>>(P_<uint64_t>(off), boff, nc, sorted, P_<uint32_t>(src));
            FMM_LAUNCH(ctx);
        }
    }
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}

// ---- P2P source runs: consecutive list entries of one target whose body ranges are
// contiguous (Morton-adjacent leaves) merge into one run {start body, flat offset in the
// target's source stream}; rtot[t] = total sources of target t.  Used by the P2P kernel to
// stream a target's sources as full fixed-size chunks.
// warp per target: a list entry starts a new run unless its body range begins where the
// previous entry's ends.  Two passes over the lists: count the runs of every target (and its
// source total), scan the per-target counts into run_off, then emit the runs at those offsets.
__device__ __forceinline__ unsigned run_starts(const uint32_t* __restrict__ bb, const uint32_t* __restrict__ bc,
                                               uint32_t sc, bool ok, uint32_t& prev_end, int lane) {
    // body range end of the previous entry: the lane before, or the last entry of the previous round
    const uint32_t b = ok ? bb[sc] : 0u, e = ok ? b + bc[sc] : 0u;
    uint32_t pe = __shfl_up_sync(0xffffffffu, e, 1);
    if (lane == 0) pe = prev_end;
    prev_end = __shfl_sync(0xffffffffu, e, 31);
    return __ballot_sync(0xffffffffu, ok && pe != b);
}

__global__ void k_run_count(const uint64_t* __restrict__ off, const uint32_t* __restrict__ src, int64_t ncell,
                            const uint32_t* __restrict__ bb, const uint32_t* __restrict__ bc,
                            uint32_t* __restrict__ nrun, uint32_t* __restrict__ rtot,
                            unsigned long long* __restrict__ inter) {
    const int lane = threadIdx.x & 31;
    unsigned long long my_inter = 0;   // lane 0: sum over this warp's targets of |T| * sources(T)
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = w0; t < ncell; t += nw) {
        const uint64_t p0 = off[t], p1 = off[t + 1];
        uint32_t prev_end = ~0u, runs = 0, tot = 0;
        for (uint64_t q0 = p0; q0 < p1; q0 += 32) {
            const uint64_t p = q0 + lane;
            const bool ok = p < p1;
            const uint32_t sc = ok ? src[p] : 0u;
            runs += __popc(run_starts(bb, bc, sc, ok, prev_end, lane));
            uint32_t c = ok ? bc[sc] : 0u;
#pragma unroll
            for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            tot += c;
        }
        if (lane == 0) {
            nrun[t] = runs;
            rtot[t] = tot;
            my_inter += (unsigned long long)tot * bc[t];
        }
    }
    if (lane == 0 && my_inter) atomicAdd(inter, my_inter);
}

// warp per target: runs at roff[t] + (rank among the round's run starts); flat source offsets
// are a warp scan of the body counts
__global__ void k_run_emit(const uint64_t* __restrict__ off, const uint32_t* __restrict__ src, int64_t ncell,
                           const uint32_t* __restrict__ bb, const uint32_t* __restrict__ bc,
                           const uint32_t* __restrict__ roff, uint2* __restrict__ runs) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = w0; t < ncell; t += nw) {
        const uint64_t p0 = off[t], p1 = off[t + 1];
        uint32_t prev_end = ~0u, carry = 0, r = roff[t];
        for (uint64_t q0 = p0; q0 < p1; q0 += 32) {
            const uint64_t p = q0 + lane;
            const bool ok = p < p1;
            const uint32_t sc = ok ? src[p] : 0u;
            const unsigned st = run_starts(bb, bc, sc, ok, prev_end, lane);
            const uint32_t c = ok ? bc[sc] : 0u;
            uint32_t x = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if ((st >> lane) & 1u) runs[r + __popc(st & lt)] = make_uint2(bb[sc], carry + x - c);
            r += __popc(st);
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
    }
}


// leaves split by size for the P2P kernel: tiny leaves (<= P2P_TINY_LEAF bodies) to a warp per
// leaf, mid-size to a 128-thread CTA with 2 target pairs per thread, big leaves
// (>= P2P_BIG_LEAF) to a CTA with 4 pairs per thread (more reuse of each staged source).  The
// tiny class is used only when it holds >= 1/16 of the leaves (else its leaves join the mid
// class): decided from this build's counts, so the kernel -- and the fp32 summation order --
// of every leaf is a function of the input alone.
__global__ void k_leaf_count(const uint32_t* __restrict__ leaf_ids, int64_t nleaf, const uint32_t* __restrict__ bc,
                             unsigned* __restrict__ counts) {
    unsigned c0 = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nleaf; i += (int64_t)gridDim.x * blockDim.x)
        c0 += bc[leaf_ids[i]] <= P2P_TINY_LEAF;
    for (int o = 16; o; o >>= 1) c0 += __shfl_xor_sync(0xffffffffu, c0, o);
    if ((threadIdx.x & 31) == 0 && c0) atomicAdd(&counts[3], c0);
}

__global__ void k_leaf_split(const uint32_t* __restrict__ leaf_ids, int64_t nleaf, const uint32_t* __restrict__ bc,
                             const unsigned* __restrict__ tiny_count, uint32_t* __restrict__ out,
                             unsigned* __restrict__ counts) {
    const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
    const bool tiny_on = (int64_t)(*tiny_count) * 16 >= nleaf;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < nleaf; i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        int c = -1;
        if (i < nleaf) {
            const uint32_t m = bc[leaf_ids[i]];
            c = (tiny_on && m <= P2P_TINY_LEAF) ? 0 : (m >= P2P_BIG_LEAF ? 2 : 1);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, c);
        unsigned base = 0;
        if (c >= 0 && (peers & lt) == 0) base = atomicAdd(&counts[c], (unsigned)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, __ffs(peers) - 1);
        if (c >= 0) out[(size_t)c * nleaf + base + __popc(peers & lt)] = leaf_ids[i];
    }
}

fmm_status build_runs(fmm_ctx* ctx, cudaStream_t s) {
    const int64_t nc = ctx->ncell;
    FMM_TRY(buf_ensure(ctx, ctx->run_tmp, (size_t)(nc + 1) * 4 + 64));
    FMM_TRY(buf_ensure(ctx, ctx->run_off, (size_t)(2 * nc + 3) * 4));
    uint32_t* nrun = P_<uint32_t>(ctx->run_tmp);
    uint32_t* roff = P_<uint32_t>(ctx->run_off);
    uint32_t* rtot = roff + nc + 2;   // see common.cuh
    const uint64_t* off = P_<uint64_t>(ctx->p2p_off);
    const uint32_t* src = P_<uint32_t>(ctx->p2p_src);
    const int g = (int)std::min<int64_t>((nc + 3) / 4, (int64_t)ctx->num_sms * 16);
    unsigned long long* d_inter = P_<unsigned long long>(ctx->dcount2) + 2;   // read lazily (fmm_get_counts)
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(d_inter, 0, 8, s));
    k_run_count<<<std::max(g, 1), 128, 0, s>>>(off, src, nc, P_<uint32_t>(ctx->c_bb), P_<uint32_t>(ctx->c_bc), nrun,
                                              rtot, d_inter);
    FMM_LAUNCH(ctx);
    FMM_TRY(scan_exclusive_u32(ctx, nrun, roff, nc, roff + nc, s));
    // P2P leaf classes (see k_leaf_split); the counts ride on the same host round trip
    FMM_TRY(buf_ensure(ctx, ctx->leaf_cls, (size_t)3 * std::max<int64_t>(ctx->nleaf, 1) * 4));
    unsigned* d_lc = P_<unsigned>(ctx->dcount2) + 16;   // u32 16..19 (0: runs, 4..5: inter, 8..12: classes)
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(d_lc, 0, 16, s));
    if (ctx->nleaf > 0) {
        const unsigned gl = (unsigned)std::min<int64_t>((ctx->nleaf + 255) / 256, (int64_t)ctx->num_sms * 8);
        k_leaf_count<<<gl, 256, 0, s>>>(P_<uint32_t>(ctx->leaf_ids), ctx->nleaf, P_<uint32_t>(ctx->c_bc), d_lc);
        k_leaf_split<<<gl, 256, 0, s>>>(P_<uint32_t>(ctx->leaf_ids), ctx->nleaf, P_<uint32_t>(ctx->c_bc), d_lc + 3,
                                        P_<uint32_t>(ctx->leaf_cls), d_lc);
        ctx->launches += 2;
    }
    uint32_t hr[4] = {0, 0, 0, 0};
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&hr[0], roff + nc, 4, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&hr[1], d_lc, 12, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    const uint32_t nr = hr[0];
    for (int c = 0; c < 3; ++c) ctx->n_leaf_cls[c] = hr[1 + c];
    ctx->n_runs = nr;
    FMM_TRY(buf_ensure(ctx, ctx->runs, (size_t)std::max<uint32_t>(nr, 1) * 8 + 64));
    k_run_emit<<<std::max(g, 1), 128, 0, s>>>(off, src, nc, P_<uint32_t>(ctx->c_bb), P_<uint32_t>(ctx->c_bc), roff,
                                             P_<uint2>(ctx->runs));
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}

}  // namespace

// Level-by-level traversal.  Fast path (a fresh traversal whose buffer sizes are known from an
// earlier build of similar size): all 2*depth+1 levels are launched back to back, each reading its
// frontier size on the device, with one host round trip at the end; on any overflow (or a deeper
// traversal) it falls back to the synchronous loop, which grows the buffers to the exact sizes.
fmm_status dtt_pass(fmm_ctx* ctx, const uint64_t* seeds, int nseeds, bool append, cudaStream_t s,
                    int max_depth_src) {
    const CellView v{P_<double4>(ctx->c_cr), P_<uint32_t>(ctx->c_cb), P_<uint32_t>(ctx->c_cc)};
    const int64_t nc = ctx->ncell;
    FMM_TRY(buf_ensure(ctx, ctx->tcnt, (size_t)nc * 2 * 4));
    uint32_t* tcnt_m2l = P_<uint32_t>(ctx->tcnt);
    uint32_t* tcnt_p2p = tcnt_m2l + nc;
    FMM_TRY(buf_ensure(ctx, ctx->dcount2, 128));
    PhaseScope ps(ctx, PH_DTT, s);
    FMM_TRY(buf_ensure(ctx, ctx->dcount, 64));
    unsigned long long* d_cnt = P_<unsigned long long>(ctx->dcount);
    const int64_t m2l0 = append ? ctx->n_m2l : 0, p2p0 = append ? ctx->n_p2p : 0;
    // list cursors restart at the entries kept from an earlier traversal (append: the local
    // lists stay, a failed fast attempt's remote entries are overwritten)
    auto reset = [&]() -> fmm_status {
        const unsigned long long c0[4] = {(unsigned long long)m2l0, (unsigned long long)p2p0, 0ull, 0ull};
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(d_cnt, c0, sizeof(c0), cudaMemcpyHostToDevice, s));
        return FMM_OK;
    };
    const int g_max = ctx->num_sms * 8;
    int64_t peak = nseeds;

    if (ctx->dtt_est_front > 0 && (!append || max_depth_src >= 0)) {
        const int L = (int)ctx->depth + (append ? max_depth_src : (int)ctx->depth) + 1;
        const uint64_t capf = (uint64_t)ctx->dtt_est_front;
        const uint64_t capm = append ? std::max<uint64_t>(ctx->lst_m2l.bytes / 8, (uint64_t)ctx->dtt_est_m2l)
                                     : (uint64_t)ctx->dtt_est_m2l;
        const uint64_t capp = append ? std::max<uint64_t>(ctx->lst_p2p.bytes / 8, (uint64_t)ctx->dtt_est_p2p)
                                     : (uint64_t)ctx->dtt_est_p2p;
        FMM_TRY(buf_ensure(ctx, ctx->fr_a, (size_t)std::max<uint64_t>(capf, (uint64_t)nseeds) * 8));
        FMM_TRY(buf_ensure(ctx, ctx->fr_b, (size_t)capf * 8));
        FMM_TRY(buf_ensure(ctx, ctx->lst_m2l, (size_t)capm * 8, append, s));
        FMM_TRY(buf_ensure(ctx, ctx->lst_p2p, (size_t)capp * 8, append, s));
        FMM_TRY(buf_ensure(ctx, ctx->dtt_lvl, (size_t)(L + 2) * 8));
        unsigned long long* lvl = P_<unsigned long long>(ctx->dtt_lvl);
        FMM_TRY(reset());
        FMM_CUDA_TRY(ctx, cudaMemsetAsync(lvl, 0, (size_t)(L + 2) * 8, s));
        const unsigned long long ns = (unsigned long long)nseeds;
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(lvl, &ns, 8, cudaMemcpyHostToDevice, s));
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->fr_a.p, seeds, (size_t)nseeds * 8, cudaMemcpyHostToDevice, s));
        for (int l = 0; l < L; ++l) {
            DevBuf& in = (l & 1) ? ctx->fr_b : ctx->fr_a;
            DevBuf& out = (l & 1) ? ctx->fr_a : ctx->fr_b;
            k_dtt_step<<<g_max, DT_THREADS, 0, s>>>(P_<uint64_t>(in), 0, lvl + l, v, ctx->theta, d_cnt, lvl + l + 1,
                                                    P_<uint64_t>(ctx->lst_m2l), P_<uint64_t>(ctx->lst_p2p),
                                                    P_<uint64_t>(out), capf, capm, capp, 0);
            FMM_LAUNCH(ctx);
        }
        unsigned long long h[4];
        std::vector<unsigned long long> hl(L + 1);
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(h, d_cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(hl.data(), lvl, (size_t)(L + 1) * 8, cudaMemcpyDeviceToHost, s));
        FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        if (h[3] & 1ull) {
            ctx->err = "dual tree traversal needed children of a remote LET cell that were not exported";
            return FMM_ERR_STATE;
        }
        for (int l = 0; l <= L; ++l) peak = std::max<int64_t>(peak, (int64_t)hl[l]);
        if (!(h[3] & 6ull) && hl[L] == 0) {
            ctx->n_m2l = (int64_t)h[0];
            ctx->n_p2p = (int64_t)h[1];
            if (!append) {
                ctx->dtt_est_front = peak + peak / 8 + 1024;
                ctx->dtt_est_m2l = ctx->n_m2l + ctx->n_m2l / 8 + 1024;
                ctx->dtt_est_p2p = ctx->n_p2p + ctx->n_p2p / 8 + 1024;
            }
            return FMM_OK;
        }
        // overflow or deeper than 2*depth+1: redo synchronously (exact sizes)
    }

    int64_t n_m2l = m2l0, n_p2p = p2p0;
    FMM_TRY(buf_ensure(ctx, ctx->fr_a, (size_t)std::max(nseeds, 128) * 8));
    FMM_TRY(reset());
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->fr_a.p, seeds, (size_t)nseeds * 8, cudaMemcpyHostToDevice, s));
    int64_t nf = nseeds;
    while (nf > 0) {
        peak = std::max(peak, nf);
        // worst case per step: one list entry or 8 children per pair
        const size_t need_m = (size_t)(n_m2l + nf) * 8, need_p = (size_t)(n_p2p + nf) * 8;
        if (need_m > ctx->lst_m2l.bytes) FMM_TRY(buf_ensure(ctx, ctx->lst_m2l, need_m + need_m / 2, true, s));
        if (need_p > ctx->lst_p2p.bytes) FMM_TRY(buf_ensure(ctx, ctx->lst_p2p, need_p + need_p / 2, true, s));
        // next frontier: at most 8 children per pair; large frontiers start from 3x and grow
        // to the exact size on overflow (keeps deep traversals of 2^24+ particles in HBM)
        const uint64_t cap = nf <= (1 << 20) ? (uint64_t)nf * 8 : (uint64_t)nf * 3;
        FMM_TRY(buf_ensure(ctx, ctx->fr_b, (size_t)cap * 8));
        FMM_CUDA_TRY(ctx, cudaMemsetAsync(d_cnt + 2, 0, 8, s));   // next-frontier cursor restarts
        const int g = (int)std::min<int64_t>((nf + DT_THREADS * DT_ITEMS - 1) / (DT_THREADS * DT_ITEMS), g_max);
        const uint64_t capm = ctx->lst_m2l.bytes / 8, capp = ctx->lst_p2p.bytes / 8;
        k_dtt_step<<<g, DT_THREADS, 0, s>>>(P_<uint64_t>(ctx->fr_a), nf, nullptr, v, ctx->theta, d_cnt, d_cnt + 2,
                                            P_<uint64_t>(ctx->lst_m2l), P_<uint64_t>(ctx->lst_p2p),
                                            P_<uint64_t>(ctx->fr_b), ctx->fr_b.bytes / 8, capm,
                                            capp, 0);
        FMM_LAUNCH(ctx);
        unsigned long long h[4];
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(h, d_cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
        FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        if (h[3] & 2ull) {
            FMM_TRY(buf_ensure(ctx, ctx->fr_b, (size_t)h[2] * 8));
            FMM_CUDA_TRY(ctx, cudaMemsetAsync(d_cnt + 2, 0, 16, s));
            k_dtt_step<<<g, DT_THREADS, 0, s>>>(P_<uint64_t>(ctx->fr_a), nf, nullptr, v, ctx->theta, d_cnt, d_cnt + 2,
                                                P_<uint64_t>(ctx->lst_m2l), P_<uint64_t>(ctx->lst_p2p),
                                                P_<uint64_t>(ctx->fr_b), ctx->fr_b.bytes / 8, capm,
                                                capp, 1);
            FMM_LAUNCH(ctx);
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync(h, d_cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
            FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        }
        if (h[3]) {
            ctx->err = "dual tree traversal needed children of a remote LET cell that were not exported";
            return FMM_ERR_STATE;
        }
        n_m2l = (int64_t)h[0];
        n_p2p = (int64_t)h[1];
        nf = (int64_t)h[2];
        std::swap(ctx->fr_a, ctx->fr_b);
    }
    ctx->n_m2l = n_m2l;
    ctx->n_p2p = n_p2p;
    if (!append) {   // sizes for the back-to-back path of the next build
        ctx->dtt_est_front = peak + peak / 8 + 1024;
        ctx->dtt_est_m2l = n_m2l + n_m2l / 8 + 1024;
        ctx->dtt_est_p2p = n_p2p + n_p2p / 8 + 1024;
    }
    return FMM_OK;
}

fmm_status lists_pass(fmm_ctx* ctx, cudaStream_t s) {
    const int64_t nc = ctx->ncell;
    uint32_t* tcnt_m2l = P_<uint32_t>(ctx->tcnt);
    uint32_t* tcnt_p2p = tcnt_m2l + nc;
    PhaseScope ps(ctx, PH_LISTS, s);
    // P2P sources are always put in ascending order (the source runs need it); the M2L
    // segments only when canonical device order is requested (fmm_copy_lists sorts on the
    // host otherwise; the set and the grouping by target are the same either way).
    if (ctx->lists_csr) {
        // the target-ordered traversal wrote the CSR lists (+ remote parts to concatenate)
        if (ctx->tc_nrem > 0) FMM_TRY(tct_concat(ctx, s));
    } else if (ctx->list_sort == 1 && ctx->canonical_m2l) {
        FMM_TRY(canonicalise_sorted(ctx, ctx->lst_m2l, ctx->n_m2l, ctx->m2l_off, ctx->m2l_src, s));
        FMM_TRY(canonicalise_sorted(ctx, ctx->lst_p2p, ctx->n_p2p, ctx->p2p_off, ctx->p2p_src, s));
    } else {
        FMM_TRY(canonicalise(ctx, ctx->lst_m2l, ctx->n_m2l, tcnt_m2l, ctx->m2l_off, ctx->m2l_src, ctx->canonical_m2l, s));
        FMM_TRY(canonicalise(ctx, ctx->lst_p2p, ctx->n_p2p, tcnt_p2p, ctx->p2p_off, ctx->p2p_src, true, s));
    }
    return lists_finish(ctx, s);
}

// the target-ordered traversal (tct.cu) already wrote the CSR lists
fmm_status lists_finish(fmm_ctx* ctx, cudaStream_t s) {
    FMM_TRY(build_runs(ctx, s));   // synchronises s; the interaction count stays on the device
    ctx->p2p_inter = -1;
    // mutual P2P (p2p_mutual.cu): on request, or (auto) for large leaves
    const bool mut = ctx->p2p_mutual == 1 ||
                     (ctx->p2p_mutual == 2 && ctx->nleaf > 0 && ctx->n >= (int64_t)P2P_BIG_LEAF * ctx->nleaf);
    ctx->mut_ready = false;
    if (mut) FMM_TRY(p2p_mutual_prep(ctx, s));
    return FMM_OK;
}

fmm_status build_lists(fmm_ctx* ctx, cudaStream_t s) {
    const uint64_t root_pair = 0;
    FMM_TRY(dtt_pass(ctx, &root_pair, 1, false, s, -1));
    return lists_pass(ctx, s);
}
