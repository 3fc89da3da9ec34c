// sort.cu -- stable LSD radix sort of 64-bit keys (optionally with a u32 payload).
//
// "HOT is analogous to radix sort, where each bit of the key is examined at each step"
// (§II-B).  Used for the Morton keys (R5: stable, so ties keep the original
// index order because the payload starts as the identity) and for the canonical
// (target, source) order of the interaction lists (R10).
//
// Onesweep form (n < 2^30): ONE read of the keys builds the 256-bin histograms of every
// digit pass at once; then each 8-bit pass is a single kernel: a tile (4096 keys) takes the
// next tile number from an atomic counter, ranks its keys (warps: ballot multi-split + per-warp
// bin counters, then per-bin prefix over warps -- stable), publishes its per-bin counts and
// finds the counts of all earlier tiles by decoupled look-back (one 32-bit status word per
// tile and bin: flag | value), then scatters to digit base + earlier tiles + in-tile rank.
// No host round trip.  Which digits are sorted: every 8-bit digit of [bit_lo, bit_hi)
// that the caller's `vary` mask touches (vary = 0: an OR/AND reduction finds the varying
// digits, one host read).  Larger n: the three-kernel pass (per-tile histograms, scan,
// scatter) of the same ranking.
#include "common.cuh"

namespace {
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 16;                       // per thread
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;     // 4096 keys per tile
constexpr int RS_BINS = 256;

__global__ void __launch_bounds__(RS_THREADS) k_histogram(const uint64_t* __restrict__ keys, int64_t n, int shift,
                                                          uint32_t* __restrict__ counts, int64_t ntiles) {
    __shared__ uint32_t h[RS_BINS];
    h[threadIdx.x] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll 4
    for (int i = 0; i < RS_ITEMS; ++i) {
        int64_t j = base + i * RS_THREADS + threadIdx.x;
        if (j < n) atomicAdd(&h[(keys[j] >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

template <bool HAS_VAL>
__global__ void __launch_bounds__(RS_THREADS) k_scatter(const uint64_t* __restrict__ kin, uint64_t* __restrict__ kout,
                                                        const uint32_t* __restrict__ vin, uint32_t* __restrict__ vout,
                                                        int64_t n, int shift, const uint32_t* __restrict__ offsets,
                                                        int64_t ntiles) {
    __shared__ uint32_t s_whist[RS_WARPS][RS_BINS];
    __shared__ uint32_t s_off[RS_BINS];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int b = lane; b < RS_BINS; b += 32) s_whist[w][b] = 0;
    s_off[threadIdx.x] = offsets[(int64_t)threadIdx.x * ntiles + blockIdx.x];
    __syncwarp();
    // warp w owns the contiguous sub-tile [base + w*512, base + (w+1)*512)
    const int64_t base = (int64_t)blockIdx.x * RS_TILE + (int64_t)w * (RS_ITEMS * 32);
    uint64_t k[RS_ITEMS];
    uint32_t v[RS_ITEMS];
    uint32_t pos[RS_ITEMS];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < RS_ITEMS; ++i) {
        int64_t j = base + i * 32 + lane;
        bool ok = j < n;
        k[i] = ok ? kin[j] : 0ull;
        if (HAS_VAL) v[i] = ok ? vin[j] : 0u;
        uint32_t d = ok ? (uint32_t)((k[i] >> shift) & 0xFF) : 0x100u;
        unsigned peers = match_digit<9>(d, 0xffffffffu);
        uint32_t rank = __popc(peers & lt);
        uint32_t cnt = __popc(peers);
        bool leader = (peers & lt) == 0;
        uint32_t before = (d < 0x100u) ? s_whist[w][d] : 0u;
        __syncwarp();
        if (leader && d < 0x100u) s_whist[w][d] = before + cnt;
        __syncwarp();
        pos[i] = ok ? (before + rank) | (d << 16) : 0xFFFFFFFFu;
    }
    __syncthreads();
    // exclusive prefix over warps for every bin (thread t owns bin t)
    {
        uint32_t run = 0;
#pragma unroll
        for (int ww = 0; ww < RS_WARPS; ++ww) {
            uint32_t c = s_whist[ww][threadIdx.x];
            s_whist[ww][threadIdx.x] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < RS_ITEMS; ++i) {
        if (pos[i] == 0xFFFFFFFFu) continue;
        uint32_t d = pos[i] >> 16;
        uint32_t dst = s_off[d] + s_whist[w][d] + (pos[i] & 0xFFFFu);
        kout[dst] = k[i];
        if (HAS_VAL) vout[dst] = v[i];
    }
}

// ---- onesweep
// Staged pass: the tile is copied into shared memory by cp.async (all of a warp's copies in
// flight at once) and ranked from there, which frees the registers the direct pass holds its
// loads in (80 instead of ~120: 3 CTAs per SM instead of 2).  Measured at 2^26 keys: loads alone
// staged at 2 CTAs per SM were slower than the direct pass (10.8 vs 10.2 ms for 8 passes); the
// third CTA is what pays (8.3 ms).
__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(a), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_4(void* smem, const void* gmem) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(a), "l"(gmem) : "memory");
}

constexpr uint32_t OS_FA = 1u << 30;         // status: tile aggregate published
constexpr uint32_t OS_FP = 2u << 30;         // status: inclusive prefix published
constexpr uint32_t OS_VAL = OS_FA - 1u;
constexpr int OS_MAXPASS = 8;
struct OsShifts {
    int s[OS_MAXPASS];
    int n;
};

__global__ void __launch_bounds__(RS_THREADS) k_os_hist(const uint64_t* __restrict__ keys, int64_t n, OsShifts sh,
                                                        uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[OS_MAXPASS][RS_BINS];
    for (int p = 0; p < sh.n; ++p) h[p][threadIdx.x] = 0;
    __syncthreads();
    // each thread counts a contiguous chunk of 8 keys per step with run-length flushes, so the
    // long equal-digit runs of nearly sorted inputs (the lists' target digits) do not pile
    // 32 lanes onto one shared-memory counter
    constexpr int CH = 8;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * CH;
    for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * CH; i0 < n; i0 += stride) {
        const int m = (int)min((int64_t)CH, n - i0);
        uint64_t k[CH];
#pragma unroll
        for (int c = 0; c < CH; ++c) k[c] = c < m ? keys[i0 + c] : 0ull;
        for (int p = 0; p < sh.n; ++p) {
            uint32_t prev = (uint32_t)(k[0] >> sh.s[p]) & 0xFF, cnt = 1;
#pragma unroll
            for (int c = 1; c < CH; ++c) {
                if (c >= m) break;
                const uint32_t d = (uint32_t)(k[c] >> sh.s[p]) & 0xFF;
                if (d == prev) {
                    ++cnt;
                } else {
                    atomicAdd(&h[p][prev], cnt);
                    prev = d;
                    cnt = 1;
                }
            }
            atomicAdd(&h[p][prev], cnt);
        }
    }
    __syncthreads();
    for (int p = 0; p < sh.n; ++p)
        if (h[p][threadIdx.x]) atomicAdd(&hist[p * RS_BINS + threadIdx.x], h[p][threadIdx.x]);
}

// exclusive scan of each pass's 256 bins, in place (block per pass)
__global__ void __launch_bounds__(RS_BINS) k_os_base(uint32_t* __restrict__ hist) {
    __shared__ uint32_t s_w[RS_BINS / 32];
    uint32_t* h = hist + blockIdx.x * RS_BINS;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t v = h[threadIdx.x];
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    uint32_t pre = 0;
    for (int i = 0; i < w; ++i) pre += s_w[i];
    h[threadIdx.x] = pre + x - v;
}

template <bool HAS_VAL>
__global__ void __launch_bounds__(RS_THREADS, 3) k_os_pass_staged(const uint64_t* __restrict__ kin, uint64_t* __restrict__ kout,
                                                        const uint32_t* __restrict__ vin, uint32_t* __restrict__ vout,
                                                        int64_t n, int shift, const uint32_t* __restrict__ base,
                                                        uint32_t* __restrict__ status, uint32_t* __restrict__ tile_ctr) {
    extern __shared__ __align__(16) uint64_t s_k[];   // [RS_TILE] keys, then [RS_TILE] values
    uint32_t* s_v = reinterpret_cast<uint32_t*>(s_k + RS_TILE);
    __shared__ uint32_t s_whist[RS_WARPS][RS_BINS];
    __shared__ uint32_t s_off[RS_BINS], s_lbase[RS_BINS], s_wsum[RS_WARPS];
    __shared__ uint32_t s_tile;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int b = lane; b < RS_BINS; b += 32) s_whist[w][b] = 0;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    // warp w ranks the contiguous sub-tile [tile*TILE + w*512, +512) in index order (stable)
    const int64_t b0 = (int64_t)tile * RS_TILE + (int64_t)w * (RS_ITEMS * 32);
    uint64_t k[RS_ITEMS];
    uint32_t v[RS_ITEMS];
    uint32_t pos[RS_ITEMS / 2];   // two 16-bit warp-local ranks per word (0xFFFF: no key)
    const unsigned lt = (1u << lane) - 1u;
    // the warp's sub-tile lands in its own slots of s_k / s_v (each lane reads back what it
    // copied, so waiting for its own copies is enough); the scatter reuses the buffers after the
    // block barrier that ends the ranking
    const int sl = w * (RS_ITEMS * 32) + lane;
#pragma unroll
    for (int i = 0; i < RS_ITEMS; ++i) {
        const int64_t j = b0 + i * 32 + lane;
        if (j < n) {
            cp_async_8(s_k + sl + i * 32, kin + j);
            if (HAS_VAL) cp_async_4(s_v + sl + i * 32, vin + j);
        }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < RS_ITEMS; ++i) {
        const int64_t j = b0 + i * 32 + lane;
        const bool ok = j < n;
        k[i] = ok ? s_k[sl + i * 32] : 0ull;
        if (HAS_VAL) v[i] = ok ? s_v[sl + i * 32] : 0u;
        const uint32_t d = ok ? (uint32_t)((k[i] >> shift) & 0xFF) : 0x100u;
        const unsigned peers = match_digit<9>(d, 0xffffffffu);
        const uint32_t rank = __popc(peers & lt);
        const uint32_t before = (d < 0x100u) ? s_whist[w][d] : 0u;
        __syncwarp();
        if ((peers & lt) == 0 && d < 0x100u) s_whist[w][d] = before + __popc(peers);
        __syncwarp();
        const uint32_t r16 = ok ? before + rank : 0xFFFFu;
        if (i & 1) pos[i >> 1] |= r16 << 16;
        else pos[i >> 1] = r16;
    }
    __syncthreads();
    uint32_t run = 0;   // thread t owns bin t: exclusive prefix over warps, tile total in run
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ++ww) {
        const uint32_t c = s_whist[ww][threadIdx.x];
        s_whist[ww][threadIdx.x] = run;
        run += c;
    }
    // decoupled look-back over the earlier tiles' status words of this bin
    volatile uint32_t* st = status + (size_t)tile * RS_BINS + threadIdx.x;
    uint32_t excl = 0;
    if (tile == 0) {
        *st = OS_FP | run;
    } else {
        *st = OS_FA | run;
        // windows of LB earlier tiles read at once (independent loads), newest first; an
        // unpublished word restarts the window there
        constexpr int LB = 16;
        int64_t j = (int64_t)tile - 1;
        bool done = false;
        while (!done) {
            uint32_t xs[LB];
#pragma unroll
            for (int u = 0; u < LB; ++u)
                xs[u] = j - u >= 0 ? ((volatile uint32_t*)status)[(size_t)(j - u) * RS_BINS + threadIdx.x] : 0x80000000u;   // before tile 0: "prefix 0"
#pragma unroll
            for (int u = 0; u < LB; ++u) {
                if (done) break;
                const uint32_t x = xs[u];
                if (!(x & (OS_FA | OS_FP))) break;   // tile j - u not published yet: re-read from it
                excl += x & OS_VAL;
                if (x & OS_FP) done = true;
                --j;
            }
        }
        *st = OS_FP | (excl + run);
    }
    // tile-local bin starts (exclusive scan of the tile's bin counts)
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[w] = x;
    __syncthreads();
    uint32_t pre = 0;
    for (int i = 0; i < w; ++i) pre += s_wsum[i];
    const uint32_t lb = pre + x - run;
    s_lbase[threadIdx.x] = lb;
    s_off[threadIdx.x] = base[threadIdx.x] + excl - lb;   // global = s_off[d] + tile-local index
    __syncthreads();
    // keys in digit order inside the tile, then written out so that consecutive threads write
    // consecutive addresses of a bin
#pragma unroll
    for (int i = 0; i < RS_ITEMS; ++i) {
        const uint32_t r16 = (pos[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu;
        if (r16 == 0xFFFFu) continue;
        const uint32_t d = (uint32_t)(k[i] >> shift) & 0xFF;
        const uint32_t lp = s_lbase[d] + s_whist[w][d] + r16;
        s_k[lp] = k[i];
        if (HAS_VAL) s_v[lp] = v[i];
    }
    __syncthreads();
    const int cnt = (int)min((int64_t)RS_TILE, n - (int64_t)tile * RS_TILE);
    for (int i = threadIdx.x; i < cnt; i += RS_THREADS) {
        const uint64_t kk = s_k[i];
        const uint32_t dst = s_off[(uint32_t)(kk >> shift) & 0xFF] + (uint32_t)i;
        kout[dst] = kk;
        if (HAS_VAL) vout[dst] = s_v[i];
    }
}

// the same pass with the keys loaded straight into registers (loads interleaved with the
// ranking, ~120 registers, 2 CTAs per SM): lower latency per tile, so it wins while the tiles
// fit in one wave of the staged kernel's 3 CTAs per SM (c2: 256 tiles, 0.210 vs 0.224 ms)
template <bool HAS_VAL>
__global__ void __launch_bounds__(RS_THREADS) k_os_pass_direct(const uint64_t* __restrict__ kin, uint64_t* __restrict__ kout,
                                                        const uint32_t* __restrict__ vin, uint32_t* __restrict__ vout,
                                                        int64_t n, int shift, const uint32_t* __restrict__ base,
                                                        uint32_t* __restrict__ status, uint32_t* __restrict__ tile_ctr) {
    extern __shared__ __align__(16) uint64_t s_k[];   // [RS_TILE] keys, then [RS_TILE] values
    uint32_t* s_v = reinterpret_cast<uint32_t*>(s_k + RS_TILE);
    __shared__ uint32_t s_whist[RS_WARPS][RS_BINS];
    __shared__ uint32_t s_off[RS_BINS], s_lbase[RS_BINS], s_wsum[RS_WARPS];
    __shared__ uint32_t s_tile;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int b = lane; b < RS_BINS; b += 32) s_whist[w][b] = 0;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    // warp w ranks the contiguous sub-tile [tile*TILE + w*512, +512) in index order (stable)
    const int64_t b0 = (int64_t)tile * RS_TILE + (int64_t)w * (RS_ITEMS * 32);
    uint64_t k[RS_ITEMS];
    uint32_t v[RS_ITEMS];
    uint32_t pos[RS_ITEMS];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < RS_ITEMS; ++i) {
        const int64_t j = b0 + i * 32 + lane;
        const bool ok = j < n;
        k[i] = ok ? kin[j] : 0ull;
        if (HAS_VAL) v[i] = ok ? vin[j] : 0u;
        const uint32_t d = ok ? (uint32_t)((k[i] >> shift) & 0xFF) : 0x100u;
        const unsigned peers = match_digit<9>(d, 0xffffffffu);
        const uint32_t rank = __popc(peers & lt);
        const uint32_t before = (d < 0x100u) ? s_whist[w][d] : 0u;
        __syncwarp();
        if ((peers & lt) == 0 && d < 0x100u) s_whist[w][d] = before + __popc(peers);
        __syncwarp();
        pos[i] = ok ? (before + rank) | (d << 16) : 0xFFFFFFFFu;
    }
    __syncthreads();
    uint32_t run = 0;   // thread t owns bin t: exclusive prefix over warps, tile total in run
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ++ww) {
        const uint32_t c = s_whist[ww][threadIdx.x];
        s_whist[ww][threadIdx.x] = run;
        run += c;
    }
    // decoupled look-back over the earlier tiles' status words of this bin
    volatile uint32_t* st = status + (size_t)tile * RS_BINS + threadIdx.x;
    uint32_t excl = 0;
    if (tile == 0) {
        *st = OS_FP | run;
    } else {
        *st = OS_FA | run;
        // windows of LB earlier tiles read at once (independent loads), newest first; an
        // unpublished word restarts the window there
        constexpr int LB = 16;
        int64_t j = (int64_t)tile - 1;
        bool done = false;
        while (!done) {
            uint32_t xs[LB];
#pragma unroll
            for (int u = 0; u < LB; ++u)
                xs[u] = j - u >= 0 ? ((volatile uint32_t*)status)[(size_t)(j - u) * RS_BINS + threadIdx.x] : 0x80000000u;   // before tile 0: "prefix 0"
#pragma unroll
            for (int u = 0; u < LB; ++u) {
                if (done) break;
                const uint32_t x = xs[u];
                if (!(x & (OS_FA | OS_FP))) break;   // tile j - u not published yet: re-read from it
                excl += x & OS_VAL;
                if (x & OS_FP) done = true;
                --j;
            }
        }
        *st = OS_FP | (excl + run);
    }
    // tile-local bin starts (exclusive scan of the tile's bin counts)
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[w] = x;
    __syncthreads();
    uint32_t pre = 0;
    for (int i = 0; i < w; ++i) pre += s_wsum[i];
    const uint32_t lb = pre + x - run;
    s_lbase[threadIdx.x] = lb;
    s_off[threadIdx.x] = base[threadIdx.x] + excl - lb;   // global = s_off[d] + tile-local index
    __syncthreads();
    // keys in digit order inside the tile, then written out so that consecutive threads write
    // consecutive addresses of a bin
#pragma unroll
    for (int i = 0; i < RS_ITEMS; ++i) {
        if (pos[i] == 0xFFFFFFFFu) continue;
        const uint32_t d = pos[i] >> 16;
        const uint32_t lp = s_lbase[d] + s_whist[w][d] + (pos[i] & 0xFFFFu);
        s_k[lp] = k[i];
        if (HAS_VAL) s_v[lp] = v[i];
    }
    __syncthreads();
    const int cnt = (int)min((int64_t)RS_TILE, n - (int64_t)tile * RS_TILE);
    for (int i = threadIdx.x; i < cnt; i += RS_THREADS) {
        const uint64_t kk = s_k[i];
        const uint32_t dst = s_off[(uint32_t)(kk >> shift) & 0xFF] + (uint32_t)i;
        kout[dst] = kk;
        if (HAS_VAL) vout[dst] = s_v[i];
    }
}

__global__ void k_or_and(const uint64_t* __restrict__ keys, int64_t n, unsigned long long* out) {
    uint64_t o = 0, a = ~0ull;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = keys[i];
        o |= k;
        a &= k;
    }
#pragma unroll
    for (int s = 16; s; s >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, s);
        a &= __shfl_xor_sync(0xffffffffu, a, s);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicOr(&out[0], (unsigned long long)o);
        atomicAnd(&out[1], (unsigned long long)a);
    }
}

__global__ void k_init_or_and(unsigned long long* out) {
    out[0] = 0ull;
    out[1] = ~0ull;
}

template <bool HAS_VAL>
fmm_status radix_sort_impl(fmm_ctx* ctx, uint64_t* k0, uint64_t* k1, uint32_t* v0, uint32_t* v1, int64_t n,
                           int bit_lo, int bit_hi, uint64_t vary, uint64_t** kout, uint32_t** vout, cudaStream_t s) {
    *kout = k0;
    if (HAS_VAL) *vout = v0;
    if (n <= 1) return FMM_OK;
    if (n >= (int64_t)1 << 32) {
        ctx->err = "radix sort: n >= 2^32 unsupported";
        return FMM_ERR_ARG;
    }
    if (vary == 0) {
        // which digits vary: OR ^ AND over all keys (one small host read)
        FMM_TRY(buf_ensure(ctx, ctx->red_tmp, 64));
        unsigned long long* d_oa = reinterpret_cast<unsigned long long*>(ctx->red_tmp.p);
        k_init_or_and<<<1, 1, 0, s>>>(d_oa);
        int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 8);
        k_or_and<<<blocks, 256, 0, s>>>(k0, n, d_oa);
        ctx->launches += 2;
        unsigned long long oa[2];
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(oa, d_oa, sizeof(oa), cudaMemcpyDeviceToHost, s));
        FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        vary = oa[0] ^ oa[1];
    }
    OsShifts sh{};
    for (int shift = bit_lo; shift < bit_hi && sh.n < OS_MAXPASS; shift += 8)
        if (vary & (0xFFull << shift)) sh.s[sh.n++] = shift;
    if (sh.n == 0) return FMM_OK;

    const int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
    uint64_t* kin = k0;
    uint64_t* kb = k1;
    uint32_t* vin = v0;
    uint32_t* vb = v1;
    if (n < (int64_t)OS_FA) {
        // [tile counters (64 B)] [hist npass x 256] [status npass x ntiles x 256], zeroed once
        const size_t words = 16 + (size_t)sh.n * RS_BINS + (size_t)sh.n * ntiles * RS_BINS;
        FMM_TRY(buf_ensure(ctx, ctx->sort_counts, words * 4));
        uint32_t* ctr = P_<uint32_t>(ctx->sort_counts);
        uint32_t* hist = ctr + 16;
        uint32_t* status = hist + (size_t)sh.n * RS_BINS;
        FMM_CUDA_TRY(ctx, cudaMemsetAsync(ctr, 0, words * 4, s));
        k_os_hist<<<(unsigned)std::min<int64_t>((n + RS_THREADS - 1) / RS_THREADS, (int64_t)ctx->num_sms * 4),
                    RS_THREADS, 0, s>>>(k0, n, sh, hist);
        FMM_LAUNCH(ctx);
        k_os_base<<<sh.n, RS_BINS, 0, s>>>(hist);
        FMM_LAUNCH(ctx);
        constexpr int smem = RS_TILE * (8 + (HAS_VAL ? 4 : 0));
        FMM_FUNC_ATTR_ONCE(ctx, cudaFuncAttributeMaxDynamicSharedMemorySize, smem, k_os_pass_staged<HAS_VAL>);
        FMM_FUNC_ATTR_ONCE(ctx, cudaFuncAttributeMaxDynamicSharedMemorySize, smem, k_os_pass_direct<HAS_VAL>);
        // staged tiles (3 CTAs per SM) once there is more than one wave of them (c4s: 8 passes
        // 10.2 -> 8.3 ms); FMM_SORT_STAGED=0/1 forces either kernel
        const bool staged = ctx->sort_staged >= 0 ? ctx->sort_staged != 0 : ntiles > (int64_t)ctx->num_sms * 3;
        for (int p = 0; p < sh.n; ++p) {
            if (staged)
                k_os_pass_staged<HAS_VAL><<<(unsigned)ntiles, RS_THREADS, smem, s>>>(
                    kin, kb, vin, vb, n, sh.s[p], hist + p * RS_BINS, status + (size_t)p * ntiles * RS_BINS, ctr + p);
            else
                k_os_pass_direct<HAS_VAL><<<(unsigned)ntiles, RS_THREADS, smem, s>>>(
                    kin, kb, vin, vb, n, sh.s[p], hist + p * RS_BINS, status + (size_t)p * ntiles * RS_BINS, ctr + p);
            FMM_LAUNCH(ctx);
            std::swap(kin, kb);
            if (HAS_VAL) std::swap(vin, vb);
        }
    } else {
        FMM_TRY(buf_ensure(ctx, ctx->sort_counts, (size_t)2 * RS_BINS * ntiles * sizeof(uint32_t)));
        uint32_t* counts = reinterpret_cast<uint32_t*>(ctx->sort_counts.p);
        uint32_t* offs = counts + RS_BINS * ntiles;
        for (int p = 0; p < sh.n; ++p) {
            k_histogram<<<(unsigned)ntiles, RS_THREADS, 0, s>>>(kin, n, sh.s[p], counts, ntiles);
            FMM_LAUNCH(ctx);
            FMM_TRY(scan_exclusive_u32(ctx, counts, offs, RS_BINS * ntiles, nullptr, s));
            k_scatter<HAS_VAL><<<(unsigned)ntiles, RS_THREADS, 0, s>>>(kin, kb, vin, vb, n, sh.s[p], offs, ntiles);
            FMM_LAUNCH(ctx);
            std::swap(kin, kb);
            if (HAS_VAL) std::swap(vin, vb);
        }
    }
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    *kout = kin;
    if (HAS_VAL) *vout = vin;
    return FMM_OK;
}
}  // namespace

fmm_status radix_sort_pairs(fmm_ctx* ctx, uint64_t* k0, uint64_t* k1, uint32_t* v0, uint32_t* v1, int64_t n,
                            int bit_lo, int bit_hi, uint64_t** kout, uint32_t** vout, cudaStream_t s, uint64_t vary) {
    return radix_sort_impl<true>(ctx, k0, k1, v0, v1, n, bit_lo, bit_hi, vary, kout, vout, s);
}

fmm_status radix_sort_keys(fmm_ctx* ctx, uint64_t* k0, uint64_t* k1, int64_t n, int bit_lo, int bit_hi,
                           uint64_t** kout, cudaStream_t s, uint64_t vary) {
    uint32_t* dummy = nullptr;
    return radix_sort_impl<false>(ctx, k0, k1, nullptr, nullptr, n, bit_lo, bit_hi, vary, kout, &dummy, s);
}
