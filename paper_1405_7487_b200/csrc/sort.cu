// sort.cu -- stable LSD radix sort of 64-bit keys (optionally with a u32 payload).
//
// "HOT is analogous to radix sort, where each bit of the key is examined at each step"
// (§II-B).  Used for the Morton keys (R5: stable, so ties keep the original
// index order because the payload starts as the identity) and for the canonical
// (target, source) order of the interaction lists (R10).
//
// Per 8-bit digit pass: (1) per-tile 256-bin histograms, (2) exclusive scan of the
// digit-major count table (digit * ntiles + tile), (3) stable scatter: inside a tile,
// warps rank their keys with __match_any_sync + per-warp bin counters, then per-bin
// prefix over warps; global position = scanned offset + warp prefix + in-warp rank.
// Passes whose digit is constant over all keys are skipped (one OR/AND reduction).
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
        unsigned peers = __match_any_sync(0xffffffffu, d);
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
                           int bit_lo, int bit_hi, uint64_t** kout, uint32_t** vout, cudaStream_t s) {
    *kout = k0;
    if (HAS_VAL) *vout = v0;
    if (n <= 1) return FMM_OK;
    if (n >= (int64_t)1 << 32) {
        ctx->err = "radix sort: n >= 2^32 unsupported";
        return FMM_ERR_ARG;
    }
    // which digits vary: OR ^ AND over all keys (one small host read; callers sync anyway)
    FMM_TRY(buf_ensure(ctx, ctx->red_tmp, 64));
    unsigned long long* d_oa = reinterpret_cast<unsigned long long*>(ctx->red_tmp.p);
    k_init_or_and<<<1, 1, 0, s>>>(d_oa);
    int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 8);
    k_or_and<<<blocks, 256, 0, s>>>(k0, n, d_oa);
    ctx->launches += 2;
    unsigned long long oa[2];
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(oa, d_oa, sizeof(oa), cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    uint64_t vary = oa[0] ^ oa[1];

    int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
    FMM_TRY(buf_ensure(ctx, ctx->sort_counts, (size_t)2 * RS_BINS * ntiles * sizeof(uint32_t)));
    uint32_t* counts = reinterpret_cast<uint32_t*>(ctx->sort_counts.p);
    uint32_t* offs = counts + RS_BINS * ntiles;
    uint64_t* kin = k0;
    uint64_t* kb = k1;
    uint32_t* vin = v0;
    uint32_t* vb = v1;
    for (int shift = bit_lo; shift < bit_hi; shift += 8) {
        uint64_t mask = 0xFFull << shift;
        if (!(vary & mask)) continue;
        k_histogram<<<(unsigned)ntiles, RS_THREADS, 0, s>>>(kin, n, shift, counts, ntiles);
        FMM_LAUNCH(ctx);
        FMM_TRY(scan_exclusive_u32(ctx, counts, offs, RS_BINS * ntiles, nullptr, s));
        k_scatter<HAS_VAL><<<(unsigned)ntiles, RS_THREADS, 0, s>>>(kin, kb, vin, vb, n, shift, offs, ntiles);
        FMM_LAUNCH(ctx);
        FMM_CUDA_TRY(ctx, cudaGetLastError());
        std::swap(kin, kb);
        if (HAS_VAL) std::swap(vin, vb);
    }
    *kout = kin;
    if (HAS_VAL) *vout = vin;
    return FMM_OK;
}
}  // namespace

fmm_status radix_sort_pairs(fmm_ctx* ctx, uint64_t* k0, uint64_t* k1, uint32_t* v0, uint32_t* v1, int64_t n,
                            int bit_lo, int bit_hi, uint64_t** kout, uint32_t** vout, cudaStream_t s) {
    return radix_sort_impl<true>(ctx, k0, k1, v0, v1, n, bit_lo, bit_hi, kout, vout, s);
}

fmm_status radix_sort_keys(fmm_ctx* ctx, uint64_t* k0, uint64_t* k1, int64_t n, int bit_lo, int bit_hi,
                           uint64_t** kout, cudaStream_t s) {
    uint32_t* dummy = nullptr;
    return radix_sort_impl<false>(ctx, k0, k1, nullptr, nullptr, n, bit_lo, bit_hi, kout, &dummy, s);
}
