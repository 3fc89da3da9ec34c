// scan.cu -- device-wide exclusive prefix sums (u32, u64) used by the tree build, the
// list CSR offsets and the radix sort.  Three-phase: per-block scan -> scan of block
// totals (recursive) -> add block offsets.  4096 items per 512-thread block.
#include "common.cuh"

namespace {
constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <typename T>
__device__ __forceinline__ T block_exclusive_sum(T v, T* s_warp, T* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        T w = lane < (SCAN_THREADS / 32) ? s_warp[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < SCAN_THREADS / 32) s_warp[lane] = w;
    }
    __syncthreads();
    T warp_prefix = wid ? s_warp[wid - 1] : T(0);
    *total = s_warp[SCAN_THREADS / 32 - 1];
    return warp_prefix + x - v;
}

template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_tiles(const T* __restrict__ in, T* __restrict__ out,
                                                             T* __restrict__ tile_sums, int64_t n) {
    __shared__ T s_warp[SCAN_THREADS / 32];
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    T v[SCAN_ITEMS];
    T sum = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        v[i] = (base + i < n) ? in[base + i] : T(0);
        sum += v[i];
    }
    T total;
    T run = block_exclusive_sum<T>(sum, s_warp, &total);
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

template <typename T>
__global__ void k_add_offsets(T* __restrict__ out, const T* __restrict__ offs, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] += offs[i / SCAN_TILE];
}

template <typename T>
__global__ void k_set_total(const T* __restrict__ last_excl, const T* __restrict__ last_in, T* total) {
    *total = *last_excl + *last_in;
}

template <typename T>
fmm_status scan_rec(fmm_ctx* ctx, const T* in, T* out, int64_t n, T* tmp, cudaStream_t s) {
    int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    T* sums = tmp;
    T* sums_scanned = tmp + tiles;
    k_scan_tiles<T><<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(in, out, sums, n);
    FMM_LAUNCH(ctx);
    if (tiles > 1) {
        FMM_TRY(scan_rec<T>(ctx, sums, sums_scanned, tiles, tmp + 2 * tiles, s));
        k_add_offsets<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(out, sums_scanned, n);
        FMM_LAUNCH(ctx);
    }
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}

template <typename T>
fmm_status scan_exclusive(fmm_ctx* ctx, const T* in, T* out, int64_t n, T* total_dev, cudaStream_t s) {
    if (n <= 0) {
        if (total_dev) FMM_CUDA_TRY(ctx, cudaMemsetAsync(total_dev, 0, sizeof(T), s));
        return FMM_OK;
    }
    // temp: 2 * tiles per level, geometric
    int64_t need = 0, m = n;
    while (m > 1) {
        m = (m + SCAN_TILE - 1) / SCAN_TILE;
        need += 2 * m;
    }
    need += 8;
    FMM_TRY(buf_ensure(ctx, ctx->scan_tmp, (size_t)need * sizeof(T)));
    T* tmp = reinterpret_cast<T*>(ctx->scan_tmp.p);
    FMM_TRY(scan_rec<T>(ctx, in, out, n, tmp, s));
    if (total_dev) {
        k_set_total<T><<<1, 1, 0, s>>>(out + n - 1, in + n - 1, total_dev);
        FMM_LAUNCH(ctx);
        FMM_CUDA_TRY(ctx, cudaGetLastError());
    }
    return FMM_OK;
}
}  // namespace

fmm_status scan_exclusive_u32(fmm_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t n, uint32_t* total_dev,
                              cudaStream_t s) {
    return scan_exclusive<uint32_t>(ctx, in, out, n, total_dev, s);
}
fmm_status scan_exclusive_u64(fmm_ctx* ctx, const uint64_t* in, uint64_t* out, int64_t n, uint64_t* total_dev,
                              cudaStream_t s) {
    return scan_exclusive<unsigned long long>(ctx, (const unsigned long long*)in, (unsigned long long*)out, n,
                                              (unsigned long long*)total_dev, s);
}
