// part.cu -- Morton-range partition of the particles over GPUs.
//
// PAPER.md:81-92 §II-B: the particles are partitioned along the space-filling curve of
// their Morton keys ("HOT is analogous to radix sort"); Eq. (1): the
// partition is weighted by the per-particle work of the previous step.  The keys here use
// the GLOBAL bounding box (R2-R4 over the union of all ranks' particles, the bounds being
// an all-reduce of fmm_bounds); each rank then builds its local tree from its local
// bounding box.
//   fmm_part_histogram: weighted histogram of `bits` key bits below a given prefix (all-reduced
//   by the caller, who refines nranks-1 splitter keys bin by bin);
//   fmm_part_assign:    destination rank of each particle = number of splitter keys <= key;
//   fmm_part_pack:      particles grouped by destination, stable, with their global ids.
#include <cmath>

#include "common.cuh"

namespace {

template <typename Real>
__global__ void k_minmax(const Real* __restrict__ pos, int64_t n, double* __restrict__ blk) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double x = (double)pos[3 * i + d];
            lo[d] = fmin(lo[d], x);
            hi[d] = fmax(hi[d], x);
        }
#pragma unroll
    for (int s = 16; s; s >>= 1)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], s));
            hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], s));
        }
    __shared__ double s_v[32][6];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0)
        for (int d = 0; d < 3; ++d) {
            s_v[w][d] = lo[d];
            s_v[w][3 + d] = hi[d];
        }
    __syncthreads();
    if (threadIdx.x < 6) {
        double v = s_v[0][threadIdx.x];
        for (int k = 1; k < nw; ++k) v = threadIdx.x < 3 ? fmin(v, s_v[k][threadIdx.x]) : fmax(v, s_v[k][threadIdx.x]);
        blk[(int64_t)blockIdx.x * 6 + threadIdx.x] = v;
    }
}

__device__ __forceinline__ uint64_t spread3p(uint32_t v) {
    uint64_t x = v & 0x1FFFFFu;
    x = (x | (x << 32)) & 0x1F00000000FFFFull;
    x = (x | (x << 16)) & 0x1F0000FF0000FFull;
    x = (x | (x << 8)) & 0x100F00F00F00F00Full;
    x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return x;
}

__device__ __forceinline__ uint32_t quantise_p(double x, double o, double s) {
    const double t = __dmul_rn(__dsub_rn(x, o), s);
    return (uint32_t)fmin(fmax(floor(t), 0.0), 2097151.0);
}

// R2 root cube of the given (global) bounds, then R3/R4 keys
template <typename Real>
__global__ void k_part_keys(const Real* __restrict__ pos, int64_t n, double lx, double ly, double lz, double hx,
                            double hy, double hz, uint64_t* __restrict__ keys) {
    const double lo[3] = {lx, ly, lz}, hi[3] = {hx, hy, hz};
    double ext = 0.0, c0[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        c0[d] = __dmul_rn(__dadd_rn(lo[d], hi[d]), 0.5);
        const double e = __dsub_rn(hi[d], lo[d]);
        if (e > ext) ext = e;
    }
    double h = __dmul_rn(0.5, ext);
    if (h == 0.0) h = 1.0;
    const double s = __ddiv_rn(1048576.0, h);
    const double o[3] = {__dsub_rn(c0[0], h), __dsub_rn(c0[1], h), __dsub_rn(c0[2], h)};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t ix = quantise_p((double)pos[3 * i], o[0], s);
        const uint32_t iy = quantise_p((double)pos[3 * i + 1], o[1], s);
        const uint32_t iz = quantise_p((double)pos[3 * i + 2], o[2], s);
        keys[i] = spread3p(ix) | (spread3p(iy) << 1) | (spread3p(iz) << 2);
    }
}

// keys whose top pbits equal prefix add their weight to the bin of their next `bits` bits
__global__ void k_part_hist(const uint64_t* __restrict__ keys, const float* __restrict__ w, int64_t n,
                            uint64_t prefix, int pbits, int bits, double* __restrict__ hist) {
    const int lo = 63 - pbits - bits;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        if (pbits > 0 && (k >> (63 - pbits)) != prefix) continue;
        atomicAdd(&hist[(k >> lo) & ((1ull << bits) - 1)], w ? (double)w[i] : 1.0);
    }
}

__global__ void k_part_assign(const uint64_t* __restrict__ keys, int64_t n, const uint64_t* __restrict__ spl, int nspl,
                              uint64_t* __restrict__ dkey, uint32_t* __restrict__ idx, unsigned long long* counts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        int lo = 0, hi = nspl;   // number of splitters <= k
        while (lo < hi) {
            const int m = (lo + hi) >> 1;
            if (spl[m] <= k) lo = m + 1;
            else hi = m;
        }
        dkey[i] = (uint64_t)lo;
        idx[i] = (uint32_t)i;
        atomicAdd(&counts[lo], 1ull);
    }
}

template <typename Real>
__global__ void k_part_gather(const Real* __restrict__ pos, const Real* __restrict__ q, const uint32_t* __restrict__ order,
                              int64_t n, int64_t gid_base, Real* __restrict__ opos, Real* __restrict__ oq,
                              int64_t* __restrict__ ogid) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t i = order[k];
#pragma unroll
        for (int d = 0; d < 3; ++d) opos[3 * k + d] = pos[3 * (int64_t)i + d];
        oq[k] = q[i];
        ogid[k] = gid_base + i;
    }
}

unsigned grid_for(const fmm_ctx* ctx, int64_t n) {
    return (unsigned)std::max<int64_t>(std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 8), 1);
}

}  // namespace

extern "C" {

fmm_status fmm_bounds(fmm_ctx* ctx, const void* pos, int64_t n, double* out, void* stream) {
    if (!ctx || !out || n < 0 || (n > 0 && !pos)) return FMM_ERR_ARG;
    DeviceGuard guard(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    for (int d = 0; d < 3; ++d) {
        out[d] = INFINITY;
        out[3 + d] = -INFINITY;
    }
    if (n == 0) return FMM_OK;
    const int nblk = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 2);
    FMM_TRY(buf_ensure(ctx, ctx->part_tmp, (size_t)nblk * 6 * 8));
    if (ctx->prec == FMM_F32) k_minmax<float><<<nblk, 256, 0, s>>>((const float*)pos, n, P_<double>(ctx->part_tmp));
    else k_minmax<double><<<nblk, 256, 0, s>>>((const double*)pos, n, P_<double>(ctx->part_tmp));
    FMM_LAUNCH(ctx);
    std::vector<double> blk((size_t)nblk * 6);
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(blk.data(), ctx->part_tmp.p, blk.size() * 8, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    for (int b = 0; b < nblk; ++b)
        for (int d = 0; d < 3; ++d) {
            out[d] = std::min(out[d], blk[6 * b + d]);
            out[3 + d] = std::max(out[3 + d], blk[6 * b + 3 + d]);
        }
    if (!std::isfinite(out[0] + out[1] + out[2] + out[3] + out[4] + out[5])) {
        ctx->err = "fmm_bounds: non-finite position";
        return FMM_ERR_NONFINITE;
    }
    return FMM_OK;
}

fmm_status fmm_part_keys(fmm_ctx* ctx, const void* pos, int64_t n, const double* bounds, uint64_t* keys, void* stream) {
    if (!ctx || !bounds || n < 0 || (n > 0 && (!pos || !keys))) return FMM_ERR_ARG;
    if (n == 0) return FMM_OK;
    DeviceGuard guard(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned g = grid_for(ctx, n);
    if (ctx->prec == FMM_F32)
        k_part_keys<float><<<g, 256, 0, s>>>((const float*)pos, n, bounds[0], bounds[1], bounds[2], bounds[3], bounds[4],
                                            bounds[5], keys);
    else
        k_part_keys<double><<<g, 256, 0, s>>>((const double*)pos, n, bounds[0], bounds[1], bounds[2], bounds[3],
                                             bounds[4], bounds[5], keys);
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}

fmm_status fmm_part_histogram(fmm_ctx* ctx, const uint64_t* keys, const float* w, int64_t n, uint64_t prefix,
                              int prefix_bits, int bits, double* hist, void* stream) {
    if (!ctx || bits < 1 || bits > 24 || prefix_bits < 0 || prefix_bits + bits > 63 || !hist || n < 0 ||
        (n > 0 && !keys))
        return FMM_ERR_ARG;
    DeviceGuard guard(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(hist, 0, ((size_t)1 << bits) * 8, s));
    if (n == 0) return FMM_OK;
    k_part_hist<<<grid_for(ctx, n), 256, 0, s>>>(keys, w, n, prefix, prefix_bits, bits, hist);
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}

fmm_status fmm_part_pack(fmm_ctx* ctx, const void* pos, const void* q, const uint64_t* keys, int64_t n,
                         const uint64_t* splitters, int nranks, int64_t gid_base, void* out_pos, void* out_q,
                         int64_t* out_gid, int64_t* counts, void* stream) {
    if (!ctx || nranks < 1 || nranks > 256 || !counts || (nranks > 1 && !splitters) || n < 0 ||
        (n > 0 && (!pos || !q || !keys || !out_pos || !out_q || !out_gid)))
        return FMM_ERR_ARG;
    for (int r = 0; r < nranks; ++r) counts[r] = 0;
    if (n == 0) return FMM_OK;
    DeviceGuard guard(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    // scratch: dkey[2n] u64 | idx[2n] u32 | splitters | counts
    const size_t need = (size_t)n * 16 + (size_t)n * 8 + 256 * 8 + 256 * 8 + 64;
    FMM_TRY(buf_ensure(ctx, ctx->part_tmp, need));
    uint64_t* k0 = P_<uint64_t>(ctx->part_tmp);
    uint64_t* k1 = k0 + n;
    uint32_t* v0 = reinterpret_cast<uint32_t*>(k1 + n);
    uint32_t* v1 = v0 + n;
    uint64_t* dspl = reinterpret_cast<uint64_t*>(v1 + n);   // byte offset 24n: 8-B aligned
    unsigned long long* dcnt = reinterpret_cast<unsigned long long*>(dspl + 256);
    if (nranks > 1)
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(dspl, splitters, (size_t)(nranks - 1) * 8, cudaMemcpyHostToDevice, s));
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(dcnt, 0, (size_t)nranks * 8, s));
    k_part_assign<<<grid_for(ctx, n), 256, 0, s>>>(keys, n, dspl, nranks - 1, k0, v0, dcnt);
    FMM_LAUNCH(ctx);
    // stable grouping by destination: one radix digit pass over the rank number
    uint64_t* kout = nullptr;
    uint32_t* order = nullptr;
    FMM_TRY(radix_sort_pairs(ctx, k0, k1, v0, v1, n, 0, 8, &kout, &order, s));
    if (ctx->prec == FMM_F32)
        k_part_gather<float><<<grid_for(ctx, n), 256, 0, s>>>((const float*)pos, (const float*)q, order, n, gid_base,
                                                             (float*)out_pos, (float*)out_q, out_gid);
    else
        k_part_gather<double><<<grid_for(ctx, n), 256, 0, s>>>((const double*)pos, (const double*)q, order, n, gid_base,
                                                              (double*)out_pos, (double*)out_q, out_gid);
    FMM_LAUNCH(ctx);
    std::vector<unsigned long long> hc(nranks);
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(hc.data(), dcnt, (size_t)nranks * 8, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    for (int r = 0; r < nranks; ++r) counts[r] = (int64_t)hc[r];
    return FMM_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- ORB multisection (§8f f3)
// PAPER.md:81, 94 §II-B: orthogonal recursive bisection along the longest axis with weighted
// cuts, generalised to any rank count: a group of K ranks is cut at the
// coordinate where the weight fraction reaches floor(K/2)/K.  Coordinates are the R3 21-bit
// quantised coordinates of the global root cube, recovered from the Morton keys, so a cut is
// exact and equal positions never separate.
namespace {
__device__ __forceinline__ uint32_t compact3(uint64_t x) {
    x &= 0x1249249249249249ull;
    x = (x | (x >> 2)) & 0x10C30C30C30C30C3ull;
    x = (x | (x >> 4)) & 0x100F00F00F00F00Full;
    x = (x | (x >> 8)) & 0x1F0000FF0000FFull;
    x = (x | (x >> 16)) & 0x1F00000000FFFFull;
    x = (x | (x >> 32)) & 0x1FFFFFull;
    return (uint32_t)x;
}

__global__ void k_orb_hist(const uint64_t* __restrict__ keys, const float* __restrict__ w,
                           const int32_t* __restrict__ grp, int64_t n, const int32_t* __restrict__ axis,
                           const uint32_t* __restrict__ prefix, int pbits, int bits, double* __restrict__ hist) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t g = grp[i];
        const int a = axis[g];
        if (a < 0) continue;
        const uint32_t c = compact3(keys[i] >> a);
        if (pbits > 0 && (c >> (21 - pbits)) != prefix[g]) continue;
        const uint32_t bin = (c >> (21 - pbits - bits)) & ((1u << bits) - 1);
        atomicAdd(&hist[((size_t)g << bits) + bin], w ? (double)w[i] : 1.0);
    }
}

__global__ void k_orb_split(const uint64_t* __restrict__ keys, int32_t* __restrict__ grp, int64_t n,
                            const int32_t* __restrict__ axis, const uint32_t* __restrict__ cut,
                            const int32_t* __restrict__ right) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t g = grp[i];
        const int a = axis[g];
        if (a < 0) continue;
        if (compact3(keys[i] >> a) >= cut[g]) grp[i] = right[g];
    }
}

template <typename Real>
__global__ void k_part_gather_dest(const Real* __restrict__ pos, const Real* __restrict__ q,
                                   const uint32_t* __restrict__ order, int64_t n, int64_t gid_base,
                                   Real* __restrict__ opos, Real* __restrict__ oq, int64_t* __restrict__ ogid) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t i = order[k];
#pragma unroll
        for (int d = 0; d < 3; ++d) opos[3 * k + d] = pos[3 * (int64_t)i + d];
        oq[k] = q[i];
        ogid[k] = gid_base + i;
    }
}

__global__ void k_dest_keys(const int32_t* __restrict__ dest, int64_t n, uint64_t* __restrict__ dkey,
                            uint32_t* __restrict__ idx, unsigned long long* counts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        dkey[i] = (uint64_t)dest[i];
        idx[i] = (uint32_t)i;
        atomicAdd(&counts[dest[i]], 1ull);
    }
}
}  // namespace

extern "C" {

fmm_status fmm_orb_histogram(fmm_ctx* ctx, const uint64_t* keys, const float* w, const int32_t* group, int64_t n,
                             int ngroups, const int32_t* axis, const uint32_t* prefix, int prefix_bits, int bits,
                             double* hist, void* stream) {
    if (!ctx || ngroups < 1 || ngroups > 256 || !axis || !prefix || !hist || bits < 1 || bits > 16 ||
        prefix_bits < 0 || prefix_bits + bits > 21 || n < 0 || (n > 0 && (!keys || !group)))
        return FMM_ERR_ARG;
    DeviceGuard guard(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    FMM_TRY(buf_ensure(ctx, ctx->orb_tmp, (size_t)256 * 12 + 64));
    int32_t* dax = P_<int32_t>(ctx->orb_tmp);
    uint32_t* dpre = reinterpret_cast<uint32_t*>(dax + 256);
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(dax, axis, (size_t)ngroups * 4, cudaMemcpyHostToDevice, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(dpre, prefix, (size_t)ngroups * 4, cudaMemcpyHostToDevice, s));
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(hist, 0, ((size_t)ngroups << bits) * 8, s));
    if (n > 0) {
        k_orb_hist<<<grid_for(ctx, n), 256, 0, s>>>(keys, w, group, n, dax, dpre, prefix_bits, bits, hist);
        FMM_LAUNCH(ctx);
    }
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));   // host arrays may be reused at return
    return FMM_OK;
}

fmm_status fmm_orb_split(fmm_ctx* ctx, const uint64_t* keys, int32_t* group, int64_t n, int ngroups,
                         const int32_t* axis, const uint32_t* cut, const int32_t* right, void* stream) {
    if (!ctx || ngroups < 1 || ngroups > 256 || !axis || !cut || !right || n < 0 || (n > 0 && (!keys || !group)))
        return FMM_ERR_ARG;
    if (n == 0) return FMM_OK;
    DeviceGuard guard(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    FMM_TRY(buf_ensure(ctx, ctx->orb_tmp, (size_t)256 * 12 + 64));
    int32_t* dax = P_<int32_t>(ctx->orb_tmp);
    uint32_t* dcut = reinterpret_cast<uint32_t*>(dax + 256);
    int32_t* drt = reinterpret_cast<int32_t*>(dcut + 256);
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(dax, axis, (size_t)ngroups * 4, cudaMemcpyHostToDevice, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(dcut, cut, (size_t)ngroups * 4, cudaMemcpyHostToDevice, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(drt, right, (size_t)ngroups * 4, cudaMemcpyHostToDevice, s));
    k_orb_split<<<grid_for(ctx, n), 256, 0, s>>>(keys, group, n, dax, dcut, drt);
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    return FMM_OK;
}

fmm_status fmm_part_pack_dest(fmm_ctx* ctx, const void* pos, const void* q, const int32_t* dest, int64_t n,
                              int nranks, int64_t gid_base, void* out_pos, void* out_q, int64_t* out_gid,
                              int64_t* counts, void* stream) {
    if (!ctx || nranks < 1 || nranks > 256 || !counts || n < 0 ||
        (n > 0 && (!pos || !q || !dest || !out_pos || !out_q || !out_gid)))
        return FMM_ERR_ARG;
    for (int r = 0; r < nranks; ++r) counts[r] = 0;
    if (n == 0) return FMM_OK;
    DeviceGuard guard(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t need = (size_t)n * 24 + 256 * 8 + 64;
    FMM_TRY(buf_ensure(ctx, ctx->part_tmp, need));
    uint64_t* k0 = P_<uint64_t>(ctx->part_tmp);
    uint64_t* k1 = k0 + n;
    uint32_t* v0 = reinterpret_cast<uint32_t*>(k1 + n);
    uint32_t* v1 = v0 + n;
    unsigned long long* dcnt = reinterpret_cast<unsigned long long*>(v1 + n);   // byte offset 24n
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(dcnt, 0, (size_t)nranks * 8, s));
    k_dest_keys<<<grid_for(ctx, n), 256, 0, s>>>(dest, n, k0, v0, dcnt);
    FMM_LAUNCH(ctx);
    uint64_t* kout = nullptr;
    uint32_t* order = nullptr;
    FMM_TRY(radix_sort_pairs(ctx, k0, k1, v0, v1, n, 0, 8, &kout, &order, s));
    if (ctx->prec == FMM_F32)
        k_part_gather_dest<float><<<grid_for(ctx, n), 256, 0, s>>>((const float*)pos, (const float*)q, order, n,
                                                                  gid_base, (float*)out_pos, (float*)out_q, out_gid);
    else
        k_part_gather_dest<double><<<grid_for(ctx, n), 256, 0, s>>>((const double*)pos, (const double*)q, order, n,
                                                                   gid_base, (double*)out_pos, (double*)out_q, out_gid);
    FMM_LAUNCH(ctx);
    std::vector<unsigned long long> hc(nranks);
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(hc.data(), dcnt, (size_t)nranks * 8, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    for (int r = 0; r < nranks; ++r) counts[r] = (int64_t)hc[r];
    return FMM_OK;
}

}  // extern "C"
