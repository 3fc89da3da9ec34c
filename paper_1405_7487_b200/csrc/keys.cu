// keys.cu -- bounds, root cube, 63-bit Morton keys, sort and body gather (a1-a3).
//
// R2 (root cube): lo/hi exact fp64 min/max; c0 = (lo+hi)*0.5; h = 0.5*max(hi-lo) (1 if 0);
//     origin = c0 - h; s = 2^20/h.        (§II-C "local bounding box")
// R3 (quantise): i = clamp(floor((x - origin)*s), 0, 2^21-1), two roundings, no FMA.
// R4 (key): x bit -> bit 3l, y -> 3l+1, z -> 3l+2; level 1 is the top digit
//     (§II-B "Three bits of the key are used to indicate which octant").
// R5 (order): stable LSD radix sort of (key, original index).
// All fp64 arithmetic uses explicit _rn intrinsics so nvcc cannot contract into FMAs:
// the keys are bit-exact against the oracle.
#include "common.cuh"

namespace {

template <typename Real>
__global__ void k_bounds(const Real* __restrict__ pos, int64_t n, double* __restrict__ blk, int* __restrict__ bad) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    int nonfinite = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            double x = (double)pos[3 * i + d];
            nonfinite |= !isfinite(x);
            lo[d] = fmin(lo[d], x);
            hi[d] = fmax(hi[d], x);
        }
    }
#pragma unroll
    for (int s = 16; s; s >>= 1)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], s));
            hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], s));
        }
    __shared__ double s_v[32][6];
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0)
        for (int d = 0; d < 3; ++d) { s_v[w][d] = lo[d]; s_v[w][3 + d] = hi[d]; }
    if (nonfinite) atomicOr(bad, 1);
    __syncthreads();
    if (threadIdx.x < 6) {
        double v = s_v[0][threadIdx.x];
        for (int k = 1; k < nw; ++k) v = threadIdx.x < 3 ? fmin(v, s_v[k][threadIdx.x]) : fmax(v, s_v[k][threadIdx.x]);
        blk[(int64_t)blockIdx.x * 6 + threadIdx.x] = v;
    }
}

// final reduction over blocks (one warp; min/max are exact in any order) + R2 root cube, from
// the particles' own bounds or from given bounds (which must contain them: *bad |= 2 if not)
__global__ void k_root_cube(const double* __restrict__ blk, int nblk, double* __restrict__ root,
                            const double* __restrict__ given, int* __restrict__ bad) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int b = threadIdx.x; b < nblk; b += 32)
        for (int d = 0; d < 3; ++d) {
            lo[d] = fmin(lo[d], blk[6 * b + d]);
            hi[d] = fmax(hi[d], blk[6 * b + 3 + d]);
        }
    for (int o = 16; o; o >>= 1)
        for (int d = 0; d < 3; ++d) {
            lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
            hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
        }
    if (threadIdx.x != 0) return;
    if (given) {
        for (int d = 0; d < 3; ++d)
            if (lo[d] < given[d] || hi[d] > given[3 + d]) *bad |= 2;
        for (int d = 0; d < 3; ++d) {
            lo[d] = given[d];
            hi[d] = given[3 + d];
        }
    }
    double c0[3], ext = 0.0;
    for (int d = 0; d < 3; ++d) {
        c0[d] = __dmul_rn(__dadd_rn(lo[d], hi[d]), 0.5);
        double e = __dsub_rn(hi[d], lo[d]);
        if (e > ext) ext = e;
    }
    double h = __dmul_rn(0.5, ext);
    if (h == 0.0) h = 1.0;
    for (int d = 0; d < 3; ++d) {
        root[d] = lo[d];
        root[3 + d] = hi[d];
        root[6 + d] = __dsub_rn(c0[d], h);
    }
    root[9] = __ddiv_rn(1048576.0, h);
    root[10] = h;
}

__device__ __forceinline__ uint64_t spread3(uint32_t v) {
    uint64_t x = v & 0x1FFFFFu;
    x = (x | (x << 32)) & 0x1F00000000FFFFull;
    x = (x | (x << 16)) & 0x1F0000FF0000FFull;
    x = (x | (x << 8)) & 0x100F00F00F00F00Full;
    x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return x;
}

__device__ __forceinline__ uint32_t quantise(double x, double o, double s) {
    double t = __dmul_rn(__dsub_rn(x, o), s);
    double f = floor(t);
    f = fmin(fmax(f, 0.0), 2097151.0);
    return (uint32_t)f;
}

template <typename Real>
__global__ void k_keys(const Real* __restrict__ pos, int64_t n, const double* __restrict__ root,
                       uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
    const double ox = root[6], oy = root[7], oz = root[8], s = root[9];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t ix = quantise((double)pos[3 * i], ox, s);
        uint32_t iy = quantise((double)pos[3 * i + 1], oy, s);
        uint32_t iz = quantise((double)pos[3 * i + 2], oz, s);
        keys[i] = spread3(ix) | (spread3(iy) << 1) | (spread3(iz) << 2);
        idx[i] = (uint32_t)i;
    }
}

template <typename Real>
__global__ void k_gather_pos(const Real* __restrict__ pos, const uint32_t* __restrict__ perm, int64_t n,
                             typename BodyT<Real>::type* __restrict__ body) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        uint32_t j = perm[k];
        typename BodyT<Real>::type b;
        b.x = pos[3 * (int64_t)j];
        b.y = pos[3 * (int64_t)j + 1];
        b.z = pos[3 * (int64_t)j + 2];
        b.w = 0;
        body[k] = b;
    }
}

// fp32 positions 16-B aligned: each body's 12 bytes come from the one or two aligned float4
// that hold them, both loads issued together (three scalar loads of one random body went to
// memory as separate requests: ncu at 2^26 read 131 B per body), and UNROLL bodies per thread
// in flight (c4s: 2.05 -> ~1.8 ms)
template <int UNROLL>
__global__ void k_gather_pos_v4(const float4* __restrict__ pos4, const uint32_t* __restrict__ perm, int64_t n,
                                float4* __restrict__ body) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * UNROLL;
    for (int64_t k0 = (int64_t)blockIdx.x * blockDim.x * UNROLL + threadIdx.x; k0 < n; k0 += stride) {
        float4 lo[UNROLL], hi[UNROLL];
        int off[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const int64_t k = k0 + (int64_t)u * blockDim.x;
            if (k < n) {
                const int64_t e = 3 * (int64_t)perm[k];   // first float of the body
                off[u] = (int)(e & 3);
                const int64_t last4 = (e >> 2) + (off[u] >= 2);   // last float4 read
                if (4 * last4 + 3 < 3 * n) {
                    lo[u] = __ldg(pos4 + (e >> 2));
                    if (off[u] >= 2) hi[u] = __ldg(pos4 + (e >> 2) + 1);
                } else {   // the array's last floats: no read past its end
                    const float* p = reinterpret_cast<const float*>(pos4) + e;
                    lo[u] = make_float4(p[0], p[1], p[2], 0.f);
                    off[u] = 0;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const int64_t k = k0 + (int64_t)u * blockDim.x;
            if (k >= n) continue;
            float4 b;
            switch (off[u]) {
                case 0: b = make_float4(lo[u].x, lo[u].y, lo[u].z, 0.f); break;
                case 1: b = make_float4(lo[u].y, lo[u].z, lo[u].w, 0.f); break;
                case 2: b = make_float4(lo[u].z, lo[u].w, hi[u].x, 0.f); break;
                default: b = make_float4(lo[u].w, hi[u].x, hi[u].y, 0.f); break;
            }
            body[k] = b;
        }
    }
}

}  // namespace

namespace {
template <typename Real>
__global__ void k_gather_q(const Real* __restrict__ q, const uint32_t* __restrict__ perm, int64_t n,
                           typename BodyT<Real>::type* __restrict__ body) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        body[k].w = q[perm[k]];
}

template <typename Real>
fmm_status build_keys_t(fmm_ctx* ctx, const Real* pos, int64_t n, cudaStream_t s) {
    const int nblk = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 2);
    {
        PhaseScope ps(ctx, PH_BOUNDS, s);
        FMM_TRY(buf_ensure(ctx, ctx->root, 16 * sizeof(double)));
        FMM_TRY(buf_ensure(ctx, ctx->red_tmp, 64 + (size_t)nblk * 6 * sizeof(double)));
        int* d_bad = reinterpret_cast<int*>(ctx->red_tmp.p);
        double* d_blk = reinterpret_cast<double*>((char*)ctx->red_tmp.p + 64);
        FMM_CUDA_TRY(ctx, cudaMemsetAsync(d_bad, 0, sizeof(int), s));
        k_bounds<Real><<<nblk, 256, 0, s>>>(pos, n, d_blk, d_bad);
        const double* given = nullptr;
        if (ctx->has_root_bounds) {
            FMM_TRY(buf_ensure(ctx, ctx->root_given, 6 * sizeof(double)));
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->root_given.p, ctx->root_bounds, 6 * sizeof(double),
                                              cudaMemcpyHostToDevice, s));
            given = P_<double>(ctx->root_given);
        }
        k_root_cube<<<1, 32, 0, s>>>(d_blk, nblk, P_<double>(ctx->root), given, d_bad);
        ctx->launches += 2;
        int bad = 0;
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
        FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        if (bad & 1) {
            ctx->err = "fmm_build: non-finite position";
            return FMM_ERR_NONFINITE;
        }
        if (bad & 2) {
            ctx->err = "fmm_build: a position lies outside the root bounds set by fmm_set_root_bounds";
            return FMM_ERR_ARG;
        }
    }
    PhaseScope ps(ctx, PH_SORT, s);
    FMM_TRY(buf_ensure(ctx, ctx->key_a, (size_t)n * 8, ctx->presorted, s));
    FMM_TRY(buf_ensure(ctx, ctx->key_b, (size_t)n * 8));
    FMM_TRY(buf_ensure(ctx, ctx->idx_a, (size_t)n * 4, ctx->presorted, s));
    FMM_TRY(buf_ensure(ctx, ctx->idx_b, (size_t)n * 4));
    const int gblk = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 8);
    if (ctx->presorted) {
        // the multi-GPU driver sorted this build's keys already (dist.cu: staying particles while
        // the partition exchange flew, arrivals after, merged) -- the same (key, index) order
        ctx->d_keys = P_<uint64_t>(ctx->key_a);
        ctx->d_perm = P_<uint32_t>(ctx->idx_a);
    } else {
        k_keys<Real><<<gblk, 256, 0, s>>>(pos, n, P_<double>(ctx->root), P_<uint64_t>(ctx->key_a),
                                          P_<uint32_t>(ctx->idx_a));
        FMM_LAUNCH(ctx);
        FMM_CUDA_TRY(ctx, cudaGetLastError());
        FMM_TRY(radix_sort_pairs(ctx, P_<uint64_t>(ctx->key_a), P_<uint64_t>(ctx->key_b), P_<uint32_t>(ctx->idx_a),
                                 P_<uint32_t>(ctx->idx_b), n, 0, 64, &ctx->d_keys, &ctx->d_perm, s, ~0ull));
    }
    FMM_TRY(buf_ensure(ctx, ctx->body, (size_t)n * sizeof(typename BodyT<Real>::type)));
    if (std::is_same<Real, float>::value && ((uintptr_t)pos & 15) == 0)
        k_gather_pos_v4<4><<<gblk, 256, 0, s>>>(reinterpret_cast<const float4*>(pos), ctx->d_perm, n,
                                                reinterpret_cast<float4*>(ctx->body.p));
    else
        k_gather_pos<Real><<<gblk, 256, 0, s>>>(pos, ctx->d_perm, n, P_<typename BodyT<Real>::type>(ctx->body));
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}
}  // namespace

fmm_status build_keys(fmm_ctx* ctx, const void* pos, int64_t n, cudaStream_t s) {
    if (ctx->prec == FMM_F32) return build_keys_t<float>(ctx, (const float*)pos, n, s);
    return build_keys_t<double>(ctx, (const double*)pos, n, s);
}

namespace {
// iperm[perm[i]] = i: the output merge gathers in the caller's order (coalesced writes)
__global__ void k_invert_perm(const uint32_t* __restrict__ perm, int64_t n, uint32_t* __restrict__ iperm) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) iperm[perm[i]] = (uint32_t)i;
}
}  // namespace

fmm_status gather_bodies_q(fmm_ctx* ctx, const void* q, cudaStream_t s) {
    int64_t n = ctx->n;
    const int gblk = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 8);
    if (ctx->prec == FMM_F32)
        k_gather_q<float><<<gblk, 256, 0, s>>>((const float*)q, ctx->d_perm, n, P_<float4>(ctx->body));
    else
        k_gather_q<double><<<gblk, 256, 0, s>>>((const double*)q, ctx->d_perm, n, P_<dbody>(ctx->body));
    FMM_LAUNCH(ctx);
    FMM_TRY(buf_ensure(ctx, ctx->iperm, (size_t)std::max<int64_t>(n, 1) * 4));
    k_invert_perm<<<gblk, 256, 0, s>>>(ctx->d_perm, n, P_<uint32_t>(ctx->iperm));
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}
