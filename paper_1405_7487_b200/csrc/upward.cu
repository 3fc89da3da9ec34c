// upward.cu -- P2M at leaves and level-by-level M2M (a6, a7), fp64 in both precisions.
//
// PAPER.md:120 §II-C: "a post-order traversal is performed ... P2M and M2M kernels are
// executed bottom up.  The P2M kernel is executed only at the leaf cells ... The M2M
// kernel ... translates the multipole expansions from its children's centers to its center."
// R12 P2M: M_beta(C) = sum_j q_j (x_j - c_C)^beta / beta!
// R13 M2M: M_alpha(par) += sum_{beta <= alpha} M_beta(ch) s^(alpha-beta)/(alpha-beta)!, s = c_ch - c_par
// Post-order is realised level-synchronously (all cells of level l+1 final before level l).
//
// P2M: warp per leaf; 32 bodies at a time, each lane builds its body's x^e/e! tables in
// shared memory, then lanes over coefficients accumulate the 32 bodies in order.
// M2M: block per parent, warp per child; the shift operator is separable, s^(a-b)/(a-b)! =
// prod_i s_i^(a_i-b_i)/(a_i-b_i)!, so each child's expansion is shifted by three 1D passes
// (x, then y, then z) through shared memory -- the same sum as R13, grouped per axis.
#include "common.cuh"

namespace {
constexpr int P2M_WARPS = 2;

__constant__ double c_inv[FMM_MAXP + 1] = {0.0,       1.0,        1.0 / 2,  1.0 / 3,  1.0 / 4,  1.0 / 5,
                                           1.0 / 6,   1.0 / 7,    1.0 / 8,  1.0 / 9,  1.0 / 10, 1.0 / 11,
                                           1.0 / 12,  1.0 / 13,   1.0 / 14, 1.0 / 15, 1.0 / 16};

template <typename Body, int NI>
__global__ void __launch_bounds__(P2M_WARPS * 32) k_p2m(const Body* __restrict__ body, const uint32_t* __restrict__ leaf_ids,
                                                        int64_t nleaf, const uint32_t* __restrict__ bb,
                                                        const uint32_t* __restrict__ bc, const double4* __restrict__ cr,
                                                        int P, int ncoef, double* __restrict__ M) {
    __shared__ uchar4 ex[816];
    __shared__ double s_pw[P2M_WARPS][3][FMM_MAXP][33];
    __shared__ double s_q[P2M_WARPS][32];
    fill_ex_table(ex, ncoef);
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t li = (int64_t)blockIdx.x * P2M_WARPS + w; li < nleaf; li += (int64_t)gridDim.x * P2M_WARPS) {
        const uint32_t c = leaf_ids[li];
        const double4 ctr = cr[c];
        double acc[NI];
        uchar4 ek[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            acc[i] = 0.0;
            ek[i] = ex[min(lane + 32 * i, ncoef - 1)];
        }
        const uint32_t b0 = bb[c], nb = bc[c];
        for (uint32_t j0 = 0; j0 < nb; j0 += 32) {
            const uint32_t m = min(32u, nb - j0);
            __syncwarp();
            if ((uint32_t)lane < m) {
                const Body p = body[b0 + j0 + lane];
                const double d[3] = {(double)p.x - ctr.x, (double)p.y - ctr.y, (double)p.z - ctr.z};
                s_q[w][lane] = (double)p.w;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    double v = 1.0;
                    s_pw[w][a][0][lane] = 1.0;
                    for (int e = 1; e < P; ++e) {
                        v = v * d[a] * c_inv[e];
                        s_pw[w][a][e][lane] = v;
                    }
                }
            }
            __syncwarp();
            // bodies outer, coefficients inner: the NI accumulators are independent chains
            // (each coefficient still sums its bodies in order)
            for (uint32_t j = 0; j < m; ++j) {
                const double qj = s_q[w][j];
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    if (lane + 32 * i < ncoef) {
                        const uchar4 e = ek[i];
                        acc[i] += qj * (s_pw[w][0][e.x][j] * s_pw[w][1][e.y][j] * s_pw[w][2][e.z][j]);
                    }
                }
            }
        }
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int k = lane + 32 * i;
            if (k < ncoef) M[(int64_t)c * ncoef + k] = acc[i];
        }
    }
}

// one separable 1D shift pass along axis `ax`: out_alpha = sum_{b <= a_ax} in_{alpha with a_ax -> b} t[a_ax - b]
__device__ __forceinline__ void shift_pass_up(const uchar4* __restrict__ ex, int ncoef, int ax, const double* in,
                                              double* out, const double* t, int lane) {
    for (int k = lane; k < ncoef; k += 32) {
        const uchar4 e = ex[k];
        int a[3] = {e.x, e.y, e.z};
        const int top = a[ax];
        double s = 0.0;
        for (int b = 0; b <= top; ++b) {
            a[ax] = b;
            s += in[cidx(a[0], a[1], a[2])] * t[top - b];
        }
        out[k] = s;
    }
}

// One block per parent, one warp per child (up to 8): each warp shifts its child's
// expansion with the three separable passes into its own shared buffers, then the block
// sums the (up to) 8 shifted expansions in child order (the same order as R13's loop).
constexpr int M2M_THREADS = 256;
__global__ void __launch_bounds__(M2M_THREADS) k_m2m(int64_t cbeg, int64_t cend, const uint32_t* __restrict__ cb,
                                                     const uint32_t* __restrict__ cc, const double4* __restrict__ cr,
                                                     int P, int ncoef, double* __restrict__ M) {
    extern __shared__ double s_dyn[];
    __shared__ uchar4 ex[816];
    __shared__ double s_t[8][3][FMM_MAXP];
    fill_ex_table(ex, ncoef);
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double* A = s_dyn + (size_t)w * 2 * ncoef;
    double* B = A + ncoef;
    for (int64_t c = cbeg + blockIdx.x; c < cend; c += gridDim.x) {
        const uint32_t nk = cc[c];
        if (nk == 0) continue;  // leaf: written by P2M (uniform over the block)
        const double4 cp = cr[c];
        if ((uint32_t)w < nk) {
            const uint32_t ch = cb[c] + w;
            const double4 q = cr[ch];
            for (int i = lane; i < ncoef; i += 32) A[i] = M[(int64_t)ch * ncoef + i];
            if (lane < 3) {
                const double sh = lane == 0 ? q.x - cp.x : lane == 1 ? q.y - cp.y : q.z - cp.z;
                double v = 1.0;
                s_t[w][lane][0] = 1.0;
                for (int e = 1; e < P; ++e) {
                    v = v * sh * c_inv[e];
                    s_t[w][lane][e] = v;
                }
            }
            __syncwarp();
            shift_pass_up(ex, ncoef, 0, A, B, s_t[w][0], lane);
            __syncwarp();
            shift_pass_up(ex, ncoef, 1, B, A, s_t[w][1], lane);
            __syncwarp();
            shift_pass_up(ex, ncoef, 2, A, B, s_t[w][2], lane);
        }
        __syncthreads();
        for (int k = threadIdx.x; k < ncoef; k += M2M_THREADS) {
            double acc = 0.0;
            for (uint32_t j = 0; j < nk; ++j) acc += s_dyn[(size_t)j * 2 * ncoef + ncoef + k];
            M[(int64_t)c * ncoef + k] = acc;
        }
        __syncthreads();
    }
}

template <typename Body>
fmm_status upward_t(fmm_ctx* ctx, cudaStream_t s) {
    PhaseScope ps(ctx, PH_UP, s);
    // remote LET cells (let.cu) take [ncell, ncell + nrem); their M arrives by fmm_let_unpack
    const int64_t nc = ctx->ncell + ctx->nrem;
    FMM_TRY(buf_ensure(ctx, ctx->M, (size_t)nc * ctx->ncoef * 8));
    double* M = P_<double>(ctx->M);
    int g = (int)std::min<int64_t>((ctx->nleaf + P2M_WARPS - 1) / P2M_WARPS, (int64_t)ctx->num_sms * 32);
    const int ni = (ctx->ncoef + 31) / 32;
    auto p2m = [&](auto tag) {
        constexpr int NI = decltype(tag)::value;
        k_p2m<Body, NI><<<std::max(g, 1), P2M_WARPS * 32, 0, s>>>(P_<Body>(ctx->body), P_<uint32_t>(ctx->leaf_ids),
                                                                 ctx->nleaf, P_<uint32_t>(ctx->c_bb),
                                                                 P_<uint32_t>(ctx->c_bc), P_<double4>(ctx->c_cr),
                                                                 ctx->P, ctx->ncoef, M);
    };
    if (ni <= 1) p2m(std::integral_constant<int, 1>());
    else if (ni <= 2) p2m(std::integral_constant<int, 2>());
    else if (ni <= 4) p2m(std::integral_constant<int, 4>());
    else if (ni <= 7) p2m(std::integral_constant<int, 7>());
    else if (ni <= 12) p2m(std::integral_constant<int, 12>());
    else if (ni <= 18) p2m(std::integral_constant<int, 18>());
    else p2m(std::integral_constant<int, 26>());
    FMM_LAUNCH(ctx);
    const size_t smem = (size_t)8 * 2 * ctx->ncoef * 8;
    if (smem > 48 * 1024) FMM_CUDA_TRY(ctx, cudaFuncSetAttribute(k_m2m, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int64_t l = ctx->depth - 1; l >= 0; --l) {
        int64_t b = ctx->level_begin[l], e = ctx->level_begin[l + 1];
        int gg = (int)std::min<int64_t>(e - b, (int64_t)ctx->num_sms * 16);
        k_m2m<<<std::max(gg, 1), M2M_THREADS, smem, s>>>(b, e, P_<uint32_t>(ctx->c_cb), P_<uint32_t>(ctx->c_cc),
                                                         P_<double4>(ctx->c_cr), ctx->P, ctx->ncoef, M);
        FMM_LAUNCH(ctx);
    }
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}
}  // namespace

fmm_status upward_pass(fmm_ctx* ctx, cudaStream_t s) {
    if (ctx->prec == FMM_F32) return upward_t<float4>(ctx, s);
    return upward_t<dbody>(ctx, s);
}
