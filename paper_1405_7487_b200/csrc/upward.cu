// upward.cu -- P2M at leaves and level-by-level M2M (a6, a7), fp64 in both precisions.
//
// PAPER.md:120 §II-C: "a post-order traversal is performed ... P2M and M2M kernels are
// executed bottom up.  The P2M kernel is executed only at the leaf cells ... The M2M
// kernel ... translates the multipole expansions from its children's centers to its center."
// R12 P2M: M_beta(C) = sum_j q_j (x_j - c_C)^beta / beta!
// R13 M2M: M_alpha(par) += sum_{beta <= alpha} M_beta(ch) s^(alpha-beta)/(alpha-beta)!, s = c_ch - c_par
// Post-order is realised level-synchronously: all cells of level l+1 are final before
// level l is formed.  Warp per cell, lanes over coefficients, per-warp power tables
// x^e/e! in shared memory, accumulators in shared memory (runtime P <= 16).
#include "common.cuh"

namespace {
constexpr int UP_WARPS = 4;

// lanes 0..P-1 of the warp fill t[e] = x^e / e! (product of x/i; same value as the
// definition up to rounding order)
__device__ __forceinline__ void pow_table(double* t, double x, int P, int lane) {
    if (lane < P) {
        double v = 1.0;
        for (int i = 1; i <= lane; ++i) v = v * x / (double)i;
        t[lane] = v;
    }
}

template <typename Body>
__global__ void __launch_bounds__(UP_WARPS * 32) k_p2m(const Body* __restrict__ body, const uint32_t* __restrict__ leaf_ids,
                                                        int64_t nleaf, const uint32_t* __restrict__ bb,
                                                        const uint32_t* __restrict__ bc, const double4* __restrict__ cr,
                                                        int P, int ncoef, double* __restrict__ M) {
    __shared__ uchar4 ex[816];
    __shared__ double s_pow[UP_WARPS][3][FMM_MAXP];
    __shared__ double s_acc[UP_WARPS][816];
    fill_ex_table(ex, ncoef);
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t li = (int64_t)blockIdx.x * UP_WARPS + w; li < nleaf; li += (int64_t)gridDim.x * UP_WARPS) {
        uint32_t c = leaf_ids[li];
        double4 ctr = cr[c];
        for (int k = lane; k < ncoef; k += 32) s_acc[w][k] = 0.0;
        uint32_t b0 = bb[c], nb = bc[c];
        for (uint32_t j = 0; j < nb; ++j) {
            Body p = body[b0 + j];
            double q = (double)p.w;
            __syncwarp();
            pow_table(s_pow[w][0], (double)p.x - ctr.x, P, lane);
            pow_table(s_pow[w][1], (double)p.y - ctr.y, P, lane);
            pow_table(s_pow[w][2], (double)p.z - ctr.z, P, lane);
            __syncwarp();
            for (int k = lane; k < ncoef; k += 32) {
                uchar4 e = ex[k];
                s_acc[w][k] += q * (s_pow[w][0][e.x] * s_pow[w][1][e.y] * s_pow[w][2][e.z]);
            }
        }
        __syncwarp();
        for (int k = lane; k < ncoef; k += 32) M[(int64_t)c * ncoef + k] = s_acc[w][k];
        __syncwarp();
    }
}

__global__ void __launch_bounds__(UP_WARPS * 32) k_m2m(int64_t cbeg, int64_t cend, const uint32_t* __restrict__ cb,
                                                        const uint32_t* __restrict__ cc, const double4* __restrict__ cr,
                                                        int P, int ncoef, double* __restrict__ M) {
    __shared__ uchar4 ex[816];
    __shared__ double s_pow[UP_WARPS][3][FMM_MAXP];
    fill_ex_table(ex, ncoef);
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t c = cbeg + (int64_t)blockIdx.x * UP_WARPS + w; c < cend; c += (int64_t)gridDim.x * UP_WARPS) {
        uint32_t nk = cc[c];
        if (nk == 0) continue;  // leaf: P2M already wrote it
        double4 cp = cr[c];
        double acc[26];
#pragma unroll
        for (int i = 0; i < 26; ++i) acc[i] = 0.0;
        for (uint32_t k = 0; k < nk; ++k) {
            uint32_t ch = cb[c] + k;
            double4 cc4 = cr[ch];
            const double* Mc = M + (int64_t)ch * ncoef;
            __syncwarp();
            pow_table(s_pow[w][0], cc4.x - cp.x, P, lane);
            pow_table(s_pow[w][1], cc4.y - cp.y, P, lane);
            pow_table(s_pow[w][2], cc4.z - cp.z, P, lane);
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 26; ++i) {
                int kk = lane + 32 * i;
                if (kk >= ncoef) break;
                uchar4 e = ex[kk];
                double sum = 0.0;
                for (int bx = 0; bx <= e.x; ++bx)
                    for (int by = 0; by <= e.y; ++by)
                        for (int bz = 0; bz <= e.z; ++bz)
                            sum += Mc[cidx(bx, by, bz)] *
                                   (s_pow[w][0][e.x - bx] * s_pow[w][1][e.y - by] * s_pow[w][2][e.z - bz]);
                acc[i] += sum;
            }
        }
#pragma unroll
        for (int i = 0; i < 26; ++i) {
            int kk = lane + 32 * i;
            if (kk >= ncoef) break;
            M[(int64_t)c * ncoef + kk] = acc[i];
        }
    }
}

template <typename Body>
fmm_status upward_t(fmm_ctx* ctx, cudaStream_t s) {
    PhaseScope ps(ctx, PH_UP, s);
    const int64_t nc = ctx->ncell;
    FMM_TRY(buf_ensure(ctx, ctx->M, (size_t)nc * ctx->ncoef * 8));
    double* M = P_<double>(ctx->M);
    int g = (int)std::min<int64_t>((ctx->nleaf + UP_WARPS - 1) / UP_WARPS, (int64_t)ctx->num_sms * 16);
    k_p2m<Body><<<std::max(g, 1), UP_WARPS * 32, 0, s>>>(P_<Body>(ctx->body), P_<uint32_t>(ctx->leaf_ids), ctx->nleaf,
                                                         P_<uint32_t>(ctx->c_bb), P_<uint32_t>(ctx->c_bc),
                                                         P_<double4>(ctx->c_cr), ctx->P, ctx->ncoef, M);
    FMM_LAUNCH(ctx);
    for (int64_t l = ctx->depth - 1; l >= 0; --l) {
        int64_t b = ctx->level_begin[l], e = ctx->level_begin[l + 1];
        int gg = (int)std::min<int64_t>((e - b + UP_WARPS - 1) / UP_WARPS, (int64_t)ctx->num_sms * 16);
        k_m2m<<<std::max(gg, 1), UP_WARPS * 32, 0, s>>>(b, e, P_<uint32_t>(ctx->c_cb), P_<uint32_t>(ctx->c_cc),
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
