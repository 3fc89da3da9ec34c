// m2l.cu -- M2L over the canonical list (a9).
//
// PAPER.md:58 §II-A: "The M2L (multipole-to-local) kernel ... translates them to local
// expansions"; M2L and P2P "make up more than 90% of the total runtime".
// R14: L_alpha(A) += sum_{|beta| <= P-1-|alpha|} (-1)^|beta| M_beta(B) D^{alpha+beta}G(c_A - c_B),
//      D^k G via the derivative form of the R14 Taylor recurrence:
//      n r^2 D_k = -(2n-1) sum_i k_i d_i D_{k-e_i} - (n-1) sum_i k_i (k_i-1) D_{k-2e_i}
//      (obtained from n r^2 t_k = (2n-1) sum d_i t_{k-e_i} - (n-1) sum t_{k-2e_i} with
//       D_k = (-1)^|k| k! t_k).
//
// This file holds the generic kernel (any P <= 16, Real = float or double): warp per
// target cell over its CSR source range, D table and signed M in shared memory, lanes
// over alpha, each pair's contribution accumulated into fp64 (R19).
#include <climits>
#include <type_traits>

#include "common.cuh"

namespace {
constexpr int ML_WARPS = 2;

// Real = float: every pair is evaluated in the target's power-of-two units (rho_A = 2^(E - level),
// 2^E >= 2 h): u = d / rho_A, M_beta / rho_A^|beta|, and L_alpha = Lhat_alpha / rho_A^(|alpha|+1) --
// exact rescalings that keep D up to order 2P-2 and the multipoles inside the fp32 range at any P
// and any level (DESIGN.md §2 reading 5); Real = double evaluates R14 as written.
template <typename Real>
__global__ void __launch_bounds__(ML_WARPS * 32) k_m2l_generic(int64_t ncell, const uint32_t* __restrict__ src,
                                                                const uint64_t* __restrict__ off,
                                                                const double4* __restrict__ cr, int P, int ncoef,
                                                                const double* __restrict__ M, double* __restrict__ L,
                                                                const int32_t* __restrict__ level,
                                                                const double* __restrict__ root) {
    constexpr bool kScaled = std::is_same<Real, float>::value;
    int E = 0;
    if (kScaled) frexp(2.0 * root[10], &E);
    // dynamic shared memory: ex[ncoef] | per warp: L (double) [ncoef], D [ncoef], M [ncoef]
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uchar4* ex = reinterpret_cast<uchar4*>(smem);
    const int ncp = (ncoef + 1) & ~1;
    double* sLw = reinterpret_cast<double*>(smem + 4 * ncp) + (size_t)w * ncp;
    Real* sDw = reinterpret_cast<Real*>(reinterpret_cast<double*>(smem + 4 * ncp) + (size_t)ML_WARPS * ncp) +
                (size_t)w * 2 * ncp;
    Real* sMw = sDw + ncp;
    fill_ex_table(ex, ncoef);
    __syncthreads();
    for (int64_t a = (int64_t)blockIdx.x * ML_WARPS + w; a < ncell; a += (int64_t)gridDim.x * ML_WARPS) {
        uint64_t p0 = off[a], p1 = off[a + 1];
        if (p0 == p1) continue;
        double4 ca = cr[a];
        const int ea = kScaled ? E - level[a] : 0;
        for (int k = lane; k < ncoef; k += 32) sLw[k] = 0.0;
        for (uint64_t p = p0; p < p1; ++p) {
            uint32_t b = src[p];
            double4 cb = cr[b];
            Real d[3] = {(Real)ldexp(ca.x - cb.x, -ea), (Real)ldexp(ca.y - cb.y, -ea), (Real)ldexp(ca.z - cb.z, -ea)};
            Real r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
            Real inv_r2 = Real(1) / r2;
            __syncwarp();
            if (lane == 0) sDw[0] = Real(1) / sqrt(r2);
            for (int k = lane; k < ncoef; k += 32) {
                Real m = (Real)ldexp(M[(int64_t)b * ncoef + k], -ea * (int)ex[k].w);
                sMw[k] = (ex[k].w & 1) ? -m : m;
            }
            __syncwarp();
            for (int n = 1; n < P; ++n) {
                int kb = ncoef_of(n), ke = ncoef_of(n + 1);
                for (int k = kb + lane; k < ke; k += 32) {
                    uchar4 e = ex[k];
                    int kk[3] = {e.x, e.y, e.z};
                    Real s1 = 0, s2 = 0;
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        if (kk[i] >= 1) {
                            int m[3] = {kk[0], kk[1], kk[2]};
                            m[i] -= 1;
                            s1 += Real(kk[i]) * d[i] * sDw[cidx(m[0], m[1], m[2])];
                        }
                        if (kk[i] >= 2) {
                            int m[3] = {kk[0], kk[1], kk[2]};
                            m[i] -= 2;
                            s2 += Real(kk[i] * (kk[i] - 1)) * sDw[cidx(m[0], m[1], m[2])];
                        }
                    }
                    sDw[k] = -(Real(2 * n - 1) * s1 + Real(n - 1) * s2) * inv_r2 / Real(n);
                }
                __syncwarp();
            }
            for (int k = lane; k < ncoef; k += 32) {
                uchar4 e = ex[k];
                int nb = ncoef_of(P - e.w);
                Real sum = 0;
                for (int j = 0; j < nb; ++j) {
                    uchar4 f = ex[j];
                    sum += sMw[j] * sDw[cidx(e.x + f.x, e.y + f.y, e.z + f.z)];
                }
                sLw[k] += (double)sum;
            }
        }
        __syncwarp();
        for (int k = lane; k < ncoef; k += 32) L[a * ncoef + k] = ldexp(sLw[k], -ea * ((int)ex[k].w + 1));
        __syncwarp();
    }
}

template <typename Real>
fmm_status m2l_generic(fmm_ctx* ctx, cudaStream_t s) {
    int g = (int)std::min<int64_t>((ctx->ncell + ML_WARPS - 1) / ML_WARPS, (int64_t)ctx->num_sms * 8);
    const int ncp = (ctx->ncoef + 1) & ~1;
    size_t smem = (size_t)4 * ncp + (size_t)ML_WARPS * ncp * (8 + 2 * sizeof(Real));
    k_m2l_generic<Real><<<std::max(g, 1), ML_WARPS * 32, smem, s>>>(ctx->ncell, P_<uint32_t>(ctx->m2l_src),
                                                                  P_<uint64_t>(ctx->m2l_off), P_<double4>(ctx->c_cr),
                                                                  ctx->P, ctx->ncoef, P_<double>(ctx->M),
                                                                  P_<double>(ctx->L), P_<int32_t>(ctx->c_level),
                                                                  P_<double>(ctx->root));
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}
__global__ void k_level_span(int64_t n, const int32_t* __restrict__ level, int* __restrict__ mm) {
    int lo = INT_MAX, hi = INT_MIN;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        lo = min(lo, level[i]);
        hi = max(hi, level[i]);
    }
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
}

// largest level difference between two cells that may meet in an M2L pair: the local tree spans
// levels 0..depth; grafted LET cells carry levels rebased to this tree's root (let.cu), so with
// remote cells the span is measured
fmm_status level_span(fmm_ctx* ctx, cudaStream_t s, int* span) {
    // (a caller-supplied tree -- fmm_debug_m2l -- has no level table: measured too)
    if (ctx->nrem == 0 && ctx->level_begin.size() >= 2 && ctx->level_begin.back() == ctx->ncell) {
        *span = (int)ctx->depth;
        return FMM_OK;
    }
    const int64_t nct = ctx->ncell + ctx->nrem;
    FMM_TRY(buf_ensure(ctx, ctx->cnt_tmp, 64));
    int* mm = P_<int>(ctx->cnt_tmp);
    const int init[2] = {INT_MAX, INT_MIN};
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(mm, init, 8, cudaMemcpyHostToDevice, s));
    k_level_span<<<(unsigned)std::min<int64_t>((nct + 255) / 256, 1024), 256, 0, s>>>(nct, P_<int32_t>(ctx->c_level), mm);
    FMM_LAUNCH(ctx);
    int h[2];
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(h, mm, 8, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    *span = h[1] - h[0];
    return FMM_OK;
}
}  // namespace

fmm_status m2l_pass(fmm_ctx* ctx, cudaStream_t s) {
    PhaseScope ps(ctx, PH_M2L, s);
    FMM_TRY(buf_ensure(ctx, ctx->L, (size_t)ctx->ncell * ctx->ncoef * 8));
    // fp32 kernels scale operands by 2^(de n) with de = the pair's level difference, n <= P-1: in
    // range for |de| <= 14 (P <= 10).  Trees spanning more levels (coincident clusters, extreme
    // adaptivity) take the fp64 generic kernel, exact in range at any level difference.
    int span = 0;
    if (ctx->prec == FMM_F32 && ctx->m2l_part != 2 && !ctx->m2l_span_fixed) {
        FMM_TRY(level_span(ctx, s, &span));
        ctx->m2l_deep = span > 14;
    }
    if (ctx->prec == FMM_F32 && ctx->m2l_deep) {
        if (ctx->m2l_part == 1) return FMM_OK;
        FMM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->L.p, 0, (size_t)ctx->ncell * ctx->ncoef * 8, s));
        PhaseScope pk(ctx, PH_M2L_KERNEL, s);
        return m2l_generic<double>(ctx, s);
    }
    if (ctx->use_fast_m2l && m2l_fast_available(ctx->P, ctx->prec)) return m2l_fast(ctx, s);
    if (ctx->m2l_part == 1) return FMM_OK;   // the generic kernel has no operand preparation
    // cells without M2L sources still need L = 0 (the generic kernel skips them)
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->L.p, 0, (size_t)ctx->ncell * ctx->ncoef * 8, s));
    PhaseScope pk(ctx, PH_M2L_KERNEL, s);
    if (ctx->prec == FMM_F32) return m2l_generic<float>(ctx, s);
    return m2l_generic<double>(ctx, s);
}
