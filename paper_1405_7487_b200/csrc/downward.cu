// downward.cu -- L2L level by level, L2P at leaves, near+far merge and un-permute (a11, a12).
//
// PAPER.md:151 §II-C: "a post-order traversal is performed and L2L and L2P kernels are
// executed to cascade the information down the tree to the particles" (pre-order,
// parent before child, realised level-synchronously).
// R15 L2L: L_alpha(ch) += sum_{beta >= alpha} L_beta(par) s^(beta-alpha)/(beta-alpha)!, s = c_ch - c_par
// R16 L2P: phi_i += sum_alpha L_alpha z^alpha/alpha!, (grad phi_i)_d += sum_{|g|<=P-2} L_{g+e_d} z^g/g!
// R18: output = near (P2P) + far (L2P), scattered to the caller's order through perm.
#include "common.cuh"

namespace {
constexpr int DN_WARPS = 4;
constexpr int LP_WARPS = 4;   // P-specialised L2P
constexpr int LPG_WARPS = 2;  // generic L2P (shared power tables)

__constant__ double c_inv[FMM_MAXP + 1] = {0.0,       1.0,        1.0 / 2,  1.0 / 3,  1.0 / 4,  1.0 / 5,
                                           1.0 / 6,   1.0 / 7,    1.0 / 8,  1.0 / 9,  1.0 / 10, 1.0 / 11,
                                           1.0 / 12,  1.0 / 13,   1.0 / 14, 1.0 / 15, 1.0 / 16};

// separable 1D "down" shift along axis ax: out_alpha = sum_{k <= P-1-|alpha|} in_{alpha + k e_ax} t[k]
// The source index starts at cidx(alpha) = kk and is stepped as a_ax grows (cidx = n(n+1)(n+2)/6 +
// m(m+1)/2 + c: +(n+1)(n+2)/2, plus m+1 on the y and z axes, plus 1 on z) -- the same terms in
// the same order as a cidx per term (upward.cu's shift_pass_up does the same).
__device__ __forceinline__ void shift_pass_down(const uchar4* __restrict__ ex, int ncoef, int P, int ax,
                                                const double* in, double* out, const double* t, int lane) {
    for (int kk = lane; kk < ncoef; kk += 32) {
        const uchar4 e = ex[kk];
        const int top = P - 1 - e.w;
        int n = e.w, m = e.y + e.z, idx = kk;
        double s = 0.0;
        for (int k = 0; k <= top; ++k) {
            s += in[idx] * t[k];
            idx += (n + 1) * (n + 2) / 2 + (ax == 0 ? 0 : m + 1) + (ax == 2 ? 1 : 0);
            ++n;
            if (ax != 0) ++m;
        }
        out[kk] = s;
    }
}

// children at level l+1 receive their parent's shifted local expansion: R15 grouped as three
// 1D passes (the shift operator s^g/g! is separable per axis)
__global__ void __launch_bounds__(DN_WARPS * 32) k_l2l(int64_t cbeg, int64_t cend, const int32_t* __restrict__ parent,
                                                        const double4* __restrict__ cr, int P, int ncoef,
                                                        double* __restrict__ L) {
    extern __shared__ double s_dyn[];
    __shared__ uchar4 ex[816];
    __shared__ double s_t[DN_WARPS][3][FMM_MAXP];
    fill_ex_table(ex, ncoef);
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double* A = s_dyn + (size_t)w * 2 * ncoef;
    double* B = A + ncoef;
    for (int64_t c = cbeg + (int64_t)blockIdx.x * DN_WARPS + w; c < cend; c += (int64_t)gridDim.x * DN_WARPS) {
        const int32_t par = parent[c];
        const double4 cc = cr[c], cp = cr[par];
        __syncwarp();
        for (int i = lane; i < ncoef; i += 32) A[i] = L[(int64_t)par * ncoef + i];
        if (lane < 3) {
            const double sh = lane == 0 ? cc.x - cp.x : lane == 1 ? cc.y - cp.y : cc.z - cp.z;
            double v = 1.0;
            s_t[w][lane][0] = 1.0;
            for (int e = 1; e < P; ++e) {
                v = v * sh * c_inv[e];
                s_t[w][lane][e] = v;
            }
        }
        __syncwarp();
        shift_pass_down(ex, ncoef, P, 0, A, B, s_t[w][0], lane);
        __syncwarp();
        shift_pass_down(ex, ncoef, P, 1, B, A, s_t[w][1], lane);
        __syncwarp();
        shift_pass_down(ex, ncoef, P, 2, A, B, s_t[w][2], lane);
        __syncwarp();
        for (int i = lane; i < ncoef; i += 32) L[(int64_t)c * ncoef + i] += B[i];
    }
}

// warp per leaf, lanes over bodies; writes the final outputs in the caller's order
template <typename Body, typename Real>
__global__ void __launch_bounds__(LPG_WARPS * 32) k_l2p(const Body* __restrict__ body, const uint32_t* __restrict__ perm,
                                                        const uint32_t* __restrict__ leaf_ids, int64_t nleaf,
                                                        const uint32_t* __restrict__ bb, const uint32_t* __restrict__ bc,
                                                        const double4* __restrict__ cr, int P, int ncoef,
                                                        const double* __restrict__ L, const Real* __restrict__ near_phi,
                                                        const Real* __restrict__ near_grad, Real* __restrict__ phi,
                                                        Real* __restrict__ grad, double4* __restrict__ far) {
    __shared__ uchar4 ex[816];
    __shared__ double s_L[LPG_WARPS][816];
    __shared__ double s_pw[LPG_WARPS][3][FMM_MAXP][32];
    fill_ex_table(ex, ncoef);
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t li = (int64_t)blockIdx.x * LPG_WARPS + w; li < nleaf; li += (int64_t)gridDim.x * LPG_WARPS) {
        uint32_t c = leaf_ids[li];
        double4 ctr = cr[c];
        __syncwarp();
        for (int k = lane; k < ncoef; k += 32) s_L[w][k] = L[(int64_t)c * ncoef + k];
        __syncwarp();
        uint32_t b0 = bb[c], nb = bc[c];
        for (uint32_t j0 = 0; j0 < nb; j0 += 32) {
            uint32_t j = j0 + lane;
            bool ok = j < nb;
            double z[3] = {0, 0, 0};
            if (ok) {
                Body p = body[b0 + j];
                z[0] = (double)p.x - ctr.x; z[1] = (double)p.y - ctr.y; z[2] = (double)p.z - ctr.z;
            }
            for (int d = 0; d < 3; ++d) {
                double v = 1.0;
                s_pw[w][d][0][lane] = 1.0;
                for (int e = 1; e < P; ++e) {
                    v = v * z[d] * c_inv[e];
                    s_pw[w][d][e][lane] = v;
                }
            }
            double f = 0.0, g0 = 0.0, g1 = 0.0, g2 = 0.0;
            for (int k = 0; k < ncoef; ++k) {
                uchar4 e = ex[k];
                double m = s_pw[w][0][e.x][lane] * s_pw[w][1][e.y][lane] * s_pw[w][2][e.z][lane];
                f += s_L[w][k] * m;
                if (e.w <= P - 2) {
                    g0 += s_L[w][cidx(e.x + 1, e.y, e.z)] * m;
                    g1 += s_L[w][cidx(e.x, e.y + 1, e.z)] * m;
                    g2 += s_L[w][cidx(e.x, e.y, e.z + 1)] * m;
                }
            }
            if (ok && far) {
                far[b0 + j] = make_double4(f, g0, g1, g2);
            } else if (ok) {
                uint32_t sj = b0 + j;
                uint32_t o = perm[sj];
                phi[o] = (Real)(f + (double)near_phi[sj]);
                grad[3 * (int64_t)o + 0] = (Real)(g0 + (double)near_grad[3 * (int64_t)sj + 0]);
                grad[3 * (int64_t)o + 1] = (Real)(g1 + (double)near_grad[3 * (int64_t)sj + 1]);
                grad[3 * (int64_t)o + 2] = (Real)(g2 + (double)near_grad[3 * (int64_t)sj + 2]);
            }
        }
    }
}

// P-specialised L2P: one lane per body, z^e/e! per axis in registers, L from a per-warp
// shared copy (broadcast reads); R16 evaluated as nested sums over (a, b, c) with
// compile-time indices.  phi uses all |alpha| <= P-1, grad_d uses L_{g+e_d}, |g| <= P-2.
template <int P>
struct InvFact {
    double v[P];
    __host__ __device__ constexpr InvFact() : v() {
        double f = 1.0;
        for (int i = 0; i < P; ++i) {
            if (i > 0) f *= (double)i;
            v[i] = 1.0 / f;
        }
    }
};

template <int P, typename Body, typename Real>
__global__ void __launch_bounds__(LP_WARPS * 32) k_l2p_t(const Body* __restrict__ body, const uint32_t* __restrict__ perm,
                                                          const uint32_t* __restrict__ leaf_ids, int64_t nleaf,
                                                          const uint32_t* __restrict__ bb,
                                                          const uint32_t* __restrict__ bc,
                                                          const double4* __restrict__ cr, const double* __restrict__ L,
                                                          const Real* __restrict__ near_phi,
                                                          const Real* __restrict__ near_grad, Real* __restrict__ phi,
                                                          Real* __restrict__ grad, double4* __restrict__ far) {
    constexpr int NC = P * (P + 1) * (P + 2) / 6;
    // two leaves per warp, a half-warp each (small Plummer leaves fill a half-warp; the halves'
    // broadcast reads of their own L copies fall in different banks, one wavefront)
    __shared__ double s_L[LP_WARPS][2][NC];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, half = lane >> 4, hl = lane & 15;
    for (int64_t lp = (int64_t)blockIdx.x * LP_WARPS + w; 2 * lp < nleaf; lp += (int64_t)gridDim.x * LP_WARPS) {
        const int64_t li = 2 * lp + half;
        const bool has = li < nleaf;
        const uint32_t c = has ? leaf_ids[li] : leaf_ids[2 * lp];
        const double4 ctr = cr[c];
        __syncwarp();
        if (has)
            for (int k = hl; k < NC; k += 16) s_L[w][half][k] = L[(int64_t)c * NC + k];
        __syncwarp();
        const double* Ls = s_L[w][half];
        const uint32_t b0 = bb[c], nb = has ? bc[c] : 0u;
        for (uint32_t j0 = 0; j0 < nb; j0 += 16) {
            const uint32_t j = j0 + hl;
            if (j >= nb) continue;
            const Body p = body[b0 + j];
            const double z[3] = {(double)p.x - ctr.x, (double)p.y - ctr.y, (double)p.z - ctr.z};
            constexpr InvFact<P> F{};
            double pw[3][P];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                double v = 1.0;
#pragma unroll
                for (int e = 0; e < P; ++e) {
                    pw[d][e] = v * F.v[e];
                    v *= z[d];
                }
            }
            double f = 0.0, g[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int a = 0; a < P; ++a) {
                double fa = 0.0, ga[3] = {0.0, 0.0, 0.0};
#pragma unroll
                for (int bq = 0; bq < P - a; ++bq) {
                    double fb = 0.0, gb[3] = {0.0, 0.0, 0.0};
#pragma unroll
                    for (int cq = 0; cq < P - a - bq; ++cq) {
                        fb = fma(Ls[cidx(a, bq, cq)], pw[2][cq], fb);
                        if (a + bq + cq <= P - 2) {
                            gb[0] = fma(Ls[cidx(a + 1, bq, cq)], pw[2][cq], gb[0]);
                            gb[1] = fma(Ls[cidx(a, bq + 1, cq)], pw[2][cq], gb[1]);
                            gb[2] = fma(Ls[cidx(a, bq, cq + 1)], pw[2][cq], gb[2]);
                        }
                    }
                    fa = fma(fb, pw[1][bq], fa);
#pragma unroll
                    for (int d = 0; d < 3; ++d) ga[d] = fma(gb[d], pw[1][bq], ga[d]);
                }
                f = fma(fa, pw[0][a], f);
#pragma unroll
                for (int d = 0; d < 3; ++d) g[d] = fma(ga[d], pw[0][a], g[d]);
            }
            const uint32_t sj = b0 + j;
            if (far) {
                far[sj] = make_double4(f, g[0], g[1], g[2]);
                continue;
            }
            const uint32_t o = perm[sj];
            phi[o] = (Real)(f + (double)near_phi[sj]);
#pragma unroll
            for (int d = 0; d < 3; ++d) grad[3 * (int64_t)o + d] = (Real)(g[d] + (double)near_grad[3 * (int64_t)sj + d]);
        }
    }
}

// R18 with the far field kept separately (L2P ran concurrently with P2P): the same sums as the
// fused L2P epilogue, (Real)(far + (double)near), in the caller's order
template <typename Real>
__global__ void k_merge_nearfar(int64_t n, const uint32_t* __restrict__ iperm, const double4* __restrict__ far,
                                const Real* __restrict__ near_phi, const Real* __restrict__ near_grad,
                                Real* __restrict__ phi, Real* __restrict__ grad) {
    // caller order o, sorted index i = iperm[o]: gathered reads, coalesced writes
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n; o += stride) {
        const int64_t i = iperm[o];
        const double4 f = far[i];
        phi[o] = (Real)(f.x + (double)near_phi[i]);
        grad[3 * o + 0] = (Real)(f.y + (double)near_grad[3 * i + 0]);
        grad[3 * o + 1] = (Real)(f.z + (double)near_grad[3 * i + 1]);
        grad[3 * o + 2] = (Real)(f.w + (double)near_grad[3 * i + 2]);
    }
}

template <typename Body, typename Real>
fmm_status downward_t(fmm_ctx* ctx, void* phi, void* grad, double4* far, cudaStream_t s) {
    PhaseScope ps(ctx, PH_DOWN, s);
    double* L = P_<double>(ctx->L);
    const size_t smem = (size_t)DN_WARPS * 2 * ctx->ncoef * 8;
    if (smem > 48 * 1024) FMM_CUDA_TRY(ctx, cudaFuncSetAttribute(k_l2l, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int64_t l = 1; l <= ctx->depth; ++l) {
        int64_t b = ctx->level_begin[l], e = ctx->level_begin[l + 1];
        int g = (int)std::min<int64_t>((e - b + DN_WARPS - 1) / DN_WARPS, (int64_t)ctx->num_sms * 16);
        k_l2l<<<std::max(g, 1), DN_WARPS * 32, smem, s>>>(b, e, P_<int32_t>(ctx->c_parent), P_<double4>(ctx->c_cr),
                                                       ctx->P, ctx->ncoef, L);
        FMM_LAUNCH(ctx);
    }
    int g = (int)std::min<int64_t>((ctx->nleaf + LP_WARPS - 1) / LP_WARPS, (int64_t)ctx->num_sms * 32);
#define FMM_L2P_T(PP)                                                                                              \
    if (ctx->P == PP) {                                                                                            \
        k_l2p_t<PP, Body, Real><<<std::max(g, 1), LP_WARPS * 32, 0, s>>>(                                          \
            P_<Body>(ctx->body), ctx->d_perm, P_<uint32_t>(ctx->leaf_ids), ctx->nleaf, P_<uint32_t>(ctx->c_bb),    \
            P_<uint32_t>(ctx->c_bc), P_<double4>(ctx->c_cr), L, P_<Real>(ctx->near_phi), P_<Real>(ctx->near_grad), \
            (Real*)phi, (Real*)grad, far);                                                                         \
        FMM_LAUNCH(ctx);                                                                                           \
        FMM_CUDA_TRY(ctx, cudaGetLastError());                                                                     \
        return FMM_OK;                                                                                             \
    }
    FMM_L2P_T(4)
    FMM_L2P_T(6)
    FMM_L2P_T(8)
    FMM_L2P_T(10)
#undef FMM_L2P_T
    g = (int)std::min<int64_t>((ctx->nleaf + LPG_WARPS - 1) / LPG_WARPS, (int64_t)ctx->num_sms * 32);
    k_l2p<Body, Real><<<std::max(g, 1), LPG_WARPS * 32, 0, s>>>(
        P_<Body>(ctx->body), ctx->d_perm, P_<uint32_t>(ctx->leaf_ids), ctx->nleaf, P_<uint32_t>(ctx->c_bb),
        P_<uint32_t>(ctx->c_bc), P_<double4>(ctx->c_cr), ctx->P, ctx->ncoef, L, P_<Real>(ctx->near_phi),
        P_<Real>(ctx->near_grad), (Real*)phi, (Real*)grad, far);
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}

template <typename Real>
fmm_status merge_t(fmm_ctx* ctx, void* phi, void* grad, cudaStream_t s) {
    PhaseScope ps(ctx, PH_DOWN, s);
    const int g = (int)std::min<int64_t>((ctx->n + 255) / 256, (int64_t)ctx->num_sms * 8);
    k_merge_nearfar<Real><<<std::max(g, 1), 256, 0, s>>>(ctx->n, P_<uint32_t>(ctx->iperm), P_<double4>(ctx->far),
                                                         P_<Real>(ctx->near_phi), P_<Real>(ctx->near_grad),
                                                         (Real*)phi, (Real*)grad);
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}
}  // namespace

fmm_status downward_pass(fmm_ctx* ctx, void* phi, void* grad, cudaStream_t s) {
    if (ctx->prec == FMM_F32) return downward_t<float4, float>(ctx, phi, grad, nullptr, s);
    return downward_t<dbody, double>(ctx, phi, grad, nullptr, s);
}

fmm_status downward_far(fmm_ctx* ctx, cudaStream_t s) {
    FMM_TRY(buf_ensure(ctx, ctx->far, (size_t)ctx->n * sizeof(double4)));
    double4* far = P_<double4>(ctx->far);
    if (ctx->prec == FMM_F32) return downward_t<float4, float>(ctx, nullptr, nullptr, far, s);
    return downward_t<dbody, double>(ctx, nullptr, nullptr, far, s);
}

fmm_status merge_nearfar(fmm_ctx* ctx, void* phi, void* grad, cudaStream_t s) {
    if (ctx->prec == FMM_F32) return merge_t<float>(ctx, phi, grad, s);
    return merge_t<double>(ctx, phi, grad, s);
}
