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
constexpr int P2M_WARPS = 4;

__constant__ double c_inv[FMM_MAXP + 1] = {0.0,       1.0,        1.0 / 2,  1.0 / 3,  1.0 / 4,  1.0 / 5,
                                           1.0 / 6,   1.0 / 7,    1.0 / 8,  1.0 / 9,  1.0 / 10, 1.0 / 11,
                                           1.0 / 12,  1.0 / 13,   1.0 / 14, 1.0 / 15, 1.0 / 16};

// M_(a,b,c) = sum_j [q_j x_j^a/a! y_j^b/b!] z_j^c/c!: per batch of 32 bodies, lane j writes its
// body's products T[(a,b)][j] = q_j x_j^a/a! y_j^b/b! (a+b <= P-1) and Z[c][j] = z_j^c/c! to the
// warp's shared tables; then every coefficient takes one FMA per body, T x Z, bodies in order
// (2 shared loads + 1 FMA per body and coefficient instead of 3 loads + 2 multiplies + 1 FMA).
__host__ __device__ __forceinline__ int p2m_smem_doubles(int P) { return (P * (P + 1) / 2 + P) * 33; }

template <typename Body, int NI>
__global__ void __launch_bounds__(P2M_WARPS * 32) k_p2m(const Body* __restrict__ body, const uint32_t* __restrict__ leaf_ids,
                                                        int64_t nleaf, const uint32_t* __restrict__ bb,
                                                        const uint32_t* __restrict__ bc, const double4* __restrict__ cr,
                                                        int P, int ncoef, double* __restrict__ M) {
    extern __shared__ double s_p2m[];
    __shared__ uchar4 ex[816];
    fill_ex_table(ex, ncoef);
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nab = P * (P + 1) / 2;
    double* T = s_p2m + (size_t)w * p2m_smem_doubles(P);   // T[(a,b)][33]
    double* Z = T + (size_t)nab * 33;                      // Z[c][33]
    int tix[NI], zc[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
        const uchar4 e = ex[min(lane + 32 * i, ncoef - 1)];
        const int s2 = e.x + e.y;
        tix[i] = (s2 * (s2 + 1) / 2 + e.y) * 33;   // (a,b) row: a+b = s2, then b
        zc[i] = e.z * 33;
    }
    for (int64_t li = (int64_t)blockIdx.x * P2M_WARPS + w; li < nleaf; li += (int64_t)gridDim.x * P2M_WARPS) {
        const uint32_t c = leaf_ids[li];
        const double4 ctr = cr[c];
        double acc[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) acc[i] = 0.0;
        const uint32_t b0 = bb[c], nb = bc[c];
        for (uint32_t j0 = 0; j0 < nb; j0 += 32) {
            const uint32_t m = min(32u, nb - j0);
            __syncwarp();
            if ((uint32_t)lane < m) {
                const Body p = body[b0 + j0 + lane];
                const double dx = (double)p.x - ctr.x, dy = (double)p.y - ctr.y, dz = (double)p.z - ctr.z;
                double qx[FMM_MAXP], yy[FMM_MAXP];
                qx[0] = (double)p.w;
                yy[0] = 1.0;
                double vz = 1.0;
                Z[lane] = 1.0;
#pragma unroll
                for (int e = 1; e < FMM_MAXP; ++e) {
                    if (e < P) {
                        qx[e] = qx[e - 1] * dx * c_inv[e];
                        yy[e] = yy[e - 1] * dy * c_inv[e];
                        vz = vz * dz * c_inv[e];
                        Z[e * 33 + lane] = vz;
                    }
                }
#pragma unroll
                for (int s2 = 0; s2 < FMM_MAXP; ++s2) {
                    if (s2 < P) {
#pragma unroll
                        for (int y = 0; y <= s2; ++y) T[(s2 * (s2 + 1) / 2 + y) * 33 + lane] = qx[s2 - y] * yy[y];
                    }
                }
            }
            __syncwarp();
            // bodies outer, coefficients inner: the NI accumulators are independent chains
            // (each coefficient still sums its bodies in order)
            for (uint32_t j = 0; j < m; ++j) {
#pragma unroll
                for (int i = 0; i < NI; ++i) acc[i] = fma(T[tix[i] + j], Z[zc[i] + j], acc[i]);
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
// The source index cidx(alpha with a_ax = b) is stepped incrementally in b (cidx = n(n+1)(n+2)/6 +
// m(m+1)/2 + c, n = |alpha|, m = a_y + a_z: raising a_ax by one adds (n+1)(n+2)/2 to the first
// term, plus m+1 to the second for the y and z axes, plus 1 for z) -- the same terms in the
// same order as evaluating cidx per term, without its multiplications and division per term.
__device__ __forceinline__ void shift_pass_up(const uchar4* __restrict__ ex, int ncoef, int ax, const double* in,
                                              double* out, const double* t, int lane) {
    for (int k = lane; k < ncoef; k += 32) {
        const uchar4 e = ex[k];
        int a[3] = {e.x, e.y, e.z};
        const int top = a[ax];
        a[ax] = 0;
        int n = a[0] + a[1] + a[2], m = a[1] + a[2];
        int idx = cidx(a[0], a[1], a[2]);
        double s = 0.0;
        for (int b = 0; b <= top; ++b) {
            s += in[idx] * t[top - b];
            idx += (n + 1) * (n + 2) / 2 + (ax == 0 ? 0 : m + 1) + (ax == 2 ? 1 : 0);
            ++n;
            if (ax != 0) ++m;
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
        const size_t sm = (size_t)P2M_WARPS * p2m_smem_doubles(ctx->P) * 8;
        if (sm > 48 * 1024)
            cudaFuncSetAttribute(k_p2m<Body, NI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_p2m<Body, NI><<<std::max(g, 1), P2M_WARPS * 32, sm, s>>>(P_<Body>(ctx->body), P_<uint32_t>(ctx->leaf_ids),
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
