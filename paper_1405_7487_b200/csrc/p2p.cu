// p2p.cu -- near-field P2P over the canonical leaf-pair list (a10).
//
// PAPER.md:58, 62, 151 §II: P2P is direct interaction between particles of neighbouring
// cells; with M2L it is >90% of the runtime.
// R17 / R1: for i in A, j in B: r^2 = |x_j - x_i|^2; skip r^2 == 0; phi_i += q_j / r;
//           grad_i += q_j (x_j - x_i) / r^3.
// Results are written in sorted order to near_phi / near_grad; L2P adds the far field.
//
// Generic kernel: warp per target leaf, 2 targets per lane (64 per pass), sources of each
// list entry staged through a per-warp shared-memory tile and read as broadcasts.
#include "common.cuh"

namespace {
constexpr int PP_WARPS = 4;
constexpr int PP_TILE = 128;

__device__ __forceinline__ float rsqrt_(float x) { return rsqrtf(x); }
__device__ __forceinline__ double rsqrt_(double x) { return 1.0 / sqrt(x); }

template <typename Body, typename Real>
__global__ void __launch_bounds__(PP_WARPS * 32) k_p2p_generic(const Body* __restrict__ body,
                                                                const uint32_t* __restrict__ leaf_ids, int64_t nleaf,
                                                                const uint64_t* __restrict__ lst,
                                                                const uint64_t* __restrict__ off,
                                                                const uint32_t* __restrict__ bb,
                                                                const uint32_t* __restrict__ bc,
                                                                Real* __restrict__ near_phi, Real* __restrict__ near_grad) {
    __shared__ Body s_src[PP_WARPS][PP_TILE];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t li = (int64_t)blockIdx.x * PP_WARPS + w; li < nleaf; li += (int64_t)gridDim.x * PP_WARPS) {
        uint32_t a = leaf_ids[li];
        uint32_t tb = bb[a], nt = bc[a];
        uint64_t p0 = off[a], p1 = off[a + 1];
        for (uint32_t t0 = 0; t0 < nt; t0 += 64) {
            Real x[2], y[2], z[2], f[2] = {0, 0}, gx[2] = {0, 0}, gy[2] = {0, 0}, gz[2] = {0, 0};
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                uint32_t t = t0 + lane + 32 * r;
                Body p = body[tb + (t < nt ? t : 0)];
                x[r] = p.x; y[r] = p.y; z[r] = p.z;
            }
            for (uint64_t pp = p0; pp < p1; ++pp) {
                uint32_t b = (uint32_t)lst[pp];
                uint32_t sb = bb[b], ns = bc[b];
                for (uint32_t s0 = 0; s0 < ns; s0 += PP_TILE) {
                    uint32_t m = min((uint32_t)PP_TILE, ns - s0);
                    __syncwarp();
                    for (uint32_t j = lane; j < m; j += 32) s_src[w][j] = body[sb + s0 + j];
                    __syncwarp();
                    for (uint32_t j = 0; j < m; ++j) {
                        Body s = s_src[w][j];
#pragma unroll
                        for (int r = 0; r < 2; ++r) {
                            Real dx = (Real)s.x - x[r], dy = (Real)s.y - y[r], dz = (Real)s.z - z[r];
                            Real r2 = dx * dx + dy * dy + dz * dz;
                            Real inv = r2 > Real(0) ? rsqrt_(r2) : Real(0);
                            Real qi = (Real)s.w * inv;
                            Real qi3 = qi * inv * inv;
                            f[r] += qi;
                            gx[r] += qi3 * dx;
                            gy[r] += qi3 * dy;
                            gz[r] += qi3 * dz;
                        }
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                uint32_t t = t0 + lane + 32 * r;
                if (t < nt) {
                    int64_t o = (int64_t)tb + t;
                    near_phi[o] = f[r];
                    near_grad[3 * o] = gx[r];
                    near_grad[3 * o + 1] = gy[r];
                    near_grad[3 * o + 2] = gz[r];
                }
            }
        }
    }
}

template <typename Body, typename Real>
fmm_status p2p_t(fmm_ctx* ctx, cudaStream_t s) {
    PhaseScope ps(ctx, PH_P2P, s);
    FMM_TRY(buf_ensure(ctx, ctx->near_phi, (size_t)ctx->n * sizeof(Real)));
    FMM_TRY(buf_ensure(ctx, ctx->near_grad, (size_t)ctx->n * 3 * sizeof(Real)));
    PhaseScope pk(ctx, PH_P2P_KERNEL, s);
    int g = (int)std::min<int64_t>((ctx->nleaf + PP_WARPS - 1) / PP_WARPS, (int64_t)ctx->num_sms * 16);
    k_p2p_generic<Body, Real><<<std::max(g, 1), PP_WARPS * 32, 0, s>>>(
        P_<Body>(ctx->body), P_<uint32_t>(ctx->leaf_ids), ctx->nleaf, P_<uint64_t>(ctx->lst_p2p),
        P_<uint64_t>(ctx->p2p_off), P_<uint32_t>(ctx->c_bb), P_<uint32_t>(ctx->c_bc), P_<Real>(ctx->near_phi),
        P_<Real>(ctx->near_grad));
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}
}  // namespace

fmm_status p2p_pass(fmm_ctx* ctx, cudaStream_t s) {
    if (ctx->prec == FMM_F32) return p2p_t<float4, float>(ctx, s);
    return p2p_t<dbody, double>(ctx, s);
}
