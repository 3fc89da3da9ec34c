// p2p_mutual.cu -- mutual (symmetric) near field, SURVEY 8(f) f2 (the
// sphere workload, ncrit 512, whose step is ~90% P2P).
//
// R17 for one leaf pair (A, B), A != B, costs the same geometry both ways: with d = x_b - x_a,
// r^-1 and r^-3 computed once, phi_a += q_b/r, grad_a += q_b d/r^3 AND phi_b += q_a/r,
// grad_b -= q_a d/r^3.  The P2P lists are symmetric ((A, B) listed iff (B, A) is: both are leaf
// pairs failing the same symmetric MAC -- checked here, the one-sided kernels run otherwise), so
// each unordered pair is evaluated once, by the warp of the smaller leaf index.
//
// Warp per target leaf A, 2*NP targets per lane (A's bodies in chunks of 64*NP), the entries
// (A, S) of A's list with S >= A in list order, S in chunks of 32 bodies, one per lane ("home").
// Systolic step s = 0..31: lane l takes body (l + s) mod 32 of the chunk by shuffle, adds its
// action to its own targets (registers) and its reaction to a running accumulator, which then
// moves one lane down -- after 32 steps every lane holds the reaction sum of its home body.
// The reaction of (A, S) is stored in a slot (one float4 per body of S, slot offsets = scan of
// |S| over the entries with S > A) and added by k_mut_react to S's near field, in S's list
// order: every sum has a fixed order, results are bit-reproducible.  The self pair (A, A) takes
// the one-sided form with the r^2 > 0 test (R17: coincident points share a leaf).
// Opt-in (FMM_P2P_MUTUAL): the mirror search scans the source's list per entry (fine for the
// sphere's ~45-entry lists, slow for c3's ~230) and slots over 8 GB fall back to one-sided P2P.
#include "common.cuh"

namespace {
constexpr int MU_WARPS = 4;

// per entry e = (T, S): w[e] = |S| if S > T (reaction slot size), mir[e] = index of (S, T) in
// S's list if S < T; err bit 0 if some mirror is missing
__global__ void k_mut_prep(const uint64_t* __restrict__ off, const uint32_t* __restrict__ src, int64_t nc,
                           const uint32_t* __restrict__ bc, uint32_t* __restrict__ mir, uint64_t* __restrict__ w,
                           unsigned* __restrict__ err) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < nc; t += nw) {
        const uint32_t T = (uint32_t)t;
        const uint64_t e0 = off[t], e1 = off[t + 1];
        for (uint64_t e = e0 + lane; e < e1; e += 32) {
            const uint32_t S = src[e];
            w[e] = S > T ? bc[S] : 0u;
            uint32_t m = ~0u;
            if (S < T) {
                const uint64_t k1 = off[S + 1];
                for (uint64_t k = off[S]; k < k1; ++k)
                    if (src[k] == T) {
                        m = (uint32_t)k;
                        break;
                    }
                if (m == ~0u) atomicOr(err, 1u);
            }
            mir[e] = m;
        }
    }
}

__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float2 shfl2(float2 v, int src) {
    return make_float2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

template <int NP>
__global__ void __launch_bounds__(MU_WARPS * 32) k_p2p_mutual(
    const float4* __restrict__ body, const uint32_t* __restrict__ leaf_ids, int64_t nleaf,
    const uint64_t* __restrict__ off, const uint32_t* __restrict__ src, const uint32_t* __restrict__ bb,
    const uint32_t* __restrict__ bc, const uint64_t* __restrict__ so, float4* __restrict__ slot,
    float* __restrict__ near_phi, float* __restrict__ near_grad, unsigned long long* __restrict__ counter) {
    constexpr int CH = 64 * NP;   // targets per lane pass: 2 NP per lane
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned long long li = 0;
        if (lane == 0) li = atomicAdd(counter, 1ull);
        li = __shfl_sync(0xffffffffu, li, 0);
        if (li >= (unsigned long long)nleaf) break;
        const uint32_t A = leaf_ids[li];
        const uint32_t ta0 = bb[A], nt_all = bc[A];
        const uint64_t e0 = off[A], e1 = off[A + 1];
        for (uint32_t t0 = 0; t0 < nt_all; t0 += CH) {
            const uint32_t nt = min(nt_all - t0, (uint32_t)CH);
            // target slot k of this lane: body t0 + lane + 32 k; slots (2h, 2h+1) form pair h.
            // Positions are held negated (d = x_b + (-x_a) is one FADD2); unused slots sit far
            // away with q = 0 (no action, no reaction)
            float2 nx[NP], ny[NP], nz[NP], qa[NP], f[NP], gx[NP], gy[NP], gz[NP];
#pragma unroll
            for (int h = 0; h < NP; ++h) {
                float px[2], py[2], pz[2], pq[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const uint32_t t = (uint32_t)lane + 32u * (2 * h + e);
                    const float4 p = body[ta0 + t0 + (t < nt ? t : 0)];
                    const bool ok = t < nt;
                    px[e] = ok ? -p.x : -1e30f;
                    py[e] = -p.y;
                    pz[e] = -p.z;
                    pq[e] = ok ? p.w : 0.f;
                }
                nx[h] = make_float2(px[0], px[1]);
                ny[h] = make_float2(py[0], py[1]);
                nz[h] = make_float2(pz[0], pz[1]);
                qa[h] = make_float2(pq[0], pq[1]);
                f[h] = gx[h] = gy[h] = gz[h] = make_float2(0.f, 0.f);
            }
            for (uint64_t e = e0; e < e1; ++e) {
                const uint32_t S = src[e];
                if (S < A) continue;   // evaluated by S's warp (reaction slot)
                const uint32_t sb = bb[S], ns = bc[S];
                if (S == A) {   // self pair: one-sided, r^2 > 0 test
                    for (uint32_t c0 = 0; c0 < ns; c0 += 32) {
                        const bool hv = c0 + lane < ns;
                        const float4 hb = hv ? body[sb + c0 + lane] : make_float4(1e30f, 0.f, 0.f, 0.f);
                        for (int s = 0; s < 32; ++s) {
                            const int sl = (lane + s) & 31;
                            const float bx = __shfl_sync(0xffffffffu, hb.x, sl), by = __shfl_sync(0xffffffffu, hb.y, sl);
                            const float bz = __shfl_sync(0xffffffffu, hb.z, sl), bq = __shfl_sync(0xffffffffu, hb.w, sl);
#pragma unroll
                            for (int h = 0; h < NP; ++h) {
                                const float2 dx = __fadd2_rn(f2(bx), nx[h]), dy = __fadd2_rn(f2(by), ny[h]),
                                             dz = __fadd2_rn(f2(bz), nz[h]);
                                const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
                                const float2 inv = make_float2(r2.x > 0.f ? rsqrtf(r2.x) : 0.f,
                                                               r2.y > 0.f ? rsqrtf(r2.y) : 0.f);
                                const float2 ta = __fmul2_rn(f2(bq), inv);
                                const float2 ta3 = __fmul2_rn(ta, __fmul2_rn(inv, inv));
                                f[h] = __fadd2_rn(f[h], ta);
                                gx[h] = __ffma2_rn(ta3, dx, gx[h]);
                                gy[h] = __ffma2_rn(ta3, dy, gy[h]);
                                gz[h] = __ffma2_rn(ta3, dz, gz[h]);
                            }
                        }
                    }
                    continue;
                }
                const uint64_t sbase = so[e];
                for (uint32_t c0 = 0; c0 < ns; c0 += 32) {
                    const bool hv = c0 + lane < ns;
                    const float4 hb = hv ? body[sb + c0 + lane] : make_float4(1e30f, 0.f, 0.f, 0.f);
                    float2 rf = make_float2(0.f, 0.f), rgx = rf, rgy = rf, rgz = rf;
                    for (int s = 0; s < 32; ++s) {
                        const int sl = (lane + s) & 31;
                        const float bx = __shfl_sync(0xffffffffu, hb.x, sl), by = __shfl_sync(0xffffffffu, hb.y, sl);
                        const float bz = __shfl_sync(0xffffffffu, hb.z, sl), bq = __shfl_sync(0xffffffffu, hb.w, sl);
                        // this step's reaction on body (l + s), summed apart from the moving
                        // accumulator: the carried chain is one FADD2 + the shuffle per step
                        float2 pf = make_float2(0.f, 0.f), pgx = pf, pgy = pf, pgz = pf;
#pragma unroll
                        for (int h = 0; h < NP; ++h) {
                            const float2 dx = __fadd2_rn(f2(bx), nx[h]), dy = __fadd2_rn(f2(by), ny[h]),
                                         dz = __fadd2_rn(f2(bz), nz[h]);
                            const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
                            const float2 inv = make_float2(rsqrtf(r2.x), rsqrtf(r2.y));
                            const float2 inv2 = __fmul2_rn(inv, inv);
                            const float2 ta = __fmul2_rn(f2(bq), inv);   // action: q_b / r
                            const float2 ta3 = __fmul2_rn(ta, inv2);
                            f[h] = __fadd2_rn(f[h], ta);
                            gx[h] = __ffma2_rn(ta3, dx, gx[h]);
                            gy[h] = __ffma2_rn(ta3, dy, gy[h]);
                            gz[h] = __ffma2_rn(ta3, dz, gz[h]);
                            const float2 tb = __fmul2_rn(qa[h], inv);   // reaction: q_a / r
                            const float2 tb3 = __fmul2_rn(tb, inv2);
                            pf = __fadd2_rn(pf, tb);
                            pgx = __ffma2_rn(make_float2(-tb3.x, -tb3.y), dx, pgx);
                            pgy = __ffma2_rn(make_float2(-tb3.x, -tb3.y), dy, pgy);
                            pgz = __ffma2_rn(make_float2(-tb3.x, -tb3.y), dz, pgz);
                        }
                        rf = __fadd2_rn(rf, pf);
                        rgx = __fadd2_rn(rgx, pgx);
                        rgy = __fadd2_rn(rgy, pgy);
                        rgz = __fadd2_rn(rgz, pgz);
                        // the accumulator of body (l + s + 1) sits in lane l + 1
                        const int nl = (lane + 1) & 31;
                        rf = shfl2(rf, nl);
                        rgx = shfl2(rgx, nl);
                        rgy = shfl2(rgy, nl);
                        rgz = shfl2(rgz, nl);
                    }
                    if (hv) {   // after 32 moves: lane l holds its home body's reaction
                        float4 v = make_float4(rf.x + rf.y, rgx.x + rgx.y, rgy.x + rgy.y, rgz.x + rgz.y);
                        float4* o = slot + sbase + c0 + lane;
                        if (t0 > 0) {   // earlier target chunks of A: added in chunk order
                            const float4 u = *o;
                            v = make_float4(u.x + v.x, u.y + v.y, u.z + v.z, u.w + v.w);
                        }
                        *o = v;
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < NP; ++h) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const uint32_t t = (uint32_t)lane + 32u * (2 * h + e);
                    if (t < nt) {
                        const int64_t o = (int64_t)ta0 + t0 + t;
                        near_phi[o] = e ? f[h].y : f[h].x;
                        near_grad[3 * o] = e ? gx[h].y : gx[h].x;
                        near_grad[3 * o + 1] = e ? gy[h].y : gy[h].x;
                        near_grad[3 * o + 2] = e ? gz[h].y : gz[h].x;
                    }
                }
            }
        }
    }
}

// reactions into the near field: target leaf T, its entries (T, S) with S < T in list order,
// each adding the slot S's warp wrote for (S, T)
__global__ void k_mut_react(const uint32_t* __restrict__ leaf_ids, int64_t nleaf, const uint64_t* __restrict__ off,
                            const uint32_t* __restrict__ src, const uint32_t* __restrict__ mir,
                            const uint64_t* __restrict__ so, const uint32_t* __restrict__ bb,
                            const uint32_t* __restrict__ bc, const float4* __restrict__ slot,
                            float* __restrict__ near_phi, float* __restrict__ near_grad) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t li = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; li < nleaf; li += nw) {
        const uint32_t T = leaf_ids[li];
        const uint32_t tb = bb[T], nt = bc[T];
        const uint64_t e0 = off[T], e1 = off[T + 1];
        for (uint32_t i = lane; i < nt; i += 32) {
            const int64_t o = (int64_t)tb + i;
            float p = near_phi[o], g0 = near_grad[3 * o], g1 = near_grad[3 * o + 1], g2 = near_grad[3 * o + 2];
            for (uint64_t e = e0; e < e1; ++e) {
                const uint32_t S = src[e];
                if (S >= T) continue;
                const float4 v = slot[so[mir[e]] + i];
                p += v.x;
                g0 += v.y;
                g1 += v.z;
                g2 += v.w;
            }
            near_phi[o] = p;
            near_grad[3 * o] = g0;
            near_grad[3 * o + 1] = g1;
            near_grad[3 * o + 2] = g2;
        }
    }
}
}  // namespace

// After the lists: mirror indices and reaction-slot offsets (one host round trip); clears
// ctx->mut_ready when a mirror is missing or the slots would exceed the budget.
fmm_status p2p_mutual_prep(fmm_ctx* ctx, cudaStream_t s) {
    ctx->mut_ready = false;
    const int64_t n = ctx->n_p2p, nc = ctx->ncell;
    if (n == 0 || ctx->prec != FMM_F32) return FMM_OK;
    FMM_TRY(buf_ensure(ctx, ctx->mut_mir, (size_t)n * 4 + 64));
    FMM_TRY(buf_ensure(ctx, ctx->mut_w, (size_t)n * 8 + 64));
    FMM_TRY(buf_ensure(ctx, ctx->mut_so, (size_t)(n + 1) * 8 + 64));
    FMM_TRY(buf_ensure(ctx, ctx->cnt_tmp2, 64));
    unsigned* err = P_<unsigned>(ctx->cnt_tmp2) + 8;
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(err, 0, 4, s));
    const unsigned g = (unsigned)std::min<int64_t>((nc + 7) / 8, (int64_t)ctx->num_sms * 8);
    k_mut_prep<<<std::max(g, 1u), 256, 0, s>>>(P_<uint64_t>(ctx->p2p_off), P_<uint32_t>(ctx->p2p_src), nc,
                                               P_<uint32_t>(ctx->c_bc), P_<uint32_t>(ctx->mut_mir),
                                               P_<uint64_t>(ctx->mut_w), err);
    FMM_LAUNCH(ctx);
    uint64_t* so = P_<uint64_t>(ctx->mut_so);
    FMM_TRY(scan_exclusive_u64(ctx, P_<uint64_t>(ctx->mut_w), so, n, so + n, s));
    uint64_t tot = 0;
    unsigned herr = 0;
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&tot, so + n, 8, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    if (herr || tot * 16 > ((uint64_t)8 << 30)) return FMM_OK;   // asymmetric lists / slots over 8 GB
    FMM_TRY(buf_ensure(ctx, ctx->mut_slot, (size_t)std::max<uint64_t>(tot, 1) * 16));
    ctx->mut_ready = true;
    return FMM_OK;
}

fmm_status p2p_mutual(fmm_ctx* ctx, cudaStream_t s) {
    FMM_TRY(buf_ensure(ctx, ctx->cnt_tmp2, 64));
    unsigned long long* counter = P_<unsigned long long>(ctx->cnt_tmp2) + 3;
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(counter, 0, 8, s));
    constexpr int NP = 4;
    int nb = 0;
    FMM_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_p2p_mutual<NP>, MU_WARPS * 32, 0));
    const int64_t g = std::min<int64_t>((int64_t)ctx->num_sms * std::max(nb, 1), (ctx->nleaf + MU_WARPS - 1) / MU_WARPS);
    k_p2p_mutual<NP><<<(unsigned)std::max<int64_t>(g, 1), MU_WARPS * 32, 0, s>>>(
        P_<float4>(ctx->body), P_<uint32_t>(ctx->leaf_ids), ctx->nleaf, P_<uint64_t>(ctx->p2p_off),
        P_<uint32_t>(ctx->p2p_src), P_<uint32_t>(ctx->c_bb), P_<uint32_t>(ctx->c_bc), P_<uint64_t>(ctx->mut_so),
        P_<float4>(ctx->mut_slot), (float*)ctx->near_phi.p, (float*)ctx->near_grad.p, counter);
    FMM_LAUNCH(ctx);
    const unsigned gr = (unsigned)std::min<int64_t>((ctx->nleaf + 7) / 8, (int64_t)ctx->num_sms * 8);
    k_mut_react<<<std::max(gr, 1u), 256, 0, s>>>(P_<uint32_t>(ctx->leaf_ids), ctx->nleaf, P_<uint64_t>(ctx->p2p_off),
                                                 P_<uint32_t>(ctx->p2p_src), P_<uint32_t>(ctx->mut_mir),
                                                 P_<uint64_t>(ctx->mut_so), P_<uint32_t>(ctx->c_bb),
                                                 P_<uint32_t>(ctx->c_bc), P_<float4>(ctx->mut_slot),
                                                 (float*)ctx->near_phi.p, (float*)ctx->near_grad.p);
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}
