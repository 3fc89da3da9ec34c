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
#include <type_traits>

#include "common.cuh"

namespace {
constexpr int PP_WARPS = 4;
constexpr int PP_TILE = 128;

__device__ __forceinline__ float rsqrt_(float x) { return rsqrtf(x); }
__device__ __forceinline__ double rsqrt_(double x) { return 1.0 / sqrt(x); }

template <typename Body, typename Real>
__global__ void __launch_bounds__(PP_WARPS * 32) k_p2p_generic(const Body* __restrict__ body,
                                                                const uint32_t* __restrict__ leaf_ids, int64_t nleaf,
                                                                const uint32_t* __restrict__ lst,
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
                uint32_t b = lst[pp];
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


// ---------------------------------------------------------------- fp32 fast path
// Warp per target leaf (dynamic: per-warp atomic counter).  The leaf's nt targets are
// spread over lpg = ceil(nt/T) lanes with T = 4 targets per lane; the warp's 32 lanes form
// G = 32/lpg groups that split the source stream (group g takes sources g, g+G, ...), so
// small leaves still fill the warp.  Source leaves are streamed through a per-warp
// double-buffered shared-memory tile with cp.async (16 B per body); in the inner loop the
// G groups read G consecutive float4 (one wavefront).  Non-self pairs skip the r^2 > 0
// test (coincident points share a key and hence a leaf, so r^2 = 0 only occurs in the
// self pair A<-A, which takes the checked loop).  Group partials are summed in shared memory.
constexpr int PF_WARPS = 8;
constexpr int PF_T = 4;
constexpr int PF_TILE = 64;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;\n" ::); }

template <bool CHECK>
__device__ __forceinline__ void p2p_body(const float4 s, const float (&x)[PF_T], const float (&y)[PF_T],
                                         const float (&z)[PF_T], float (&f)[PF_T], float (&gx)[PF_T],
                                         float (&gy)[PF_T], float (&gz)[PF_T]) {
#pragma unroll
    for (int k = 0; k < PF_T; ++k) {
        const float dx = s.x - x[k], dy = s.y - y[k], dz = s.z - z[k];
        const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        float inv = rsqrtf(r2);
        if (CHECK) inv = r2 > 0.f ? inv : 0.f;
        const float qi = s.w * inv;
        const float qi3 = qi * (inv * inv);
        f[k] += qi;
        gx[k] = fmaf(qi3, dx, gx[k]);
        gy[k] = fmaf(qi3, dy, gy[k]);
        gz[k] = fmaf(qi3, dz, gz[k]);
    }
}

__global__ void __launch_bounds__(PF_WARPS * 32) k_p2p_f32(const float4* __restrict__ body,
                                                           const uint32_t* __restrict__ leaf_ids, int64_t nleaf,
                                                           const uint32_t* __restrict__ lst,
                                                           const uint64_t* __restrict__ off,
                                                           const uint32_t* __restrict__ bb,
                                                           const uint32_t* __restrict__ bc, float* __restrict__ near_phi,
                                                           float* __restrict__ near_grad,
                                                           unsigned long long* __restrict__ counter) {
    __shared__ __align__(16) float4 s_tile[PF_WARPS][2][PF_TILE];
    __shared__ float4 s_red[PF_WARPS][32 * PF_T];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float4 (*tile)[PF_TILE] = s_tile[w];
    for (;;) {
        unsigned long long li = 0;
        if (lane == 0) li = atomicAdd(counter, 1ull);
        li = __shfl_sync(0xffffffffu, li, 0);
        if (li >= (unsigned long long)nleaf) break;
        const uint32_t a = leaf_ids[li];
        const uint32_t tb = bb[a], nt_all = bc[a];
        const uint64_t p0 = off[a], p1 = off[a + 1];
        for (uint32_t t0 = 0; t0 < nt_all; t0 += 32 * PF_T) {
            const uint32_t nt = min(nt_all - t0, (uint32_t)(32 * PF_T));
            const int lpg = (int)((nt + PF_T - 1) / PF_T);
            const int G = min(32 / lpg, 16);
            const int g = lane / lpg, j = lane - g * lpg;
            const bool active = g < G;
            float x[PF_T], y[PF_T], z[PF_T], f[PF_T], gx[PF_T], gy[PF_T], gz[PF_T];
#pragma unroll
            for (int k = 0; k < PF_T; ++k) {
                const uint32_t t = (uint32_t)(j + k * lpg);
                const float4 p = body[tb + t0 + (t < nt ? t : 0)];
                // unused slots sit far away so they never produce r^2 = 0
                x[k] = t < nt ? p.x : 1e30f; y[k] = p.y; z[k] = p.z;
                f[k] = gx[k] = gy[k] = gz[k] = 0.f;
            }
            // chunk iterator over (list entry, offset in source leaf)
            uint64_t cp_ = p0;
            uint32_t cs = 0;
            auto chunk = [&](uint64_t pp, uint32_t s0, uint32_t& src, uint32_t& m, bool& self) {
                const uint32_t b = lst[pp];
                src = bb[b] + s0;
                m = min((uint32_t)PF_TILE, bc[b] - s0);
                self = b == a;
            };
            auto advance = [&](uint64_t& pp, uint32_t& s0) {
                const uint32_t b = lst[pp];
                s0 += PF_TILE;
                if (s0 >= bc[b]) { ++pp; s0 = 0; }
            };
            int buf = 0;
            uint32_t src_c = 0, m_c = 0;
            bool self_c = false;
            if (cp_ < p1) {
                chunk(cp_, cs, src_c, m_c, self_c);
                for (uint32_t i = lane; i < m_c; i += 32) cp_async16(&tile[0][i], body + src_c + i);
            }
            cp_async_commit();
            while (cp_ < p1) {
                // prefetch the next chunk into the other buffer
                uint64_t np_ = cp_;
                uint32_t ns_ = cs;
                advance(np_, ns_);
                uint32_t src_n = 0, m_n = 0;
                bool self_n = false;
                if (np_ < p1) {
                    chunk(np_, ns_, src_n, m_n, self_n);
                    for (uint32_t i = lane; i < m_n; i += 32) cp_async16(&tile[buf ^ 1][i], body + src_n + i);
                }
                cp_async_commit();
                cp_async_wait_1();
                __syncwarp();
                if (active) {
                    const float4* tl = tile[buf];
                    if (self_c) {
                        for (uint32_t i = g; i < m_c; i += G) p2p_body<true>(tl[i], x, y, z, f, gx, gy, gz);
                    } else {
                        for (uint32_t i = g; i < m_c; i += G) p2p_body<false>(tl[i], x, y, z, f, gx, gy, gz);
                    }
                }
                __syncwarp();
                cp_ = np_;
                cs = ns_;
                m_c = m_n;
                self_c = self_n;
                buf ^= 1;
            }
            cp_async_wait_0();
            // sum the G group partials per target
            __syncwarp();
#pragma unroll
            for (int k = 0; k < PF_T; ++k) s_red[w][lane * PF_T + k] = make_float4(f[k], gx[k], gy[k], gz[k]);
            __syncwarp();
            if (g == 0) {
#pragma unroll
                for (int k = 0; k < PF_T; ++k) {
                    const uint32_t t = (uint32_t)(j + k * lpg);
                    if (t < nt) {
                        float4 acc = s_red[w][lane * PF_T + k];
                        for (int gg = 1; gg < G; ++gg) {
                            const float4 v = s_red[w][(gg * lpg + j) * PF_T + k];
                            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
                        }
                        const int64_t o = (int64_t)tb + t0 + t;
                        near_phi[o] = acc.x;
                        near_grad[3 * o] = acc.y;
                        near_grad[3 * o + 1] = acc.z;
                        near_grad[3 * o + 2] = acc.w;
                    }
                }
            }
            __syncwarp();
        }
    }
}


// Packed form of p2p_body for the CTA path: the thread's 4 targets are held as 2 float2 pairs
// (positions stored NEGATED so dx = s.x + (-x) is one FADD2 with a broadcast operand), and
// every FP32 step is an f32x2 instruction (FADD2/FMUL2/FFMA2, sm_100): the FMA pipe does the
// same 13 lane-ops per interaction, but the issue slots they take halve, which leaves room
// for the LDS, MUFU.RSQ and loop instructions (the scalar form was issue-bound).
template <bool CHECK, int NP>
__device__ __forceinline__ void p2p_body2(const float4 s, const float2 (&nx)[NP], const float2 (&ny)[NP],
                                          const float2 (&nz)[NP], float2 (&f)[NP], float2 (&gx)[NP],
                                          float2 (&gy)[NP], float2 (&gz)[NP]) {
    const float2 sx = make_float2(s.x, s.x), sy = make_float2(s.y, s.y), sz = make_float2(s.z, s.z);
    const float2 sq = make_float2(s.w, s.w);
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        const float2 dx = __fadd2_rn(sx, nx[k]), dy = __fadd2_rn(sy, ny[k]), dz = __fadd2_rn(sz, nz[k]);
        const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
        float2 inv = make_float2(rsqrtf(r2.x), rsqrtf(r2.y));
        if (CHECK) {
            inv.x = r2.x > 0.f ? inv.x : 0.f;
            inv.y = r2.y > 0.f ? inv.y : 0.f;
        }
        const float2 qi = __fmul2_rn(sq, inv);
        const float2 qi3 = __fmul2_rn(qi, __fmul2_rn(inv, inv));
        f[k] = __fadd2_rn(f[k], qi);
        gx[k] = __ffma2_rn(qi3, dx, gx[k]);
        gy[k] = __ffma2_rn(qi3, dy, gy[k]);
        gz[k] = __ffma2_rn(qi3, dz, gz[k]);
    }
}

// ------------------------------------------------------- fp32 CTA-per-leaf path
// One CTA (128 threads) per target leaf, taken from an atomic counter in leaf order.  The
// leaf's nt targets occupy lpg = ceil(nt/4) threads x 4 registers; the CTA's 128 threads form
// G = 128/lpg groups that split the target's source stream (512 slots per CTA keeps the
// slot use ~90-100% for the ragged occupancies around ncrit/2).  The source stream is the
// target's P2P list flattened into Morton-contiguous body runs (build_runs); it is cut into
// chunks of CH = G*floor(256/G) bodies, loaded with cp.async into a double-buffered shared
// tile (thread i fetches flat indices i and i+128, locating its run with a forward cursor),
// and group g consumes entries g, g+G, ... (G consecutive float4 per step).  Only chunks
// that overlap the target's own leaf take the r^2 > 0 test.
constexpr int PC_THREADS = 128;
// GT threads ("team") per target leaf; a block of PC_THREADS holds PC_THREADS/GT teams that
// work independently (GT = 32: a warp per leaf for small leaves, synchronised with
// __syncwarp; GT = 128: the whole block).
template <int GT, int PC_TILE, int NP>
__global__ void __launch_bounds__(PC_THREADS) k_p2p_cta(const float4* __restrict__ body,
                                                         const uint32_t* __restrict__ leaf_ids, int64_t nleaf,
                                                         const uint2* __restrict__ runs,
                                                         const uint32_t* __restrict__ roff,
                                                         const uint32_t* __restrict__ rtot,
                                                         const uint32_t* __restrict__ bb, const uint32_t* __restrict__ bc,
                                                         float* __restrict__ near_phi, float* __restrict__ near_grad,
                                                         unsigned long long* __restrict__ counter) {
    constexpr int TEAMS = PC_THREADS / GT;
    __shared__ __align__(16) float4 s_tile_all[TEAMS][2][PC_TILE];
    __shared__ float4 s_red_all[TEAMS][GT * (2 * NP)];
    __shared__ unsigned long long s_leaf_all[TEAMS];
    __shared__ uint32_t s_self_all[TEAMS];
    const int team = threadIdx.x / GT, tid = threadIdx.x - team * GT;
    float4 (*s_tile)[PC_TILE] = s_tile_all[team];
    float4* s_red = s_red_all[team];
    unsigned long long& s_leaf = s_leaf_all[team];
    uint32_t& s_self = s_self_all[team];
    auto team_sync = [team] {
        if constexpr (GT == 32) __syncwarp();
        else if constexpr (GT == PC_THREADS) __syncthreads();
        else asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "r"(GT) : "memory");   // named barrier per team
    };
    for (;;) {
        team_sync();
        if (tid == 0) s_leaf = atomicAdd(counter, 1ull);
        team_sync();
        const unsigned long long li = s_leaf;
        if (li >= (unsigned long long)nleaf) break;
        const uint32_t a = leaf_ids[li];
        const uint32_t tb = bb[a], nt_all = bc[a];
        const uint32_t r0 = roff[a], r1 = roff[a + 1], ns = rtot[a];
        // flat offset of the target's own bodies in its source stream
        for (uint32_t r = r0 + tid; r < r1; r += GT) {
            const uint2 ru = runs[r];
            const uint32_t end = (r + 1 < r1) ? runs[r + 1].y : ns;
            if (ru.x <= tb && tb < ru.x + (end - ru.y)) s_self = ru.y + (tb - ru.x);
        }
        team_sync();
        const uint32_t selfF = s_self;
        for (uint32_t t0 = 0; t0 < nt_all; t0 += GT * (2 * NP)) {
            const uint32_t nt = min(nt_all - t0, (uint32_t)(GT * (2 * NP)));
            const int lpg = (int)((nt + (2 * NP) - 1) / (2 * NP));
            const int G = min(GT / lpg, 64);
            const int g = tid / lpg, j = tid - g * lpg;
            const bool active = g < G;
            const uint32_t CH = (uint32_t)(G * (PC_TILE / G));
            // target slot k of this thread is t = j + k*lpg; slots (2h, 2h+1) form pair h
            float2 nx[NP], ny[NP], nz[NP], f[NP], gx[NP], gy[NP], gz[NP];
#pragma unroll
            for (int h = 0; h < NP; ++h) {
                float px[2], py[2], pz[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const uint32_t t = (uint32_t)(j + (2 * h + e) * lpg);
                    const float4 p = body[tb + t0 + (t < nt ? t : 0)];
                    // unused slots sit far away so they never produce r^2 = 0
                    px[e] = t < nt ? -p.x : -1e30f; py[e] = -p.y; pz[e] = -p.z;
                }
                nx[h] = make_float2(px[0], px[1]); ny[h] = make_float2(py[0], py[1]);
                nz[h] = make_float2(pz[0], pz[1]);
                f[h] = gx[h] = gy[h] = gz[h] = make_float2(0.f, 0.f);
            }
            // loader cursors for flat indices tid, tid + GT, ... of every chunk
            constexpr int NH = PC_TILE / GT;
            uint32_t cur[NH];
#pragma unroll
            for (int h = 0; h < NH; ++h) cur[h] = r0;
            auto load_chunk = [&](uint32_t k, int buf) {
                const uint32_t f0 = k * CH;
                const uint32_t len = min(CH, ns - f0);
#pragma unroll
                for (int h = 0; h < NH; ++h) {
                    const uint32_t i = (uint32_t)tid + (uint32_t)h * GT;
                    if (i < len) {
                        const uint32_t fl = f0 + i;
                        while (cur[h] + 1 < r1 && runs[cur[h] + 1].y <= fl) ++cur[h];
                        const uint2 ru = runs[cur[h]];
                        cp_async16(&s_tile[buf][i], body + ru.x + (fl - ru.y));
                    }
                }
            };
            const uint32_t nch = (ns + CH - 1) / CH;
            if (nch > 0) load_chunk(0, 0);
            cp_async_commit();
            for (uint32_t k = 0; k < nch; ++k) {
                if (k + 1 < nch) load_chunk(k + 1, (k + 1) & 1);
                cp_async_commit();
                cp_async_wait_1();
                team_sync();
                const uint32_t f0 = k * CH;
                const uint32_t len = min(CH, ns - f0);
                if (active) {
                    const float4* tl = s_tile[k & 1];
                    const bool self = f0 < selfF + nt_all && selfF < f0 + len;
                    if (self) {
                        for (uint32_t i = g; i < len; i += G) p2p_body2<true, NP>(tl[i], nx, ny, nz, f, gx, gy, gz);
                    } else {
                        for (uint32_t i = g; i < len; i += G) p2p_body2<false, NP>(tl[i], nx, ny, nz, f, gx, gy, gz);
                    }
                }
                team_sync();
            }
            cp_async_wait_0();
#pragma unroll
            for (int h = 0; h < NP; ++h) {
                s_red[tid * (2 * NP) + 2 * h] = make_float4(f[h].x, gx[h].x, gy[h].x, gz[h].x);
                s_red[tid * (2 * NP) + 2 * h + 1] = make_float4(f[h].y, gx[h].y, gy[h].y, gz[h].y);
            }
            team_sync();
            if (g == 0) {
#pragma unroll
                for (int k = 0; k < (2 * NP); ++k) {
                    const uint32_t t = (uint32_t)(j + k * lpg);
                    if (t < nt) {
                        float4 acc = s_red[tid * (2 * NP) + k];
                        for (int gg = 1; gg < G; ++gg) {
                            const float4 v = s_red[(gg * lpg + j) * (2 * NP) + k];
                            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
                        }
                        const int64_t o = (int64_t)tb + t0 + t;
                        near_phi[o] = acc.x;
                        near_grad[3 * o] = acc.y;
                        near_grad[3 * o + 1] = acc.z;
                        near_grad[3 * o + 2] = acc.w;
                    }
                }
            }
            team_sync();
        }
    }
}

// ---------------------------------------------------------------- TMA bulk-copy variant
// Same work layout as k_p2p_cta<128, TILE, NP>, but the source chunks are staged with 1D bulk
// copies (cp.async.bulk, the TMA engine) of whole Morton runs issued by one thread, with
// mbarrier completion: consumers wait on the chunk's "full" barrier (transaction bytes), each
// warp arrives on the buffer's "empty" barrier when done, and the issuing thread waits on that
// before refilling -- no CTA-wide barrier per chunk (ncu: ~10% barrier stalls).
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(b);
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                     "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                 "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}

template <int PC_TILE, int NP, int NS = 2>
__global__ void __launch_bounds__(PC_THREADS) k_p2p_tma(const float4* __restrict__ body,
                                                         const uint32_t* __restrict__ leaf_ids, int64_t nleaf,
                                                         const uint2* __restrict__ runs,
                                                         const uint32_t* __restrict__ roff,
                                                         const uint32_t* __restrict__ rtot,
                                                         const uint32_t* __restrict__ bb, const uint32_t* __restrict__ bc,
                                                         float* __restrict__ near_phi, float* __restrict__ near_grad,
                                                         unsigned long long* __restrict__ counter) {
    constexpr int NW = PC_THREADS / 32;
    __shared__ __align__(128) float4 s_tile[NS][PC_TILE];
    __shared__ float4 s_red[PC_THREADS * (2 * NP)];
    __shared__ __align__(8) uint64_t full[NS], empty[NS];
    __shared__ unsigned long long s_leaf;
    __shared__ uint32_t s_self;
    // the leaf's source runs, loaded coalesced once per leaf: the issuing thread walks them from
    // shared memory instead of with dependent global loads (ncu: warp 0 -- the producer -- was the
    // straggler every other warp waited for at the chunk barriers)
    constexpr int RUN_CAP = 256;
    __shared__ uint2 s_runs[RUN_CAP];
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t kk = 0;   // chunks issued by this CTA so far (buffer kk % NS, use parity (kk / NS) & 1)
    for (;;) {
        __syncthreads();
        if (tid == 0) s_leaf = atomicAdd(counter, 1ull);
        __syncthreads();
        const unsigned long long li = s_leaf;
        if (li >= (unsigned long long)nleaf) break;
        const uint32_t a = leaf_ids[li];
        const uint32_t tb = bb[a], nt_all = bc[a];
        const uint32_t r0 = roff[a], r1 = roff[a + 1], ns = rtot[a];
        const bool runs_in_smem = r1 - r0 <= (uint32_t)RUN_CAP;
        for (uint32_t r = r0 + tid; r < r1; r += PC_THREADS) {
            const uint2 ru = runs[r];
            const uint32_t end = (r + 1 < r1) ? runs[r + 1].y : ns;
            if (ru.x <= tb && tb < ru.x + (end - ru.y)) s_self = ru.y + (tb - ru.x);
            if (runs_in_smem) s_runs[r - r0] = ru;
        }
        __syncthreads();
        const uint32_t selfF = s_self;
        const uint2* lruns = runs_in_smem ? s_runs - r0 : runs;   // indexed by the global run number
        for (uint32_t t0 = 0; t0 < nt_all; t0 += PC_THREADS * (2 * NP)) {
            const uint32_t nt = min(nt_all - t0, (uint32_t)(PC_THREADS * (2 * NP)));
            const int lpg = (int)((nt + (2 * NP) - 1) / (2 * NP));
            const int G = min(PC_THREADS / lpg, 64);
            const int g = tid / lpg, j = tid - g * lpg;
            const bool active = g < G;
            const uint32_t CH = (uint32_t)(G * (PC_TILE / G));
            float2 nx[NP], ny[NP], nz[NP], f[NP], gx[NP], gy[NP], gz[NP];
#pragma unroll
            for (int h = 0; h < NP; ++h) {
                float px[2], py[2], pz[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const uint32_t t = (uint32_t)(j + (2 * h + e) * lpg);
                    const float4 p = body[tb + t0 + (t < nt ? t : 0)];
                    px[e] = t < nt ? -p.x : -1e30f; py[e] = -p.y; pz[e] = -p.z;
                }
                nx[h] = make_float2(px[0], px[1]); ny[h] = make_float2(py[0], py[1]);
                nz[h] = make_float2(pz[0], pz[1]);
                f[h] = gx[h] = gy[h] = gz[h] = make_float2(0.f, 0.f);
            }
            const uint32_t nch = (ns + CH - 1) / CH;
            uint32_t cur = r0;   // thread 0's run cursor
            // thread 0 issues chunk c (global number kk0 + c) as bulk copies of its run pieces
            const uint32_t kk0 = kk;
            auto issue = [&](uint32_t c) {
                const uint32_t q = kk0 + c, buf = q % NS;
                if (q >= NS) mbar_wait(&empty[buf], (q / NS - 1) & 1);   // chunk q-NS consumed
                const uint32_t f0 = c * CH, len = min(CH, ns - f0);
                mbar_expect_tx(&full[buf], len * 16u);
                uint32_t fl = f0, dst = 0;
                while (dst < len) {
                    while (cur + 1 < r1 && lruns[cur + 1].y <= fl) ++cur;
                    const uint2 ru = lruns[cur];
                    const uint32_t end = (cur + 1 < r1) ? lruns[cur + 1].y : ns;
                    const uint32_t m = min(end - fl, len - dst);
                    bulk_g2s(&s_tile[buf][dst], body + ru.x + (fl - ru.y), m * 16u, &full[buf]);
                    fl += m;
                    dst += m;
                }
            };
            if (tid == 0)
                for (uint32_t c = 0; c + 1 < NS && c < nch; ++c) issue(c);
            for (uint32_t c = 0; c < nch; ++c) {
                const uint32_t q = kk0 + c, buf = q % NS;
                if (tid == 0 && c + NS - 1 < nch) issue(c + NS - 1);
                mbar_wait(&full[buf], (q / NS) & 1);
                const uint32_t f0 = c * CH;
                const uint32_t len = min(CH, ns - f0);
                if (active) {
                    const float4* tl = s_tile[buf];
                    const bool self = f0 < selfF + nt_all && selfF < f0 + len;
                    if (self) {
                        for (uint32_t i = g; i < len; i += G) p2p_body2<true, NP>(tl[i], nx, ny, nz, f, gx, gy, gz);
                    } else {
                        for (uint32_t i = g; i < len; i += G) p2p_body2<false, NP>(tl[i], nx, ny, nz, f, gx, gy, gz);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[buf]);
            }
            kk += nch;
#pragma unroll
            for (int h = 0; h < NP; ++h) {
                s_red[tid * (2 * NP) + 2 * h] = make_float4(f[h].x, gx[h].x, gy[h].x, gz[h].x);
                s_red[tid * (2 * NP) + 2 * h + 1] = make_float4(f[h].y, gx[h].y, gy[h].y, gz[h].y);
            }
            __syncthreads();
            if (g == 0) {
#pragma unroll
                for (int k = 0; k < (2 * NP); ++k) {
                    const uint32_t t = (uint32_t)(j + k * lpg);
                    if (t < nt) {
                        float4 acc = s_red[tid * (2 * NP) + k];
                        for (int gg = 1; gg < G; ++gg) {
                            const float4 v = s_red[(gg * lpg + j) * (2 * NP) + k];
                            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
                        }
                        const int64_t o = (int64_t)tb + t0 + t;
                        near_phi[o] = acc.x;
                        near_grad[3 * o] = acc.y;
                        near_grad[3 * o + 1] = acc.z;
                        near_grad[3 * o + 2] = acc.w;
                    }
                }
            }
            __syncthreads();
        }
    }
}

template <typename Body, typename Real>
fmm_status p2p_t(fmm_ctx* ctx, cudaStream_t s) {
    PhaseScope ps(ctx, PH_P2P, s);
    FMM_TRY(buf_ensure(ctx, ctx->near_phi, (size_t)ctx->n * sizeof(Real)));
    FMM_TRY(buf_ensure(ctx, ctx->near_grad, (size_t)ctx->n * 3 * sizeof(Real)));
    PhaseScope pk(ctx, PH_P2P_KERNEL, s);
    if (std::is_same<Real, float>::value && ctx->mut_ready) return p2p_mutual(ctx, s);
    if (std::is_same<Real, float>::value && ctx->use_fast_p2p && ctx->p2p_variant == 0) {
        // three leaf classes (k_leaf_split): tiny (<= P2P_TINY_LEAF) a warp per leaf, mid a CTA with
        // 2 target pairs per thread, big (>= P2P_BIG_LEAF) a CTA with 4 (measured: mean-8 leaves
        // 1.9x faster per warp than per CTA; c2's ~32-body leaves best at 2 pairs, sphere's ~234 at 4)
        FMM_TRY(buf_ensure(ctx, ctx->cnt_tmp2, 64));
        unsigned long long* counter = P_<unsigned long long>(ctx->cnt_tmp2);
        FMM_CUDA_TRY(ctx, cudaMemsetAsync(counter, 0, 24, s));
        const uint2* runs = P_<uint2>(ctx->runs);
        const uint32_t* rtot = P_<uint32_t>(ctx->run_off) + ctx->ncell + 2;
        const uint32_t* lists = P_<uint32_t>(ctx->leaf_cls);
        auto launch = [&](auto kern, const uint32_t* ids, int64_t cnt, unsigned long long* ctr) -> fmm_status {
            if (cnt == 0) return FMM_OK;
            int nb = 0;
            FMM_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, PC_THREADS, 0));
            const int64_t g = std::min<int64_t>((int64_t)ctx->num_sms * std::max(nb, 1), (cnt + 3) / 4 * 4);
            kern<<<(unsigned)g, PC_THREADS, 0, s>>>(P_<float4>(ctx->body), ids, cnt, runs, P_<uint32_t>(ctx->run_off),
                                                   rtot, P_<uint32_t>(ctx->c_bb), P_<uint32_t>(ctx->c_bc),
                                                   (float*)ctx->near_phi.p, (float*)ctx->near_grad.p, ctr);
            FMM_LAUNCH(ctx);
            return FMM_OK;
        };
        FMM_TRY(launch(k_p2p_cta<32, 64, 1>, lists, ctx->n_leaf_cls[0], counter));
        // mid leaves: TMA bulk-copy staging (measured 3% faster at c2/c3) of 512-body chunks
        // (1.5% faster than 256, 1024 and 3 stages slower); big leaves: cp.async (bulk copies,
        // also of 512-body chunks, measured 3-5% slower for the sphere's ~234-body leaves)
        FMM_TRY(launch(k_p2p_tma<512, 2>, lists + ctx->nleaf, ctx->n_leaf_cls[1], counter + 1));
        FMM_TRY(launch(k_p2p_cta<128, 256, 4>, lists + 2 * ctx->nleaf, ctx->n_leaf_cls[2], counter + 2));
        FMM_CUDA_TRY(ctx, cudaGetLastError());
        return FMM_OK;
    }
    if (std::is_same<Real, float>::value && ctx->use_fast_p2p) {
        FMM_TRY(buf_ensure(ctx, ctx->cnt_tmp2, 64));
        unsigned long long* counter = P_<unsigned long long>(ctx->cnt_tmp2);
        FMM_CUDA_TRY(ctx, cudaMemsetAsync(counter, 0, 8, s));
        int nb = 0;
        FMM_CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_p2p_f32, PF_WARPS * 32, 0));
        k_p2p_f32<<<ctx->num_sms * std::max(nb, 1), PF_WARPS * 32, 0, s>>>(
            P_<float4>(ctx->body), P_<uint32_t>(ctx->leaf_ids), ctx->nleaf, P_<uint32_t>(ctx->p2p_src),
            P_<uint64_t>(ctx->p2p_off), P_<uint32_t>(ctx->c_bb), P_<uint32_t>(ctx->c_bc), (float*)ctx->near_phi.p,
            (float*)ctx->near_grad.p, counter);
        FMM_LAUNCH(ctx);
        FMM_CUDA_TRY(ctx, cudaGetLastError());
        return FMM_OK;
    }
    int g = (int)std::min<int64_t>((ctx->nleaf + PP_WARPS - 1) / PP_WARPS, (int64_t)ctx->num_sms * 16);
    k_p2p_generic<Body, Real><<<std::max(g, 1), PP_WARPS * 32, 0, s>>>(
        P_<Body>(ctx->body), P_<uint32_t>(ctx->leaf_ids), ctx->nleaf, P_<uint32_t>(ctx->p2p_src),
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
