// let.cu -- local essential tree (LET) export and graft for the multi-GPU path.
//
// PAPER.md:122 §II-C: "the LET is constructed by sending the necessary parts of the local
// tree to the other processes"; the received parts are grafted onto the local
// tree and traversed; §II-B: the MAC decides what a remote process needs.
// The rule is sender-initiated and conservative:
//   receiver j publishes a cover of <= 73 entries of its local tree:
//     summary: every cell at level 2 and every leaf at levels 0-1, with Rleafmax = the
//              largest leaf radius in its subtree (a leaf: its own R);
//     guard:   every internal cell at levels 0-1, with its own R.
//   sender i marks cell C "opened for j" iff
//     some summary b: theta * dist(c_C, box_b) <= R_C + max(R_C, Rleafmax_b), or
//     some guard T:   R_T <= R_C and theta * dist(c_C, box_T) <= R_T + R_C
//   (both with a 1e-9 relative margin, so fp64 rounding can only over-open), closes the set
//   upwards (an opened cell's ancestors are opened), and exports the root plus every child of
//   an opened cell.  Opened leaves ship their bodies.  Every exported cell keeps its original
//   child and body counts, so R9's "is B a leaf" reads exactly as in the sender's tree; a cell
//   whose children were not exported carries child_begin = FMM_LET_ABSENT, and the traversal
//   raises FMM_ERR_STATE if it ever needs them (it cannot when the cover argument holds).
// Structure (geometry, counts, body positions) is exchanged at build time; multipoles and
// body charges (data) after the upward pass.
#include <cstring>

#include "common.cuh"

namespace {

struct __align__(16) LetCell {
    double4 cr;         // centre, radius (fp64, bit-exact copies)
    int32_t e;          // sender's scale exponent E - level (M2L operand scaling)
    uint32_t cb;        // first child inside this LET, or FMM_LET_ABSENT
    uint32_t cc;        // original child count (0: leaf)
    uint32_t bb;        // first body inside this LET's body block, or FMM_LET_ABSENT
    uint32_t bc;        // original body count
    uint32_t orig;      // cell index in the sender's tree
    uint32_t pad[2];
};
static_assert(sizeof(LetCell) == 64, "LetCell is 64 B");

struct LetHeader {
    int64_t ncell, nbody, ncoef, prec, magic, depth, pad[2];   // depth: sender's deepest level
};
static_assert(sizeof(LetHeader) == 64, "LetHeader is 64 B");
constexpr int64_t LET_MAGIC = 0x4c45543031ll;   // "LET01"

size_t let_body_size(int prec) { return prec == FMM_F32 ? sizeof(float4) : sizeof(dbody); }
// bytes per shipped multipole coefficient: fp32 contexts ship the fp32 operand precision the M2L
// reads (R19), scaled by the cell's power-of-two rho^-|beta| (exact, keeps the fp32 range);
// fp64 contexts ship fp64
size_t let_m_size(int prec) { return prec == FMM_F32 ? 4 : 8; }
// data message: header | M [ncell][ncoef] fp64 | q [nbody]; each part padded to 16 B
size_t let_round16(size_t b) { return (b + 15) / 16 * 16; }

__device__ __forceinline__ unsigned long long dbits(double x) { return (unsigned long long)__double_as_longlong(x); }

// Rleafmax of every level-2 cell: each leaf at level >= 2 raises its level-2 ancestor
// (radii are >= 0, so the IEEE bit patterns order like the values)
__global__ void k_rleafmax(int64_t nc, const uint32_t* __restrict__ cc, const int32_t* __restrict__ level,
                           const int32_t* __restrict__ parent, const double4* __restrict__ cr, int64_t l2b,
                           unsigned long long* __restrict__ rl) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc || cc[c] != 0 || level[c] < 2) return;
    int64_t a = c;
    while (level[a] > 2) a = parent[a];
    atomicMax(&rl[a - l2b], dbits(cr[c].w));
}

__device__ __forceinline__ double dist_box(const double4 c, const double* e) {
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double x = d == 0 ? c.x : (d == 1 ? c.y : c.z);
        const double lo = e[2 + d], hi = e[5 + d];
        const double t = x < lo ? lo - x : (x > hi ? x - hi : 0.0);
        s += t * t;
    }
    return sqrt(s);
}

// cover entry: [kind (0 summary, 1 guard), R, lo xyz, hi xyz]
__global__ void k_let_mark(int64_t nc, const double4* __restrict__ cr, const double* __restrict__ cover, int ncover,
                           double theta, uint32_t* __restrict__ opened) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const double4 C = cr[c];
    const double slack = 1.0 + 1e-9;
    uint32_t o = 0;
    for (int k = 0; k < ncover && !o; ++k) {
        const double* e = cover + 8 * k;
        const double Rb = e[1];
        const double td = theta * dist_box(C, e);
        if (e[0] == 0.0) o = td <= (C.w + fmax(C.w, Rb)) * slack;
        else o = Rb <= C.w * slack && td <= (Rb + C.w) * slack;
    }
    opened[c] = o;
}

__global__ void k_let_close(int64_t nc, const int32_t* __restrict__ parent, uint32_t* __restrict__ opened) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc || !opened[c]) return;
    for (int32_t a = parent[c]; a >= 0 && !opened[a]; a = parent[a]) opened[a] = 1;   // idempotent writes
}

// exported: root, or a child of an opened cell; body count shipped: opened leaves
__global__ void k_let_flags(int64_t nc, const int32_t* __restrict__ parent, const uint32_t* __restrict__ cc,
                            const uint32_t* __restrict__ bc, const uint32_t* __restrict__ opened,
                            uint32_t* __restrict__ eflag, uint32_t* __restrict__ bflag) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const uint32_t ex = c == 0 || opened[parent[c]];
    eflag[c] = ex;
    bflag[c] = (ex && opened[c] && cc[c] == 0) ? bc[c] : 0u;
}

__global__ void k_let_pack_cells(int64_t nc, const double4* __restrict__ cr, const int32_t* __restrict__ level,
                                 const uint32_t* __restrict__ cb, const uint32_t* __restrict__ cc,
                                 const uint32_t* __restrict__ bc, const uint32_t* __restrict__ opened,
                                 const uint32_t* __restrict__ eflag, const uint32_t* __restrict__ eidx,
                                 const uint32_t* __restrict__ bflag, const uint32_t* __restrict__ boff,
                                 const double* __restrict__ root, LetCell* __restrict__ out) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc || !eflag[c]) return;
    int E;
    frexp(2.0 * root[10], &E);
    LetCell r;
    r.cr = cr[c];
    r.e = E - level[c];
    r.cc = cc[c];
    r.cb = (opened[c] && cc[c] > 0) ? eidx[cb[c]] : FMM_LET_ABSENT;
    r.bc = bc[c];
    r.bb = bflag[c] ? boff[c] : FMM_LET_ABSENT;
    r.orig = (uint32_t)c;
    r.pad[0] = r.pad[1] = 0;
    out[eidx[c]] = r;
}

template <typename Body>
__global__ void k_let_pack_bodies(int64_t nc, const Body* __restrict__ body, const uint32_t* __restrict__ bb,
                                  const uint32_t* __restrict__ bflag, const uint32_t* __restrict__ boff,
                                  Body* __restrict__ out, bool with_q) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = w; c < nc; c += nw) {
        const uint32_t m = bflag[c];
        if (!m) continue;
        const uint32_t s0 = bb[c], d0 = boff[c];
        for (uint32_t i = lane; i < m; i += 32) {
            Body b = body[s0 + i];
            if (!with_q) b.w = 0;
            out[d0 + i] = b;
        }
    }
}

template <typename Real, typename Body>
__global__ void k_let_pack_q(int64_t nc, const Body* __restrict__ body, const uint32_t* __restrict__ bb,
                             const uint32_t* __restrict__ bflag, const uint32_t* __restrict__ boff,
                             Real* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = w; c < nc; c += nw) {
        const uint32_t m = bflag[c];
        if (!m) continue;
        const uint32_t s0 = bb[c], d0 = boff[c];
        for (uint32_t i = lane; i < m; i += 32) out[d0 + i] = body[s0 + i].w;
    }
}

__global__ void k_let_pack_M(int64_t nc, int ncoef, const uint32_t* __restrict__ eflag,
                             const uint32_t* __restrict__ eidx, const double* __restrict__ M, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = w; c < nc; c += nw) {
        if (!eflag[c]) continue;
        const double* src = M + (size_t)c * ncoef;
        double* dst = out + (size_t)eidx[c] * ncoef;
        for (int k = lane; k < ncoef; k += 32) dst[k] = src[k];
    }
}

__device__ __forceinline__ int coef_degree(int k) {
    int n = 0;
    while (ncoef_of(n + 1) <= k) ++n;
    return n;
}

// fp32 mode: M_beta / rho^|beta| as float, rho = 2^(E - level) of the sender's cell
__global__ void k_let_pack_M32(int64_t nc, int ncoef, const uint32_t* __restrict__ eflag,
                               const uint32_t* __restrict__ eidx, const int32_t* __restrict__ level,
                               const double* __restrict__ root, const double* __restrict__ M, float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int E;
    frexp(2.0 * root[10], &E);
    for (int64_t c = w; c < nc; c += nw) {
        if (!eflag[c]) continue;
        const int e = E - level[c];
        const double* src = M + (size_t)c * ncoef;
        float* dst = out + (size_t)eidx[c] * ncoef;
        for (int k = lane; k < ncoef; k += 32) dst[k] = (float)ldexp(src[k], -e * coef_degree(k));
    }
}

// receiver: the grafted cell's level' = E_local - e_sender (k_let_graft_cells) gives back e exactly
__global__ void k_let_unpack_M32(int64_t m, int ncoef, const float* __restrict__ in, const int32_t* __restrict__ level,
                                 const double* __restrict__ root, double* __restrict__ M) {
    int E;
    frexp(2.0 * root[10], &E);
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m * ncoef; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = t / ncoef;
        const int k = (int)(t - c * ncoef);
        M[t] = ldexp((double)in[t], (E - level[c]) * coef_degree(k));
    }
}

// graft one peer's cells at [base, base + m): indices rebased, scale exponent re-expressed as
// a level of this tree (E_local - e) so the M2L operand preparation reproduces it exactly
__global__ void k_let_graft_cells(int64_t m, const LetCell* __restrict__ in, int64_t base, int64_t bbase,
                                  const double* __restrict__ root, double4* __restrict__ cr, int32_t* __restrict__ level,
                                  uint32_t* __restrict__ cb, uint32_t* __restrict__ cc, uint32_t* __restrict__ bb,
                                  uint32_t* __restrict__ bc, int32_t* __restrict__ parent, uint64_t* __restrict__ key,
                                  uint32_t* __restrict__ orig) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    int E;
    frexp(2.0 * root[10], &E);
    const LetCell c = in[r];
    const int64_t i = base + r;
    cr[i] = c.cr;
    level[i] = E - c.e;
    cb[i] = c.cb == FMM_LET_ABSENT ? FMM_LET_ABSENT : (uint32_t)(base + c.cb);
    cc[i] = c.cc;
    bb[i] = c.bb == FMM_LET_ABSENT ? FMM_LET_ABSENT : (uint32_t)(bbase + c.bb);
    bc[i] = c.bc;
    parent[i] = -1;
    key[i] = 0;
    orig[i] = c.orig;
}

template <typename Body>
__global__ void k_let_graft_bodies(int64_t m, const Body* __restrict__ in, Body* __restrict__ body) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) body[i] = in[i];
}

template <typename Real, typename Body>
__global__ void k_let_unpack_q(int64_t m, const Real* __restrict__ q, Body* __restrict__ body) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) body[i].w = q[i];
}

unsigned blocks_for(int64_t n, int t) { return (unsigned)std::max<int64_t>((n + t - 1) / t, 1); }

}  // namespace

// ---------------------------------------------------------------- internal entry points
fmm_status let_cover(fmm_ctx* ctx, double* cover, int* ncover, cudaStream_t s) {
    *ncover = 0;
    const int64_t nc = ctx->ncell;
    if (nc == 0) return FMM_OK;
    const int64_t l2b = ctx->level_begin.size() > 3 ? ctx->level_begin[2] : nc;
    const int64_t l2e = ctx->level_begin.size() > 3 ? ctx->level_begin[3] : nc;
    const int64_t nshallow = std::min<int64_t>(l2e, FMM_LET_MAX_COVER);
    FMM_TRY(buf_ensure(ctx, ctx->let_tmp, (size_t)(l2e - l2b + 1) * 8));
    unsigned long long* rl = P_<unsigned long long>(ctx->let_tmp);
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(rl, 0, (size_t)(l2e - l2b + 1) * 8, s));
    if (l2e > l2b) {
        k_rleafmax<<<blocks_for(nc, 256), 256, 0, s>>>(nc, P_<uint32_t>(ctx->c_cc), P_<int32_t>(ctx->c_level),
                                                      P_<int32_t>(ctx->c_parent), P_<double4>(ctx->c_cr), l2b, rl);
        FMM_LAUNCH(ctx);
    }
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    std::vector<uint32_t> cc(nshallow);
    std::vector<int32_t> lev(nshallow);
    std::vector<double> lo(3 * nshallow), hi(3 * nshallow), cr(4 * nshallow);
    std::vector<unsigned long long> rlh(std::max<int64_t>(l2e - l2b, 1));
    FMM_CUDA_TRY(ctx, cudaMemcpy(cc.data(), ctx->c_cc.p, nshallow * 4, cudaMemcpyDeviceToHost));
    FMM_CUDA_TRY(ctx, cudaMemcpy(lev.data(), ctx->c_level.p, nshallow * 4, cudaMemcpyDeviceToHost));
    FMM_CUDA_TRY(ctx, cudaMemcpy(lo.data(), ctx->c_bmin.p, nshallow * 24, cudaMemcpyDeviceToHost));
    FMM_CUDA_TRY(ctx, cudaMemcpy(hi.data(), ctx->c_bmax.p, nshallow * 24, cudaMemcpyDeviceToHost));
    FMM_CUDA_TRY(ctx, cudaMemcpy(cr.data(), ctx->c_cr.p, nshallow * 32, cudaMemcpyDeviceToHost));
    if (l2e > l2b) FMM_CUDA_TRY(ctx, cudaMemcpy(rlh.data(), rl, (l2e - l2b) * 8, cudaMemcpyDeviceToHost));
    int k = 0;
    for (int64_t c = 0; c < nshallow; ++c) {
        double* e = cover + 8 * k;
        double R = cr[4 * c + 3];
        if (lev[c] == 2) {
            e[0] = 0.0;
            const unsigned long long b = cc[c] == 0 ? 0ull : rlh[c - l2b];
            double rm;
            memcpy(&rm, &b, 8);
            e[1] = cc[c] == 0 ? R : rm;
        } else if (lev[c] < 2) {
            e[0] = cc[c] == 0 ? 0.0 : 1.0;
            e[1] = R;
        } else {
            continue;
        }
        for (int d = 0; d < 3; ++d) {
            e[2 + d] = lo[3 * c + d];
            e[5 + d] = hi[3 * c + d];
        }
        ++k;
    }
    *ncover = k;
    return FMM_OK;
}

fmm_status let_plan(fmm_ctx* ctx, int peer, const double* cover, int ncover, int64_t* sbytes, int64_t* dbytes,
                    cudaStream_t s) {
    const int64_t nc = ctx->ncell;
    if ((int)ctx->let_peers.size() <= peer) ctx->let_peers.resize(peer + 1);
    LetPeer& lp = ctx->let_peers[peer];
    FMM_TRY(buf_ensure(ctx, lp.opened, (size_t)(nc + 1) * 4));
    FMM_TRY(buf_ensure(ctx, lp.eflag, (size_t)(nc + 1) * 4));
    FMM_TRY(buf_ensure(ctx, lp.eidx, (size_t)(nc + 1) * 4));
    FMM_TRY(buf_ensure(ctx, lp.bflag, (size_t)(nc + 1) * 4));
    FMM_TRY(buf_ensure(ctx, lp.boff, (size_t)(nc + 1) * 4));
    FMM_TRY(buf_ensure(ctx, ctx->let_cov, FMM_LET_MAX_COVER * 8 * 8));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->let_cov.p, cover, (size_t)ncover * 64, cudaMemcpyHostToDevice, s));
    uint32_t* opened = P_<uint32_t>(lp.opened);
    k_let_mark<<<blocks_for(nc, 256), 256, 0, s>>>(nc, P_<double4>(ctx->c_cr), P_<double>(ctx->let_cov), ncover,
                                                  ctx->theta, opened);
    k_let_close<<<blocks_for(nc, 256), 256, 0, s>>>(nc, P_<int32_t>(ctx->c_parent), opened);
    k_let_flags<<<blocks_for(nc, 256), 256, 0, s>>>(nc, P_<int32_t>(ctx->c_parent), P_<uint32_t>(ctx->c_cc),
                                                   P_<uint32_t>(ctx->c_bc), opened, P_<uint32_t>(lp.eflag),
                                                   P_<uint32_t>(lp.bflag));
    ctx->launches += 3;
    uint32_t* tot = P_<uint32_t>(lp.eidx) + nc;
    uint32_t* btot = P_<uint32_t>(lp.boff) + nc;
    FMM_TRY(scan_exclusive_u32(ctx, P_<uint32_t>(lp.eflag), P_<uint32_t>(lp.eidx), nc, tot, s));
    FMM_TRY(scan_exclusive_u32(ctx, P_<uint32_t>(lp.bflag), P_<uint32_t>(lp.boff), nc, btot, s));
    uint32_t h[2];
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&h[0], tot, 4, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&h[1], btot, 4, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    lp.ncell = h[0];
    lp.nbody = h[1];
    lp.planned = true;
    const size_t bs = let_body_size(ctx->prec), rs = ctx->prec == FMM_F32 ? 4 : 8;
    *sbytes = (int64_t)(sizeof(LetHeader) + (size_t)lp.ncell * sizeof(LetCell) + (size_t)lp.nbody * bs);
    *dbytes = (int64_t)(sizeof(LetHeader) + let_round16((size_t)lp.ncell * ctx->ncoef * let_m_size(ctx->prec)) +
                        let_round16((size_t)lp.nbody * rs));
    return FMM_OK;
}

fmm_status let_pack(fmm_ctx* ctx, int peer, int part, void* dst, cudaStream_t s) {
    if (peer < 0 || peer >= (int)ctx->let_peers.size() || !ctx->let_peers[peer].planned) {
        ctx->err = "fmm_let_pack: peer not planned";
        return FMM_ERR_STATE;
    }
    LetPeer& lp = ctx->let_peers[peer];
    const int64_t nc = ctx->ncell;
    LetHeader h{};
    h.ncell = lp.ncell;
    h.nbody = lp.nbody;
    h.ncoef = ctx->ncoef;
    h.prec = ctx->prec;
    h.magic = LET_MAGIC + part;
    h.depth = ctx->depth;
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(dst, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    char* p = (char*)dst + sizeof(LetHeader);
    const unsigned gw = (unsigned)std::min<int64_t>((nc + 7) / 8, (int64_t)ctx->num_sms * 16);
    if (part == 0) {
        k_let_pack_cells<<<blocks_for(nc, 256), 256, 0, s>>>(
            nc, P_<double4>(ctx->c_cr), P_<int32_t>(ctx->c_level), P_<uint32_t>(ctx->c_cb), P_<uint32_t>(ctx->c_cc),
            P_<uint32_t>(ctx->c_bc), P_<uint32_t>(lp.opened), P_<uint32_t>(lp.eflag), P_<uint32_t>(lp.eidx),
            P_<uint32_t>(lp.bflag), P_<uint32_t>(lp.boff), P_<double>(ctx->root), (LetCell*)p);
        p += (size_t)lp.ncell * sizeof(LetCell);
        if (ctx->prec == FMM_F32)
            k_let_pack_bodies<float4><<<gw, 256, 0, s>>>(nc, P_<float4>(ctx->body), P_<uint32_t>(ctx->c_bb),
                                                        P_<uint32_t>(lp.bflag), P_<uint32_t>(lp.boff), (float4*)p, false);
        else
            k_let_pack_bodies<dbody><<<gw, 256, 0, s>>>(nc, P_<dbody>(ctx->body), P_<uint32_t>(ctx->c_bb),
                                                       P_<uint32_t>(lp.bflag), P_<uint32_t>(lp.boff), (dbody*)p, false);
    } else {
        if (!ctx->upward_done) {
            ctx->err = "fmm_let_pack_data: run fmm_upward first";
            return FMM_ERR_STATE;
        }
        if (ctx->prec == FMM_F32)
            k_let_pack_M32<<<gw, 256, 0, s>>>(nc, ctx->ncoef, P_<uint32_t>(lp.eflag), P_<uint32_t>(lp.eidx),
                                              P_<int32_t>(ctx->c_level), P_<double>(ctx->root), P_<double>(ctx->M),
                                              (float*)p);
        else
            k_let_pack_M<<<gw, 256, 0, s>>>(nc, ctx->ncoef, P_<uint32_t>(lp.eflag), P_<uint32_t>(lp.eidx),
                                            P_<double>(ctx->M), (double*)p);
        p += let_round16((size_t)lp.ncell * ctx->ncoef * let_m_size(ctx->prec));
        if (ctx->prec == FMM_F32)
            k_let_pack_q<float, float4><<<gw, 256, 0, s>>>(nc, P_<float4>(ctx->body), P_<uint32_t>(ctx->c_bb),
                                                          P_<uint32_t>(lp.bflag), P_<uint32_t>(lp.boff), (float*)p);
        else
            k_let_pack_q<double, dbody><<<gw, 256, 0, s>>>(nc, P_<dbody>(ctx->body), P_<uint32_t>(ctx->c_bb),
                                                          P_<uint32_t>(lp.bflag), P_<uint32_t>(lp.boff), (double*)p);
    }
    ctx->launches += 2;
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}

fmm_status let_graft(fmm_ctx* ctx, int npeers, const void* const* src, const int64_t* bytes, cudaStream_t s) {
    const int64_t nc = ctx->ncell, n = ctx->n;
    std::vector<LetHeader> hs(npeers);
    int64_t add_c = 0, add_b = 0;
    for (int k = 0; k < npeers; ++k) {
        if (!src[k] || bytes[k] < (int64_t)sizeof(LetHeader)) {
            ctx->err = "fmm_let_graft: short buffer";
            return FMM_ERR_ARG;
        }
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&hs[k], src[k], sizeof(LetHeader), cudaMemcpyDeviceToHost, s));
    }
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    const size_t bs = let_body_size(ctx->prec);
    for (int k = 0; k < npeers; ++k) {
        const LetHeader& h = hs[k];
        if (h.magic != LET_MAGIC || h.ncoef != ctx->ncoef || h.prec != ctx->prec ||
            bytes[k] < (int64_t)(sizeof(LetHeader) + h.ncell * sizeof(LetCell) + h.nbody * bs)) {
            ctx->err = "fmm_let_graft: LET structure does not match this context";
            return FMM_ERR_ARG;
        }
        add_c += h.ncell;
        add_b += h.nbody;
    }
    // grafts append after the LETs already grafted in this build (one fragment at a time)
    const int64_t ctot = nc + ctx->nrem + add_c, btot = n + ctx->nrem_body + add_b;
    if (ctot >= (int64_t)FMM_LET_ABSENT || btot >= (int64_t)FMM_LET_ABSENT) {
        ctx->err = "fmm_let_graft: more than 2^32-1 cells or bodies";
        return FMM_ERR_ARG;
    }
    // grow the cell arrays the traversal and the M2L/P2P kernels read, keeping the local part
    DevBuf* u32s[] = {&ctx->c_cb, &ctx->c_cc, &ctx->c_bb, &ctx->c_bc};
    for (DevBuf* b : u32s) FMM_TRY(buf_ensure(ctx, *b, (size_t)ctot * 4, true, s));
    FMM_TRY(buf_ensure(ctx, ctx->c_level, (size_t)ctot * 4, true, s));
    FMM_TRY(buf_ensure(ctx, ctx->c_parent, (size_t)ctot * 4, true, s));
    FMM_TRY(buf_ensure(ctx, ctx->c_key, (size_t)ctot * 8, true, s));
    FMM_TRY(buf_ensure(ctx, ctx->c_cr, (size_t)ctot * 32, true, s));
    FMM_TRY(buf_ensure(ctx, ctx->c_orig, (size_t)std::max<int64_t>(ctot, 1) * 4, true, s));
    FMM_TRY(buf_ensure(ctx, ctx->body, (size_t)btot * bs, true, s));
    int64_t cbase = nc + ctx->nrem, bbase = n + ctx->nrem_body;
    for (int k = 0; k < npeers; ++k) {
        const LetHeader& h = hs[k];
        const char* p = (const char*)src[k] + sizeof(LetHeader);
        if (h.ncell > 0) {
            k_let_graft_cells<<<blocks_for(h.ncell, 256), 256, 0, s>>>(
                h.ncell, (const LetCell*)p, cbase, bbase, P_<double>(ctx->root), P_<double4>(ctx->c_cr),
                P_<int32_t>(ctx->c_level), P_<uint32_t>(ctx->c_cb), P_<uint32_t>(ctx->c_cc), P_<uint32_t>(ctx->c_bb),
                P_<uint32_t>(ctx->c_bc), P_<int32_t>(ctx->c_parent), P_<uint64_t>(ctx->c_key),
                P_<uint32_t>(ctx->c_orig));
            FMM_LAUNCH(ctx);
        }
        p += (size_t)h.ncell * sizeof(LetCell);
        if (h.nbody > 0) {
            if (ctx->prec == FMM_F32)
                k_let_graft_bodies<float4><<<blocks_for(h.nbody, 256), 256, 0, s>>>(
                    h.nbody, (const float4*)p, P_<float4>(ctx->body) + bbase);
            else
                k_let_graft_bodies<dbody><<<blocks_for(h.nbody, 256), 256, 0, s>>>(
                    h.nbody, (const dbody*)p, P_<dbody>(ctx->body) + bbase);
            FMM_LAUNCH(ctx);
        }
        ctx->let_remote.push_back({cbase, h.ncell, bbase, h.nbody, (int)h.depth});
        cbase += h.ncell;
        bbase += h.nbody;
    }
    ctx->nrem += add_c;
    ctx->nrem_body += add_b;
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}

fmm_status let_unpack(fmm_ctx* ctx, int first, int npeers, const void* const* src, const int64_t* bytes,
                      cudaStream_t s) {
    if (first < 0 || first + npeers > (int)ctx->let_remote.size()) {
        ctx->err = "fmm_let_unpack: more data messages than grafted LETs";
        return FMM_ERR_STATE;
    }
    const int64_t ctot = ctx->ncell + ctx->nrem;
    FMM_TRY(buf_ensure(ctx, ctx->M, (size_t)ctot * ctx->ncoef * 8, true, s));
    for (int k = 0; k < npeers; ++k) {
        const LetRemote& r = ctx->let_remote[first + k];
        const size_t need = sizeof(LetHeader) + let_round16((size_t)r.ncell * ctx->ncoef * let_m_size(ctx->prec)) +
                            (size_t)r.nbody * (ctx->prec == FMM_F32 ? 4 : 8);
        if (!src[k] || bytes[k] < (int64_t)need) {
            ctx->err = "fmm_let_unpack: short buffer";
            return FMM_ERR_ARG;
        }
        const char* p = (const char*)src[k] + sizeof(LetHeader);
        if (r.ncell && ctx->prec == FMM_F32) {
            k_let_unpack_M32<<<blocks_for(r.ncell * ctx->ncoef, 256), 256, 0, s>>>(
                r.ncell, ctx->ncoef, (const float*)p, P_<int32_t>(ctx->c_level) + r.base, P_<double>(ctx->root),
                P_<double>(ctx->M) + (size_t)r.base * ctx->ncoef);
            FMM_LAUNCH(ctx);
        } else if (r.ncell)
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync(P_<double>(ctx->M) + (size_t)r.base * ctx->ncoef, p,
                                              (size_t)r.ncell * ctx->ncoef * 8, cudaMemcpyDeviceToDevice, s));
        p += let_round16((size_t)r.ncell * ctx->ncoef * let_m_size(ctx->prec));
        if (r.nbody) {
            if (ctx->prec == FMM_F32)
                k_let_unpack_q<float, float4><<<blocks_for(r.nbody, 256), 256, 0, s>>>(
                    r.nbody, (const float*)p, P_<float4>(ctx->body) + r.bbase);
            else
                k_let_unpack_q<double, dbody><<<blocks_for(r.nbody, 256), 256, 0, s>>>(
                    r.nbody, (const double*)p, P_<dbody>(ctx->body) + r.bbase);
            FMM_LAUNCH(ctx);
        }
    }
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}

// ---------------------------------------------------------------- Eq. (1) work weights
// PAPER.md:108-115 Eq. (1): w_i = l_i + alpha * r_i, l_i / r_i the local / remote interaction
// list sizes of particle i.  Here a list entry is weighted by its work:
//   P2P: every source body of i's leaf counts 1 (one interaction);
//   M2L: every pair (C <- B) of i's leaf or any ancestor C counts c_m2l / |C| (the pair's work,
//        in P2P-interaction units, shared by the |C| particles below C);
// local: sources of this rank's tree, remote: sources in grafted LETs (index >= ncell).
namespace {
__global__ void k_work_cells(int64_t nc, const uint64_t* __restrict__ off, const uint32_t* __restrict__ src,
                             const uint32_t* __restrict__ bc, double c_m2l, double2* __restrict__ share) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const uint64_t p0 = off[c], p1 = off[c + 1];
    uint64_t nl = 0;
    for (uint64_t p = p0; p < p1; ++p) nl += src[p] < (uint32_t)nc;
    const double inv = bc[c] ? c_m2l / (double)bc[c] : 0.0;
    share[c] = make_double2(inv * (double)nl, inv * (double)(p1 - p0 - nl));
}

template <typename Real>
__global__ void k_work_leaves(int64_t nc, const uint32_t* __restrict__ leaf_ids, int64_t nleaf,
                              const uint64_t* __restrict__ poff, const uint32_t* __restrict__ psrc,
                              const uint32_t* __restrict__ bb, const uint32_t* __restrict__ bc,
                              const int32_t* __restrict__ parent, const double2* __restrict__ share,
                              const uint32_t* __restrict__ perm, float alpha, float* __restrict__ w,
                              double* __restrict__ sums) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double sl = 0.0, sr = 0.0;
    for (int64_t li = w0; li < nleaf; li += nw) {
        const uint32_t a = leaf_ids[li];
        double pl = 0.0, pr = 0.0;
        for (uint64_t p = poff[a] + lane; p < poff[a + 1]; p += 32) {
            const uint32_t b = psrc[p];
            if (b < (uint32_t)nc) pl += bc[b];
            else pr += bc[b];
        }
        for (int o = 16; o; o >>= 1) {
            pl += __shfl_xor_sync(0xffffffffu, pl, o);
            pr += __shfl_xor_sync(0xffffffffu, pr, o);
        }
        double ml = 0.0, mr = 0.0;
        for (int32_t c = (int32_t)a; c >= 0; c = parent[c]) {
            const double2 s = share[c];
            ml += s.x;
            mr += s.y;
        }
        const double l = pl + ml, r = pr + mr;
        const uint32_t b0 = bb[a], m = bc[a];
        for (uint32_t k = lane; k < m; k += 32) w[perm[b0 + k]] = (float)(l + (double)alpha * r);
        if (lane == 0) {
            sl += l * m;
            sr += r * m;
        }
    }
    if (lane == 0 && (sl != 0.0 || sr != 0.0)) {
        atomicAdd(&sums[0], sl);
        atomicAdd(&sums[1], sr);
    }
}
}  // namespace

extern "C" fmm_status fmm_work(fmm_ctx* ctx, double c_m2l, float alpha, float* w, double* lr_sums, void* stream) {
    if (!ctx || c_m2l < 0 || (ctx->n > 0 && !w)) return FMM_ERR_ARG;
    if (!ctx->built) {
        ctx->err = "fmm_work: needs the lists of a build";
        return FMM_ERR_STATE;
    }
    if (lr_sums) lr_sums[0] = lr_sums[1] = 0.0;
    if (ctx->n == 0) return FMM_OK;
    DeviceGuard guard(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nc = ctx->ncell;
    FMM_TRY(buf_ensure(ctx, ctx->let_tmp, (size_t)nc * 16 + 64));
    double2* share = P_<double2>(ctx->let_tmp);
    double* sums = reinterpret_cast<double*>(share + nc);
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(sums, 0, 16, s));
    k_work_cells<<<blocks_for(nc, 256), 256, 0, s>>>(nc, P_<uint64_t>(ctx->m2l_off), P_<uint32_t>(ctx->m2l_src),
                                                     P_<uint32_t>(ctx->c_bc), c_m2l, share);
    const unsigned g = (unsigned)std::min<int64_t>((ctx->nleaf + 3) / 4, (int64_t)ctx->num_sms * 16);
    k_work_leaves<float><<<std::max(g, 1u), 128, 0, s>>>(nc, P_<uint32_t>(ctx->leaf_ids), ctx->nleaf,
                                                        P_<uint64_t>(ctx->p2p_off), P_<uint32_t>(ctx->p2p_src),
                                                        P_<uint32_t>(ctx->c_bb), P_<uint32_t>(ctx->c_bc),
                                                        P_<int32_t>(ctx->c_parent), share, ctx->d_perm, alpha, w, sums);
    ctx->launches += 2;
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    if (lr_sums) {
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(lr_sums, sums, 16, cudaMemcpyDeviceToHost, s));
        FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    }
    return FMM_OK;
}
