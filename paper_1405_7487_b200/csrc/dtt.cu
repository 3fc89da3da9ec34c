// dtt.cu -- dual tree traversal producing explicit M2L and P2P lists (a8).
//
// PAPER.md:151 §II-C: "the M2L and P2P kernels are processed ... by using the dual tree
// traversal [Dehnen]"; north_star asks for the traversal to emit explicit lists.
// R8 MAC: accept (A <- B) iff (R_A + R_B) < theta * sqrt((dx*dx + dy*dy) + dz*dz) over
//         the tight-box centres; fp64 with _rn intrinsics so it is bit-exact with the oracle.
// R9 from (root, root): MAC -> M2L; both leaves -> P2P; else split A if B is a leaf or
//         (A internal and R_A >= R_B), else split B.  The rule is a pure function of the
//         pair, so this breadth-first frontier emits the same SETS as the oracle's recursion.
// R10 canonical order: ascending (target, source) -- radix sort of the packed u64
//         (target << 32 | source); CSR offsets per target cell by binary search.
// Each frontier step: a count kernel (3 warp-aggregated counters), one host read to size
// the buffers, then an emit kernel appending with warp-aggregated atomics.
#include "common.cuh"

namespace {

struct CellView {
    const double4* __restrict__ cr;
    const uint32_t* __restrict__ cb;
    const uint32_t* __restrict__ cc;
};

// outcome: 0 = M2L, 1 = P2P, 2 = split A, 3 = split B; nchild = children emitted
__device__ __forceinline__ int classify(const CellView& v, uint32_t a, uint32_t b, double theta, uint32_t& nchild) {
    double4 A = v.cr[a], B = v.cr[b];
    double dx = __dsub_rn(A.x, B.x), dy = __dsub_rn(A.y, B.y), dz = __dsub_rn(A.z, B.z);
    double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    nchild = 0;
    if (__dadd_rn(A.w, B.w) < __dmul_rn(theta, __dsqrt_rn(d2))) return 0;
    uint32_t ca = v.cc[a], cbn = v.cc[b];
    if (ca == 0 && cbn == 0) return 1;
    if (cbn == 0 || (ca != 0 && A.w >= B.w)) { nchild = ca; return 2; }
    nchild = cbn;
    return 3;
}

__device__ __forceinline__ unsigned long long warp_append(unsigned long long* counter, uint32_t cnt) {
    // exclusive warp scan of cnt, one atomic per warp; returns this lane's base
    const int lane = threadIdx.x & 31;
    uint32_t x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    uint32_t total = __shfl_sync(0xffffffffu, x, 31);
    unsigned long long base = 0;
    if (lane == 31 && total) base = atomicAdd(counter, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 31);
    return base + (x - cnt);
}

__global__ void k_dtt_count(const uint64_t* __restrict__ fr, int64_t nf, CellView v, double theta,
                            unsigned long long* __restrict__ cnt /* [3]: m2l, p2p, next */) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    unsigned long long m = 0, p = 0, c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += stride) {
        uint64_t pr = fr[i];
        uint32_t nch;
        int o = classify(v, (uint32_t)(pr >> 32), (uint32_t)pr, theta, nch);
        m += (o == 0);
        p += (o == 1);
        c += nch;
    }
#pragma unroll
    for (int s = 16; s; s >>= 1) {
        m += __shfl_xor_sync(0xffffffffu, m, s);
        p += __shfl_xor_sync(0xffffffffu, p, s);
        c += __shfl_xor_sync(0xffffffffu, c, s);
    }
    if ((threadIdx.x & 31) == 0) {
        if (m) atomicAdd(&cnt[0], m);
        if (p) atomicAdd(&cnt[1], p);
        if (c) atomicAdd(&cnt[2], c);
    }
}

__global__ void k_dtt_emit(const uint64_t* __restrict__ fr, int64_t nf, CellView v, double theta,
                           unsigned long long* __restrict__ cnt, uint64_t* __restrict__ m2l, uint64_t* __restrict__ p2p,
                           uint64_t* __restrict__ next) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // grid-stride with warp-uniform trip count so every lane joins the shuffles
    int64_t nfr = (nf + 31) / 32 * 32;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nfr; i += stride) {
        bool ok = i < nf;
        uint32_t a = 0, b = 0, nch = 0;
        int o = -1;
        if (ok) {
            uint64_t pr = fr[i];
            a = (uint32_t)(pr >> 32);
            b = (uint32_t)pr;
            o = classify(v, a, b, theta, nch);
        }
        unsigned long long pm = warp_append(&cnt[0], o == 0);
        unsigned long long pp = warp_append(&cnt[1], o == 1);
        unsigned long long pc = warp_append(&cnt[2], nch);
        const uint64_t packed = ((uint64_t)a << 32) | b;
        if (o == 0) m2l[pm] = packed;
        else if (o == 1) p2p[pp] = packed;
        else if (o == 2) {
            uint32_t k0 = v.cb[a];
            for (uint32_t k = 0; k < nch; ++k) next[pc + k] = ((uint64_t)(k0 + k) << 32) | b;
        } else if (o == 3) {
            uint32_t k0 = v.cb[b];
            for (uint32_t k = 0; k < nch; ++k) next[pc + k] = ((uint64_t)a << 32) | (k0 + k);
        }
    }
}

__global__ void k_init_frontier(uint64_t* fr) { fr[0] = 0; }

// CSR offsets: off[c] = first list index with target >= c (sorted packed keys)
__global__ void k_csr(const uint64_t* __restrict__ lst, int64_t n, int64_t ncell, uint64_t* __restrict__ off) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c > ncell) return;
    int64_t lo = 0, hi = n;
    const uint64_t key = (uint64_t)c << 32;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (lst[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    off[c] = (uint64_t)lo;
}

__global__ void k_p2p_inter(const uint64_t* __restrict__ lst, int64_t n, const uint32_t* __restrict__ bc,
                            unsigned long long* out) {
    unsigned long long s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t pr = lst[i];
        s += (unsigned long long)bc[pr >> 32] * bc[(uint32_t)pr];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

fmm_status sort_and_index(fmm_ctx* ctx, DevBuf& lst, int64_t n, DevBuf& off, cudaStream_t s) {
    FMM_TRY(buf_ensure(ctx, ctx->lst_tmp, (size_t)std::max<int64_t>(n, 1) * 8));
    FMM_TRY(buf_ensure(ctx, off, (size_t)(ctx->ncell + 1) * 8));
    int nb = 0;
    while (((int64_t)1 << nb) < ctx->ncell) ++nb;
    uint64_t* sorted = nullptr;
    FMM_TRY(radix_sort_keys(ctx, P_<uint64_t>(lst), P_<uint64_t>(ctx->lst_tmp), n, 0, 32 + nb, &sorted, s));
    if (sorted != P_<uint64_t>(lst)) std::swap(lst, ctx->lst_tmp);
    k_csr<<<(unsigned)((ctx->ncell + 1 + 255) / 256), 256, 0, s>>>(P_<uint64_t>(lst), n, ctx->ncell,
                                                                   P_<uint64_t>(off));
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}

__global__ void k_widen(const uint32_t* __restrict__ in, int64_t n, uint64_t* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[i];
}

// ---- P2P source runs: consecutive list entries of one target whose body ranges are
// contiguous (Morton-adjacent leaves) merge into one run {start body, flat offset in the
// target's source stream}; rtot[t] = total sources of target t.  Used by the P2P kernel to
// stream a target's sources as full fixed-size chunks.
__global__ void k_run_flags(const uint64_t* __restrict__ lst, int64_t n, const uint32_t* __restrict__ bb,
                            const uint32_t* __restrict__ bc, uint32_t* __restrict__ flag) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t cur = lst[i];
    uint32_t f = 1;
    if (i > 0) {
        const uint64_t prv = lst[i - 1];
        const uint32_t sp = (uint32_t)prv, sc = (uint32_t)cur;
        f = ((prv >> 32) != (cur >> 32)) || (bb[sp] + bc[sp] != bb[sc]);
    }
    flag[i] = f;
}

__global__ void k_run_emit(const uint64_t* __restrict__ lst, int64_t n, const uint32_t* __restrict__ bb,
                           const uint32_t* __restrict__ bc, const uint32_t* __restrict__ flag,
                           const uint32_t* __restrict__ rid, uint32_t* __restrict__ rstart, uint32_t* __restrict__ rlen,
                           uint32_t* __restrict__ rtarget) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t cur = lst[i];
    const uint32_t sc = (uint32_t)cur, r = rid[i] + flag[i] - 1;   // run containing entry i
    if (flag[i]) {
        rstart[r] = bb[sc];
        rtarget[r] = (uint32_t)(cur >> 32);
    }
    if (i + 1 == n || flag[i + 1]) rlen[r] = bb[sc] + bc[sc];   // end body; converted to length below
}

__global__ void k_run_len(int64_t nr, const uint32_t* __restrict__ rstart, uint32_t* __restrict__ rlen) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < nr) rlen[r] -= rstart[r];
}

// per target: roff (first run), then each run's flat offset within its target and the total
__global__ void k_run_csr(const uint32_t* __restrict__ rtarget, int64_t nr, int64_t ncell, uint32_t* __restrict__ roff) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c > ncell) return;
    int64_t lo = 0, hi = nr;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (rtarget[mid] < (uint32_t)c) lo = mid + 1;
        else hi = mid;
    }
    roff[c] = (uint32_t)lo;
}

__global__ void k_run_flat(int64_t nr, int64_t ncell, const uint32_t* __restrict__ rtarget,
                           const uint32_t* __restrict__ roff, const uint32_t* __restrict__ rstart,
                           const uint64_t* __restrict__ gpre, const uint32_t* __restrict__ rlen,
                           uint2* __restrict__ runs, uint32_t* __restrict__ rtot) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < nr) {
        const uint32_t t = rtarget[r];
        runs[r] = make_uint2(rstart[r], (uint32_t)(gpre[r] - gpre[roff[t]]));
    }
    if (r < ncell) {
        const uint32_t a = roff[r], b = roff[r + 1];
        rtot[r] = (a == b) ? 0u : (uint32_t)(gpre[b - 1] + rlen[b - 1] - gpre[a]);
    }
}

fmm_status build_runs(fmm_ctx* ctx, cudaStream_t s) {
    const int64_t n = ctx->n_p2p, nc = ctx->ncell;
    FMM_TRY(buf_ensure(ctx, ctx->run_tmp, (size_t)std::max<int64_t>(n, 1) * 4 * 5 + 64));
    uint32_t* flag = P_<uint32_t>(ctx->run_tmp);
    uint32_t* rid = flag + n;
    uint32_t* rstart = rid + n;
    uint32_t* rlen = rstart + n;
    uint32_t* rtarget = rlen + n;
    FMM_TRY(buf_ensure(ctx, ctx->dcount2, 64));
    uint32_t* d_nr = P_<uint32_t>(ctx->dcount2);
    const unsigned g = (unsigned)((n + 255) / 256);
    k_run_flags<<<g, 256, 0, s>>>(P_<uint64_t>(ctx->lst_p2p), n, P_<uint32_t>(ctx->c_bb), P_<uint32_t>(ctx->c_bc), flag);
    FMM_LAUNCH(ctx);
    FMM_TRY(scan_exclusive_u32(ctx, flag, rid, n, d_nr, s));
    k_run_emit<<<g, 256, 0, s>>>(P_<uint64_t>(ctx->lst_p2p), n, P_<uint32_t>(ctx->c_bb), P_<uint32_t>(ctx->c_bc),
                                 flag, rid, rstart, rlen, rtarget);
    FMM_LAUNCH(ctx);
    uint32_t nr = 0;
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&nr, d_nr, 4, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    ctx->n_runs = nr;
    k_run_len<<<(unsigned)((nr + 255) / 256), 256, 0, s>>>(nr, rstart, rlen);
    FMM_LAUNCH(ctx);
    FMM_TRY(buf_ensure(ctx, ctx->run_off, (size_t)(nc + 2) * 4));
    FMM_TRY(buf_ensure(ctx, ctx->runs, (size_t)std::max<int64_t>(nr, 1) * 8 + (size_t)(nc + 1) * 4 + 64));
    FMM_TRY(buf_ensure(ctx, ctx->run_pre, (size_t)std::max<int64_t>(nr, 1) * 8));
    k_run_csr<<<(unsigned)((nc + 1 + 255) / 256), 256, 0, s>>>(rtarget, nr, nc, P_<uint32_t>(ctx->run_off));
    FMM_LAUNCH(ctx);
    // 64-bit exclusive scan of the run lengths (widen on the fly)
    FMM_TRY(buf_ensure(ctx, ctx->run_len64, (size_t)std::max<int64_t>(nr, 1) * 8));
    k_widen<<<(unsigned)((nr + 255) / 256), 256, 0, s>>>(rlen, nr, P_<uint64_t>(ctx->run_len64));
    FMM_LAUNCH(ctx);
    FMM_TRY(scan_exclusive_u64(ctx, P_<uint64_t>(ctx->run_len64), P_<uint64_t>(ctx->run_pre), nr, nullptr, s));
    uint2* runs = P_<uint2>(ctx->runs);
    uint32_t* rtot = reinterpret_cast<uint32_t*>(runs + std::max<int64_t>(nr, 1));
    k_run_flat<<<(unsigned)((std::max<int64_t>(nr, nc) + 255) / 256), 256, 0, s>>>(
        nr, nc, rtarget, P_<uint32_t>(ctx->run_off), rstart, P_<uint64_t>(ctx->run_pre), rlen, runs, rtot);
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}

}  // namespace

fmm_status build_lists(fmm_ctx* ctx, cudaStream_t s) {
    CellView v{P_<double4>(ctx->c_cr), P_<uint32_t>(ctx->c_cb), P_<uint32_t>(ctx->c_cc)};
    int64_t n_m2l = 0, n_p2p = 0;
    {
        PhaseScope ps(ctx, PH_DTT, s);
        FMM_TRY(buf_ensure(ctx, ctx->fr_a, 1024 * 8));
        FMM_TRY(buf_ensure(ctx, ctx->dcount, 64));
        if (ctx->lst_m2l.bytes == 0) FMM_TRY(buf_ensure(ctx, ctx->lst_m2l, (size_t)ctx->ncell * 256 * 8));
        if (ctx->lst_p2p.bytes == 0) FMM_TRY(buf_ensure(ctx, ctx->lst_p2p, (size_t)ctx->nleaf * 32 * 8));
        unsigned long long* d_cnt = P_<unsigned long long>(ctx->dcount);   // [0..2] step counts, [4..6] emit cursors
        k_init_frontier<<<1, 1, 0, s>>>(P_<uint64_t>(ctx->fr_a));
        FMM_LAUNCH(ctx);
        int64_t nf = 1;
        FMM_CUDA_TRY(ctx, cudaMemsetAsync(d_cnt + 4, 0, 3 * 8, s));
        while (nf > 0) {
            FMM_CUDA_TRY(ctx, cudaMemsetAsync(d_cnt, 0, 3 * 8, s));
            int g = (int)std::min<int64_t>((nf + 255) / 256, (int64_t)ctx->num_sms * 16);
            k_dtt_count<<<g, 256, 0, s>>>(P_<uint64_t>(ctx->fr_a), nf, v, ctx->theta, d_cnt);
            FMM_LAUNCH(ctx);
            unsigned long long h[3];
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync(h, d_cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
            FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
            size_t need_m = (size_t)(n_m2l + h[0]) * 8, need_p = (size_t)(n_p2p + h[1]) * 8;
            if (need_m > ctx->lst_m2l.bytes) FMM_TRY(buf_ensure(ctx, ctx->lst_m2l, need_m + need_m / 2, true, s));
            if (need_p > ctx->lst_p2p.bytes) FMM_TRY(buf_ensure(ctx, ctx->lst_p2p, need_p + need_p / 2, true, s));
            FMM_TRY(buf_ensure(ctx, ctx->fr_b, (size_t)std::max<unsigned long long>(h[2], 1) * 8));
            // the next-frontier cursor restarts at 0 each step
            FMM_CUDA_TRY(ctx, cudaMemsetAsync(d_cnt + 6, 0, 8, s));
            k_dtt_emit<<<g, 256, 0, s>>>(P_<uint64_t>(ctx->fr_a), nf, v, ctx->theta, d_cnt + 4,
                                         P_<uint64_t>(ctx->lst_m2l), P_<uint64_t>(ctx->lst_p2p),
                                         P_<uint64_t>(ctx->fr_b));
            FMM_LAUNCH(ctx);
            FMM_CUDA_TRY(ctx, cudaGetLastError());
            n_m2l += h[0];
            n_p2p += h[1];
            nf = (int64_t)h[2];
            std::swap(ctx->fr_a, ctx->fr_b);
        }
    }
    ctx->n_m2l = n_m2l;
    ctx->n_p2p = n_p2p;
    PhaseScope ps(ctx, PH_LISTS, s);
    FMM_TRY(sort_and_index(ctx, ctx->lst_m2l, n_m2l, ctx->m2l_off, s));
    FMM_TRY(sort_and_index(ctx, ctx->lst_p2p, n_p2p, ctx->p2p_off, s));
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(P_<unsigned long long>(ctx->dcount) + 7, 0, 8, s));
    k_p2p_inter<<<ctx->num_sms * 4, 256, 0, s>>>(P_<uint64_t>(ctx->lst_p2p), n_p2p, P_<uint32_t>(ctx->c_bc),
                                                  P_<unsigned long long>(ctx->dcount) + 7);
    FMM_LAUNCH(ctx);
    unsigned long long inter = 0;
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&inter, P_<unsigned long long>(ctx->dcount) + 7, 8, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    ctx->p2p_inter = (int64_t)inter;
    return build_runs(ctx, s);
}
