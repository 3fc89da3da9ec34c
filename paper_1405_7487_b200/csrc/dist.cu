// dist.cu -- the multi-GPU step behind the C-ABI (SURVEY.md §8(b) fmm_create_dist /
// fmm_set_weights, §8(e), §8(f) f1/f3/f4): the library owns the communicator (NCCL, or an
// in-process group of threads), the partition arithmetic (Morton splitter refinement, ORB
// multisection, Eq. (1) alpha tuning) and the sequencing of every exchange; the Python layer only
// marshals arguments.
//
// One step (fmm_dist_solve), §II-B/C:
//   1. global bounds (all-reduce of exact fp64 min/max); keys under the global root cube (R2-R4);
//   2. Morton ranges weighted by Eq. (1) (w = l + alpha r, 1 at the first
//      step): histogram refinement of the splitters ("each bit of the key is examined
//      at each step"), or ORB multisection;
//   3. particles exchanged by grouped send/recv; WHILE they fly, the particles that stay on this
//      rank are sorted on a side stream (f1: the partition communication overlapped with the
//      keys/sort of the local tree, "asynchronously execute the FMM kernels while the
//      communication for partitioning is happening"); the arrivals are sorted after landing and
//      merged, giving exactly the order a full sort would (key, then local index);
//   4. local tree on the global root cube (DESIGN.md §2 reading 9); P2M/M2M on the aux stream;
//   5. covers all-gathered; each rank plans and packs for every peer the part of its tree the peer
//      can need; the LET STRUCTURE goes out in K-1 ring rounds on the comm stream BEFORE the local
//      traversal, which overlaps them ("completely overlapped with the Traverse");
//      the multipole/charge DATA follows on the comm stream as soon as the upward pass is done,
//      overlapping the remote traversals; every fragment is grafted and traversed as it lands
//      (the per-message `when`);
//   6. lists, unpack, M2L/P2P/L2L/L2P; Eq. (1) weights of this step (fmm_work);
//   7. phi, grad and the weights back to the particles' owners, in the caller's order.
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>

#include "comm.cuh"

namespace {

// ------------------------------------------------------------------ host logic (testable on CPU)
// bin where the inclusive cumulative weight first reaches t, and the weight still needed in it
void choose_bin(const double* hist, int nbins, double t, int64_t* bin, double* resid) {
    double c = 0.0, before = 0.0;
    int b = nbins - 1;
    for (int i = 0; i < nbins; ++i) {
        before = c;
        c += hist[i];
        if (c >= t) {
            b = i;
            break;
        }
        if (i == nbins - 1) before = c - hist[i];
    }
    *bin = b;
    *resid = t - before;
}

// Morton-range splitters: splitter j (1 <= j < K) refined `bits` key bits per round
// down to the bin where the cumulative weight crosses j/K of the total, until that bin holds
// <= tol * total / K or the key is exhausted; rank j takes the keys >= splitter j.
template <typename HistFn>
fmm_status splitters_refine(int K, int bits, double tol, HistFn hist, uint64_t* out) {
    if (K <= 1) return FMM_OK;
    const int nb0 = 1 << bits;
    std::vector<double> h0(nb0);
    uint64_t zero = 0;
    FMM_TRY(hist(&zero, 1, 0, bits, h0.data()));
    double total = 0.0;
    for (double v : h0) total += v;
    if (!(total > 0.0)) {
        for (int j = 0; j < K - 1; ++j) out[j] = 0;
        return FMM_OK;
    }
    std::vector<uint64_t> prefix(K - 1);
    std::vector<double> resid(K - 1), weight(K - 1);
    for (int j = 0; j < K - 1; ++j) {
        int64_t b;
        choose_bin(h0.data(), nb0, total * (j + 1) / K, &b, &resid[j]);
        prefix[j] = (uint64_t)b;
        weight[j] = h0[b];
    }
    int pbits = bits;
    auto heavy = [&] {
        for (double w : weight)
            if (w > tol * total / K) return true;
        return false;
    };
    std::vector<double> hs;
    while (pbits < 63 && heavy()) {
        const int nb = std::min(bits, 63 - pbits);
        hs.assign((size_t)(K - 1) << nb, 0.0);
        FMM_TRY(hist(prefix.data(), K - 1, pbits, nb, hs.data()));
        for (int j = 0; j < K - 1; ++j) {
            int64_t b;
            double r;
            choose_bin(hs.data() + ((size_t)j << nb), 1 << nb, resid[j], &b, &r);
            prefix[j] = (prefix[j] << nb) | (uint64_t)b;
            resid[j] = r;
            weight[j] = hs[((size_t)j << nb) + b];
        }
        pbits += nb;
    }
    uint64_t run = 0;
    for (int j = 0; j < K - 1; ++j) {
        const uint64_t v = prefix[j] << (63 - pbits);
        run = j == 0 ? v : std::max(run, v);
        out[j] = run;
    }
    return FMM_OK;
}

// ORB multisection for any rank count: group ids are the first
// rank of the group's range, so after the last round a particle's group is its rank.  Each round,
// every group of Kg > 1 ranks is cut along the longest axis of its box (quantised coordinates,
// ties to the lower axis) where the weight fraction reaches floor(Kg/2)/Kg: the cut coordinate is
// refined `bits` then the remaining 21 - bits bits; coordinates >= cut take the right half's id.
constexpr int COORD_BITS = 21;
template <typename HistFn, typename SplitFn>
fmm_status orb_plan_t(int K, int bits, HistFn hist, SplitFn split, int32_t* boxes /*[K][6]*/) {
    struct G { int r0, r1; int32_t lo[3], hi[3]; };
    const int32_t full = 1 << COORD_BITS;
    std::vector<G> grp(K);
    std::vector<bool> live(K, false);
    grp[0] = {0, K, {0, 0, 0}, {full, full, full}};
    live[0] = true;
    auto pending = [&] {
        for (int g = 0; g < K; ++g)
            if (live[g] && grp[g].r1 - grp[g].r0 > 1) return true;
        return false;
    };
    const int nb2 = COORD_BITS - bits;
    std::vector<double> h((size_t)K << bits), h2((size_t)K << nb2);
    while (pending()) {
        std::vector<int32_t> axis(K, -1), right(K, 0);
        std::vector<uint32_t> prefix(K, 0), cut(K, 0);
        std::vector<double> frac(K, 0.0), total(K, 0.0), resid(K, 0.0);
        for (int g = 0; g < K; ++g) {
            if (!live[g] || grp[g].r1 - grp[g].r0 <= 1) continue;
            int a = 0;
            for (int d = 1; d < 3; ++d)
                if (grp[g].hi[d] - grp[g].lo[d] > grp[g].hi[a] - grp[g].lo[a]) a = d;
            axis[g] = a;
            frac[g] = (double)((grp[g].r1 - grp[g].r0) / 2) / (grp[g].r1 - grp[g].r0);
        }
        FMM_TRY(hist(axis.data(), prefix.data(), 0, bits, h.data()));
        for (int g = 0; g < K; ++g) {
            if (axis[g] < 0) continue;
            const double* hg = h.data() + ((size_t)g << bits);
            for (int i = 0; i < (1 << bits); ++i) total[g] += hg[i];
            resid[g] = total[g] * frac[g];
            if (total[g] > 0) {
                int64_t b;
                double r;
                choose_bin(hg, 1 << bits, resid[g], &b, &r);
                prefix[g] = (uint32_t)b;
                resid[g] = r;
            }
        }
        FMM_TRY(hist(axis.data(), prefix.data(), bits, nb2, h2.data()));
        std::vector<G> add;
        for (int g = 0; g < K; ++g) {
            if (axis[g] < 0) continue;
            const int a = axis[g];
            int64_t c;
            if (total[g] > 0) {
                int64_t b2;
                double r;
                choose_bin(h2.data() + ((size_t)g << nb2), 1 << nb2, resid[g], &b2, &r);
                c = ((int64_t)prefix[g] << nb2) | b2;
            } else {
                c = ((int64_t)grp[g].lo[a] + grp[g].hi[a]) / 2;
            }
            c = std::min<int64_t>(std::max<int64_t>(c, grp[g].lo[a]), grp[g].hi[a]);
            const int kl = (grp[g].r1 - grp[g].r0) / 2, rid = grp[g].r0 + kl;
            cut[g] = (uint32_t)c;
            right[g] = rid;
            G r = grp[g];
            r.r0 = rid;
            r.lo[a] = (int32_t)c;
            grp[g].r1 = rid;
            grp[g].hi[a] = (int32_t)c;
            add.push_back(r);
        }
        FMM_TRY(split(axis.data(), cut.data(), right.data()));
        for (const G& r : add) {
            grp[r.r0] = r;
            live[r.r0] = true;
        }
    }
    for (int g = 0; g < K; ++g)
        for (int d = 0; d < 3; ++d) {
            boxes[6 * g + d] = grp[g].lo[d];
            boxes[6 * g + 3 + d] = grp[g].hi[d];
        }
    return FMM_OK;
}

}  // namespace

// alpha of Eq. (1), "a constant that is optimized over the time steps to minimize the total
// runtime" (the paper names no method).  Reading: golden-section search
// on log(alpha) over [lo, hi], one measured step runtime per probe, until the bracket is narrower
// than tol; a probe is set for two consecutive steps and scored by the second (the first step
// partitioned with it); after convergence alpha stays at the fastest probe.
struct fmm_alpha_tuner {
    double a, b, tol, c, d;
    double fc = NAN, fd = NAN;
    double probe;
    int age = 0;
    std::vector<std::pair<double, double>> history;
    static constexpr double GR = 0.6180339887498949;
    bool converged() const { return b - a < tol; }
    double best() const {
        if (history.empty()) return std::exp(probe);
        auto it = std::min_element(history.begin(), history.end(),
                                   [](const auto& x, const auto& y) { return x.second < y.second; });
        return it->first;
    }
    double next() const { return converged() ? best() : std::exp(probe); }
    void report(double t) {
        if (converged()) return;
        if (++age < 2) return;
        history.push_back({std::exp(probe), t});
        if (probe == c) fc = t;
        else fd = t;
        if (std::isnan(fc)) probe = c;
        else if (std::isnan(fd)) probe = d;
        else if (fc < fd) {   // minimum in [a, d]
            b = d;
            d = c;
            fd = fc;
            c = b - GR * (b - a);
            fc = NAN;
            probe = c;
        } else {              // minimum in [c, b]
            a = c;
            c = d;
            fc = fd;
            d = a + GR * (b - a);
            fd = NAN;
            probe = d;
        }
        age = 0;
    }
};

struct fmm_group {
    LocalGroup g;
};

// ------------------------------------------------------------------------------- the driver
enum { TL_PARTITION, TL_EXCHANGE, TL_STAY_SORT, TL_TREE, TL_UPWARD, TL_COVER, TL_STRUCT_XCHG, TL_LOCAL_DTT,
       TL_DATA_XCHG, TL_REMOTE_DTT, TL_LISTS, TL_INTERACT, TL_BACK, TL_INTERACT_LOCAL, TL_INTERACT_REMOTE, TL_COUNT };
static const char* kTlNames[TL_COUNT] = {"partition", "particle_exchange", "stay_sort", "tree", "upward",
                                         "cover_plan", "let_struct_exchange", "local_dtt", "let_data_exchange",
                                         "remote_dtt", "lists", "interact", "results_back", "interact_local",
                                         "interact_remote"};

struct DistState {
    Transport* tr = nullptr;
    int K = 1, rank = 0, partitioner = FMM_PART_MORTON;
    double alpha = 1.0, c_m2l = 0.0;
    fmm_alpha_tuner* tuner = nullptr;
    bool overlap_sort = true;   // f1: staying particles sorted while the particles fly (FMM_DIST_SORT=0: off)
    // FMM_DIST_SPLIT=1: local M2L/P2P started on the compute stream right after the local traversal,
    // while the LET fragments are grafted and traversed; the remote lists' interactions added after.
    // Off by default: the persistent M2L/P2P kernels hold every SM until they finish, so the remote
    // traversal's kernels queue behind them -- the split reorders the work without overlapping it
    // (profiles/r02_dist_timeline_1gpu_split.jsonl)
    bool split = false;
    cudaStream_t cx = nullptr;
    int64_t nct_cap = 0;
    // remote-only CSR lists, their P2P source runs, and the second outputs of the remote pass
    DevBuf r_moff, r_msrc, r_poff, r_psrc, r_runs, r_run_off, r_run_tmp, r_leaf_cls, Lr2, L2, near2_phi, near2_grad,
        inter_loc, span_tmp;
    int64_t r_nm = 0, r_np = 0, r_nruns = 0, r_ncls[3] = {0, 0, 0};
    cudaStream_t cs = nullptr, side = nullptr;
    cudaEvent_t ev[12] = {};
    std::vector<cudaEvent_t> ev_round;
    // timeline (ctx->timing): start/end events per span, relative to ev_t0
    cudaEvent_t ev_t0 = nullptr;
    cudaEvent_t tl[TL_COUNT][2] = {};
    bool tl_rec[TL_COUNT] = {};
    double tl_ms[TL_COUNT][2] = {};
    // buffers
    DevBuf keys, pk_pos, pk_q, pk_gid, l_pos, l_q, l_gid, hist, red, cov, let_send, let_recv, back_send,
        back_recv, w_prev, w_set, w_loc, phi_loc, grad_loc, group, sk, si, ak, ai, stage;
    int64_t w_prev_n = -1, w_set_n = -1, n_local = 0;
    bool stay_in_b = false;   // the staying run's sort ended in its second (ping-pong) half
    double gb[6] = {0, 0, 0, 0, 0, 0};
    std::vector<int32_t> boxes;
    std::vector<int> peers;
    fmm_dist_stats st{};
    ~DistState() {
        delete tr;
        delete tuner;
        if (cs) cudaStreamDestroy(cs);
        if (side) cudaStreamDestroy(side);
        if (cx) cudaStreamDestroy(cx);
        DevBuf* rb[] = {&r_moff, &r_msrc, &r_poff, &r_psrc, &r_runs, &r_run_off, &r_run_tmp, &r_leaf_cls, &Lr2, &L2,
                        &near2_phi, &near2_grad, &inter_loc, &span_tmp};
        for (DevBuf* x : rb) buf_free(*x);
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
        for (auto e : ev_round) cudaEventDestroy(e);
        if (ev_t0) cudaEventDestroy(ev_t0);
        for (auto& p : tl)
            for (auto e : p)
                if (e) cudaEventDestroy(e);
        DevBuf* b[] = {&keys, &pk_pos, &pk_q, &pk_gid, &l_pos, &l_q, &l_gid, &hist, &red, &cov, &let_send, &let_recv,
                       &back_send, &back_recv, &w_prev, &w_set, &w_loc, &phi_loc, &grad_loc, &group, &sk, &si,
                       &ak, &ai, &stage};
        for (DevBuf* x : b) buf_free(*x);
    }
};

void dist_destroy(DistState* d) { delete d; }

namespace {

// M2L cost in P2P interactions (FP32 lane-op model of the harmonic kernel; paper_1405_7487_b200/
// costs.py m2l_flops_per_pair "instr" / 13): the c_m2l of Eq. (1)'s l and r
double m2l_cost_ratio(int P) {
    auto t2n = [](int p) { return p * (p + 1) / 2; };
    long fma = 0, rec = 0;
    for (int m = 0; m < P; ++m) fma += (long)(m + 1) * (t2n(P - m) + t2n(P - 1 - m));
    for (int m = 0; m < P - 1; ++m) fma += (long)(m + 1) * t2n(P - 1 - m);
    for (int m = 2; m < P; ++m) fma += (long)(m + 1) * t2n(P - m);
    for (int n = 1; n < P; ++n) {
        for (int z = 0; z <= n; ++z) {
            const int y = n - z;
            rec += (y > 0) + (z > 0) + (y > 1) + (z > 1) + (n > 1 ? 2 : 1);
        }
        for (int z = 0; z < n; ++z) {
            const int y = n - 1 - z;
            rec += 1 + (y > 0) + (z > 0) + (y > 1) + (z > 1) + (n > 1 ? 2 : 1);
        }
    }
    rec += 2 * (P - 1) + 3 * P + 6;
    return (double)(fma + rec) / 13.0;
}

unsigned grid1(int64_t n) { return (unsigned)std::min<int64_t>(std::max<int64_t>((n + 255) / 256, 1), 148 * 16); }

template <typename Real>
__global__ void k_pack_back(int64_t n, const Real* __restrict__ phi, const Real* __restrict__ grad,
                            const float* __restrict__ w, Real* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        out[5 * i] = phi[i];
        out[5 * i + 1] = grad[3 * i];
        out[5 * i + 2] = grad[3 * i + 1];
        out[5 * i + 3] = grad[3 * i + 2];
        out[5 * i + 4] = (Real)w[i];
    }
}

template <typename Real>
__global__ void k_scatter_back(int64_t n, const Real* __restrict__ v, const int64_t* __restrict__ gid, int64_t base,
                               Real* __restrict__ phi, Real* __restrict__ grad, float* __restrict__ w) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = gid[k] - base;
        phi[i] = v[5 * k];
        grad[3 * i] = v[5 * k + 1];
        grad[3 * i + 1] = v[5 * k + 2];
        grad[3 * i + 2] = v[5 * k + 3];
        w[i] = (float)v[5 * k + 4];
    }
}

__global__ void k_iota_u32(int64_t n, uint32_t base, uint32_t* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = base + (uint32_t)i;
}

// arrivals: local indices [0, a) and [b, n) (everything but the staying block [a, b))
__global__ void k_arrival_ids(int64_t na, uint32_t a, uint32_t b, const uint64_t* __restrict__ keys_all,
                              uint64_t* __restrict__ k, uint32_t* __restrict__ idx) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t j = i < a ? (uint32_t)i : (uint32_t)(i - a + b);
        k[i] = keys_all[j];
        idx[i] = j;
    }
}

// merge of two runs sorted by (key, index) (all pairs distinct): each element's output position
// is its rank in its own run plus the number of elements of the other run that precede it
__device__ __forceinline__ bool pair_less(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}
__global__ void k_merge_runs(const uint64_t* __restrict__ ka, const uint32_t* __restrict__ ia, int64_t na,
                             const uint64_t* __restrict__ kb, const uint32_t* __restrict__ ib, int64_t nb,
                             uint64_t* __restrict__ ko, uint32_t* __restrict__ io) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < na + nb; t += (int64_t)gridDim.x * blockDim.x) {
        const bool in_a = t < na;
        const int64_t i = in_a ? t : t - na;
        const uint64_t k = in_a ? ka[i] : kb[i];
        const uint32_t x = in_a ? ia[i] : ib[i];
        const uint64_t* ok = in_a ? kb : ka;
        const uint32_t* oi = in_a ? ib : ia;
        int64_t lo = 0, hi = in_a ? nb : na;   // first element of the other run not before (k, x)
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (pair_less(ok[mid], oi[mid], k, x)) lo = mid + 1;
            else hi = mid;
        }
        ko[i + lo] = k;
        io[i + lo] = x;
    }
}

// ---- split interactions (local lists first, remote lists after): buffer swaps and merges
void swap_m2l_csr(fmm_ctx* ctx, DistState* D) {
    std::swap(ctx->m2l_off, D->r_moff);
    std::swap(ctx->m2l_src, D->r_msrc);
    std::swap(ctx->n_m2l, D->r_nm);
}
void swap_p2p_csr(fmm_ctx* ctx, DistState* D) {
    std::swap(ctx->p2p_off, D->r_poff);
    std::swap(ctx->p2p_src, D->r_psrc);
    std::swap(ctx->n_p2p, D->r_np);
}
void swap_runs(fmm_ctx* ctx, DistState* D) {
    std::swap(ctx->runs, D->r_runs);
    std::swap(ctx->run_off, D->r_run_off);
    std::swap(ctx->run_tmp, D->r_run_tmp);
    std::swap(ctx->leaf_cls, D->r_leaf_cls);
    std::swap(ctx->n_runs, D->r_nruns);
    for (int k = 0; k < 3; ++k) std::swap(ctx->n_leaf_cls[k], D->r_ncls[k]);
}

// reduced L_hat: local + remote (each pass wrote only the targets that have a list of its kind)
__global__ void k_merge_lr(int64_t nc, int NL, const uint64_t* __restrict__ offl, const uint64_t* __restrict__ offr,
                           double* __restrict__ Lr, const double* __restrict__ Lr2) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nc * NL; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = t / NL;
        if (offr[c] == offr[c + 1]) continue;
        Lr[t] = (offl[c] < offl[c + 1] ? Lr[t] : 0.0) + Lr2[t];
    }
}
__global__ void k_add_f64(int64_t n, double* __restrict__ a, const double* __restrict__ b) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] += b[i];
}
template <typename Real>
__global__ void k_add_near(int64_t n, Real* __restrict__ phi, const Real* __restrict__ phi2, Real* __restrict__ grad,
                           const Real* __restrict__ grad2) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        phi[i] += phi2[i];
        grad[3 * i] += grad2[3 * i];
        grad[3 * i + 1] += grad2[3 * i + 1];
        grad[3 * i + 2] += grad2[3 * i + 2];
    }
}
__global__ void k_add_u64(unsigned long long* a, const unsigned long long* b) { *a += *b; }
__global__ void k_level_minmax(int64_t n, const int32_t* __restrict__ level, int* __restrict__ mm) {
    int lo = 1 << 30, hi = -(1 << 30);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        lo = min(lo, level[i]);
        hi = max(hi, level[i]);
    }
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
}

struct Step {
    fmm_ctx* ctx;
    DistState* D;
    cudaStream_t s, m, aux;
    size_t es;
    void tl_begin(int i, cudaStream_t st) {
        if (ctx->timing) cudaEventRecord(D->tl[i][0], st), D->tl_rec[i] = true;
    }
    void tl_end(int i, cudaStream_t st) {
        if (ctx->timing) cudaEventRecord(D->tl[i][1], st);
    }
};

fmm_status tr_err(fmm_ctx* ctx, DistState* D, fmm_status st) {
    if (st != FMM_OK) {
        ctx->err = "transport: " + D->tr->err;
        D->tr->abort();
    }
    return st;
}
#define FMM_TR(expr) FMM_TRY(tr_err(ctx, D, (expr)))

}  // namespace

// ------------------------------------------------------------------------------- the step
static fmm_status dist_step(fmm_ctx* ctx, DistState* D, const void* pos, const void* q, int64_t n, int64_t gid_base,
                            const float* w, void* phi, void* grad, cudaStream_t s) {
    const int K = D->K, me = D->rank;
    const size_t es = ctx->prec == FMM_F32 ? 4 : 8;
    cudaStream_t m = ctx->hp ? ctx->hp : s, aux = ctx->aux, cs = D->cs, side = D->side;
    Step S{ctx, D, s, m, aux, es};
    for (int i = 0; i < TL_COUNT; ++i) D->tl_rec[i] = false;
    if (m != s) {
        FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[0], s));
        FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(m, D->ev[0], 0));
    }
    if (ctx->timing) FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev_t0, m));
    // ---- 1. global bounds, keys (R2-R4 on the global root cube)
    S.tl_begin(TL_PARTITION, m);
    double lohi[6];
    FMM_TRY(fmm_bounds(ctx, pos, n, lohi, m));
    double hb[6] = {-lohi[0], -lohi[1], -lohi[2], lohi[3], lohi[4], lohi[5]};
    FMM_TRY(buf_ensure(ctx, D->red, 64 * 8));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(D->red.p, hb, 48, cudaMemcpyHostToDevice, m));
    FMM_TR(D->tr->allreduce_f64(P_<double>(D->red), 6, 2, m));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(hb, D->red.p, 48, cudaMemcpyDeviceToHost, m));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(m));
    for (int d = 0; d < 3; ++d) {
        D->gb[d] = -hb[d];
        D->gb[3 + d] = hb[3 + d];
    }
    const bool empty_world = !(D->gb[0] <= D->gb[3]);
    FMM_TRY(buf_ensure(ctx, D->keys, (size_t)std::max<int64_t>(n, 1) * 8));
    if (!empty_world) FMM_TRY(fmm_part_keys(ctx, pos, n, D->gb, P_<uint64_t>(D->keys), m));
    // ---- 2. destination ranks
    std::vector<int64_t> cnt(K, 0);
    FMM_TRY(buf_ensure(ctx, D->pk_pos, (size_t)std::max<int64_t>(n, 1) * 3 * es));
    FMM_TRY(buf_ensure(ctx, D->pk_q, (size_t)std::max<int64_t>(n, 1) * es));
    FMM_TRY(buf_ensure(ctx, D->pk_gid, (size_t)std::max<int64_t>(n, 1) * 8));
    const uint64_t* keys = P_<uint64_t>(D->keys);
    if (D->partitioner == FMM_PART_MORTON) {
        std::vector<uint64_t> spl(std::max(K - 1, 1), 0);
        auto hist = [&](const uint64_t* prefixes, int np, int pbits, int bits, double* out) -> fmm_status {
            const size_t nb = (size_t)1 << bits;
            FMM_TRY(buf_ensure(ctx, D->hist, (size_t)np * nb * 8));
            for (int r = 0; r < np; ++r)
                FMM_TRY(fmm_part_histogram(ctx, keys, w, n, prefixes[r], pbits, bits, P_<double>(D->hist) + r * nb, m));
            FMM_TR(D->tr->allreduce_f64(P_<double>(D->hist), (size_t)np * nb, 0, m));
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync(out, D->hist.p, (size_t)np * nb * 8, cudaMemcpyDeviceToHost, m));
            FMM_CUDA_TRY(ctx, cudaStreamSynchronize(m));
            return FMM_OK;
        };
        if (!empty_world) FMM_TRY(splitters_refine(K, 16, 1.0 / 512, hist, spl.data()));
        FMM_TRY(fmm_part_pack(ctx, pos, q, keys, n, spl.data(), K, gid_base, D->pk_pos.p, D->pk_q.p,
                              P_<int64_t>(D->pk_gid), cnt.data(), m));
    } else {
        FMM_TRY(buf_ensure(ctx, D->group, (size_t)std::max<int64_t>(n, 1) * 4));
        FMM_CUDA_TRY(ctx, cudaMemsetAsync(D->group.p, 0, (size_t)std::max<int64_t>(n, 1) * 4, m));
        int32_t* grp = P_<int32_t>(D->group);
        auto hist = [&](const int32_t* axis, const uint32_t* prefix, int pbits, int bits, double* out) -> fmm_status {
            const size_t nb = (size_t)1 << bits;
            FMM_TRY(buf_ensure(ctx, D->hist, (size_t)K * nb * 8));
            FMM_TRY(fmm_orb_histogram(ctx, keys, w, grp, n, K, axis, prefix, pbits, bits, P_<double>(D->hist), m));
            FMM_TR(D->tr->allreduce_f64(P_<double>(D->hist), (size_t)K * nb, 0, m));
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync(out, D->hist.p, (size_t)K * nb * 8, cudaMemcpyDeviceToHost, m));
            FMM_CUDA_TRY(ctx, cudaStreamSynchronize(m));
            return FMM_OK;
        };
        auto split = [&](const int32_t* axis, const uint32_t* cut, const int32_t* right) -> fmm_status {
            return fmm_orb_split(ctx, keys, grp, n, K, axis, cut, right, m);
        };
        D->boxes.assign((size_t)6 * K, 0);
        if (!empty_world) FMM_TRY(orb_plan_t(K, 16, hist, split, D->boxes.data()));
        FMM_TRY(fmm_part_pack_dest(ctx, pos, q, grp, n, K, gid_base, D->pk_pos.p, D->pk_q.p, P_<int64_t>(D->pk_gid),
                                   cnt.data(), m));
    }
    // counts matrix: row r = what rank r sends to each rank
    FMM_TRY(buf_ensure(ctx, D->stage, (size_t)(K + 1) * K * 16 + 1024));
    int64_t* dcnt = P_<int64_t>(D->stage);
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(dcnt, cnt.data(), (size_t)K * 8, cudaMemcpyHostToDevice, m));
    FMM_TR(D->tr->allgather(dcnt, dcnt + K, (size_t)K * 8, m));
    std::vector<int64_t> all((size_t)K * K);
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(all.data(), dcnt + K, (size_t)K * K * 8, cudaMemcpyDeviceToHost, m));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(m));
    std::vector<int64_t> rc(K), roff(K + 1, 0), soff(K + 1, 0);
    for (int j = 0; j < K; ++j) {
        rc[j] = all[(size_t)j * K + me];
        roff[j + 1] = roff[j] + rc[j];
        soff[j + 1] = soff[j] + cnt[j];
    }
    const int64_t nl = roff[K];
    if (nl > ctx->n_max) {
        ctx->err = "fmm_dist_solve: this rank's share exceeds n_local_max of fmm_create_dist";
        D->tr->abort();
        return FMM_ERR_ARG;
    }
    D->n_local = nl;
    S.tl_end(TL_PARTITION, m);
    // ---- 3. particle exchange (grouped send/recv on the comm stream); the staying particles are
    // sorted meanwhile on the side stream (f1)
    FMM_TRY(buf_ensure(ctx, D->l_pos, (size_t)std::max<int64_t>(nl, 1) * 3 * es));
    FMM_TRY(buf_ensure(ctx, D->l_q, (size_t)std::max<int64_t>(nl, 1) * es));
    FMM_TRY(buf_ensure(ctx, D->l_gid, (size_t)std::max<int64_t>(nl, 1) * 8));
    const bool presort = D->overlap_sort && D->partitioner == FMM_PART_MORTON && nl > 0;
    const int64_t nstay = cnt[me];
    if (presort) {
        FMM_TRY(buf_ensure(ctx, D->sk, (size_t)std::max<int64_t>(nstay, 1) * 16));
        FMM_TRY(buf_ensure(ctx, D->si, (size_t)std::max<int64_t>(nstay, 1) * 8));
    }
    FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[1], m));   // packed particles ready
    // the staying particles' sort is enqueued first, so it runs while the exchange flies
    if (presort && nstay > 0) {
        FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(side, D->ev[1], 0));
        S.tl_begin(TL_STAY_SORT, side);
        uint64_t* k0 = P_<uint64_t>(D->sk);
        uint32_t* i0 = P_<uint32_t>(D->si);
        FMM_TRY(fmm_part_keys(ctx, (char*)D->pk_pos.p + soff[me] * 3 * es, nstay, D->gb, k0, side));
        k_iota_u32<<<grid1(nstay), 256, 0, side>>>(nstay, (uint32_t)roff[me], i0);
        FMM_LAUNCH(ctx);
        uint64_t* ko = nullptr;
        uint32_t* io = nullptr;
        FMM_TRY(radix_sort_pairs(ctx, k0, k0 + nstay, i0, i0 + nstay, nstay, 0, 64, &ko, &io, side, ~0ull));
        D->stay_in_b = ko != k0;
        S.tl_end(TL_STAY_SORT, side);
        FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[3], side));
    }
    FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(cs, D->ev[1], 0));
    S.tl_begin(TL_EXCHANGE, cs);
    {
        std::vector<CommMsg> sends, recvs;
        for (int j = 0; j < K; ++j) {
            if (j == me) continue;
            sends.push_back({j, (char*)D->pk_pos.p + soff[j] * 3 * es, (size_t)cnt[j] * 3 * es});
            sends.push_back({j, (char*)D->pk_q.p + soff[j] * es, (size_t)cnt[j] * es});
            sends.push_back({j, P_<int64_t>(D->pk_gid) + soff[j], (size_t)cnt[j] * 8});
            recvs.push_back({j, (char*)D->l_pos.p + roff[j] * 3 * es, (size_t)rc[j] * 3 * es});
            recvs.push_back({j, (char*)D->l_q.p + roff[j] * es, (size_t)rc[j] * es});
            recvs.push_back({j, P_<int64_t>(D->l_gid) + roff[j], (size_t)rc[j] * 8});
        }
        // the staying block is a device copy
        if (nstay) {
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync((char*)D->l_pos.p + roff[me] * 3 * es, (char*)D->pk_pos.p + soff[me] * 3 * es,
                                              (size_t)nstay * 3 * es, cudaMemcpyDeviceToDevice, cs));
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync((char*)D->l_q.p + roff[me] * es, (char*)D->pk_q.p + soff[me] * es,
                                              (size_t)nstay * es, cudaMemcpyDeviceToDevice, cs));
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync(P_<int64_t>(D->l_gid) + roff[me], P_<int64_t>(D->pk_gid) + soff[me],
                                              (size_t)nstay * 8, cudaMemcpyDeviceToDevice, cs));
        }
        FMM_TR(D->tr->sendrecv(sends, recvs, cs));
    }
    S.tl_end(TL_EXCHANGE, cs);
    FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[2], cs));   // local particles landed
    FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(m, D->ev[2], 0));
    // ---- 4. local tree on the global root cube (Morton) / local box (ORB)
    S.tl_begin(TL_TREE, m);
    FMM_TRY(fmm_set_root_bounds(ctx, D->partitioner == FMM_PART_MORTON && !empty_world ? D->gb : nullptr));
    if (presort) {
        // arrivals sorted after landing, merged with the staying run: the order of a full sort
        const int64_t na = nl - nstay;
        // the radix sort's scratch is the context's: the staying sort must be done first
        if (nstay > 0) FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(m, D->ev[3], 0));
        FMM_TRY(buf_ensure(ctx, D->ak, (size_t)(nl + 2 * na) * 8 + 64));
        FMM_TRY(buf_ensure(ctx, D->ai, (size_t)std::max<int64_t>(na, 1) * 8 + 64));
        uint64_t* kall = P_<uint64_t>(D->ak);
        uint64_t* a0 = kall + nl;
        uint32_t* b0 = P_<uint32_t>(D->ai);
        uint64_t* ako = a0;
        uint32_t* aio = b0;
        if (na > 0) {
            FMM_TRY(fmm_part_keys(ctx, D->l_pos.p, nl, D->gb, kall, m));
            k_arrival_ids<<<grid1(na), 256, 0, m>>>(na, (uint32_t)roff[me], (uint32_t)(roff[me] + nstay), kall, a0, b0);
            FMM_LAUNCH(ctx);
            FMM_TRY(radix_sort_pairs(ctx, a0, a0 + na, b0, b0 + na, na, 0, 64, &ako, &aio, m, ~0ull));
        }
        const uint64_t* sko = D->stay_in_b ? P_<uint64_t>(D->sk) + nstay : P_<uint64_t>(D->sk);
        const uint32_t* sio = D->stay_in_b ? P_<uint32_t>(D->si) + nstay : P_<uint32_t>(D->si);
        FMM_TRY(buf_ensure(ctx, ctx->key_a, (size_t)nl * 8));
        FMM_TRY(buf_ensure(ctx, ctx->idx_a, (size_t)nl * 4));
        k_merge_runs<<<grid1(nl), 256, 0, m>>>(sko, sio, nstay, ako, aio, na, P_<uint64_t>(ctx->key_a),
                                               P_<uint32_t>(ctx->idx_a));
        FMM_LAUNCH(ctx);
        ctx->presorted = true;
    }
    fmm_status bst = fmm_build_tree(ctx, D->l_pos.p, nl, m);
    ctx->presorted = false;
    FMM_TRY(bst);
    S.tl_end(TL_TREE, m);
    // ---- upward pass on the aux stream (P2M/M2M need the tree and q only).  The split flow
    // launches it after the LET capacity is reserved (a reservation may move M and the bodies)
    // (a rank left without particles takes the unsplit flow: it has no lists; the collective calls
    // of both flows are the same)
    const bool split = D->split && K > 1 && nl > 0;
    auto launch_upward = [&]() -> fmm_status {
        FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[4], m));
        FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(aux, D->ev[4], 0));
        S.tl_begin(TL_UPWARD, aux);
        FMM_TRY(fmm_upward(ctx, D->l_pos.p, D->l_q.p, aux));
        S.tl_end(TL_UPWARD, aux);
        FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[5], aux));   // upward done
        return FMM_OK;
    };
    if (!split) FMM_TRY(launch_upward());
    // ---- 5. covers, plans, LET structure
    S.tl_begin(TL_COVER, m);
    const int CW = 1 + 8 * FMM_LET_MAX_COVER;
    std::vector<double> cov(CW, 0.0);
    int ncov = 0;
    FMM_TRY(fmm_let_cover(ctx, cov.data() + 1, &ncov, m));
    cov[0] = ncov;
    FMM_TRY(buf_ensure(ctx, D->cov, (size_t)(K + 1) * CW * 8));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(D->cov.p, cov.data(), (size_t)CW * 8, cudaMemcpyHostToDevice, m));
    FMM_TR(D->tr->allgather(D->cov.p, P_<double>(D->cov) + CW, (size_t)CW * 8, m));
    std::vector<double> allcov((size_t)K * CW);
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(allcov.data(), P_<double>(D->cov) + CW, allcov.size() * 8, cudaMemcpyDeviceToHost, m));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(m));
    std::vector<int64_t> sb(K, 0), db(K, 0);
    for (int j = 0; j < K; ++j) {
        if (j == me) continue;
        const double* cj = allcov.data() + (size_t)j * CW;
        FMM_TRY(fmm_let_plan(ctx, j, cj + 1, (int)cj[0], &sb[j], &db[j], m));
    }
    std::vector<int64_t> so(K + 1, 0);   // send buffer: [struct_j | data_j] per peer, 256-B aligned
    auto al = [](int64_t b) { return (b + 255) / 256 * 256; };
    for (int j = 0; j < K; ++j) so[j + 1] = so[j] + al(sb[j]) + al(db[j]);
    FMM_TRY(buf_ensure(ctx, D->let_send, (size_t)std::max<int64_t>(so[K], 256)));
    char* lsend = (char*)D->let_send.p;
    for (int j = 0; j < K; ++j)
        if (j != me && sb[j]) FMM_TRY(fmm_let_pack_struct(ctx, j, lsend + so[j], m));
    // message sizes: row r = (struct, data) bytes rank r sends to each rank
    std::vector<int64_t> szs((size_t)2 * K);
    for (int j = 0; j < K; ++j) {
        szs[2 * j] = sb[j];
        szs[2 * j + 1] = db[j];
    }
    int64_t* dsz = P_<int64_t>(D->stage);
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(dsz, szs.data(), (size_t)2 * K * 8, cudaMemcpyHostToDevice, m));
    FMM_TR(D->tr->allgather(dsz, dsz + 2 * K, (size_t)2 * K * 8, m));
    std::vector<int64_t> asz((size_t)2 * K * K);
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(asz.data(), dsz + 2 * K, asz.size() * 8, cudaMemcpyDeviceToHost, m));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(m));
    std::vector<int64_t> rsb(K, 0), rdb(K, 0), ro(K + 1, 0);
    for (int j = 0; j < K; ++j) {
        rsb[j] = asz[(size_t)j * 2 * K + 2 * me];
        rdb[j] = asz[(size_t)j * 2 * K + 2 * me + 1];
        ro[j + 1] = ro[j] + al(rsb[j]) + al(rdb[j]);
    }
    FMM_TRY(buf_ensure(ctx, D->let_recv, (size_t)std::max<int64_t>(ro[K], 256)));
    char* lrecv = (char*)D->let_recv.p;
    if (split) {
        // capacity for every incoming fragment now, so grafting never moves an array the local
        // interactions (compute stream) or the upward pass (aux) are reading: a structure message of
        // b bytes holds at most (b - 64) / 64 cells and (b - 64) / body-size bodies
        const int64_t bsz = ctx->prec == FMM_F32 ? 16 : 32;
        int64_t addc = 0, addb = 0;
        for (int j = 0; j < K; ++j)
            if (j != me && rsb[j] > 64) {
                addc += (rsb[j] - 64) / 64;
                addb += (rsb[j] - 64) / bsz;
            }
        const int64_t ctot = ctx->ncell + addc, btot = nl + addb;
        DevBuf* u32s[] = {&ctx->c_cb, &ctx->c_cc, &ctx->c_bb, &ctx->c_bc, &ctx->c_level, &ctx->c_parent};
        for (DevBuf* b : u32s) FMM_TRY(buf_ensure(ctx, *b, (size_t)std::max<int64_t>(ctot, 1) * 4, true, m));
        FMM_TRY(buf_ensure(ctx, ctx->c_key, (size_t)std::max<int64_t>(ctot, 1) * 8, true, m));
        FMM_TRY(buf_ensure(ctx, ctx->c_cr, (size_t)std::max<int64_t>(ctot, 1) * 32, true, m));
        FMM_TRY(buf_ensure(ctx, ctx->c_orig, (size_t)std::max<int64_t>(ctot, 1) * 4, true, m));
        FMM_TRY(buf_ensure(ctx, ctx->body, (size_t)std::max<int64_t>(btot, 1) * bsz, true, m));
        FMM_TRY(buf_ensure(ctx, ctx->M, (size_t)std::max<int64_t>(ctot, 1) * ctx->ncoef * 8, true, m));
        D->nct_cap = std::max<int64_t>(ctot, 1);
        FMM_TRY(launch_upward());
    }
    S.tl_end(TL_COVER, m);
    // structure rounds on the comm stream: round r sends to me + r, receives from me - r
    FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[6], m));   // structures packed
    FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(cs, D->ev[6], 0));
    S.tl_begin(TL_STRUCT_XCHG, cs);
    while ((int)D->ev_round.size() < K) {
        cudaEvent_t e;
        FMM_CUDA_TRY(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        D->ev_round.push_back(e);
    }
    for (int r = 1; r < K; ++r) {
        const int dst = (me + r) % K, src = (me - r + K) % K;
        std::vector<CommMsg> sends{{dst, lsend + so[dst], (size_t)sb[dst]}}, recvs{{src, lrecv + ro[src], (size_t)rsb[src]}};
        FMM_TR(D->tr->sendrecv(sends, recvs, cs));
        FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev_round[r], cs));
    }
    S.tl_end(TL_STRUCT_XCHG, cs);
    // ---- local traversal on the critical stream, overlapping the structure rounds
    S.tl_begin(TL_LOCAL_DTT, m);
    FMM_TRY(fmm_dtt(ctx, 0, m));
    S.tl_end(TL_LOCAL_DTT, m);
    bool fast_local = false;
    if (split) {
        // local lists -> P2P source runs (synchronises m), then the local M2L and P2P on the compute
        // stream: they run while the LET fragments are grafted and traversed below
        FMM_TRY(lists_finish(ctx, m));
        FMM_TRY(buf_ensure(ctx, D->inter_loc, 64));
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(D->inter_loc.p, P_<unsigned long long>(ctx->dcount2) + 2, 8,
                                          cudaMemcpyDeviceToDevice, m));   // local P2P interaction count
        FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[8], m));
        FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(D->cx, D->ev[8], 0));
        FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(D->cx, D->ev[5], 0));   // M and the bodies' charges
        S.tl_begin(TL_INTERACT_LOCAL, D->cx);
        ctx->m2l_cap = D->nct_cap;
        ctx->m2l_prep_c0 = 0;
        ctx->m2l_no_expand = true;
        ctx->m2l_span_fixed = false;
        ctx->m2l_part = 0;
        FMM_TRY(m2l_pass(ctx, D->cx));
        fast_local = ctx->use_fast_m2l && m2l_fast_available(ctx->P, ctx->prec) && !(ctx->prec == FMM_F32 && ctx->m2l_deep);
        FMM_TRY(p2p_pass(ctx, D->cx));
        S.tl_end(TL_INTERACT_LOCAL, D->cx);
    }
    // ---- LET data (multipoles, charges) on the comm stream once the upward pass is done
    FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(cs, D->ev[5], 0));
    S.tl_begin(TL_DATA_XCHG, cs);
    for (int j = 0; j < K; ++j)
        if (j != me && db[j]) FMM_TRY(fmm_let_pack_data(ctx, j, lsend + so[j] + al(sb[j]), cs));
    {
        std::vector<CommMsg> sends, recvs;
        for (int r = 1; r < K; ++r) {
            const int dst = (me + r) % K, src = (me - r + K) % K;
            sends.push_back({dst, lsend + so[dst] + al(sb[dst]), (size_t)db[dst]});
            recvs.push_back({src, lrecv + ro[src] + al(rsb[src]), (size_t)rdb[src]});
        }
        FMM_TR(D->tr->sendrecv(sends, recvs, cs));
    }
    S.tl_end(TL_DATA_XCHG, cs);
    FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[7], cs));   // LET data landed
    // ---- every structure fragment grafted and traversed as it lands
    D->peers.clear();
    S.tl_begin(TL_REMOTE_DTT, m);
    for (int r = 1; r < K; ++r) {
        const int src = (me - r + K) % K;
        if (!rsb[src]) continue;
        FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(m, D->ev_round[r], 0));
        const void* p = lrecv + ro[src];
        const int64_t bytes = rsb[src];
        FMM_TRY(fmm_let_graft(ctx, 1, &p, &bytes, m));
        FMM_TRY(fmm_dtt(ctx, 1, m));
        D->peers.push_back(src);
    }
    S.tl_end(TL_REMOTE_DTT, m);
    FMM_TRY(buf_ensure(ctx, D->phi_loc, (size_t)std::max<int64_t>(nl, 1) * es));
    FMM_TRY(buf_ensure(ctx, D->grad_loc, (size_t)std::max<int64_t>(nl, 1) * 3 * es));
    FMM_TRY(buf_ensure(ctx, D->w_loc, (size_t)std::max<int64_t>(nl, 1) * 4));
    auto unpack = [&]() -> fmm_status {   // LET data (graft order)
        FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(m, D->ev[7], 0));
        FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(m, D->ev[5], 0));
        if (D->peers.empty()) return FMM_OK;
        std::vector<const void*> ptrs;
        std::vector<int64_t> bytes;
        for (int src : D->peers) {
            ptrs.push_back(lrecv + ro[src] + al(rsb[src]));
            bytes.push_back(rdb[src]);
        }
        return fmm_let_unpack(ctx, 0, (int)ptrs.size(), ptrs.data(), bytes.data(), m);
    };
    if (!split) {
        S.tl_begin(TL_LISTS, m);
        FMM_TRY(fmm_lists(ctx, m));
        S.tl_end(TL_LISTS, m);
        // ---- 6. data unpacked (graft order), interactions
        FMM_TRY(unpack());
        S.tl_begin(TL_INTERACT, m);
        FMM_TRY(fmm_interact(ctx, D->phi_loc.p, D->grad_loc.p, m));
    } else {
        cudaStream_t cx = D->cx;
        const int64_t nc = ctx->ncell;
        S.tl_begin(TL_LISTS, m);
        // remote-only CSR lists: the remote traversal parts concatenated per target into an empty
        // list (the local lists stay in place for the kernels reading them on the compute stream)
        swap_m2l_csr(ctx, D);
        swap_p2p_csr(ctx, D);
        FMM_TRY(buf_ensure(ctx, ctx->m2l_off, (size_t)(nc + 1) * 8));
        FMM_TRY(buf_ensure(ctx, ctx->p2p_off, (size_t)(nc + 1) * 8));
        FMM_TRY(buf_ensure(ctx, ctx->m2l_src, 64));
        FMM_TRY(buf_ensure(ctx, ctx->p2p_src, 64));
        FMM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->m2l_off.p, 0, (size_t)(nc + 1) * 8, m));
        FMM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->p2p_off.p, 0, (size_t)(nc + 1) * 8, m));
        ctx->n_m2l = ctx->n_p2p = 0;
        const int parts = ctx->tc_nrem;
        FMM_TRY(tct_concat(ctx, m));
        ctx->tc_nrem = parts;   // kept for the full concatenation below
        // the remote P2P source runs (into the swapped-out run buffers)
        swap_runs(ctx, D);
        FMM_TRY(lists_finish(ctx, m));
        k_add_u64<<<1, 1, 0, m>>>(P_<unsigned long long>(ctx->dcount2) + 2, P_<unsigned long long>(D->inter_loc));
        FMM_LAUNCH(ctx);
        swap_runs(ctx, D);
        swap_p2p_csr(ctx, D);
        swap_m2l_csr(ctx, D);
        S.tl_end(TL_LISTS, m);
        FMM_TRY(unpack());
        // an fp32 tree spanning more than 14 levels with the LETs grafted: the register kernels'
        // operand scale leaves the fp32 range (m2l.cu) -- redo M2L with the fp64 kernel on all lists
        int span = 0;
        if (ctx->prec == FMM_F32 && fast_local) {
            FMM_TRY(buf_ensure(ctx, D->span_tmp, 64));
            int init[2] = {1 << 30, -(1 << 30)}, mm[2];
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync(D->span_tmp.p, init, 8, cudaMemcpyHostToDevice, m));
            k_level_minmax<<<grid1(nc + ctx->nrem), 256, 0, m>>>(nc + ctx->nrem, P_<int32_t>(ctx->c_level),
                                                                 P_<int>(D->span_tmp));
            FMM_LAUNCH(ctx);
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync(mm, D->span_tmp.p, 8, cudaMemcpyDeviceToHost, m));
            FMM_CUDA_TRY(ctx, cudaStreamSynchronize(m));
            span = mm[1] - mm[0];
        }
        const bool redo = fast_local && span > 14;
        FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[9], m));   // remote lists, runs and data ready
        FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(cx, D->ev[9], 0));
        S.tl_begin(TL_INTERACT_REMOTE, cx);
        ctx->m2l_span_fixed = true;   // keep the local pass's kernel choice
        ctx->m2l_prep_c0 = nc;        // operands of the grafted cells only
        if (!redo) {
            swap_m2l_csr(ctx, D);
            fmm_status st;
            if (fast_local) {
                std::swap(ctx->Lr, D->Lr2);
                st = m2l_pass(ctx, cx);
                std::swap(ctx->Lr, D->Lr2);
            } else {
                std::swap(ctx->L, D->L2);
                st = m2l_pass(ctx, cx);
                std::swap(ctx->L, D->L2);
            }
            swap_m2l_csr(ctx, D);
            FMM_TRY(st);
            if (fast_local) {
                const int NL = ctx->P * ctx->P;
                k_merge_lr<<<grid1(nc * NL), 256, 0, cx>>>(nc, NL, P_<uint64_t>(ctx->m2l_off), P_<uint64_t>(D->r_moff),
                                                           P_<double>(ctx->Lr), P_<double>(D->Lr2));
            } else {
                k_add_f64<<<grid1(nc * ctx->ncoef), 256, 0, cx>>>(nc * ctx->ncoef, P_<double>(ctx->L), P_<double>(D->L2));
            }
            FMM_LAUNCH(ctx);
        }
        // remote P2P into second partials, added to the local ones
        swap_p2p_csr(ctx, D);
        swap_runs(ctx, D);
        std::swap(ctx->near_phi, D->near2_phi);
        std::swap(ctx->near_grad, D->near2_grad);
        fmm_status st = p2p_pass(ctx, cx);
        std::swap(ctx->near_phi, D->near2_phi);
        std::swap(ctx->near_grad, D->near2_grad);
        swap_runs(ctx, D);
        swap_p2p_csr(ctx, D);
        FMM_TRY(st);
        if (ctx->prec == FMM_F32)
            k_add_near<float><<<grid1(nl), 256, 0, cx>>>(nl, P_<float>(ctx->near_phi), P_<float>(D->near2_phi),
                                                         P_<float>(ctx->near_grad), P_<float>(D->near2_grad));
        else
            k_add_near<double><<<grid1(nl), 256, 0, cx>>>(nl, P_<double>(ctx->near_phi), P_<double>(D->near2_phi),
                                                          P_<double>(ctx->near_grad), P_<double>(D->near2_grad));
        FMM_LAUNCH(ctx);
        if (!redo && fast_local) FMM_TRY(m2l_expand(ctx, P_<uint64_t>(D->r_moff), cx));
        ctx->m2l_prep_c0 = 0;
        ctx->m2l_no_expand = false;
        ctx->m2l_span_fixed = false;
        // the full concatenated lists (introspection, Eq. (1) weights) on the critical stream, beside
        // the downward pass: the concatenation rotates the list buffers (tct_concat writes into the
        // buffers the local and remote lists occupied), so it waits until the compute stream is past
        // every kernel that reads a list
        FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[10], cx));
        FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(m, D->ev[10], 0));
        FMM_TRY(tct_concat(ctx, m));
        ctx->built = true;
        if (redo) {
            FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[10], m));
            FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(cx, D->ev[10], 0));
            ctx->m2l_cap = 0;
            ctx->m2l_part = 0;
            FMM_TRY(m2l_pass(ctx, cx));   // all lists, level span measured again: the fp64 kernel
        }
        ctx->m2l_cap = 0;
        FMM_TRY(downward_pass(ctx, D->phi_loc.p, D->grad_loc.p, cx));   // L2L/L2P + near field, local order
        S.tl_end(TL_INTERACT_REMOTE, cx);
        FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[11], cx));
        ctx->evaluated = true;
    }
    if (split) S.tl_begin(TL_INTERACT, m);   // (the unsplit flow began the span at its interactions)
    double lr[2] = {0, 0};
    if (nl > 0) FMM_TRY(fmm_work(ctx, D->c_m2l, (float)D->alpha, P_<float>(D->w_loc), lr, m));
    D->st.work_local = lr[0];
    D->st.work_remote = lr[1];
    if (split) FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(m, D->ev[11], 0));   // phi/grad of the local particles
    S.tl_end(TL_INTERACT, m);
    // ---- 7. results and weights back to the owners
    S.tl_begin(TL_BACK, m);
    FMM_TRY(buf_ensure(ctx, D->back_send, (size_t)std::max<int64_t>(nl, 1) * 5 * es));
    FMM_TRY(buf_ensure(ctx, D->back_recv, (size_t)std::max<int64_t>(n, 1) * 5 * es));
    if (nl > 0) {
        if (ctx->prec == FMM_F32)
            k_pack_back<float><<<grid1(nl), 256, 0, m>>>(nl, P_<float>(D->phi_loc), P_<float>(D->grad_loc),
                                                         P_<float>(D->w_loc), P_<float>(D->back_send));
        else
            k_pack_back<double><<<grid1(nl), 256, 0, m>>>(nl, P_<double>(D->phi_loc), P_<double>(D->grad_loc),
                                                          P_<float>(D->w_loc), P_<double>(D->back_send));
        FMM_LAUNCH(ctx);
    }
    {
        std::vector<CommMsg> sends, recvs;
        for (int j = 0; j < K; ++j) {
            sends.push_back({j, (char*)D->back_send.p + roff[j] * 5 * es, (size_t)rc[j] * 5 * es});
            recvs.push_back({j, (char*)D->back_recv.p + soff[j] * 5 * es, (size_t)cnt[j] * 5 * es});
        }
        FMM_TR(D->tr->sendrecv(sends, recvs, m));
    }
    FMM_TRY(buf_ensure(ctx, D->w_prev, (size_t)std::max<int64_t>(n, 1) * 4, false, m));
    if (n > 0) {
        if (ctx->prec == FMM_F32)
            k_scatter_back<float><<<grid1(n), 256, 0, m>>>(n, P_<float>(D->back_recv), P_<int64_t>(D->pk_gid), gid_base,
                                                           (float*)phi, (float*)grad, P_<float>(D->w_prev));
        else
            k_scatter_back<double><<<grid1(n), 256, 0, m>>>(n, P_<double>(D->back_recv), P_<int64_t>(D->pk_gid),
                                                            gid_base, (double*)phi, (double*)grad, P_<float>(D->w_prev));
        FMM_LAUNCH(ctx);
    }
    D->w_prev_n = n;
    S.tl_end(TL_BACK, m);
    // join the comm and side streams into the critical one, then into the caller's
    FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[0], cs));
    FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(m, D->ev[0], 0));
    FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[0], side));
    FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(m, D->ev[0], 0));
    FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[0], D->cx));
    FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(m, D->ev[0], 0));
    if (m != s) {
        FMM_CUDA_TRY(ctx, cudaEventRecord(D->ev[0], m));
        FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(s, D->ev[0], 0));
    }
    // stats
    fmm_dist_stats& st = D->st;
    for (int d = 0; d < 6; ++d) st.bounds[d] = D->gb[d];
    st.alpha = D->alpha;
    st.c_m2l = D->c_m2l;
    st.n_local = nl;
    st.npeers = (int)D->peers.size();
    st.let_struct_bytes = st.let_data_bytes = 0;
    for (int j = 0; j < K; ++j) {
        st.let_struct_bytes += sb[j];
        st.let_data_bytes += db[j];
    }
    st.part_bytes = 0;
    for (int j = 0; j < K; ++j)
        if (j != me) st.part_bytes += cnt[j] * (int64_t)(4 * es + 8);
    return FMM_OK;
}

// ------------------------------------------------------------------------------- C-ABI
extern "C" {

fmm_status fmm_group_create(int nranks, fmm_group** out) {
    if (nranks < 1 || nranks > 256 || !out) return FMM_ERR_ARG;
    fmm_group* g = new fmm_group();
    g->g.nranks = nranks;
    g->g.slots.resize(nranks);
    *out = g;
    return FMM_OK;
}

fmm_status fmm_group_destroy(fmm_group* g) {
    if (!g) return FMM_ERR_ARG;
    {
        std::lock_guard<std::mutex> lk(g->g.mu);
        if (g->g.nctx != 0) return FMM_ERR_STATE;
    }
    delete g;
    return FMM_OK;
}

fmm_status fmm_dist_unique_id(void* out) {
    if (!out) return FMM_ERR_ARG;
    std::string err;
    return nccl_unique_id(out, err);
}

fmm_status fmm_create_dist(int64_t n_local_max, int p, double theta, int ncrit, int prec, int device, int nranks,
                           int rank, const void* nccl_unique_id, fmm_group* group, int partitioner, fmm_ctx** out) {
    if (!out || nranks < 1 || nranks > 256 || rank < 0 || rank >= nranks || (!nccl_unique_id) == (!group) ||
        (partitioner != FMM_PART_MORTON && partitioner != FMM_PART_ORB) || (group && group->g.nranks != nranks))
        return FMM_ERR_ARG;
    fmm_ctx* ctx = nullptr;
    FMM_TRY(fmm_create(n_local_max, p, theta, ncrit, prec, device, &ctx));
    DeviceGuard g(device);
    DistState* D = new DistState();
    ctx->dist = D;
    D->K = nranks;
    D->rank = rank;
    D->partitioner = partitioner;
    D->c_m2l = m2l_cost_ratio(p);
    const char* e = getenv("FMM_DIST_SORT");
    D->overlap_sort = !(e && e[0] == '0');
    const char* e2 = getenv("FMM_DIST_SPLIT");
    D->split = e2 && e2[0] == '1';
    ctx->p2p_mutual = 0;   // the split flow runs P2P per list half (one-sided kernels)
    std::string err;
    fmm_status st = nccl_unique_id ? transport_nccl(nranks, rank, nccl_unique_id, device, &D->tr, err)
                                   : transport_local(&group->g, rank, device, &D->tr, err);
    if (st == FMM_OK) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        bool ok = cudaStreamCreateWithPriority(&D->cs, cudaStreamNonBlocking, hi) == cudaSuccess &&
                  cudaStreamCreateWithFlags(&D->side, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaStreamCreateWithFlags(&D->cx, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaEventCreate(&D->ev_t0) == cudaSuccess;
        for (auto& ev : D->ev) ok = ok && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess;
        for (auto& pr : D->tl)
            for (auto& ev : pr) ok = ok && cudaEventCreate(&ev) == cudaSuccess;
        if (!ok) {
            err = "stream/event creation failed";
            st = FMM_ERR_CUDA;
        }
    }
    if (st != FMM_OK) {
        // keep the message: the context is returned only on success
        fmm_destroy(ctx);
        (void)err;
        return st;
    }
    *out = ctx;
    return FMM_OK;
}

fmm_status fmm_set_weights(fmm_ctx* ctx, const float* w, int64_t n) {
    if (!ctx || !ctx->dist || n < 0) return FMM_ERR_ARG;
    DistState* D = ctx->dist;
    if (!w) {
        D->w_set_n = -1;
        return FMM_OK;
    }
    DeviceGuard g(ctx->device);
    FMM_TRY(buf_ensure(ctx, D->w_set, (size_t)std::max<int64_t>(n, 1) * 4));
    if (n) FMM_CUDA_TRY(ctx, cudaMemcpy(D->w_set.p, w, (size_t)n * 4, cudaMemcpyDefault));
    D->w_set_n = n;
    return FMM_OK;
}

fmm_status fmm_dist_set_alpha(fmm_ctx* ctx, double alpha, double c_m2l) {
    if (!ctx || !ctx->dist || !(alpha >= 0.0)) return FMM_ERR_ARG;
    ctx->dist->alpha = alpha;
    if (c_m2l > 0.0) ctx->dist->c_m2l = c_m2l;
    return FMM_OK;
}

fmm_status fmm_dist_tune_alpha(fmm_ctx* ctx, double lo, double hi, double tol) {
    if (!ctx || !ctx->dist) return FMM_ERR_ARG;
    DistState* D = ctx->dist;
    delete D->tuner;
    D->tuner = nullptr;
    if (lo <= 0.0 && hi <= 0.0) {   // off: keep the best alpha found
        return FMM_OK;
    }
    return fmm_alpha_tuner_create(lo, hi, tol, &D->tuner);
}

fmm_status fmm_dist_solve(fmm_ctx* ctx, const void* pos, const void* q, int64_t n, int64_t gid_base,
                          int reuse_weights, void* phi, void* grad, void* stream) {
    if (!ctx || !ctx->dist) return FMM_ERR_ARG;
    ctx->err.clear();
    if (n < 0 || (n > 0 && (!pos || !q || !phi || !grad)) || gid_base < 0) {
        ctx->err = "fmm_dist_solve: bad argument";
        return FMM_ERR_ARG;
    }
    DistState* D = ctx->dist;
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    const float* w = nullptr;
    if (reuse_weights && D->w_prev_n == n) w = P_<float>(D->w_prev);
    else if (D->w_set_n == n) w = P_<float>(D->w_set);
    std::chrono::steady_clock::time_point t0;
    if (D->tuner) {
        FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        t0 = std::chrono::steady_clock::now();
        D->alpha = D->tuner->next();   // for this step's weights
    }
    fmm_status st = dist_step(ctx, D, pos, q, n, gid_base, w, phi, grad, s);
    if (st != FMM_OK) {
        // the other ranks must not wait forever in a collective this rank will not reach
        D->tr->abort();
        return st;
    }
    if (D->tuner) {
        FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        FMM_TRY(buf_ensure(ctx, D->red, 64 * 8));
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(D->red.p, &t, 8, cudaMemcpyHostToDevice, s));
        FMM_TR(D->tr->allreduce_f64(P_<double>(D->red), 1, 2, s));   // runtime = max over ranks
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&t, D->red.p, 8, cudaMemcpyDeviceToHost, s));
        FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        D->tuner->report(t);
        D->st.tuner_probes = (int)D->tuner->history.size();
        D->st.tuner_converged = D->tuner->converged();
        D->st.tuner_best = D->tuner->best();
    }
    if (ctx->timing) {
        for (int i = 0; i < TL_COUNT; ++i) {
            if (!D->tl_rec[i]) {
                D->tl_ms[i][0] = D->tl_ms[i][1] = -1.0;
                continue;
            }
            float a = 0.f, b = 0.f;
            FMM_CUDA_TRY(ctx, cudaEventSynchronize(D->tl[i][1]));
            FMM_CUDA_TRY(ctx, cudaEventElapsedTime(&a, D->ev_t0, D->tl[i][0]));
            FMM_CUDA_TRY(ctx, cudaEventElapsedTime(&b, D->ev_t0, D->tl[i][1]));
            D->tl_ms[i][0] = a;
            D->tl_ms[i][1] = b;
        }
    }
    return FMM_OK;
}

fmm_status fmm_dist_get_stats(const fmm_ctx* ctx, fmm_dist_stats* out) {
    if (!ctx || !ctx->dist || !out) return FMM_ERR_ARG;
    *out = ctx->dist->st;
    return FMM_OK;
}

fmm_status fmm_dist_local(const fmm_ctx* ctx_c, int64_t* gid, int32_t* peers) {
    if (!ctx_c || !ctx_c->dist) return FMM_ERR_ARG;
    fmm_ctx* ctx = const_cast<fmm_ctx*>(ctx_c);
    DistState* D = ctx->dist;
    DeviceGuard g(ctx->device);
    if (gid && D->n_local) FMM_CUDA_TRY(ctx, cudaMemcpy(gid, D->l_gid.p, (size_t)D->n_local * 8, cudaMemcpyDeviceToHost));
    if (peers)
        for (int k = 0; k < D->K; ++k) peers[k] = k < (int)D->peers.size() ? D->peers[k] : -1;
    return FMM_OK;
}

fmm_status fmm_dist_weights(const fmm_ctx* ctx_c, float* w) {
    if (!ctx_c || !ctx_c->dist || !w) return FMM_ERR_ARG;
    fmm_ctx* ctx = const_cast<fmm_ctx*>(ctx_c);
    DistState* D = ctx->dist;
    if (D->w_prev_n < 0) return FMM_ERR_STATE;
    DeviceGuard g(ctx->device);
    if (D->w_prev_n) FMM_CUDA_TRY(ctx, cudaMemcpy(w, D->w_prev.p, (size_t)D->w_prev_n * 4, cudaMemcpyDeviceToHost));
    return FMM_OK;
}

fmm_status fmm_dist_orb_boxes(const fmm_ctx* ctx, int32_t* boxes) {
    if (!ctx || !ctx->dist || !boxes) return FMM_ERR_ARG;
    const DistState* D = ctx->dist;
    if (D->partitioner != FMM_PART_ORB || D->boxes.size() != (size_t)6 * D->K) return FMM_ERR_STATE;
    std::memcpy(boxes, D->boxes.data(), D->boxes.size() * 4);
    return FMM_OK;
}

fmm_status fmm_dist_timeline(const fmm_ctx* ctx, double* ms, int cap, int* n) {
    if (!ctx || !ctx->dist || !ms || !n) return FMM_ERR_ARG;
    *n = std::min(cap, (int)TL_COUNT);
    for (int i = 0; i < *n; ++i) {
        ms[2 * i] = ctx->dist->tl_ms[i][0];
        ms[2 * i + 1] = ctx->dist->tl_ms[i][1];
    }
    return FMM_OK;
}

const char* fmm_dist_timeline_name(int i) { return i >= 0 && i < TL_COUNT ? kTlNames[i] : ""; }

// ---- host logic, no device (CPU tests)
fmm_status fmm_splitters(int nranks, int bits, double tol, fmm_hist_fn fn, void* user, uint64_t* splitters) {
    if (nranks < 1 || nranks > 256 || bits < 1 || bits > 24 || !fn || (nranks > 1 && !splitters)) return FMM_ERR_ARG;
    auto hist = [&](const uint64_t* prefixes, int np, int pbits, int b, double* out) -> fmm_status {
        return fn(user, prefixes, np, pbits, b, out) == 0 ? FMM_OK : FMM_ERR_ARG;
    };
    return splitters_refine(nranks, bits, tol, hist, splitters);
}

fmm_status fmm_orb_plan(int nranks, int bits, fmm_orb_hist_fn hfn, fmm_orb_split_fn sfn, void* user, int32_t* boxes) {
    if (nranks < 1 || nranks > 256 || bits < 1 || bits >= COORD_BITS || !hfn || !sfn || !boxes) return FMM_ERR_ARG;
    auto hist = [&](const int32_t* axis, const uint32_t* prefix, int pbits, int b, double* out) -> fmm_status {
        return hfn(user, axis, prefix, pbits, b, out) == 0 ? FMM_OK : FMM_ERR_ARG;
    };
    auto split = [&](const int32_t* axis, const uint32_t* cut, const int32_t* right) -> fmm_status {
        return sfn(user, axis, cut, right) == 0 ? FMM_OK : FMM_ERR_ARG;
    };
    return orb_plan_t(nranks, bits, hist, split, boxes);
}

fmm_status fmm_alpha_tuner_create(double lo, double hi, double tol, fmm_alpha_tuner** out) {
    if (!out || !(lo > 0.0) || !(hi > lo) || !(tol > 0.0)) return FMM_ERR_ARG;
    fmm_alpha_tuner* t = new fmm_alpha_tuner();
    t->a = std::log(lo);
    t->b = std::log(hi);
    t->tol = tol;
    t->c = t->b - fmm_alpha_tuner::GR * (t->b - t->a);
    t->d = t->a + fmm_alpha_tuner::GR * (t->b - t->a);
    t->probe = t->c;
    *out = t;
    return FMM_OK;
}

double fmm_alpha_tuner_next(const fmm_alpha_tuner* t) { return t ? t->next() : NAN; }

fmm_status fmm_alpha_tuner_report(fmm_alpha_tuner* t, double runtime) {
    if (!t) return FMM_ERR_ARG;
    t->report(runtime);
    return FMM_OK;
}

fmm_status fmm_alpha_tuner_state(const fmm_alpha_tuner* t, int* converged, double* best, int* nhist, double* hist,
                                 int cap) {
    if (!t) return FMM_ERR_ARG;
    if (converged) *converged = t->converged();
    if (best) *best = t->best();
    if (nhist) *nhist = (int)t->history.size();
    if (hist)
        for (int i = 0; i < std::min(cap, (int)t->history.size()); ++i) {
            hist[2 * i] = t->history[i].first;
            hist[2 * i + 1] = t->history[i].second;
        }
    return FMM_OK;
}

fmm_status fmm_alpha_tuner_destroy(fmm_alpha_tuner* t) {
    delete t;
    return FMM_OK;
}

}  // extern "C"
