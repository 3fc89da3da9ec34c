// capi.cu -- the extern "C" boundary of libfmm (include/fmm.h): context, build, evaluate,
// introspection, timing.  Every step of the path runs in this library's kernels; there is
// no CPU fallback (a missing device is an FMM_ERR_CUDA).
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cmath>
#include <map>
#include <mutex>

#include "common.cuh"

#define FMM_VERSION 1

namespace {
const char* kPhaseNames[PH_COUNT] = {"bounds", "sort", "tree", "geometry", "dtt", "lists",
                                      "upward", "m2l", "p2p", "downward", "copy", "m2l_kernel", "p2p_kernel"};

fmm_status check_ctx(const fmm_ctx* ctx) { return ctx ? FMM_OK : FMM_ERR_ARG; }

}  // namespace

// ---- memory checking without compute-sanitizer (closed on this pool): with FMM_GUARD=1 every
// buffer a context allocates gets a 4 KiB guard zone after its usable bytes, filled with a
// pattern that fmm_debug_check verifies (out-of-bounds writes past any buffer end); with
// FMM_POISON=1 fresh allocations are filled with 0xFF bytes (NaN floats, huge indices), so a
// kernel reading memory no kernel wrote shows up as NaN / wrong structure in the parity tests.
constexpr size_t kGuardBytes = 4096;
constexpr unsigned char kGuardByte = 0xA5;
std::mutex g_guard_mu;
std::map<void*, size_t>& guard_registry() {   // device pointer -> usable bytes
    static std::map<void*, size_t> m;
    return m;
}

fmm_status buf_ensure(fmm_ctx* ctx, DevBuf& b, size_t bytes, bool keep, cudaStream_t s) {
    if (bytes <= b.bytes) return FMM_OK;
    void* p = nullptr;
    size_t nb = std::max(bytes, (size_t)256);
    cudaError_t e = cudaMalloc(&p, nb + (ctx->guard ? kGuardBytes : 0));
    if (e != cudaSuccess) {
        cudaGetLastError();
        ctx->err = "cudaMalloc(" + std::to_string(nb) + " B) failed: " + cudaGetErrorString(e);
        return FMM_ERR_OOM;
    }
    if (ctx->poison) FMM_CUDA_TRY(ctx, cudaMemsetAsync(p, 0xFF, nb, s));
    if (ctx->guard) {
        FMM_CUDA_TRY(ctx, cudaMemsetAsync((char*)p + nb, kGuardByte, kGuardBytes, s));
        std::lock_guard<std::mutex> lk(g_guard_mu);
        guard_registry()[p] = nb;
    }
    if (keep && b.p && b.bytes) {
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(p, b.p, b.bytes, cudaMemcpyDeviceToDevice, s));
        FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    }
    if (ctx->poison || ctx->guard) FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    buf_free(b);
    b.p = p;
    b.bytes = nb;
    return FMM_OK;
}

void buf_free(DevBuf& b) {
    if (b.p) {
        {
            std::lock_guard<std::mutex> lk(g_guard_mu);
            guard_registry().erase(b.p);
        }
        cudaFree(b.p);
    }
    b.p = nullptr;
    b.bytes = 0;
}

PhaseScope::PhaseScope(fmm_ctx* c, int ph, cudaStream_t st) : ctx(c), phase(ph), s(st) {
    if (!ctx->timing) return;
    if (ctx->event_pool.empty()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        ctx->event_pool.push_back(e);
    }
    a = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    cudaEventRecord(a, s);
}

PhaseScope::~PhaseScope() {
    if (!ctx->timing || !a) return;
    cudaEvent_t b;
    if (ctx->event_pool.empty()) cudaEventCreate(&b);
    else {
        b = ctx->event_pool.back();
        ctx->event_pool.pop_back();
    }
    cudaEventRecord(b, s);
    ctx->pending.push_back({phase, a, b});
}

extern "C" {

int fmm_version(void) { return FMM_VERSION; }

fmm_status fmm_create(int64_t n_max, int p, double theta, int ncrit, int prec, int device, fmm_ctx** out) {
    if (!out) return FMM_ERR_ARG;
    *out = nullptr;
    if (n_max < 0 || n_max >= ((int64_t)1 << 32) || p < 1 || p > FMM_MAXP || !(theta > 0.0 && theta < 1.0) ||
        ncrit < 1 || (prec != FMM_F32 && prec != FMM_F64))
        return FMM_ERR_ARG;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return FMM_ERR_CUDA;
    }
    fmm_ctx* ctx = new fmm_ctx();
    ctx->n_max = n_max;
    ctx->P = p;
    ctx->ncoef = ncoef_of(p);
    ctx->theta = theta;
    ctx->ncrit = ncrit;
    ctx->prec = prec;
    ctx->device = device;
    DeviceGuard g(device);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
        delete ctx;
        return FMM_ERR_CUDA;
    }
    ctx->num_sms = prop.multiProcessorCount;
    {
        const char* g = getenv("FMM_M2L_GENERIC");
        ctx->use_fast_m2l = !(g && g[0] == '1');
        const char* g2 = getenv("FMM_P2P_GENERIC");
        ctx->use_fast_p2p = !(g2 && g2[0] == '1');
        const char* g3 = getenv("FMM_P2P_VARIANT");
        ctx->p2p_variant = g3 ? atoi(g3) : 0;
        const char* gm = getenv("FMM_P2P_MUTUAL");
        ctx->p2p_mutual = gm ? atoi(gm) : 0;
        const char* g4 = getenv("FMM_OVERLAP");
        ctx->overlap = !(g4 && g4[0] == '0');
        const char* g5 = getenv("FMM_CANONICAL_M2L");
        ctx->canonical_m2l = !(g5 && g5[0] == '0');
        const char* g16 = getenv("FMM_TCT_SINGLE");
        ctx->tc_single = !(g16 && g16[0] == '0');
        const char* g17 = getenv("FMM_TCT_CAP");
        ctx->tc_scap = g17 ? atoi(g17) : 0;
        const char* g18 = getenv("FMM_TCT_TIGHT");
        ctx->tc_tight = g18 && g18[0] == '1';
        const char* g19 = getenv("FMM_TCT_SKIP");
        ctx->tc_force_skip = g19 && g19[0] == '1';
        const char* g21 = getenv("FMM_TREE_FAST");
        ctx->tree_fast = !(g21 && g21[0] == '0');
        const char* g22 = getenv("FMM_SORT_STAGED");
        ctx->sort_staged = g22 ? atoi(g22) : -1;
        const char* g15 = getenv("FMM_DTT");
        ctx->dtt_mode = (g15 && std::string(g15) == "bfs") ? 1 : 0;
        const char* g7 = getenv("FMM_LIST_SORT");
        ctx->list_sort = g7 ? atoi(g7) : 0;
        const char* g6 = getenv("FMM_M2L_VARIANT");
        ctx->m2l_variant = g6 ? atoi(g6) : 0;
        const char* gg = getenv("FMM_GUARD");
        ctx->guard = gg && gg[0] == '1';
        const char* gp = getenv("FMM_POISON");
        ctx->poison = gp && gp[0] == '1';
    }
    if (cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_up, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_done, cudaEventDisableTiming) != cudaSuccess) {
        delete ctx;
        return FMM_ERR_CUDA;
    }
    {
        const char* g11 = getenv("FMM_PRIO");
        int lo = 0, hi = 0;
        if (!(g11 && g11[0] == '0') && cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess && hi < lo) {
            if (cudaStreamCreateWithPriority(&ctx->hp, cudaStreamNonBlocking, hi) != cudaSuccess) ctx->hp = nullptr;
        }
    }
    *out = ctx;
    return FMM_OK;
}

fmm_status fmm_destroy(fmm_ctx* ctx) {
    if (!ctx) return FMM_ERR_ARG;
    DeviceGuard g(ctx->device);
    cudaDeviceSynchronize();
    if (ctx->dist) dist_destroy(ctx->dist);
    ctx->dist = nullptr;
    DevBuf* bufs[] = {&ctx->root, &ctx->key_a, &ctx->key_b, &ctx->idx_a, &ctx->idx_b, &ctx->sort_counts,
                      &ctx->scan_tmp, &ctx->red_tmp, &ctx->body, &ctx->c_key, &ctx->c_level, &ctx->c_bb,
                      &ctx->c_bc, &ctx->c_cb, &ctx->c_cc, &ctx->c_parent, &ctx->c_bmin, &ctx->c_bmax, &ctx->c_cr,
                      &ctx->split_tmp, &ctx->split_cnt, &ctx->leaf_ids, &ctx->fr_a, &ctx->fr_b, &ctx->lst_m2l,
                      &ctx->lst_p2p, &ctx->lst_tmp, &ctx->m2l_src, &ctx->p2p_src, &ctx->m2l_off, &ctx->p2p_off,
                      &ctx->cnt_tmp, &ctx->cnt_tmp2, &ctx->dcount, &ctx->runs, &ctx->run_off, &ctx->run_tmp, &ctx->run_pre,
                      &ctx->run_len64, &ctx->dcount2, &ctx->tcnt, &ctx->cnt64, &ctx->big_off, &ctx->M, &ctx->L, &ctx->Mr, &ctx->Lr, &ctx->near_phi, &ctx->near_grad,
                      &ctx->far, &ctx->h_stage, &ctx->mut_mir, &ctx->mut_w, &ctx->mut_so, &ctx->mut_slot, &ctx->iperm, &ctx->m2l_mix};
    for (DevBuf* b : bufs) buf_free(*b);
    DevBuf* tbufs[] = {&ctx->tc_cnt, &ctx->tc_voff, &ctx->tc_lb, &ctx->tc_d[0], &ctx->tc_d[1], &ctx->tc_doff[0],
                       &ctx->tc_doff[1], &ctx->tc_glob, &ctx->tc_slab, &ctx->tc_bsum, &ctx->tc_cat_off,
                       &ctx->tc_cat_src, &ctx->tc_rec, &ctx->tree_lb, &ctx->tc_mixflag};
    for (auto& pt : ctx->tc_rem) {
        DevBuf* pb[] = {&pt.off_m, &pt.src_m, &pt.off_p, &pt.src_p};
        for (DevBuf* b : pb) buf_free(*b);
    }
    for (DevBuf* b : tbufs) buf_free(*b);
    DevBuf* lbufs[] = {&ctx->let_tmp, &ctx->let_cov, &ctx->c_orig, &ctx->part_tmp, &ctx->seg_lists, &ctx->orb_tmp, &ctx->root_given, &ctx->fold_tab, &ctx->leaf_cls, &ctx->dtt_lvl};
    for (DevBuf* b : lbufs) buf_free(*b);
    for (auto& lp : ctx->let_peers) {
        DevBuf* pb[] = {&lp.opened, &lp.eflag, &lp.eidx, &lp.bflag, &lp.boff};
        for (DevBuf* b : pb) buf_free(*b);
    }
    for (auto& t : ctx->pending) {
        cudaEventDestroy(t.a);
        cudaEventDestroy(t.b);
    }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    if (ctx->aux) cudaStreamDestroy(ctx->aux);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->ev_up) cudaEventDestroy(ctx->ev_up);
    if (ctx->ev_done) cudaEventDestroy(ctx->ev_done);
    if (ctx->hp) cudaStreamDestroy(ctx->hp);
    delete ctx;
    return FMM_OK;
}

const char* fmm_last_error(const fmm_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

fmm_status fmm_build_tree(fmm_ctx* ctx, const void* pos, int64_t n, void* stream) {
    FMM_TRY(check_ctx(ctx));
    ctx->err.clear();
    if (n < 0 || n > ctx->n_max) {
        ctx->err = "fmm_build: n out of range";
        return FMM_ERR_ARG;
    }
    if (n > 0 && !pos) {
        ctx->err = "fmm_build: null pos";
        return FMM_ERR_ARG;
    }
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    ctx->built = ctx->tree_built = false;
    ctx->lists_csr = false;
    ctx->tc_mix_ncell = -1;
    ctx->tc_nrem = 0;
    ctx->evaluated = ctx->upward_done = false;
    ctx->n = n;
    ctx->built_pos = pos;
    ctx->ncell = ctx->nleaf = ctx->depth = ctx->n_m2l = ctx->n_p2p = ctx->p2p_inter = 0;
    ctx->nrem = ctx->nrem_body = 0;
    ctx->let_remote.clear();
    ctx->let_traversed = 0;
    for (auto& lp : ctx->let_peers) lp.planned = false;
    ctx->level_begin.clear();
    if (n > 0) {
        FMM_TRY(build_keys(ctx, pos, n, s));
        FMM_TRY(build_tree(ctx, s));
    }
    ctx->tree_built = true;
    return FMM_OK;
}

fmm_status fmm_set_root_bounds(fmm_ctx* ctx, const double* bounds) {
    FMM_TRY(check_ctx(ctx));
    if (!bounds) {
        ctx->has_root_bounds = false;
        return FMM_OK;
    }
    for (int d = 0; d < 3; ++d)
        if (!std::isfinite(bounds[d]) || !std::isfinite(bounds[3 + d]) || bounds[d] > bounds[3 + d]) return FMM_ERR_ARG;
    for (int d = 0; d < 6; ++d) ctx->root_bounds[d] = bounds[d];
    ctx->has_root_bounds = true;
    return FMM_OK;
}

fmm_status fmm_dtt(fmm_ctx* ctx, int remote, void* stream) {
    FMM_TRY(check_ctx(ctx));
    ctx->err.clear();
    if (!ctx->tree_built) {
        ctx->err = "fmm_dtt: no tree (fmm_build_tree first)";
        return FMM_ERR_STATE;
    }
    ctx->built = ctx->evaluated = false;
    if (ctx->n == 0) return FMM_OK;
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    if (!remote) {
        ctx->lists_csr = false;
        ctx->tc_mix_ncell = -1;   // set again by the target-ordered traversal
        if (ctx->dtt_mode == 0) {
            PhaseScope ps(ctx, PH_DTT, s);
            FMM_TRY(tct_lists(ctx, s));
            ctx->lists_csr = true;
            return FMM_OK;
        }
        const uint64_t root_pair = 0;
        return dtt_pass(ctx, &root_pair, 1, false, s, -1);
    }
    if (ctx->lists_csr) {
        // target-ordered: one more CSR part per batch of grafted LETs (concatenated by fmm_lists)
        std::vector<uint32_t> roots;
        for (size_t k = ctx->let_traversed; k < ctx->let_remote.size(); ++k)
            if (ctx->let_remote[k].ncell > 0) roots.push_back((uint32_t)ctx->let_remote[k].base);
        ctx->let_traversed = ctx->let_remote.size();
        if (roots.empty()) return FMM_OK;
        PhaseScope ps(ctx, PH_DTT, s);
        return tct_remote(ctx, roots, s);
    }
    // (local root 0, remote root) of every LET grafted since the last remote traversal
    std::vector<uint64_t> seeds;
    int dmax = 0;
    for (size_t k = ctx->let_traversed; k < ctx->let_remote.size(); ++k)
        if (ctx->let_remote[k].ncell > 0) {
            seeds.push_back((uint64_t)ctx->let_remote[k].base);
            dmax = std::max(dmax, ctx->let_remote[k].depth);
        }
    ctx->let_traversed = ctx->let_remote.size();
    if (seeds.empty()) return FMM_OK;
    return dtt_pass(ctx, seeds.data(), (int)seeds.size(), true, s, dmax);
}

fmm_status fmm_lists(fmm_ctx* ctx, void* stream) {
    FMM_TRY(check_ctx(ctx));
    ctx->err.clear();
    if (!ctx->tree_built) {
        ctx->err = "fmm_lists: no tree (fmm_build_tree first)";
        return FMM_ERR_STATE;
    }
    DeviceGuard g(ctx->device);
    if (ctx->n > 0) FMM_TRY(lists_pass(ctx, (cudaStream_t)stream));
    ctx->built = true;
    return FMM_OK;
}

fmm_status fmm_build(fmm_ctx* ctx, const void* pos, int64_t n, void* stream) {
    FMM_TRY(fmm_build_tree(ctx, pos, n, stream));
    FMM_TRY(fmm_dtt(ctx, 0, stream));
    return fmm_lists(ctx, stream);
}

fmm_status fmm_upward(fmm_ctx* ctx, const void* pos, const void* q, void* stream) {
    FMM_TRY(check_ctx(ctx));
    ctx->err.clear();
    if (!ctx->tree_built || pos != ctx->built_pos) {
        ctx->err = "fmm_upward: no matching fmm_build for these positions";
        return FMM_ERR_STATE;
    }
    ctx->evaluated = false;
    if (ctx->n == 0) {
        ctx->upward_done = true;
        return FMM_OK;
    }
    if (!q) {
        ctx->err = "fmm_upward: null pointer";
        return FMM_ERR_ARG;
    }
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    FMM_TRY(gather_bodies_q(ctx, q, s));
    FMM_TRY(upward_pass(ctx, s));
    ctx->upward_done = true;
    return FMM_OK;
}

fmm_status fmm_interact(fmm_ctx* ctx, void* phi, void* grad, void* stream) {
    FMM_TRY(check_ctx(ctx));
    ctx->err.clear();
    if (!ctx->built || !ctx->upward_done) {
        ctx->err = "fmm_interact: needs fmm_lists and fmm_upward first";
        return FMM_ERR_STATE;
    }
    if (ctx->n == 0) return FMM_OK;
    if (!phi || !grad) {
        ctx->err = "fmm_interact: null pointer";
        return FMM_ERR_ARG;
    }
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    FMM_TRY(m2l_pass(ctx, s));
    if (!ctx->overlap) {
        FMM_TRY(p2p_pass(ctx, s));
        FMM_TRY(downward_pass(ctx, phi, grad, s));
    } else {
        // L2L/L2P (level-synchronous, latency-bound) on the aux stream while P2P fills the GPU;
        // the far field waits in ctx->far and the merge adds the P2P partials
        FMM_CUDA_TRY(ctx, cudaEventRecord(ctx->ev_fork, s));
        FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->aux, ctx->ev_fork, 0));
        FMM_TRY(downward_far(ctx, ctx->aux));
        FMM_CUDA_TRY(ctx, cudaEventRecord(ctx->ev_join, ctx->aux));
        FMM_TRY(p2p_pass(ctx, s));
        FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_join, 0));
        FMM_TRY(merge_nearfar(ctx, phi, grad, s));
    }
    ctx->evaluated = true;
    return FMM_OK;
}

fmm_status fmm_evaluate(fmm_ctx* ctx, const void* pos, const void* q, void* phi, void* grad, void* stream) {
    FMM_TRY(check_ctx(ctx));
    if (!ctx->built || pos != ctx->built_pos) {
        ctx->err = "fmm_evaluate: no matching fmm_build for these positions";
        return FMM_ERR_STATE;
    }
    if (ctx->n > 0 && (!q || !phi || !grad)) {
        ctx->err = "fmm_evaluate: null pointer";
        return FMM_ERR_ARG;
    }
    FMM_TRY(fmm_upward(ctx, pos, q, stream));
    return fmm_interact(ctx, phi, grad, stream);
}

fmm_status fmm_solve(fmm_ctx* ctx, const void* pos, const void* q, int64_t n, void* phi, void* grad, void* stream) {
    FMM_TRY(check_ctx(ctx));
    if (n > 0 && (!q || !phi || !grad)) {
        ctx->err = "fmm_solve: null pointer";
        return FMM_ERR_ARG;
    }
    if (n == 0 || !ctx->overlap) {
        FMM_TRY(fmm_build_tree(ctx, pos, n, stream));
        FMM_TRY(fmm_dtt(ctx, 0, stream));
        FMM_TRY(fmm_lists(ctx, stream));
        return fmm_evaluate(ctx, pos, q, phi, grad, stream);
    }
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    // the critical path runs on the library's high-priority stream (joined back into `stream`
    // at the end), the aux stream has the lowest priority: its blocks only take SM slots the
    // critical path leaves free
    cudaStream_t m = ctx->hp ? ctx->hp : s;
    if (m != s) {
        FMM_CUDA_TRY(ctx, cudaEventRecord(ctx->ev_fork, s));
        FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(m, ctx->ev_fork, 0));
    }
    FMM_TRY(fmm_build_tree(ctx, pos, n, m));
    // P2M/M2M need the tree and q only: on the aux stream while the traversal and the list
    // grouping (latency-bound, with host round trips) run on the critical-path stream
    FMM_CUDA_TRY(ctx, cudaEventRecord(ctx->ev_fork, m));
    FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->aux, ctx->ev_fork, 0));
    FMM_TRY(gather_bodies_q(ctx, q, ctx->aux));
    FMM_TRY(upward_pass(ctx, ctx->aux));
    ctx->m2l_part = 1;   // the M2L operand (fp32 folded copy of M) is prepared there too
    fmm_status st = m2l_pass(ctx, ctx->aux);
    ctx->m2l_part = 0;
    FMM_TRY(st);
    FMM_CUDA_TRY(ctx, cudaEventRecord(ctx->ev_up, ctx->aux));
    FMM_TRY(fmm_dtt(ctx, 0, m));
    FMM_TRY(fmm_lists(ctx, m));
    FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(m, ctx->ev_up, 0));
    ctx->upward_done = true;
    ctx->m2l_part = 2;
    st = fmm_interact(ctx, phi, grad, m);
    ctx->m2l_part = 0;
    FMM_TRY(st);
    if (m != s) {
        FMM_CUDA_TRY(ctx, cudaEventRecord(ctx->ev_done, m));
        FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(s, ctx->ev_done, 0));
    }
    return FMM_OK;
}

// ---- multi-GPU: LET (let.cu)
fmm_status fmm_let_cover(fmm_ctx* ctx, double* cover, int* ncover, void* stream) {
    FMM_TRY(check_ctx(ctx));
    ctx->err.clear();
    if (!cover || !ncover) return FMM_ERR_ARG;
    if (!ctx->tree_built) return FMM_ERR_STATE;
    DeviceGuard g(ctx->device);
    return let_cover(ctx, cover, ncover, (cudaStream_t)stream);
}

fmm_status fmm_let_plan(fmm_ctx* ctx, int peer, const double* cover, int ncover, int64_t* struct_bytes,
                        int64_t* data_bytes, void* stream) {
    FMM_TRY(check_ctx(ctx));
    ctx->err.clear();
    if (peer < 0 || ncover < 0 || ncover > FMM_LET_MAX_COVER || (ncover > 0 && !cover) || !struct_bytes ||
        !data_bytes)
        return FMM_ERR_ARG;
    if (!ctx->tree_built) return FMM_ERR_STATE;
    DeviceGuard g(ctx->device);
    if (ctx->n == 0) {
        if ((int)ctx->let_peers.size() <= peer) ctx->let_peers.resize(peer + 1);
        ctx->let_peers[peer].ncell = ctx->let_peers[peer].nbody = 0;
        ctx->let_peers[peer].planned = false;
        *struct_bytes = *data_bytes = 0;
        return FMM_OK;
    }
    return let_plan(ctx, peer, cover, ncover, struct_bytes, data_bytes, (cudaStream_t)stream);
}

fmm_status fmm_let_pack_struct(fmm_ctx* ctx, int peer, void* dst, void* stream) {
    FMM_TRY(check_ctx(ctx));
    ctx->err.clear();
    if (!dst) return FMM_ERR_ARG;
    DeviceGuard g(ctx->device);
    return let_pack(ctx, peer, 0, dst, (cudaStream_t)stream);
}

fmm_status fmm_let_pack_data(fmm_ctx* ctx, int peer, void* dst, void* stream) {
    FMM_TRY(check_ctx(ctx));
    ctx->err.clear();
    if (!dst) return FMM_ERR_ARG;
    DeviceGuard g(ctx->device);
    return let_pack(ctx, peer, 1, dst, (cudaStream_t)stream);
}

fmm_status fmm_let_graft(fmm_ctx* ctx, int npeers, const void* const* src, const int64_t* bytes, void* stream) {
    FMM_TRY(check_ctx(ctx));
    ctx->err.clear();
    if (npeers < 0 || (npeers > 0 && (!src || !bytes))) return FMM_ERR_ARG;
    if (!ctx->tree_built) return FMM_ERR_STATE;
    if (ctx->n == 0) return FMM_OK;
    DeviceGuard g(ctx->device);
    ctx->built = ctx->evaluated = false;
    return let_graft(ctx, npeers, src, bytes, (cudaStream_t)stream);
}

fmm_status fmm_let_unpack(fmm_ctx* ctx, int first, int npeers, const void* const* src, const int64_t* bytes,
                          void* stream) {
    FMM_TRY(check_ctx(ctx));
    ctx->err.clear();
    if (first < 0 || npeers < 0 || (npeers > 0 && (!src || !bytes))) return FMM_ERR_ARG;
    if (ctx->n == 0) return FMM_OK;
    DeviceGuard g(ctx->device);
    return let_unpack(ctx, first, npeers, src, bytes, (cudaStream_t)stream);
}

fmm_status fmm_let_remote(const fmm_ctx* ctx_c, int k, int64_t* base, int64_t* ncell, int64_t* nbody, uint32_t* orig) {
    FMM_TRY(check_ctx(ctx_c));
    fmm_ctx* ctx = const_cast<fmm_ctx*>(ctx_c);
    if (k < 0 || k >= (int)ctx->let_remote.size()) return FMM_ERR_ARG;
    const LetRemote& r = ctx->let_remote[k];
    if (base) *base = r.base;
    if (ncell) *ncell = r.ncell;
    if (nbody) *nbody = r.nbody;
    if (orig && r.ncell) {
        DeviceGuard g(ctx->device);
        FMM_CUDA_TRY(ctx, cudaDeviceSynchronize());
        FMM_CUDA_TRY(ctx, cudaMemcpy(orig, P_<uint32_t>(ctx->c_orig) + r.base, r.ncell * 4, cudaMemcpyDeviceToHost));
    }
    return FMM_OK;
}

fmm_status fmm_solve_host(fmm_ctx* ctx, const void* pos_h, const void* q_h, int64_t n, void* phi_h, void* grad_h,
                          void* stream) {
    FMM_TRY(check_ctx(ctx));
    if (n < 0 || n > ctx->n_max || (n > 0 && (!pos_h || !q_h || !phi_h || !grad_h))) return FMM_ERR_ARG;
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t es = ctx->prec == FMM_F32 ? 4 : 8;
    const size_t bpos = (size_t)n * 3 * es, bq = (size_t)n * es;
    // staging: pos | q | phi | grad, each 256-B aligned
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    FMM_TRY(buf_ensure(ctx, ctx->h_stage, al(bpos) * 2 + al(bq) * 2 + 1024));
    char* base = (char*)ctx->h_stage.p;
    void* dpos = base;
    void* dq = base + al(bpos);
    void* dphi = base + al(bpos) + al(bq);
    void* dgrad = base + al(bpos) + 2 * al(bq);
    {
        PhaseScope ps(ctx, PH_COPY, s);
        if (n) FMM_CUDA_TRY(ctx, cudaMemcpyAsync(dpos, pos_h, bpos, cudaMemcpyHostToDevice, s));
        if (n && ctx->overlap) {
            // q is first needed by P2M on the aux stream: copy it there, behind the caller's
            // earlier work, while the tree is built from the positions
            FMM_CUDA_TRY(ctx, cudaEventRecord(ctx->ev_fork, s));
            FMM_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->aux, ctx->ev_fork, 0));
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync(dq, q_h, bq, cudaMemcpyHostToDevice, ctx->aux));
        } else if (n) {
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync(dq, q_h, bq, cudaMemcpyHostToDevice, s));
        }
    }
    FMM_TRY(fmm_solve(ctx, dpos, dq, n, dphi, dgrad, stream));
    {
        PhaseScope ps(ctx, PH_COPY, s);
        if (n) FMM_CUDA_TRY(ctx, cudaMemcpyAsync(phi_h, dphi, bq, cudaMemcpyDeviceToHost, s));
        if (n) FMM_CUDA_TRY(ctx, cudaMemcpyAsync(grad_h, dgrad, bpos, cudaMemcpyDeviceToHost, s));
    }
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    return FMM_OK;
}

fmm_status fmm_get_counts(const fmm_ctx* ctx, fmm_counts* out) {
    FMM_TRY(check_ctx(ctx));
    if (!out) return FMM_ERR_ARG;
    out->n = ctx->n;
    out->ncell = ctx->ncell;
    out->nleaf = ctx->nleaf;
    out->depth = ctx->depth;
    out->n_m2l = ctx->n_m2l;
    out->n_p2p = ctx->n_p2p;
    if (ctx->p2p_inter < 0) {   // counted by the P2P run builder on the device; read once
        fmm_ctx* c = const_cast<fmm_ctx*>(ctx);
        DeviceGuard g(c->device);
        unsigned long long v = 0;
        FMM_CUDA_TRY(c, cudaDeviceSynchronize());
        FMM_CUDA_TRY(c, cudaMemcpy(&v, P_<unsigned long long>(c->dcount2) + 2, 8, cudaMemcpyDeviceToHost));
        c->p2p_inter = (int64_t)v;
    }
    out->p2p_interactions = ctx->p2p_inter;
    return FMM_OK;
}

fmm_status fmm_copy_sorted(const fmm_ctx* ctx_c, uint64_t* keys, uint32_t* perm) {
    FMM_TRY(check_ctx(ctx_c));
    fmm_ctx* ctx = const_cast<fmm_ctx*>(ctx_c);
    if (!ctx->built) return FMM_ERR_STATE;
    DeviceGuard g(ctx->device);
    FMM_CUDA_TRY(ctx, cudaDeviceSynchronize());
    if (ctx->n == 0) return FMM_OK;
    if (keys) FMM_CUDA_TRY(ctx, cudaMemcpy(keys, ctx->d_keys, ctx->n * 8, cudaMemcpyDeviceToHost));
    if (perm) FMM_CUDA_TRY(ctx, cudaMemcpy(perm, ctx->d_perm, ctx->n * 4, cudaMemcpyDeviceToHost));
    return FMM_OK;
}

fmm_status fmm_copy_cells(const fmm_ctx* ctx_c, int32_t* level, uint64_t* key, uint32_t* body_begin,
                          uint32_t* body_count, uint32_t* child_begin, uint32_t* child_count, int32_t* parent,
                          double* bmin, double* bmax, double* center, double* radius) {
    FMM_TRY(check_ctx(ctx_c));
    fmm_ctx* ctx = const_cast<fmm_ctx*>(ctx_c);
    if (!ctx->built) return FMM_ERR_STATE;
    DeviceGuard g(ctx->device);
    FMM_CUDA_TRY(ctx, cudaDeviceSynchronize());
    const int64_t nc = ctx->ncell;
    if (nc == 0) return FMM_OK;
    if (level) FMM_CUDA_TRY(ctx, cudaMemcpy(level, ctx->c_level.p, nc * 4, cudaMemcpyDeviceToHost));
    if (key) FMM_CUDA_TRY(ctx, cudaMemcpy(key, ctx->c_key.p, nc * 8, cudaMemcpyDeviceToHost));
    if (body_begin) FMM_CUDA_TRY(ctx, cudaMemcpy(body_begin, ctx->c_bb.p, nc * 4, cudaMemcpyDeviceToHost));
    if (body_count) FMM_CUDA_TRY(ctx, cudaMemcpy(body_count, ctx->c_bc.p, nc * 4, cudaMemcpyDeviceToHost));
    if (child_begin) FMM_CUDA_TRY(ctx, cudaMemcpy(child_begin, ctx->c_cb.p, nc * 4, cudaMemcpyDeviceToHost));
    if (child_count) FMM_CUDA_TRY(ctx, cudaMemcpy(child_count, ctx->c_cc.p, nc * 4, cudaMemcpyDeviceToHost));
    if (parent) FMM_CUDA_TRY(ctx, cudaMemcpy(parent, ctx->c_parent.p, nc * 4, cudaMemcpyDeviceToHost));
    if (bmin) FMM_CUDA_TRY(ctx, cudaMemcpy(bmin, ctx->c_bmin.p, nc * 24, cudaMemcpyDeviceToHost));
    if (bmax) FMM_CUDA_TRY(ctx, cudaMemcpy(bmax, ctx->c_bmax.p, nc * 24, cudaMemcpyDeviceToHost));
    if (center || radius) {
        std::vector<double> cr((size_t)nc * 4);
        FMM_CUDA_TRY(ctx, cudaMemcpy(cr.data(), ctx->c_cr.p, nc * 32, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < nc; ++i) {
            if (center)
                for (int d = 0; d < 3; ++d) center[3 * i + d] = cr[4 * i + d];
            if (radius) radius[i] = cr[4 * i + 3];
        }
    }
    return FMM_OK;
}

fmm_status fmm_copy_lists(const fmm_ctx* ctx_c, uint32_t* m2l, uint32_t* p2p) {
    FMM_TRY(check_ctx(ctx_c));
    fmm_ctx* ctx = const_cast<fmm_ctx*>(ctx_c);
    if (!ctx->built) return FMM_ERR_STATE;
    DeviceGuard g(ctx->device);
    FMM_CUDA_TRY(ctx, cudaDeviceSynchronize());
    struct {
        uint32_t* dst;
        DevBuf* off;
        DevBuf* src;
        int64_t n;
    } jobs[2] = {{m2l, &ctx->m2l_off, &ctx->m2l_src, ctx->n_m2l}, {p2p, &ctx->p2p_off, &ctx->p2p_src, ctx->n_p2p}};
    for (auto& j : jobs) {
        if (!j.dst || j.n == 0) continue;
        std::vector<uint64_t> off((size_t)ctx->ncell + 1);
        std::vector<uint32_t> src((size_t)j.n);
        FMM_CUDA_TRY(ctx, cudaMemcpy(off.data(), j.off->p, off.size() * 8, cudaMemcpyDeviceToHost));
        FMM_CUDA_TRY(ctx, cudaMemcpy(src.data(), j.src->p, src.size() * 4, cudaMemcpyDeviceToHost));
        for (int64_t t = 0; t < ctx->ncell; ++t) {
            std::sort(src.begin() + off[t], src.begin() + off[t + 1]);   // canonical (target, source) order
            for (uint64_t p = off[t]; p < off[t + 1]; ++p) {
                j.dst[2 * p] = (uint32_t)t;
                j.dst[2 * p + 1] = src[p];
            }
        }
    }
    return FMM_OK;
}

fmm_status fmm_copy_expansions(const fmm_ctx* ctx_c, double* M, double* L) {
    FMM_TRY(check_ctx(ctx_c));
    fmm_ctx* ctx = const_cast<fmm_ctx*>(ctx_c);
    if (!ctx->evaluated) return FMM_ERR_STATE;
    DeviceGuard g(ctx->device);
    FMM_CUDA_TRY(ctx, cudaDeviceSynchronize());
    size_t sz = (size_t)ctx->ncell * ctx->ncoef * 8;
    if (M && sz) FMM_CUDA_TRY(ctx, cudaMemcpy(M, ctx->M.p, sz, cudaMemcpyDeviceToHost));
    if (L && sz) FMM_CUDA_TRY(ctx, cudaMemcpy(L, ctx->L.p, sz, cudaMemcpyDeviceToHost));
    return FMM_OK;
}

fmm_status fmm_debug_check(fmm_ctx* ctx, int64_t* nbad) {
    FMM_TRY(check_ctx(ctx));
    DeviceGuard g(ctx->device);
    FMM_CUDA_TRY(ctx, cudaDeviceSynchronize());
    int64_t bad = 0, checked = 0;
    std::vector<unsigned char> h(kGuardBytes);
    std::lock_guard<std::mutex> lk(g_guard_mu);
    for (const auto& kv : guard_registry()) {
        cudaPointerAttributes a;
        if (cudaPointerGetAttributes(&a, kv.first) != cudaSuccess || a.device != ctx->device) {
            cudaGetLastError();
            continue;
        }
        FMM_CUDA_TRY(ctx, cudaMemcpy(h.data(), (char*)kv.first + kv.second, kGuardBytes, cudaMemcpyDeviceToHost));
        ++checked;
        for (unsigned char c : h)
            if (c != kGuardByte) {
                ++bad;
                break;
            }
    }
    if (nbad) *nbad = bad;
    if (bad) {
        ctx->err = "fmm_debug_check: " + std::to_string(bad) + " of " + std::to_string(checked) +
                   " guarded buffers written past their end";
        return FMM_ERR_STATE;
    }
    return FMM_OK;
}

fmm_status fmm_set_timing(fmm_ctx* ctx, int enable) {
    FMM_TRY(check_ctx(ctx));
    ctx->timing = enable != 0;
    return FMM_OK;
}

fmm_status fmm_phase_times(fmm_ctx* ctx, double* ms, int cap, int* n, int reset) {
    FMM_TRY(check_ctx(ctx));
    DeviceGuard g(ctx->device);
    for (auto& t : ctx->pending) {
        FMM_CUDA_TRY(ctx, cudaEventSynchronize(t.b));
        float e = 0.f;
        FMM_CUDA_TRY(ctx, cudaEventElapsedTime(&e, t.a, t.b));
        ctx->phase_ms[t.phase] += e;
        ctx->event_pool.push_back(t.a);
        ctx->event_pool.push_back(t.b);
    }
    ctx->pending.clear();
    if (ms)
        for (int i = 0; i < cap && i < PH_COUNT; ++i) ms[i] = ctx->phase_ms[i];
    if (n) *n = PH_COUNT;
    if (reset)
        for (int i = 0; i < PH_COUNT; ++i) ctx->phase_ms[i] = 0.0;
    return FMM_OK;
}

const char* fmm_phase_name(int phase) { return (phase >= 0 && phase < PH_COUNT) ? kPhaseNames[phase] : ""; }

int64_t fmm_launch_count(fmm_ctx* ctx, int reset) {
    if (!ctx) return -1;
    int64_t v = ctx->launches;
    if (reset) ctx->launches = 0;
    return v;
}

}  // extern "C"
