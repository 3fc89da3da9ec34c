// debug.cu -- stage entry points on a CALLER-SUPPLIED tree and interaction list (SURVEY.md
// §8(b) "debug stage entry points: run P2P / M2L on caller-supplied tree + lists"): the hot
// kernels of fmm_evaluate (P2P: the leaf-class TMA/cp.async kernels with their source runs;
// M2L: the register kernels with their fp32 operand preparation) run on the view's data, so
// the parity tests can feed them the ORACLE's tree and lists and compare stage by stage.
//   P2P (R17, §II-A "P2P"), M2L (R14, "M2L").
#include "common.cuh"

namespace {

template <typename Real, typename Body>
__global__ void k_dbg_pack_bodies(int64_t n, const Real* __restrict__ pos, const Real* __restrict__ q,
                                  Body* __restrict__ body) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Body b;
    b.x = pos[3 * i];
    b.y = pos[3 * i + 1];
    b.z = pos[3 * i + 2];
    b.w = q[i];
    body[i] = b;
}

// per-target list lengths of (target, source) pairs sorted by target; flags a pair out of order
// or out of range
__global__ void k_dbg_count(int64_t npairs, const uint32_t* __restrict__ pairs, int64_t ncell,
                            uint64_t* __restrict__ cnt, unsigned* __restrict__ bad) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= npairs) return;
    const uint32_t t = pairs[2 * k], s = pairs[2 * k + 1];
    if (t >= ncell || s >= ncell) {
        atomicOr(bad, 1u);
        return;
    }
    if (k > 0) {
        const uint32_t tp = pairs[2 * k - 2], sp = pairs[2 * k - 1];
        if (tp > t || (tp == t && sp >= s)) atomicOr(bad, 2u);   // not ascending (target, source)
    }
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt + t), 1ull);
}

__global__ void k_dbg_src(int64_t npairs, const uint32_t* __restrict__ pairs, uint32_t* __restrict__ src) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < npairs) src[k] = pairs[2 * k + 1];
}

__global__ void k_dbg_leaf_flags(int64_t ncell, const uint32_t* __restrict__ cc, uint32_t* __restrict__ flag) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < ncell) flag[c] = cc[c] == 0 ? 1u : 0u;
}

__global__ void k_dbg_leaf_compact(int64_t ncell, const uint32_t* __restrict__ cc, const uint32_t* __restrict__ off,
                                   uint32_t* __restrict__ leaf_ids) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < ncell && cc[c] == 0) leaf_ids[off[c]] = (uint32_t)c;
}

__global__ void k_dbg_cr(int64_t ncell, const double* __restrict__ center, double4* __restrict__ cr) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < ncell) cr[c] = make_double4(center[3 * c], center[3 * c + 1], center[3 * c + 2], 0.0);
}

unsigned blocks(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>((n + t - 1) / t, 1); }

// the view's pairs -> ctx CSR (off[ncell+1] u64, src u32); FMM_ERR_ARG when unsorted / out of range
fmm_status load_pairs(fmm_ctx* ctx, const uint32_t* pairs, int64_t npairs, DevBuf& off, DevBuf& src, cudaStream_t s) {
    const int64_t nc = ctx->ncell;
    FMM_TRY(buf_ensure(ctx, off, (size_t)(nc + 1) * 8));
    FMM_TRY(buf_ensure(ctx, src, (size_t)std::max<int64_t>(npairs, 1) * 4));
    FMM_TRY(buf_ensure(ctx, ctx->cnt64, (size_t)(nc + 1) * 8 + 64));
    uint64_t* cnt = P_<uint64_t>(ctx->cnt64);
    unsigned* bad = reinterpret_cast<unsigned*>(cnt + nc + 1);
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(cnt, 0, (size_t)(nc + 1) * 8 + 8, s));
    if (npairs > 0) {
        k_dbg_count<<<blocks(npairs), 256, 0, s>>>(npairs, pairs, nc, cnt, bad);
        k_dbg_src<<<blocks(npairs), 256, 0, s>>>(npairs, pairs, P_<uint32_t>(src));
        ctx->launches += 2;
    }
    FMM_TRY(scan_exclusive_u64(ctx, cnt, P_<uint64_t>(off), nc, P_<uint64_t>(off) + nc, s));
    unsigned hb = 0;
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    if (hb) {
        ctx->err = hb & 1u ? "fmm_debug: a pair names a cell >= ncell"
                           : "fmm_debug: pairs not in ascending (target, source) order";
        return FMM_ERR_ARG;
    }
    return FMM_OK;
}

fmm_status check_view(fmm_ctx* ctx, const fmm_tree_view* v, const void* pairs, int64_t npairs) {
    if (!v || v->n < 0 || v->ncell < 0 || npairs < 0 || (npairs > 0 && !pairs) || v->n > ctx->n_max ||
        v->ncell > 0xFFFFFFFFll) {
        ctx->err = "fmm_debug: bad view or pair list";
        return FMM_ERR_ARG;
    }
    return FMM_OK;
}

// invalidate the build state: a debug call leaves no usable tree behind
void drop_build(fmm_ctx* ctx) {
    ctx->built = ctx->tree_built = ctx->evaluated = ctx->upward_done = false;
    ctx->built_pos = nullptr;
    ctx->lists_csr = false;
    ctx->tc_mix_ncell = -1;     // the caller's lists: m2l_fast.cu scans them for mixed levels
    ctx->nrem = ctx->nrem_body = 0;
    ctx->let_remote.clear();
    ctx->level_begin.clear();   // the caller's cells need not be level-ordered (m2l_fast.cu: all "mixed")
    ctx->depth = 0;
}

}  // namespace

extern "C" {

fmm_status fmm_debug_p2p(fmm_ctx* ctx, const fmm_tree_view* v, const uint32_t* p2p, int64_t n_pairs, void* phi,
                         void* grad, void* stream) {
    if (!ctx) return FMM_ERR_ARG;
    ctx->err.clear();
    FMM_TRY(check_view(ctx, v, p2p, n_pairs));
    if (v->n > 0 && (!v->pos || !v->q || !phi || !grad || !v->body_begin || !v->body_count || !v->child_count)) {
        ctx->err = "fmm_debug_p2p: null pointer";
        return FMM_ERR_ARG;
    }
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    drop_build(ctx);
    ctx->n = v->n;
    ctx->ncell = v->ncell;
    if (v->n == 0 || v->ncell == 0) return FMM_OK;
    const int64_t n = v->n, nc = v->ncell;
    const size_t es = ctx->prec == FMM_F32 ? 4 : 8;
    FMM_TRY(buf_ensure(ctx, ctx->body, (size_t)n * 4 * es + 64));
    if (ctx->prec == FMM_F32)
        k_dbg_pack_bodies<float, float4><<<blocks(n), 256, 0, s>>>(n, (const float*)v->pos, (const float*)v->q,
                                                                   P_<float4>(ctx->body));
    else
        k_dbg_pack_bodies<double, dbody><<<blocks(n), 256, 0, s>>>(n, (const double*)v->pos, (const double*)v->q,
                                                                   P_<dbody>(ctx->body));
    FMM_LAUNCH(ctx);
    FMM_TRY(buf_ensure(ctx, ctx->c_bb, (size_t)nc * 4));
    FMM_TRY(buf_ensure(ctx, ctx->c_bc, (size_t)nc * 4));
    FMM_TRY(buf_ensure(ctx, ctx->c_cc, (size_t)nc * 4));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->c_bb.p, v->body_begin, (size_t)nc * 4, cudaMemcpyDeviceToDevice, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->c_bc.p, v->body_count, (size_t)nc * 4, cudaMemcpyDeviceToDevice, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->c_cc.p, v->child_count, (size_t)nc * 4, cudaMemcpyDeviceToDevice, s));
    // leaves = cells without children, in cell order
    FMM_TRY(buf_ensure(ctx, ctx->split_tmp, (size_t)(nc + 1) * 8 + 64));
    uint32_t* flag = P_<uint32_t>(ctx->split_tmp);
    uint32_t* off = flag + nc + 1;
    k_dbg_leaf_flags<<<blocks(nc), 256, 0, s>>>(nc, P_<uint32_t>(ctx->c_cc), flag);
    FMM_LAUNCH(ctx);
    FMM_TRY(scan_exclusive_u32(ctx, flag, off, nc, off + nc, s));
    uint32_t nleaf = 0;
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(&nleaf, off + nc, 4, cudaMemcpyDeviceToHost, s));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    ctx->nleaf = nleaf;
    FMM_TRY(buf_ensure(ctx, ctx->leaf_ids, (size_t)std::max<uint32_t>(nleaf, 1) * 4));
    k_dbg_leaf_compact<<<blocks(nc), 256, 0, s>>>(nc, P_<uint32_t>(ctx->c_cc), off, P_<uint32_t>(ctx->leaf_ids));
    FMM_LAUNCH(ctx);
    FMM_TRY(load_pairs(ctx, p2p, n_pairs, ctx->p2p_off, ctx->p2p_src, s));
    ctx->n_p2p = n_pairs;
    FMM_TRY(buf_ensure(ctx, ctx->dcount2, 128));
    FMM_TRY(lists_finish(ctx, s));   // P2P source runs and leaf size classes, as after a traversal
    // the near-field partials are zero for bodies no leaf list touches
    FMM_TRY(buf_ensure(ctx, ctx->near_phi, (size_t)n * es));
    FMM_TRY(buf_ensure(ctx, ctx->near_grad, (size_t)n * 3 * es));
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->near_phi.p, 0, (size_t)n * es, s));
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->near_grad.p, 0, (size_t)n * 3 * es, s));
    FMM_TRY(p2p_pass(ctx, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(phi, ctx->near_phi.p, (size_t)n * es, cudaMemcpyDeviceToDevice, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(grad, ctx->near_grad.p, (size_t)n * 3 * es, cudaMemcpyDeviceToDevice, s));
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}

fmm_status fmm_debug_m2l(fmm_ctx* ctx, const fmm_tree_view* v, const uint32_t* m2l, int64_t n_pairs, double* L,
                         void* stream) {
    if (!ctx) return FMM_ERR_ARG;
    ctx->err.clear();
    FMM_TRY(check_view(ctx, v, m2l, n_pairs));
    if (v->ncell > 0 && (!v->center || !v->level || !v->M || !L || !(v->root_half_width > 0.0))) {
        ctx->err = "fmm_debug_m2l: null pointer or root_half_width <= 0";
        return FMM_ERR_ARG;
    }
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    drop_build(ctx);
    ctx->n = v->n;
    ctx->ncell = v->ncell;
    if (v->ncell == 0) return FMM_OK;
    const int64_t nc = v->ncell;
    const size_t lbytes = (size_t)nc * ctx->ncoef * 8;
    FMM_TRY(buf_ensure(ctx, ctx->c_cr, (size_t)nc * 32));
    FMM_TRY(buf_ensure(ctx, ctx->c_level, (size_t)nc * 4));
    FMM_TRY(buf_ensure(ctx, ctx->M, lbytes));
    FMM_TRY(buf_ensure(ctx, ctx->root, 16 * 8));
    k_dbg_cr<<<blocks(nc), 256, 0, s>>>(nc, v->center, P_<double4>(ctx->c_cr));
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->c_level.p, v->level, (size_t)nc * 4, cudaMemcpyDeviceToDevice, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->M.p, v->M, lbytes, cudaMemcpyDeviceToDevice, s));
    double root[16] = {0};
    root[10] = v->root_half_width;   // the expansion scale rho = 2^(E - level), 2^E >= 2 h (DESIGN.md §2 reading 5)
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->root.p, root, sizeof(root), cudaMemcpyHostToDevice, s));
    FMM_TRY(load_pairs(ctx, m2l, n_pairs, ctx->m2l_off, ctx->m2l_src, s));   // synchronises s
    ctx->n_m2l = n_pairs;
    ctx->m2l_part = 0;
    FMM_TRY(m2l_pass(ctx, s));
    FMM_CUDA_TRY(ctx, cudaMemcpyAsync(L, ctx->L.p, lbytes, cudaMemcpyDeviceToDevice, s));
    FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));   // `root` is a host temporary
    return FMM_OK;
}

}  // extern "C"
