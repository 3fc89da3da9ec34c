// m2l_tc.cu -- tensor-core experiment for BASELINE configs[4]'s M2L microbench (SURVEY §8(d) item 2
// "Tensor cores"): on the UNIFORM level-7 grid the classic interaction list repeats 316 distinct
// displacements v, so M2L (R14) is a dense batched contraction with shared operators:
//   Lhat_alpha(T) += sum_{|beta| <= P-1-|alpha|} H_v[alpha, beta] Shat_beta(T + v),
//   H_v[alpha, beta] = D^{alpha+beta} G(v)   (v in cell widths),
//   Shat_beta = (-1)^|beta| M_beta / w^|beta|, L_alpha = Lhat_alpha / w^(|alpha|+1)   (exact rescaling).
// Cells are split into the 8 parity classes p (coordinate parities): a target of class p has
// displacement set V_p (189 vectors), its source T+v lies in class p ^ (v & 1) at sub-grid offset
// floor((p+v)/2).  Each class is a 64^3 sub-grid stored with a 2-cell zero halo (68^3 columns), so
// for every (p, v) and every target degree a one GEMM covers all targets of the class:
//   L_p[rows of degree a, interior columns] += H_v[rows a, cols 0..ncoef(P-a)) * S_{p'}[.., cols + shift]
// (M = (a+1)(a+2)/2, K = ncoef(P-a), N = 64 * 68^2 columns: zero padding waste in K, ~20% halo in N).
// The GEMMs run through cuBLAS -- plain library GEMMs -- in FP32 (CUDA cores), TF32 and FP32 emulated
// with BF16x9 on the tensor cores (Blackwell, cuBLAS 12.9), one grouped call per displacement.
// Experiment only (tools/): the adaptive trees of the product path have no repeated operators.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC tools/m2l_tc.cu -lcublas
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

namespace {

constexpr int LEVEL = 7, G = 1 << LEVEL, H = G / 2, HP = H + 4;   // class sub-grid 64^3, padded 68^3
constexpr int64_t NC = (int64_t)G * G * G;
constexpr int64_t NPAD = (int64_t)HP * HP * HP;

int ncoef_of(int P) { return P * (P + 1) * (P + 2) / 6; }

struct Problem {
    int P = 0, nco = 0;
    double* M = nullptr;   // [NC][nco] fp64, Morton order
    double* L = nullptr;   // [NC][nco] fp64 result
    float* S = nullptr;    // [8][NPAD][nco]
    float* Lp = nullptr;   // [8][NPAD][nco]
    float* Hm = nullptr;   // [nv][nco][nco] column-major
    std::vector<int> vx, vy, vz;   // the 316 displacements
    cublasHandle_t h = nullptr;
};
Problem g_pb;
bool g_grouped = true;   // the last run used grouped calls

__host__ __device__ int cidx(int a, int b, int c) {
    int n = a + b + c, m = b + c;
    return n * (n + 1) * (n + 2) / 6 + m * (m + 1) / 2 + c;
}

__device__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// M_beta = u * w^|beta| / beta!, u ~ U[-1, 1)  (SURVEY §8(d) c5-M2L "cell-size-scaled M")
__global__ void k_make_M(int nco, const int* __restrict__ ex, const double* __restrict__ scale, uint64_t seed,
                         double* __restrict__ M) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < NC * nco; t += (int64_t)gridDim.x * blockDim.x) {
        const double u = (double)(mix64(seed + 0x9E3779B97F4A7C15ull * (uint64_t)(t + 1)) >> 11) * 0x1.0p-53;
        M[t] = (2.0 * u - 1.0) * scale[t % nco];
    }
}

__device__ void morton_xyz(int64_t m, int& x, int& y, int& z) {
    x = y = z = 0;
    for (int l = 0; l < LEVEL; ++l) {
        x |= (int)((m >> (3 * l)) & 1) << l;
        y |= (int)((m >> (3 * l + 1)) & 1) << l;
        z |= (int)((m >> (3 * l + 2)) & 1) << l;
    }
}

__device__ int64_t pad_index(int x, int y, int z) {   // class sub-grid coordinate of a cell
    const int tx = x >> 1, ty = y >> 1, tz = z >> 1;
    return ((int64_t)(tz + 2) * HP + (ty + 2)) * HP + (tx + 2);
}

// S_p = (-1)^|beta| M / w^|beta| in fp32, class-major padded columns (halo stays zero)
__global__ void k_to_classes(int nco, const int* __restrict__ deg, const double* __restrict__ M, double w,
                             float* __restrict__ S) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < NC * nco; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = t / nco;
        const int k = (int)(t - m * nco);
        int x, y, z;
        morton_xyz(m, x, y, z);
        const int p = (x & 1) | (y & 1) << 1 | (z & 1) << 2;
        const double v = M[t] * pow(w, -(double)deg[k]) * ((deg[k] & 1) ? -1.0 : 1.0);
        S[((int64_t)p * NPAD + pad_index(x, y, z)) * nco + k] = (float)v;
    }
}

__global__ void k_from_classes(int nco, const int* __restrict__ deg, const float* __restrict__ Lp, double w,
                               double* __restrict__ L) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < NC * nco; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = t / nco;
        const int k = (int)(t - m * nco);
        int x, y, z;
        morton_xyz(m, x, y, z);
        const int p = (x & 1) | (y & 1) << 1 | (z & 1) << 2;
        L[t] = (double)Lp[((int64_t)p * NPAD + pad_index(x, y, z)) * nco + k] * pow(w, -(double)(deg[k] + 1));
    }
}

// D^gamma G(v) for |gamma| <= 2P-2 in fp64 (R14's Taylor table, derivative form:
// n r^2 D_k = -(2n-1) sum_i k_i v_i D_{k-e_i} - (n-1) sum_i k_i (k_i - 1) D_{k-2e_i})
void derivs(int Q, double vx, double vy, double vz, std::vector<double>& D) {
    D.assign(ncoef_of(Q), 0.0);
    const double r2 = vx * vx + vy * vy + vz * vz;
    D[0] = 1.0 / std::sqrt(r2);
    const double v[3] = {vx, vy, vz};
    for (int n = 1; n < Q; ++n)
        for (int a = n; a >= 0; --a)
            for (int b = n - a; b >= 0; --b) {
                const int c = n - a - b, k[3] = {a, b, c};
                double s1 = 0.0, s2 = 0.0;
                for (int i = 0; i < 3; ++i) {
                    int m[3] = {a, b, c};
                    if (k[i] >= 1) {
                        m[i] -= 1;
                        s1 += k[i] * v[i] * D[cidx(m[0], m[1], m[2])];
                        m[i] += 1;
                    }
                    if (k[i] >= 2) {
                        m[i] -= 2;
                        s2 += (double)k[i] * (k[i] - 1) * D[cidx(m[0], m[1], m[2])];
                    }
                }
                D[cidx(a, b, c)] = -((2.0 * n - 1.0) * s1 + (n - 1.0) * s2) / (n * r2);
            }
}

}  // namespace

extern "C" {

// Build the problem for P (M random with `seed`); returns 0 on success.
int m2ltc_setup(int P, uint64_t seed) {
    Problem& pb = g_pb;
    if (pb.M) {
        cudaFree(pb.M); cudaFree(pb.L); cudaFree(pb.S); cudaFree(pb.Lp); cudaFree(pb.Hm);
        pb.M = nullptr;
    }
    if (!pb.h && cublasCreate(&pb.h) != CUBLAS_STATUS_SUCCESS) return 1;
    pb.P = P;
    pb.nco = ncoef_of(P);
    const int nco = pb.nco;
    std::vector<int> ex(3 * nco), deg(nco);
    std::vector<double> scale(nco);
    const double w = 1.0 / G;
    for (int n = 0, k = 0; n < P; ++n)
        for (int a = n; a >= 0; --a)
            for (int b = n - a; b >= 0; --b, ++k) {
                const int c = n - a - b;
                ex[3 * k] = a; ex[3 * k + 1] = b; ex[3 * k + 2] = c;
                deg[k] = n;
                scale[k] = std::pow(w, n) / (std::tgamma(a + 1.0) * std::tgamma(b + 1.0) * std::tgamma(c + 1.0));
            }
    int *dex, *ddeg;
    double* dscale;
    cudaMalloc(&dex, ex.size() * 4); cudaMalloc(&ddeg, deg.size() * 4); cudaMalloc(&dscale, nco * 8);
    cudaMemcpy(dex, ex.data(), ex.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(ddeg, deg.data(), deg.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dscale, scale.data(), nco * 8, cudaMemcpyHostToDevice);
    if (cudaMalloc(&pb.M, NC * nco * 8) || cudaMalloc(&pb.L, NC * nco * 8) ||
        cudaMalloc(&pb.S, 8 * NPAD * nco * 4) || cudaMalloc(&pb.Lp, 8 * NPAD * nco * 4))
        return 2;
    cudaMemset(pb.S, 0, 8 * NPAD * nco * 4);
    k_make_M<<<4096, 256>>>(nco, dex, dscale, seed, pb.M);
    k_to_classes<<<4096, 256>>>(nco, ddeg, pb.M, w, pb.S);
    // displacements: union over parities of [-2-p, 3-p]^3 minus the 27 neighbours = [-3, 3]^3 minus them
    pb.vx.clear(); pb.vy.clear(); pb.vz.clear();
    for (int z = -3; z <= 3; ++z)
        for (int y = -3; y <= 3; ++y)
            for (int x = -3; x <= 3; ++x)
                if (std::max(std::abs(x), std::max(std::abs(y), std::abs(z))) > 1) {
                    pb.vx.push_back(x); pb.vy.push_back(y); pb.vz.push_back(z);
                }
    const int nv = (int)pb.vx.size();
    std::vector<float> Hh((size_t)nv * nco * nco, 0.0f);
    std::vector<double> D;
    for (int i = 0; i < nv; ++i) {
        // d = c_target - c_source = -v cell widths (the source is the target shifted by +v)
        derivs(2 * P - 1, -pb.vx[i], -pb.vy[i], -pb.vz[i], D);
        float* Hv = Hh.data() + (size_t)i * nco * nco;
        for (int al = 0; al < nco; ++al)
            for (int be = 0; be < nco; ++be) {
                if (deg[al] + deg[be] > P - 1) continue;
                Hv[(size_t)be * nco + al] = (float)D[cidx(ex[3 * al] + ex[3 * be], ex[3 * al + 1] + ex[3 * be + 1],
                                                          ex[3 * al + 2] + ex[3 * be + 2])];
            }
    }
    if (cudaMalloc(&pb.Hm, Hh.size() * 4)) return 3;
    cudaMemcpy(pb.Hm, Hh.data(), Hh.size() * 4, cudaMemcpyHostToDevice);
    cudaFree(dex); cudaFree(ddeg); cudaFree(dscale);
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : 4;
}

// One M2L over the whole grid with the given GEMM precision (0 FP32 CUDA cores, 1 TF32, 2 FP32
// emulated with BF16x9 on the tensor cores), `reps` times; *ms = mean CUDA-event time per M2L
// (all GEMMs; the class layout conversion is outside); the result lands in L (fp64, Morton).
int m2ltc_run(int mode, int reps, float* ms) {
    Problem& pb = g_pb;
    const int P = pb.P, nco = pb.nco, nv = (int)pb.vx.size();
    cublasComputeType_t ct = mode == 0 ? CUBLAS_COMPUTE_32F : mode == 1 ? CUBLAS_COMPUTE_32F_FAST_TF32
                                                                       : CUBLAS_COMPUTE_32F_EMULATED_16BFX9;
    if (mode == 2) cublasSetEmulationStrategy(pb.h, CUBLAS_EMULATION_STRATEGY_EAGER);
    cublasSetMathMode(pb.h, mode == 2 ? CUBLAS_FP32_EMULATED_BF16X9_MATH : CUBLAS_DEFAULT_MATH);
    // grouped GEMM per displacement: every (class p having v, target degree a)
    const int64_t j0 = ((int64_t)2 * HP + 2) * HP + 2;                      // first interior column
    const int64_t ncol = ((int64_t)(H + 1) * HP + (H + 1)) * HP + (H + 1) - j0 + 1;
    std::vector<std::vector<const void*>> A(nv), B(nv);
    std::vector<std::vector<void*>> C(nv);
    std::vector<std::vector<int>> m(nv), k(nv);
    for (int i = 0; i < nv; ++i) {
        const int v[3] = {pb.vx[i], pb.vy[i], pb.vz[i]};
        for (int p = 0; p < 8; ++p) {
            int s[3], q = 0;
            bool ok = true;
            for (int d = 0; d < 3; ++d) {
                const int pd = (p >> d) & 1;
                if (v[d] < -2 - pd || v[d] > 3 - pd) ok = false;
                const int t = pd + v[d];
                s[d] = (int)std::floor(t / 2.0);
                q |= (t & 1) << d;
            }
            if (!ok) continue;
            const int64_t shift = ((int64_t)s[2] * HP + s[1]) * HP + s[0];
            for (int a = 0; a < P; ++a) {
                const int r0 = a * (a + 1) * (a + 2) / 6, na = (a + 1) * (a + 2) / 2, ka = ncoef_of(P - a);
                A[i].push_back(pb.Hm + (size_t)i * nco * nco + r0);
                B[i].push_back(pb.S + ((int64_t)q * NPAD + j0 + shift) * nco);
                C[i].push_back(pb.Lp + ((int64_t)p * NPAD + j0) * nco + r0);
                m[i].push_back(na);
                k[i].push_back(ka);
            }
        }
    }
    // pointer arrays of the grouped calls live in device memory
    std::vector<void**> dA(nv), dB(nv), dC(nv);
    for (int i = 0; i < nv; ++i) {
        const size_t ng = A[i].size();
        cudaMalloc(&dA[i], ng * 8); cudaMalloc(&dB[i], ng * 8); cudaMalloc(&dC[i], ng * 8);
        cudaMemcpy(dA[i], A[i].data(), ng * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dB[i], B[i].data(), ng * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dC[i], C[i].data(), ng * 8, cudaMemcpyHostToDevice);
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float total = 0.f;
    bool grouped = true;
    for (int r = 0; r < reps + 1; ++r) {
        cudaMemset(pb.Lp, 0, 8 * NPAD * nco * 4);
        cudaEventRecord(e0);
        for (int i = 0; i < nv; ++i) {
            const int ng = (int)A[i].size();
            std::vector<cublasOperation_t> tn(ng, CUBLAS_OP_N);
            std::vector<int> nn(ng, (int)ncol), ld(ng, nco), one(ng, 1);
            std::vector<float> al(ng, 1.0f), be(ng, 1.0f);
            cublasStatus_t st = CUBLAS_STATUS_NOT_SUPPORTED;
            if (grouped)
                st = cublasGemmGroupedBatchedEx(pb.h, tn.data(), tn.data(), m[i].data(), nn.data(), k[i].data(),
                                                al.data(), (const void* const*)dA[i], CUDA_R_32F, ld.data(),
                                                (const void* const*)dB[i], CUDA_R_32F, ld.data(), be.data(),
                                                (void* const*)dC[i], CUDA_R_32F, ld.data(), ng, one.data(), ct);
            if (st == CUBLAS_STATUS_NOT_SUPPORTED) {   // e.g. emulated FP32: one GEMM per (p, degree)
                grouped = false;
                const float one_f = 1.0f;
                for (int g = 0; g < ng; ++g) {
                    st = cublasGemmEx(pb.h, CUBLAS_OP_N, CUBLAS_OP_N, m[i][g], (int)ncol, k[i][g], &one_f, A[i][g],
                                      CUDA_R_32F, nco, B[i][g], CUDA_R_32F, nco, &one_f, C[i][g], CUDA_R_32F, nco, ct,
                                      CUBLAS_GEMM_DEFAULT);
                    if (st != CUBLAS_STATUS_SUCCESS) break;
                }
            }
            if (st != CUBLAS_STATUS_SUCCESS) {
                fprintf(stderr, "cuBLAS GEMM failed: %d (mode %d)\n", (int)st, mode);
                return 10 + (int)st;
            }
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float t = 0.f;
        cudaEventElapsedTime(&t, e0, e1);
        if (r > 0) total += t;   // the first run is a warm-up
    }
    for (int i = 0; i < nv; ++i) {
        cudaFree(dA[i]); cudaFree(dB[i]); cudaFree(dC[i]);
    }
    g_grouped = grouped;
    *ms = total / reps;
    // back to Morton order, unscaled
    std::vector<int> deg(nco);
    for (int n = 0, kk = 0; n < P; ++n)
        for (int c = 0; c < (n + 1) * (n + 2) / 2; ++c, ++kk) deg[kk] = n;
    int* ddeg;
    cudaMalloc(&ddeg, nco * 4);
    cudaMemcpy(ddeg, deg.data(), nco * 4, cudaMemcpyHostToDevice);
    k_from_classes<<<4096, 256>>>(nco, ddeg, pb.Lp, 1.0 / G, pb.L);
    cudaFree(ddeg);
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : 5;
}

int m2ltc_grouped() { return g_grouped ? 1 : 0; }

// fp64 M or L rows of the given Morton cell ids into out [n][ncoef]
int m2ltc_rows(int which, int n, const int64_t* ids, double* out) {
    const Problem& pb = g_pb;
    for (int i = 0; i < n; ++i)
        if (cudaMemcpy(out + (size_t)i * pb.nco, (which ? pb.L : pb.M) + ids[i] * pb.nco, pb.nco * 8,
                       cudaMemcpyDeviceToHost) != cudaSuccess)
            return 1;
    return 0;
}

}  // extern "C"
