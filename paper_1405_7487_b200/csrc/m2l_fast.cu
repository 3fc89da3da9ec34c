// m2l_fast.cu -- register-resident M2L for P <= 10 (fp32) / P <= 6 (fp64)  (a9, the hot kernel).
//
// Same mathematics as R14 (L_alpha = sum_beta (-1)^|beta| M_beta D^{alpha+beta}G), evaluated
// in the harmonic ("trace-reduced") Cartesian form, which is exact because G = 1/r is
// harmonic (sum_i D^{gamma+2e_i}G = 0 for every gamma; pinned in tests/test_oracle.py):
//   * D_gamma with gamma_x >= 2 is never formed: only D0 = D_(0,y,z) (|.| <= P-1) and
//     D1 = D_(1,y,z) (|.| <= P-2) -- P^2 values instead of P(P+1)(P+2)/6;
//   * the signed multipole S_beta = (-1)^|beta| M_beta is folded onto beta_x in {0,1} once
//     per source cell (S_beta -> S_{beta-2e_x+2e_y}, S_{beta-2e_x+2e_z} with weight -1),
//     which leaves every contraction with D unchanged;
//   * only L_alpha with alpha_x in {0,1} is computed; L is harmonic to truncation order
//     (the |beta| range depends on |alpha| only), so L_alpha for alpha_x >= 2 is rebuilt
//     exactly as -L_{alpha-2e_x+2e_y} - L_{alpha-2e_x+2e_z} (k_l_expand).
//   With a+b = 2 folded into N[q'] = -S1[q'-2e_y] - S1[q'-2e_z], the four products are
//     L0[p] += S0[q] D0[p+q]   (|p|+|q| <= P-1)     L0[p] += S1[q] D1[p+q] (<= P-2)
//     L1[p] += S0[q] D1[p+q]   (<= P-2)             L1[p] += N[q'] D0[p+q'] (<= P-1)
//   i.e. 2275 FMA per pair at P=10 instead of 5005, and a 100-entry recurrence instead of 220.
// Scaling (fp32 range, SURVEY §7 hard part 5): every cell has rho = 2^e (e = E - level, an
// exact power of two near the octant width).  Stored S_hat = S / rho_B^|beta|, D is evaluated
// at u = d / rho_A, each streamed S_hat is multiplied by (rho_B/rho_A)^|beta|, and the
// accumulators hold L_hat = L rho_A^(|alpha|+1).
// All scalings are exact powers of two.
// Work layout: one warp per target cell (CSR range), ONE PAIR PER LANE; the derivative
// table (D0, D1) and the lane's L accumulators live in registers (compile-time indices,
// fully unrolled); S_hat of the lane's source is streamed with 16-B loads.  Lanes
// accumulate their pairs (same target) in Real, then the warp reduces in fp64 and stores
// the reduced L_hat (no atomics).  Targets are handed to warps through an atomic counter.
#include <type_traits>
#include <utility>

#include "common.cuh"

namespace {

// compile-time loop B..E-1 in order (a fold over an index sequence: no recursion-depth limit)
template <int B, typename F, int... I>
__device__ __forceinline__ void sfor_seq(F&& f, std::integer_sequence<int, I...>) {
    (f(std::integral_constant<int, B + I>{}), ...);
}
template <int B, int E, typename F>
__device__ __forceinline__ void sfor(F&& f) {
    if constexpr (B < E) sfor_seq<B>(f, std::make_integer_sequence<int, E - B>{});
}

__host__ __device__ constexpr int t2(int y, int z) { return (y + z) * (y + z + 1) / 2 + z; }
__host__ __device__ constexpr int deg2(int e) {
    int m = 0;
    while ((m + 1) * (m + 2) / 2 <= e) ++m;
    return m;
}
__host__ __device__ constexpr int zof(int e) { return e - deg2(e) * (deg2(e) + 1) / 2; }
__host__ __device__ constexpr int yof(int e) { return deg2(e) - zof(e); }

template <int P>
struct RF {
    static constexpr int N0 = P * (P + 1) / 2;   // 2D indices of degree <= P-1
    static constexpr int N1 = (P - 1) * P / 2;   // degree <= P-2
    static constexpr int NS = 2 * N0 + N1;       // S0 | S1 | N
    static constexpr int NSP = (NS + 3) / 4 * 4;
    static constexpr int NL = N0 + N1;           // L0 | L1
};

__device__ __forceinline__ float fma_(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float rsqrt_(float x) { return rsqrtf(x); }
__device__ __forceinline__ double rsqrt_(double x) { return 1.0 / sqrt(x); }
__device__ __forceinline__ float rcp_(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double rcp_(double x) { return 1.0 / x; }

template <typename R> struct Vec4;
template <> struct Vec4<float> { using type = float4; };
template <> struct Vec4<double> { using type = double4; };

// D0[t2(y,z)] = D_(0,y,z)(u), D1[t2(y,z)] = D_(1,y,z)(u): derivative form of the R14 recurrence
//   n r^2 D_k = -(2n-1) sum_i k_i u_i D_{k-e_i} - (n-1) sum_i k_i (k_i - 1) D_{k-2e_i}
template <int P, typename R>
__device__ __forceinline__ void derivs(R ux, R uy, R uz, R (&D0)[RF<P>::N0], R (&D1)[RF<P>::N1]) {
    const R r2 = ux * ux + uy * uy + uz * uz;
    const R ir2 = rcp_(r2);
    R yu[P], zu[P];
#pragma unroll
    for (int m = 1; m < P; ++m) {
        yu[m] = R(m) * uy;
        zu[m] = R(m) * uz;
    }
    D0[0] = rsqrt_(r2);
#pragma unroll
    for (int n = 1; n < P; ++n) {
        const R A = R(-(2.0 * n - 1.0) / n) * ir2;
        const R B = R(-(n - 1.0) / n) * ir2;
#pragma unroll
        for (int z = 0; z <= n; ++z) {
            const int y = n - z;
            R s1 = R(0);
            if (y > 0) s1 = yu[y] * D0[t2(y - 1, z)];
            if (z > 0) s1 = (y > 0) ? fma_(zu[z], D0[t2(y, z - 1)], s1) : zu[z] * D0[t2(y, z - 1)];
            R s2 = R(0);
            if (y > 1) s2 = R(y * (y - 1)) * D0[t2(y - 2, z)];
            if (z > 1) s2 = fma_(R(z * (z - 1)), D0[t2(y, z - 2)], s2);
            D0[t2(y, z)] = (n > 1) ? fma_(A, s1, B * s2) : A * s1;
        }
#pragma unroll
        for (int z = 0; z <= n - 1; ++z) {
            const int y = n - 1 - z;
            R s1 = ux * D0[t2(y, z)];
            if (y > 0) s1 = fma_(yu[y], D1[t2(y - 1, z)], s1);
            if (z > 0) s1 = fma_(zu[z], D1[t2(y, z - 1)], s1);
            R s2 = R(0);
            if (y > 1) s2 = R(y * (y - 1)) * D1[t2(y - 2, z)];
            if (z > 1) s2 = fma_(R(z * (z - 1)), D1[t2(y, z - 2)], s2);
            D1[t2(y, z)] = (n > 1) ? fma_(A, s1, B * s2) : A * s1;
        }
    }
}

// degree |beta| of stored element E (S0: |q|, S1: |q|+1, N: |q'|-1); -1 for padding
template <int P>
__host__ __device__ constexpr int elem_deg(int e) {
    return e < RF<P>::N0 ? deg2(e)
           : e < RF<P>::N0 + RF<P>::N1 ? deg2(e - RF<P>::N0) + 1
           : e < RF<P>::NS ? deg2(e - RF<P>::N0 - RF<P>::N1) - 1
                           : -1;
}

// one streamed element s = S_hat[E] into the accumulators
template <int P, int E, typename R>
__device__ __forceinline__ void apply_elem(R s, const R (&D0)[RF<P>::N0], const R (&D1)[RF<P>::N1],
                                           R (&L0)[RF<P>::N0], R (&L1)[RF<P>::N1]) {
    constexpr int N0 = RF<P>::N0, N1 = RF<P>::N1;
    if constexpr (E < N0) {
        constexpr int qy = yof(E), qz = zof(E), m = qy + qz;
#pragma unroll
        for (int pm = 0; pm <= P - 1 - m; ++pm)
#pragma unroll
            for (int pz = 0; pz <= pm; ++pz) {
                const int py = pm - pz;
                L0[t2(py, pz)] = fma_(s, D0[t2(py + qy, pz + qz)], L0[t2(py, pz)]);
            }
#pragma unroll
        for (int pm = 0; pm <= P - 2 - m; ++pm)
#pragma unroll
            for (int pz = 0; pz <= pm; ++pz) {
                const int py = pm - pz;
                L1[t2(py, pz)] = fma_(s, D1[t2(py + qy, pz + qz)], L1[t2(py, pz)]);
            }
    } else if constexpr (E < N0 + N1) {
        constexpr int e = E - N0, qy = yof(e), qz = zof(e), m = qy + qz;
#pragma unroll
        for (int pm = 0; pm <= P - 2 - m; ++pm)
#pragma unroll
            for (int pz = 0; pz <= pm; ++pz) {
                const int py = pm - pz;
                L0[t2(py, pz)] = fma_(s, D1[t2(py + qy, pz + qz)], L0[t2(py, pz)]);
            }
    } else if constexpr (E < RF<P>::NS) {
        constexpr int e = E - N0 - N1, qy = yof(e), qz = zof(e), m = qy + qz;
        if constexpr (m >= 2) {
#pragma unroll
            for (int pm = 0; pm <= P - 1 - m; ++pm)
#pragma unroll
                for (int pz = 0; pz <= pm; ++pz) {
                    const int py = pm - pz;
                    L1[t2(py, pz)] = fma_(s, D0[t2(py + qy, pz + qz)], L1[t2(py, pz)]);
                }
        }
    }
}

template <int P, typename R>
__global__ void __launch_bounds__(128, 2)
    k_m2l_fast(int64_t ncell, const uint32_t* __restrict__ src, const uint64_t* __restrict__ off,
               const double4* __restrict__ cr, const int* __restrict__ sexp,
               const typename Vec4<R>::type* __restrict__ Sv, double* __restrict__ Lr,
               unsigned long long* __restrict__ counter) {
    using V4 = typename Vec4<R>::type;
    constexpr int N0 = RF<P>::N0, N1 = RF<P>::N1, NCH = RF<P>::NSP / 4, NL = RF<P>::NL;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    (void)w;
    for (;;) {
        unsigned long long an = 0;
        if (lane == 0) an = atomicAdd(counter, 1ull);
        const long long a = (long long)__shfl_sync(0xffffffffu, an, 0);
        if (a >= ncell) break;
        const uint64_t p0 = off[a], p1 = off[a + 1];
        if (p0 == p1) continue;
        const double4 ca = cr[a];
        const int ea = sexp[a];
        const double sa = exp2((double)-ea);   // 1/rho_A, exact
        R L0[N0], L1[N1];
#pragma unroll
        for (int i = 0; i < N0; ++i) L0[i] = R(0);
#pragma unroll
        for (int i = 0; i < N1; ++i) L1[i] = R(0);
        for (uint64_t p = p0 + lane; p < p1; p += 32) {
            const uint32_t b = src[p];
            const double4 cb = cr[b];
            const int eb = sexp[b];
            const R ux = (R)((ca.x - cb.x) * sa);
            const R uy = (R)((ca.y - cb.y) * sa);
            const R uz = (R)((ca.z - cb.z) * sa);
            R D0[N0], D1[N1];
            derivs<P, R>(ux, uy, uz, D0, D1);
            // (rho_B / rho_A)^n per degree, exact powers of two
            const int de = eb - ea;
            // (rho_B/rho_A)^n: all pairs of a uniform tree have de = 0; the scaling runs only
            // in chunks of pairs where some lane of the warp needs it (warp-uniform branch)
            const bool need = __any_sync(__activemask(), de != 0);
            R pw[P];
            pw[0] = R(1);
            pw[1] = (R)exp2((double)de);
#pragma unroll
            for (int n = 2; n < P; ++n) pw[n] = pw[n - 1] * pw[1];
            const V4* sv = Sv + (size_t)b * NCH;
            sfor<0, NCH>([&](auto c) {
                constexpr int C4 = decltype(c)::value;
                const V4 v = sv[C4];
                R vv[4] = {v.x, v.y, v.z, v.w};
                if (need) {
                    sfor<0, 4>([&](auto j) {
                        constexpr int dg = elem_deg<P>(4 * C4 + decltype(j)::value);
                        if constexpr (dg > 0) vv[decltype(j)::value] *= pw[dg];
                    });
                }
                sfor<0, 4>([&](auto j) {
                    constexpr int E = 4 * C4 + decltype(j)::value;
                    constexpr int dg = elem_deg<P>(E);
                    if constexpr (dg >= 0) apply_elem<P, E, R>(vv[decltype(j)::value], D0, D1, L0, L1);
                });
            });
        }
        // warp reduction in fp64, lane (k mod 32) stores entry k of the reduced L_hat
        sfor<0, NL>([&](auto kk) {
            constexpr int k = decltype(kk)::value;
            double v;
            if constexpr (k < N0) v = (double)L0[k];
            else v = (double)L1[k - N0];
#pragma unroll
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == (k & 31)) Lr[(size_t)a * NL + k] = v;
        });
    }
}

// Harmonic fold in closed form (operand preparation, per source cell): repeatedly moving
// S_beta (beta_x >= 2) onto beta - 2e_x + 2e_y and beta - 2e_x + 2e_z with weight -1 gives
//   S~(b,y,z) = sum_k (-1)^k sum_{j<=k} C(k,j) S(b+2k, y-2j, z-2(k-j)),  S = (-1)^|beta| M;
// the streamed operand is S0 = S~(0,.,.) | S1 = S~(1,.,.) | N[q] = -S1[q-2e_y] - S1[q-2e_z]
// (|q| >= 2), each scaled by rho^-|beta| (exact powers of two) and rounded to R.
// The preparation is a sparse linear map built once per P from the rules above: output
// element i = sum over table entries (k, w) of w * M[k] (the sign (-1)^|beta| and the fold's
// binomial weights in w), then scaled by rho^(-e dg_i).  The kernel is a warp per cell with M
// staged in shared memory and lanes over outputs (the per-element decode-and-recurse version
// took 0.26 ms at c2 and 4.1 ms at c3; profiles/r01_c3 launch list).
struct FoldTable {
    std::vector<int> off;      // [NSP + 1]
    std::vector<int> k;        // coefficient index (R11 order)
    std::vector<double> w;     // weight
    std::vector<int> dg;       // [NSP] degree |beta| for the rho scaling, -1 for padding
};

void fold_terms_host(int b, int y, int z, double sgn, std::vector<std::pair<int, double>>& out) {
    // S~(b,y,z) = sum_k (-1)^k sum_{j<=k} C(k,j) S(b+2k, y-2j, z-2(k-j)), S = (-1)^|beta| M
    for (int k = 0; 2 * k <= y + z; ++k) {
        double binom = 1.0;
        for (int j = 0; j <= k; ++j) {
            if (j > 0) binom = binom * (double)(k - j + 1) / (double)j;
            const int yy = y - 2 * j, zz = z - 2 * (k - j);
            if (yy >= 0 && zz >= 0) {
                const int a = b + 2 * k;
                const double sM = ((a + yy + zz) & 1) ? -1.0 : 1.0;
                out.push_back({cidx(a, yy, zz), sgn * ((k & 1) ? -binom : binom) * sM});
            }
        }
    }
}

FoldTable build_fold_table(int P, int NS, int NSP) {
    FoldTable t;
    const int N0 = P * (P + 1) / 2, N1 = (P - 1) * P / 2;
    t.off.assign(NSP + 1, 0);
    t.dg.assign(NSP, -1);
    auto decode = [](int ii, int& m, int& y, int& z) {
        m = 0;
        while ((m + 1) * (m + 2) / 2 <= ii) ++m;
        z = ii - m * (m + 1) / 2;
        y = m - z;
    };
    for (int i = 0; i < NSP; ++i) {
        std::vector<std::pair<int, double>> e;
        int m, y, z;
        if (i < N0) {            // S0: S~(0, q)
            decode(i, m, y, z);
            fold_terms_host(0, y, z, 1.0, e);
            t.dg[i] = m;
        } else if (i < N0 + N1) {   // S1: S~(1, q)
            decode(i - N0, m, y, z);
            fold_terms_host(1, y, z, 1.0, e);
            t.dg[i] = m + 1;
        } else if (i < NS) {        // N[q] = -S1[q - 2e_y] - S1[q - 2e_z]
            decode(i - N0 - N1, m, y, z);
            if (m >= 2) {
                if (y >= 2) fold_terms_host(1, y - 2, z, -1.0, e);
                if (z >= 2) fold_terms_host(1, y, z - 2, -1.0, e);
            }
            t.dg[i] = m - 1;
        }
        for (auto& x : e) {
            t.k.push_back(x.first);
            t.w.push_back(x.second);
        }
        t.off[i + 1] = (int)t.k.size();
    }
    return t;
}

// 2^k as a double for |k| <= 1000 (exponent bits), else ldexp's general path
__device__ __forceinline__ double scale2(double v, int k) {
    return (k >= -1000 && k <= 1000) ? v * __longlong_as_double((long long)(k + 1023) << 52) : ldexp(v, k);
}

// the fold table (nt terms) is copied to shared memory once per block: every output entry reads
// its terms there instead of through L1 per cell
template <typename R>
__global__ void k_m2l_prep_table(int64_t c0, int64_t ncell, int ncoef, int NSP, const int* __restrict__ toff,
                                 const int* __restrict__ tk, const double* __restrict__ tw,
                                 const int* __restrict__ tdg, const double* __restrict__ M,
                                 const int32_t* __restrict__ level, const double* __restrict__ root,
                                 int* __restrict__ sexp, R* __restrict__ Sv, int64_t copy_stride, int nt) {
    extern __shared__ double s_M[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double* s_tw = s_M + (size_t)nw * ncoef;
    int* s_tk = reinterpret_cast<int*>(s_tw + nt);
    int* s_toff = s_tk + nt;
    int* s_tdg = s_toff + NSP + 1;
    for (int i = threadIdx.x; i < nt; i += blockDim.x) {
        s_tw[i] = tw[i];
        s_tk[i] = tk[i];
    }
    for (int i = threadIdx.x; i <= NSP; i += blockDim.x) s_toff[i] = toff[i];
    for (int i = threadIdx.x; i < NSP; i += blockDim.x) s_tdg[i] = tdg[i];
    __syncthreads();
    double* Mw = s_M + (size_t)w * ncoef;
    int E;
    frexp(2.0 * root[10], &E);
    for (int64_t c = c0 + (int64_t)blockIdx.x * nw + w; c < ncell; c += (int64_t)gridDim.x * nw) {
        const int e = E - level[c];
        for (int k = lane; k < ncoef; k += 32) Mw[k] = M[(size_t)c * ncoef + k];
        if (lane == 0) sexp[c] = e;
        __syncwarp();
        R* out = Sv + (size_t)c * NSP;
        for (int i = lane; i < NSP; i += 32) {
            double v = 0.0;
            for (int t = s_toff[i]; t < s_toff[i + 1]; ++t) v += s_tw[t] * Mw[s_tk[t]];
            const int dg = s_tdg[i];
            out[i] = dg < 0 ? R(0) : (R)scale2(v, -e * dg);
            if (copy_stride) {   // the operand as the pair scaling 2^(de dg) leaves it, de = -1 and +1
                out[i - copy_stride] = dg < 0 ? R(0) : (R)scale2(v, -(e + 1) * dg);
                out[i + copy_stride] = dg < 0 ? R(0) : (R)scale2(v, -(e - 1) * dg);
            }
        }
        __syncwarp();
    }
}

// reduced, scaled L_hat -> full fp64 L (R11 order) by harmonicity, zero for cells without M2L.
// The index maps are decoded once per block into shared tables (per element before: a search
// loop for the degree and a cidx per term, ~8x the kernel's memory time):
//   t_red[i] = {cidx of reduced entry i, its scale degree ax+m+1}, i < P^2 (L0 | L1, t2 order);
//   t_fill[j] = {dst, src1, src2}: L[ax,y,z] = -L[ax-2,y+2,z] - L[ax-2,y,z+2], ax = 2..P-1 in order,
//   with fill_off[ax] the first entry of level ax.
__global__ void k_l_expand(int64_t ncell, int P, int ncoef, const uint64_t* __restrict__ off,
                           const uint64_t* __restrict__ off2, const int* __restrict__ sexp,
                           const double* __restrict__ Lr, double* __restrict__ L) {
    extern __shared__ double s_L[];
    __shared__ ushort2 t_red[FMM_MAXP * FMM_MAXP];
    __shared__ ushort4 t_fill[816];
    __shared__ int fill_off[FMM_MAXP + 1];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int N0 = P * (P + 1) / 2, NL = P * P;
    for (int i = threadIdx.x; i < NL; i += blockDim.x) {
        const int ax = i < N0 ? 0 : 1, ii = i < N0 ? i : i - N0;
        int m = 0;
        while ((m + 1) * (m + 2) / 2 <= ii) ++m;
        const int z = ii - m * (m + 1) / 2, y = m - z;
        t_red[i] = make_ushort2((unsigned short)cidx(ax, y, z), (unsigned short)(ax + m + 1));
    }
    if (threadIdx.x < FMM_MAXP + 1) {   // level ax starts after sum_{a=2}^{ax-1} (P-a)(P-a+1)/2 entries
        int o = 0;
        for (int a2 = 2; a2 < (int)threadIdx.x && a2 < P; ++a2) o += (P - a2) * (P - a2 + 1) / 2;
        fill_off[threadIdx.x] = o;
    }
    __syncthreads();
    for (int ax = 2; ax < P; ++ax) {
        const int cnt = (P - ax) * (P - ax + 1) / 2, o = fill_off[ax];
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            int m = 0;
            while ((m + 1) * (m + 2) / 2 <= i) ++m;
            const int z = i - m * (m + 1) / 2, y = m - z;
            t_fill[o + i] = make_ushort4((unsigned short)cidx(ax, y, z), (unsigned short)cidx(ax - 2, y + 2, z),
                                         (unsigned short)cidx(ax - 2, y, z + 2), 0);
        }
    }
    __syncthreads();
    double* Lf = s_L + (size_t)w * ncoef;
    for (int64_t c = (int64_t)blockIdx.x * nw + w; c < ncell; c += (int64_t)gridDim.x * nw) {
        double* out = L + (size_t)c * ncoef;
        if (off[c] == off[c + 1] && (!off2 || off2[c] == off2[c + 1])) {   // no list (local or remote)
            for (int k = lane; k < ncoef; k += 32) out[k] = 0.0;
            continue;
        }
        const int e = sexp[c];
        for (int i = lane; i < NL; i += 32) {
            const ushort2 t = t_red[i];
            Lf[t.x] = ldexp(Lr[(size_t)c * NL + i], -e * (int)t.y);
        }
        __syncwarp();
        for (int ax = 2; ax < P; ++ax) {
            const int o0 = fill_off[ax], cnt = (P - ax) * (P - ax + 1) / 2;
            for (int i = lane; i < cnt; i += 32) {
                const ushort4 t = t_fill[o0 + i];
                Lf[t.x] = -Lf[t.y] - Lf[t.z];
            }
            __syncwarp();
        }
        for (int k = lane; k < ncoef; k += 32) out[k] = Lf[k];
        __syncwarp();
    }
}

template <int P, typename R>
fmm_status m2l_fast_t(fmm_ctx* ctx, cudaStream_t s) {
    constexpr int NSP = RF<P>::NSP, NL = RF<P>::NL;
    const int64_t nc = ctx->ncell;
    const int64_t nct = ctx->ncell + ctx->nrem;   // sources include grafted LET cells
    // operand layout capacity (the split multi-GPU flow prepares local and remote cells in two
    // passes, so the layout must not move between them) and the first cell to prepare
    const int64_t lay = ctx->m2l_cap > 0 ? ctx->m2l_cap : nct, c0 = ctx->m2l_prep_c0;
    FMM_TRY(buf_ensure(ctx, ctx->Mr, (size_t)lay * NSP * sizeof(R) + (size_t)lay * 4 + 256));
    FMM_TRY(buf_ensure(ctx, ctx->Lr, (size_t)nc * NL * 8));
    FMM_TRY(buf_ensure(ctx, ctx->cnt_tmp, 64));
    R* Sv = P_<R>(ctx->Mr);
    int* sexp = reinterpret_cast<int*>(reinterpret_cast<char*>(ctx->Mr.p) + (size_t)lay * NSP * sizeof(R));
    ctx->m2l_sexp = sexp;
    const int nw = 4;
    int g = (int)std::min<int64_t>((nc + nw - 1) / nw, (int64_t)ctx->num_sms * 16);
    const int gp = (int)std::min<int64_t>((nct - c0 + nw - 1) / nw, (int64_t)ctx->num_sms * 16);
    if (ctx->fold_P != P) {   // scalar layout table (the mirror kernel keys its own as 1000 + P)
        const FoldTable t = build_fold_table(P, RF<P>::NS, NSP);
        const size_t nt = t.k.size();
        FMM_TRY(buf_ensure(ctx, ctx->fold_tab, (NSP + 1) * 4 + NSP * 4 + nt * 4 + nt * 8 + 64));
        char* b = (char*)ctx->fold_tab.p;
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(b, t.w.data(), nt * 8, cudaMemcpyHostToDevice, s));
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(b + nt * 8, t.off.data(), (NSP + 1) * 4, cudaMemcpyHostToDevice, s));
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(b + nt * 8 + (NSP + 1) * 4, t.dg.data(), NSP * 4, cudaMemcpyHostToDevice, s));
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(b + nt * 8 + (2 * NSP + 1) * 4, t.k.data(), nt * 4, cudaMemcpyHostToDevice, s));
        FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));   // pageable sources: complete before reuse
        ctx->fold_P = P;
        ctx->fold_nt = (int64_t)nt;
    }
    if (ctx->m2l_part != 2) {
        char* b = (char*)ctx->fold_tab.p;
        const size_t nt = (size_t)ctx->fold_nt;
        const size_t psm = (size_t)nw * ctx->ncoef * 8 + nt * 12 + (size_t)(2 * NSP + 1) * 4;
        if (psm > 48 * 1024)
            FMM_CUDA_TRY(ctx, cudaFuncSetAttribute(k_m2l_prep_table<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm));
        k_m2l_prep_table<R><<<std::max(gp, 1), nw * 32, psm, s>>>(
            c0, nct, ctx->ncoef, NSP, reinterpret_cast<const int*>(b + nt * 8),
            reinterpret_cast<const int*>(b + nt * 8 + (2 * NSP + 1) * 4), reinterpret_cast<const double*>(b),
            reinterpret_cast<const int*>(b + nt * 8 + (NSP + 1) * 4), P_<double>(ctx->M), P_<int32_t>(ctx->c_level),
            P_<double>(ctx->root), sexp, Sv, (int64_t)0, (int)nt);
        FMM_LAUNCH(ctx);
    }
    if (ctx->m2l_part == 1) return FMM_OK;
    unsigned long long* counter = P_<unsigned long long>(ctx->cnt_tmp);
    FMM_CUDA_TRY(ctx, cudaMemsetAsync(counter, 0, 8, s));
    {
        PhaseScope ps(ctx, PH_M2L_KERNEL, s);
        k_m2l_fast<P, R><<<ctx->num_sms * 2, 128, 0, s>>>(nc, P_<uint32_t>(ctx->m2l_src), P_<uint64_t>(ctx->m2l_off),
                                                         P_<double4>(ctx->c_cr), sexp,
                                                         reinterpret_cast<const typename Vec4<R>::type*>(Sv),
                                                         P_<double>(ctx->Lr), counter);
        FMM_LAUNCH(ctx);
    }
    if (!ctx->m2l_no_expand) {
        k_l_expand<<<std::max(g, 1), nw * 32, (size_t)nw * ctx->ncoef * 8, s>>>(
            nc, P, ctx->ncoef, P_<uint64_t>(ctx->m2l_off), ctx->m2l_off2, sexp, P_<double>(ctx->Lr),
            P_<double>(ctx->L));
        FMM_LAUNCH(ctx);
    }
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}

// ================================================================ mirror-paired M2L (fp32)
// The harmonic 2D correlations are symmetric under the y <-> z mirror M(y,z) = (z,y): the
// recurrence gives D at M(k) from the recurrence at k with u_y and u_z exchanged, and
// M(p) + M(q) = M(p+q).  So every off-diagonal canonical index (y > z) holds the PAIR
// {X[y,z], X[z,y]} of D0, D1, L0, L1 and of the streamed S0, S1, N, and one f32x2 instruction
// (FFMA2/FMUL2, sm_100) does the work for an index and its mirror:
//   recurrence:  DP[y,z] = A ({y uy, y uz} * DP(y-1,z) + {z uz, z uy} * DP(y,z-1)) + B (...)
//   contraction: LP[p] += SP[q] * DP(p+q)  (element q)   and   LP[p] += swap(SP[q]) * DP(p+Mq)
//                (element Mq); DP(k) of a non-canonical k is swap(DP[Mk]); diagonal indices
//                (y == z) are scalars used through the .F32 broadcast operand.
// All swaps and broadcasts are FFMA2 operand modifiers (no extra instructions).  The pair body is
// ~1,500 instructions at P=10 (the scalar kernel: ~3,100), within the 32 KB L1.5 I-cache.
namespace mir {
__host__ __device__ constexpr int t2m(int y, int z) { return (y + z) * (y + z + 1) / 2 + z; }
// off-diagonal canonical (y > z) slots of degree <= D, in t2 order of (y, z)
__host__ __device__ constexpr int noff(int D) {
    int c = 0;
    for (int n = 0; n <= D; ++n) c += (n + 1) / 2;
    return c;
}
__host__ __device__ constexpr int ndia(int D) { return D / 2 + 1; }
__host__ __device__ constexpr int off(int y, int z) {   // y > z
    int c = noff(y + z - 1);
    for (int zz = 0; zz < z; ++zz)
        if (y + z - zz > zz) ++c;
    return c;
}

template <int P>
struct L {
    static constexpr int D0 = P - 1, D1 = P - 2;
    static constexpr int O0 = noff(D0), O1 = noff(D1 < 0 ? 0 : D1), G0 = ndia(D0), G1 = ndia(D1 < 0 ? 0 : D1);
    // stream (floats): S0 pairs | S1 pairs | N pairs | S0 diag | S1 diag | N diag
    static constexpr int BS0 = 0, BS1 = 2 * O0, BN = BS1 + 2 * O1, BD0 = BN + 2 * O0, BD1 = BD0 + G0,
                         BDN = BD1 + G1, NS = BDN + G0, NSP = (NS + 3) / 4 * 4, NCH = NSP / 4;
    static constexpr int NL = P * (P + 1) / 2 + (P - 1) * P / 2;   // reduced L: L0 | L1 (t2 order)
};

template <int P>
struct Regs {
    using K = L<P>;
    float2 D0p[K::O0];
    float D0d[K::G0];
    float2 D1p[K::O1 > 0 ? K::O1 : 1];
    float D1d[K::G1];
    float2 L0p[K::O0];
    float2 L0d[K::G0];   // diagonal outputs as two partial sums (one FFMA2 per element pair)
    float2 L1p[K::O1 > 0 ? K::O1 : 1];
    float2 L1d[K::G1];
};

__device__ __forceinline__ float2 sw(float2 v) { return make_float2(v.y, v.x); }
__device__ __forceinline__ float2 bc(float v) { return make_float2(v, v); }

// {X[y,z], X[z,y]} of a paired array for any (y, z)
template <int Y, int Z>
__device__ __forceinline__ float2 pr(const float2* p, const float* d) {
    if constexpr (Y > Z) return p[off(Y, Z)];
    else if constexpr (Y < Z) return sw(p[off(Z, Y)]);
    else return bc(d[Y]);
}

template <int P>
__device__ __forceinline__ void derivs_mir(float ux, float uy, float uz, Regs<P>& R) {
    const float r2 = ux * ux + uy * uy + uz * uz;
    const float ir2 = __frcp_rn(r2);
    float2 YU[P];   // {m uy, m uz}
#pragma unroll
    for (int m = 1; m < P; ++m) YU[m] = make_float2(float(m) * uy, float(m) * uz);
    R.D0d[0] = rsqrtf(r2);
    sfor<1, P>([&](auto nn) {
        constexpr int n = decltype(nn)::value;
        const float A = float(-(2.0 * n - 1.0) / n) * ir2;
        const float B = float(-(n - 1.0) / n) * ir2;
        // D0, degree n: canonical (y >= z), y + z = n
        sfor<0, n / 2 + 1>([&](auto zz) {
            constexpr int z = decltype(zz)::value, y = n - z;
            if constexpr (y > z) {
                float2 s1;
                if constexpr (z > 0)
                    s1 = __ffma2_rn(sw(YU[z]), pr<y, z - 1>(R.D0p, R.D0d), __fmul2_rn(YU[y], pr<y - 1, z>(R.D0p, R.D0d)));
                else
                    s1 = __fmul2_rn(YU[y], pr<y - 1, z>(R.D0p, R.D0d));
                float2 v;
                if constexpr (n > 1) {
                    float2 s2 = make_float2(0.f, 0.f);
                    if constexpr (y > 1) s2 = __fmul2_rn(bc(float(y * (y - 1))), pr<y - 2, z>(R.D0p, R.D0d));
                    if constexpr (z > 1) s2 = __ffma2_rn(bc(float(z * (z - 1))), pr<y, z - 2>(R.D0p, R.D0d), s2);
                    v = __ffma2_rn(bc(A), s1, __fmul2_rn(bc(B), s2));
                } else {
                    v = __fmul2_rn(bc(A), s1);
                }
                R.D0p[off(y, z)] = v;
            } else {   // diagonal: D0[y,y] = A y (uy D0[y-1,y] + uz D0[y,y-1]) + B y(y-1) (D0[y-2,y] + D0[y,y-2])
                const float2 q1 = R.D0p[off(y, y - 1)];
                const float s1 = fmaf(YU[y].y, q1.x, YU[y].x * q1.y);
                float v;
                if constexpr (y > 1) {
                    const float2 q2 = R.D0p[off(y, y - 2)];
                    v = fmaf(A, s1, B * (float(y * (y - 1)) * (q2.x + q2.y)));
                } else {
                    v = A * s1;
                }
                R.D0d[y] = v;
            }
        });
        // D1, total degree n: canonical (y >= z), y + z = n - 1
        sfor<0, (n - 1) / 2 + 1>([&](auto zz) {
            constexpr int z = decltype(zz)::value, y = n - 1 - z;
            if constexpr (y > z) {
                float2 s1 = __fmul2_rn(bc(ux), pr<y, z>(R.D0p, R.D0d));
                if constexpr (y > 0) s1 = __ffma2_rn(YU[y], pr<y - 1, z>(R.D1p, R.D1d), s1);
                if constexpr (z > 0) s1 = __ffma2_rn(sw(YU[z]), pr<y, z - 1>(R.D1p, R.D1d), s1);
                float2 v;
                if constexpr (n > 1) {
                    float2 s2 = make_float2(0.f, 0.f);
                    if constexpr (y > 1) s2 = __fmul2_rn(bc(float(y * (y - 1))), pr<y - 2, z>(R.D1p, R.D1d));
                    if constexpr (z > 1) s2 = __ffma2_rn(bc(float(z * (z - 1))), pr<y, z - 2>(R.D1p, R.D1d), s2);
                    v = __ffma2_rn(bc(A), s1, __fmul2_rn(bc(B), s2));
                } else {
                    v = __fmul2_rn(bc(A), s1);
                }
                R.D1p[off(y, z)] = v;
            } else {   // diagonal y == z
                float s1 = ux * R.D0d[y];
                if constexpr (y > 0) {
                    const float2 q1 = R.D1p[off(y, y - 1)];
                    s1 = fmaf(YU[y].x, q1.y, s1);
                    s1 = fmaf(YU[y].y, q1.x, s1);
                }
                float v;
                if constexpr (y > 1) {
                    const float2 q2 = R.D1p[off(y, y - 2)];
                    v = fmaf(A, s1, B * (float(y * (y - 1)) * (q2.x + q2.y)));
                } else if constexpr (n > 1) {
                    v = A * s1;
                } else {
                    v = A * s1;
                }
                R.D1d[y] = v;
            }
        });
    });
}

// element pair {S[q], S[Mq]} (q = (QY, QZ), QY > QZ) into L += S (x) D for |p| + |q| <= DMAX
template <int DMAX, int QY, int QZ, int NO, int NG, int DO, int DG>
__device__ __forceinline__ void corr_pair(float2 sp, float2 (&Lp)[NO], float2 (&Ld)[NG], const float2 (&Dp)[DO],
                                          const float (&Dd)[DG]) {
    constexpr int m = QY + QZ;
    // element q (and the diagonal outputs), then element Mq: the two updates of one accumulator
    // are a whole sweep apart (no back-to-back dependent FFMA2)
    sfor<0, DMAX - m + 1>([&](auto pp) {
        constexpr int pn = decltype(pp)::value;
        sfor<0, pn / 2 + 1>([&](auto zz) {
            constexpr int pz = decltype(zz)::value, py = pn - pz;
            if constexpr (py > pz) {
                Lp[off(py, pz)] = __ffma2_rn(sp, pr<py + QY, pz + QZ>(Dp, Dd), Lp[off(py, pz)]);
            } else {   // diagonal p: k = p + q is canonical off-diagonal; .x element q, .y element Mq
                Ld[py] = __ffma2_rn(sp, Dp[off(py + QY, pz + QZ)], Ld[py]);
            }
        });
    });
    sfor<0, DMAX - m + 1>([&](auto pp) {
        constexpr int pn = decltype(pp)::value;
        sfor<0, pn / 2 + 1>([&](auto zz) {
            constexpr int pz = decltype(zz)::value, py = pn - pz;
            if constexpr (py > pz)
                Lp[off(py, pz)] = __ffma2_rn(sw(sp), pr<py + QZ, pz + QY>(Dp, Dd), Lp[off(py, pz)]);
        });
    });
}

// diagonal element S[q] (q = (Q, Q)) into L += S (x) D for |p| + |q| <= DMAX
template <int DMAX, int Q, int NO, int NG, int DO, int DG>
__device__ __forceinline__ void corr_diag(float s, float2 (&Lp)[NO], float2 (&Ld)[NG], const float2 (&Dp)[DO],
                                          const float (&Dd)[DG]) {
    constexpr int m = 2 * Q;
    sfor<0, DMAX - m + 1>([&](auto pp) {
        constexpr int pn = decltype(pp)::value;
        sfor<0, pn / 2 + 1>([&](auto zz) {
            constexpr int pz = decltype(zz)::value, py = pn - pz;
            if constexpr (py > pz) Lp[off(py, pz)] = __ffma2_rn(bc(s), pr<py + Q, pz + Q>(Dp, Dd), Lp[off(py, pz)]);
            else Ld[py].x = fmaf(s, Dd[py + Q], Ld[py].x);
        });
    });
}

// canonical off-diagonal slot index j of degree <= D -> (y, z)
__host__ __device__ constexpr int slot_y(int j) {
    for (int n = 0;; ++n)
        for (int z = 0; 2 * z < n; ++z)
            if (j-- == 0) return n - z;
}
__host__ __device__ constexpr int slot_z(int j) {
    for (int n = 0;; ++n)
        for (int z = 0; 2 * z < n; ++z)
            if (j-- == 0) return z;
}

// SC = false: only the targets whose sources are all within one level of their own
// (mixed[a] == 0; a uniform tree: every target), reading the operand copy prepared at the pair's
// scale 2^(de n), de in {-1, 0, 1}, so the kernel has no scaling code at all (~8% fewer
// instructions per pair); SC = true: the other targets (every target if mixed == nullptr), de = 0
// copy scaled in registers
template <int P, bool SC>
__global__ void __launch_bounds__(128, 2)
    k_m2l_mir(int64_t ncell, const uint32_t* __restrict__ src, const uint64_t* __restrict__ offs,
              const double4* __restrict__ cr, const int* __restrict__ sexp, const float4* __restrict__ Sv,
              double* __restrict__ Lr, unsigned long long* __restrict__ counter,
              const uint8_t* __restrict__ mixed, int64_t lay, const uint32_t* __restrict__ tlist = nullptr,
              const unsigned long long* __restrict__ tcount = nullptr) {
    using K = L<P>;
    constexpr int NCH = K::NCH;
    const int lane = threadIdx.x & 31;
    // next pair's source centre, fetched with cp.async one pair ahead (ncu: the src -> cr load
    // chain at every pair start was the top long-scoreboard stall)
    __shared__ __align__(16) double4 s_cb[128];
    __shared__ int s_eb[128];
    double4* my_cb = s_cb + threadIdx.x;
    int* my_eb = s_eb + threadIdx.x;
    auto fetch_cb = [&](uint32_t bn) {
        const unsigned sa_ = (unsigned)__cvta_generic_to_shared(my_cb);
        const unsigned se_ = (unsigned)__cvta_generic_to_shared(my_eb);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa_), "l"(cr + bn) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa_ + 16), "l"(reinterpret_cast<const char*>(cr + bn) + 16) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(se_), "l"(sexp + bn) : "memory");
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    // work: every target (skipping the other kernel's), or the listed ones (tlist: the scaled
    // kernel after k_m2l_mixed)
    const long long nwork = tlist ? (long long)*tcount : (long long)ncell;
    for (;;) {
        unsigned long long an = 0;
        if (lane == 0) an = atomicAdd(counter, 1ull);
        const long long wi = (long long)__shfl_sync(0xffffffffu, an, 0);
        if (wi >= nwork) break;
        const long long a = tlist ? (long long)tlist[wi] : wi;
        const uint64_t p0 = offs[a], p1 = offs[a + 1];
        if (p0 == p1) continue;
        if (!tlist && mixed && (mixed[a] != 0) != SC) continue;   // the other kernel's target
        const double4 ca = cr[a];
        const int ea = sexp[a];
        const double sa = exp2((double)-ea);   // 1/rho_A, exact
        Regs<P> R;
#pragma unroll
        for (int i = 0; i < K::O0; ++i) R.L0p[i] = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < K::G0; ++i) R.L0d[i] = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < K::O1; ++i) R.L1p[i] = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < K::G1; ++i) R.L1d[i] = make_float2(0.f, 0.f);
        uint32_t bnext = 0;
        if (p0 + lane < p1) {
            bnext = src[p0 + lane];
            fetch_cb(bnext);
        }
        for (uint64_t p = p0 + lane; p < p1; p += 32) {
            const uint32_t b = bnext;
            bnext = p + 32 < p1 ? src[p + 32] : b;
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            const double4 cb = *my_cb;
            const int de = *my_eb - ea;
            const float ux = (float)((ca.x - cb.x) * sa);
            const float uy = (float)((ca.y - cb.y) * sa);
            const float uz = (float)((ca.z - cb.z) * sa);
            derivs_mir<P>(ux, uy, uz, R);
            if (p + 32 < p1) fetch_cb(bnext);   // after the recurrence: bnext has landed
            // (rho_B/rho_A)^n: only in warps where some lane needs it (uniform trees: never)
            const bool need = SC && __any_sync(__activemask(), de != 0);
            // 2^(de*n) from exponent bits: |de| <= 14 is guaranteed by m2l_pass, which routes trees
            // spanning more than 14 levels to the fp64 kernel (|de * n| <= 126 for n <= 9)
            auto pw = [&](int n) { return __int_as_float((127 + de * n) << 23); };
            // SC = false: |de| <= 1 for every pair of this target, and the operand comes from the
            // copy prepared at that scale (rows -lay .. +lay of the de = 0 copy Sv)
            const float4* sv = Sv + ((SC ? 0 : (int64_t)de * lay) + (int64_t)b) * NCH;
            sfor<0, NCH>([&](auto cc) {
                constexpr int C = decltype(cc)::value;
                const float4 v = sv[C];
                const float vv[4] = {v.x, v.y, v.z, v.w};
                sfor<0, 4>([&](auto jj) {
                    constexpr int F = 4 * C + decltype(jj)::value;
                    if constexpr (F < K::BD0) {
                        if constexpr (F % 2 == 0) {
                            constexpr int kind = F < K::BS1 ? 0 : (F < K::BN ? 1 : 2);
                            constexpr int j = (F - (kind == 0 ? K::BS0 : kind == 1 ? K::BS1 : K::BN)) / 2;
                            constexpr int qy = slot_y(j), qz = slot_z(j), m = qy + qz;
                            float2 sp = make_float2(vv[F % 4], vv[F % 4 + 1]);
                            if constexpr (kind == 0) {          // S0: L0 += S0 D0 (<= P-1), L1 += S0 D1 (<= P-2)
                                if constexpr (m > 0) {
                                    if (need) sp = __fmul2_rn(bc(pw(m)), sp);
                                }
                                corr_pair<P - 1, qy, qz>(sp, R.L0p, R.L0d, R.D0p, R.D0d);
                                if constexpr (m <= P - 2) corr_pair<P - 2, qy, qz>(sp, R.L1p, R.L1d, R.D1p, R.D1d);
                            } else if constexpr (kind == 1) {   // S1 (degree m+1): L0 += S1 D1 (<= P-2)
                                if (need) sp = __fmul2_rn(bc(pw(m + 1)), sp);
                                corr_pair<P - 2, qy, qz>(sp, R.L0p, R.L0d, R.D1p, R.D1d);
                            } else if constexpr (m >= 2) {      // N (degree m-1): L1 += N D0 (<= P-1)
                                if (need) sp = __fmul2_rn(bc(pw(m - 1)), sp);
                                corr_pair<P - 1, qy, qz>(sp, R.L1p, R.L1d, R.D0p, R.D0d);
                            }
                        }
                    } else if constexpr (F < K::NS) {
                        constexpr int kind = F < K::BD1 ? 0 : (F < K::BDN ? 1 : 2);
                        constexpr int Q = F - (kind == 0 ? K::BD0 : kind == 1 ? K::BD1 : K::BDN);
                        float sd = vv[F % 4];
                        if constexpr (kind == 0) {
                            if constexpr (Q > 0) {
                                if (need) sd *= pw(2 * Q);
                            }
                            corr_diag<P - 1, Q>(sd, R.L0p, R.L0d, R.D0p, R.D0d);
                            if constexpr (2 * Q <= P - 2) corr_diag<P - 2, Q>(sd, R.L1p, R.L1d, R.D1p, R.D1d);
                        } else if constexpr (kind == 1) {
                            if (need) sd *= pw(2 * Q + 1);
                            corr_diag<P - 2, Q>(sd, R.L0p, R.L0d, R.D1p, R.D1d);
                        } else if constexpr (2 * Q >= 2) {
                            if (need) sd *= pw(2 * Q - 1);
                            corr_diag<P - 1, Q>(sd, R.L1p, R.L1d, R.D0p, R.D0d);
                        }
                    }
                });
            });
        }
        // warp reduction in fp64; reduced L_hat in (L0 | L1) t2 order for k_l_expand
        constexpr int N0 = P * (P + 1) / 2;
        auto val = [&](auto kk) -> float {   // this lane's partial sum of reduced index k
            constexpr int k = decltype(kk)::value;
            constexpr int x1 = k >= N0, e = x1 ? k - N0 : k;
            constexpr int n = deg2(e), z = zof(e), y = n - z;
            if constexpr (!x1) {
                if constexpr (y > z) return R.L0p[off(y, z)].x;
                else if constexpr (y < z) return R.L0p[off(z, y)].y;
                else return R.L0d[y].x + R.L0d[y].y;
            } else {
                if constexpr (y > z) return R.L1p[off(y, z)].x;
                else if constexpr (y < z) return R.L1p[off(z, y)].y;
                else return R.L1d[y].x + R.L1d[y].y;
            }
        };
        if constexpr (K::NL <= 128) {
            // reduce-scatter over the NLP (padded: 32, 64 or 128) values: each xor stage keeps the
            // half of the block this lane's bit selects and adds the partner's copy of it, so
            // lane l ends with the totals of k = Q l .. Q l + Q-1, Q = NLP / 32 (~1/5 of the
            // shuffles of one butterfly per value)
            constexpr int NLP = K::NL <= 32 ? 32 : (K::NL <= 64 ? 64 : 128), Q = NLP / 32;
            double v1[NLP / 2], v2[NLP / 4], v3[NLP / 8], v4[NLP / 16], v5[Q];
            const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2, b0 = lane & 1;
            sfor<0, NLP / 2>([&](auto jj) {
                constexpr int j = decltype(jj)::value;
                double lo = 0.0, hi = 0.0;
                if constexpr (j < K::NL) lo = (double)val(std::integral_constant<int, j>{});
                if constexpr (j + NLP / 2 < K::NL) hi = (double)val(std::integral_constant<int, j + NLP / 2>{});
                v1[j] = (b4 ? hi : lo) + __shfl_xor_sync(0xffffffffu, b4 ? lo : hi, 16);
            });
            sfor<0, NLP / 4>([&](auto jj) {
                constexpr int j = decltype(jj)::value, h = NLP / 4;
                v2[j] = (b3 ? v1[j + h] : v1[j]) + __shfl_xor_sync(0xffffffffu, b3 ? v1[j] : v1[j + h], 8);
            });
            sfor<0, NLP / 8>([&](auto jj) {
                constexpr int j = decltype(jj)::value, h = NLP / 8;
                v3[j] = (b2 ? v2[j + h] : v2[j]) + __shfl_xor_sync(0xffffffffu, b2 ? v2[j] : v2[j + h], 4);
            });
            sfor<0, NLP / 16>([&](auto jj) {
                constexpr int j = decltype(jj)::value, h = NLP / 16;
                v4[j] = (b1 ? v3[j + h] : v3[j]) + __shfl_xor_sync(0xffffffffu, b1 ? v3[j] : v3[j + h], 2);
            });
            sfor<0, Q>([&](auto jj) {
                constexpr int j = decltype(jj)::value;
                v5[j] = (b0 ? v4[j + Q] : v4[j]) + __shfl_xor_sync(0xffffffffu, b0 ? v4[j] : v4[j + Q], 1);
            });
#pragma unroll
            for (int j = 0; j < Q; ++j) {
                const int k = Q * lane + j;
                if (k < K::NL) Lr[(size_t)a * K::NL + k] = v5[j];
            }
        } else {
            sfor<0, K::NL>([&](auto kk) {
                constexpr int k = decltype(kk)::value;
                double v = (double)val(kk);
#pragma unroll
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == (k & 31)) Lr[(size_t)a * K::NL + k] = v;
            });
        }
    }
}

// mixed[a] = 1 iff target a's M2L list holds a source more than one level away (no prepared
// operand copy at that scale); those targets are also listed (any order) for the scaled kernel.
// Local cells are level-ordered, so a local source is within one level of a iff its index lies
// in lvl[level(a) - 1] .. lvl[level(a) + 2] (no gather); grafted LET cells (index >= nloc), and
// every cell of a caller-supplied tree without level ranges (fmm_debug_m2l), compare exponents.
// Warp per target.
__global__ void k_m2l_mixed(int64_t ncell, int64_t nloc, const uint32_t* __restrict__ src,
                            const uint64_t* __restrict__ offs, const int32_t* __restrict__ level,
                            const int64_t* __restrict__ lvl, int nlvl, const int* __restrict__ sexp,
                            uint8_t* __restrict__ mixed, uint32_t* __restrict__ mlist,
                            unsigned long long* __restrict__ mcount) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t a = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); a < ncell; a += nw) {
        const uint64_t p0 = offs[a], p1 = offs[a + 1];
        const int la = level[a];
        const bool ok = la + 1 < nlvl;   // level ranges describe the local cells
        const int64_t lo = ok ? lvl[max(la - 1, 0)] : 0, hi = ok ? lvl[min(la + 2, nlvl - 1)] : 0;
        const int64_t nl = ok ? nloc : 0;
        const int ea = sexp[a];
        bool mix = false;
        for (uint64_t p = p0 + lane; p < p1; p += 32) {
            const int64_t b = src[p];
            mix |= b < nl ? (b < lo || b >= hi) : abs(sexp[b] - ea) > 1;
        }
        mix = __any_sync(0xffffffffu, mix);
        if (lane == 0) {
            mixed[a] = mix ? 1 : 0;
            if (mix) mlist[atomicAdd(mcount, 1ull)] = (uint32_t)a;   // the scaled kernel's work list
        }
    }
}

// the same split from the traversal's per-target flags (tct.cu: an M2L source outside levels
// l-1 .. l+1 of a local target) -- a pass over the cells instead of over the M2L list
__global__ void k_m2l_mixed_flags(int64_t ncell, const uint32_t* __restrict__ flag, uint8_t* __restrict__ mixed,
                                  uint32_t* __restrict__ mlist, unsigned long long* __restrict__ mcount) {
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= ncell) return;
    const bool mix = flag[a] != 0;
    mixed[a] = mix ? 1 : 0;
    if (mix) mlist[atomicAdd(mcount, 1ull)] = (uint32_t)a;   // the scaled kernel's work list
}

// operand layout of the mirror kernel as a fold table: output float i -> (kind, 2D index, degree)
FoldTable build_fold_table_mir(int P, int NS, int NSP) {
    const int O0 = noff(P - 1), O1 = noff(P - 2 < 0 ? 0 : P - 2), G0 = ndia(P - 1), G1 = ndia(P - 2 < 0 ? 0 : P - 2);
    const int BS1 = 2 * O0, BN = BS1 + 2 * O1, BD0 = BN + 2 * O0, BD1 = BD0 + G0, BDN = BD1 + G1;
    FoldTable t;
    t.off.assign(NSP + 1, 0);
    t.dg.assign(NSP, -1);
    for (int i = 0; i < NSP; ++i) {
        std::vector<std::pair<int, double>> e;
        int kind = -1, y = 0, z = 0;
        if (i < BD0) {
            const int base = i < BS1 ? 0 : (i < BN ? BS1 : BN);
            kind = i < BS1 ? 0 : (i < BN ? 1 : 2);
            const int j = (i - base) / 2;
            y = slot_y(j);
            z = slot_z(j);
            if ((i - base) & 1) std::swap(y, z);   // .y of the pair: the mirror element
        } else if (i < NS) {
            kind = i < BD1 ? 0 : (i < BDN ? 1 : 2);
            const int Q = i - (kind == 0 ? BD0 : kind == 1 ? BD1 : BDN);
            y = z = Q;
        }
        const int m = y + z;
        if (kind == 0) {
            fold_terms_host(0, y, z, 1.0, e);
            t.dg[i] = m;
        } else if (kind == 1) {
            fold_terms_host(1, y, z, 1.0, e);
            t.dg[i] = m + 1;
        } else if (kind == 2) {
            if (m >= 2) {
                if (y >= 2) fold_terms_host(1, y - 2, z, -1.0, e);
                if (z >= 2) fold_terms_host(1, y, z - 2, -1.0, e);
            }
            t.dg[i] = m - 1;
        }
        for (auto& x : e) {
            t.k.push_back(x.first);
            t.w.push_back(x.second);
        }
        t.off[i + 1] = (int)t.k.size();
    }
    return t;
}
}  // namespace mir

template <int P>
fmm_status m2l_mir_t(fmm_ctx* ctx, cudaStream_t s) {
    using K = mir::L<P>;
    constexpr int NSP = K::NSP, NL = K::NL;
    const int64_t nc = ctx->ncell;
    const int64_t nct = ctx->ncell + ctx->nrem;   // sources include grafted LET cells
    // operand layout capacity (the split multi-GPU flow prepares local and remote cells in two
    // passes, so the layout must not move between them) and the first cell to prepare
    const int64_t lay = ctx->m2l_cap > 0 ? ctx->m2l_cap : nct, c0 = ctx->m2l_prep_c0;
    // operand: three copies [de = -1 | de = 0 | de = +1] of lay cells each, then the exponents
    const size_t lstride = (size_t)lay * NSP;   // floats per copy
    FMM_TRY(buf_ensure(ctx, ctx->Mr, 3 * lstride * 4 + (size_t)lay * 4 + 256));
    FMM_TRY(buf_ensure(ctx, ctx->Lr, (size_t)nc * NL * 8));
    FMM_TRY(buf_ensure(ctx, ctx->cnt_tmp, 64));
    float* Sv = P_<float>(ctx->Mr) + lstride;   // the de = 0 copy
    int* sexp = reinterpret_cast<int*>(reinterpret_cast<char*>(ctx->Mr.p) + 3 * lstride * 4);
    ctx->m2l_sexp = sexp;
    const int nw = 4;
    const int g = (int)std::min<int64_t>((nc + nw - 1) / nw, (int64_t)ctx->num_sms * 16);
    const int gp = (int)std::min<int64_t>((nct - c0 + nw - 1) / nw, (int64_t)ctx->num_sms * 16);
    if (ctx->fold_P != 1000 + P) {
        const FoldTable t = mir::build_fold_table_mir(P, K::NS, NSP);
        const size_t nt = t.k.size();
        FMM_TRY(buf_ensure(ctx, ctx->fold_tab, (NSP + 1) * 4 + NSP * 4 + nt * 4 + nt * 8 + 64));
        char* b = (char*)ctx->fold_tab.p;
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(b, t.w.data(), nt * 8, cudaMemcpyHostToDevice, s));
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(b + nt * 8, t.off.data(), (NSP + 1) * 4, cudaMemcpyHostToDevice, s));
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(b + nt * 8 + (NSP + 1) * 4, t.dg.data(), NSP * 4, cudaMemcpyHostToDevice, s));
        FMM_CUDA_TRY(ctx, cudaMemcpyAsync(b + nt * 8 + (2 * NSP + 1) * 4, t.k.data(), nt * 4, cudaMemcpyHostToDevice, s));
        FMM_CUDA_TRY(ctx, cudaStreamSynchronize(s));   // pageable sources: complete before reuse
        ctx->fold_P = 1000 + P;
        ctx->fold_nt = (int64_t)nt;
    }
    if (ctx->m2l_part != 2) {
        char* b = (char*)ctx->fold_tab.p;
        const size_t nt = (size_t)ctx->fold_nt;
        const size_t psm = (size_t)nw * ctx->ncoef * 8 + nt * 12 + (size_t)(2 * NSP + 1) * 4;
        if (psm > 48 * 1024)
            FMM_CUDA_TRY(ctx, cudaFuncSetAttribute(k_m2l_prep_table<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm));
        k_m2l_prep_table<float><<<std::max(gp, 1), nw * 32, psm, s>>>(
            c0, nct, ctx->ncoef, NSP, reinterpret_cast<const int*>(b + nt * 8),
            reinterpret_cast<const int*>(b + nt * 8 + (2 * NSP + 1) * 4), reinterpret_cast<const double*>(b),
            reinterpret_cast<const int*>(b + nt * 8 + (NSP + 1) * 4), P_<double>(ctx->M), P_<int32_t>(ctx->c_level),
            P_<double>(ctx->root), sexp, Sv, (int64_t)lstride, (int)nt);
        FMM_LAUNCH(ctx);
    }
    if (ctx->m2l_part == 1) return FMM_OK;   // operand preparation only (fmm_solve: aux stream)
    unsigned long long* counter = P_<unsigned long long>(ctx->cnt_tmp);
    {
        PhaseScope ps(ctx, PH_M2L_KERNEL, s);
        // split the targets by whether every source is within one level: those run the kernel
        // without scaling code, the others the scaled kernel (a uniform tree: none of them)
        // (level ranges only when they describe these cells; else the exponents are compared)
        const bool ranges = ctx->level_begin.size() >= 2 && ctx->level_begin.back() == ctx->ncell;
        const int nlvl = ranges ? (int)ctx->level_begin.size() : 0;
        FMM_TRY(buf_ensure(ctx, ctx->m2l_mix, (size_t)nlvl * 8 + (size_t)nc * 4 + (size_t)nc + 64));
        int64_t* lvl = P_<int64_t>(ctx->m2l_mix);
        uint32_t* mlist = reinterpret_cast<uint32_t*>(lvl + nlvl);
        uint8_t* mixed = reinterpret_cast<uint8_t*>(mlist + nc);
        if (nlvl > 0)   // pageable source: staged at the call, ordered on s
            FMM_CUDA_TRY(ctx, cudaMemcpyAsync(lvl, ctx->level_begin.data(), (size_t)nlvl * 8, cudaMemcpyHostToDevice, s));
        FMM_CUDA_TRY(ctx, cudaMemsetAsync(counter, 0, 24, s));   // two work counters + the list length
        if (ranges && ctx->tc_mix_ncell == nc && ctx->nrem == 0) {   // (no grafted LET sources)
            // the target-ordered traversal flagged these targets while emitting the lists
            mir::k_m2l_mixed_flags<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(
                nc, P_<uint32_t>(ctx->tc_mixflag), mixed, mlist, counter + 2);
        } else {
            mir::k_m2l_mixed<<<std::max(g, 1), nw * 32, 0, s>>>(nc, ctx->ncell, P_<uint32_t>(ctx->m2l_src),
                                                                P_<uint64_t>(ctx->m2l_off), P_<int32_t>(ctx->c_level),
                                                                lvl, nlvl, sexp, mixed, mlist, counter + 2);
        }
        FMM_LAUNCH(ctx);
        mir::k_m2l_mir<P, false><<<ctx->num_sms * 2, 128, 0, s>>>(
            nc, P_<uint32_t>(ctx->m2l_src), P_<uint64_t>(ctx->m2l_off), P_<double4>(ctx->c_cr), sexp,
            reinterpret_cast<const float4*>(Sv), P_<double>(ctx->Lr), counter, mixed, lay);
        FMM_LAUNCH(ctx);
        mir::k_m2l_mir<P, true><<<ctx->num_sms * 2, 128, 0, s>>>(
            nc, P_<uint32_t>(ctx->m2l_src), P_<uint64_t>(ctx->m2l_off), P_<double4>(ctx->c_cr), sexp,
            reinterpret_cast<const float4*>(Sv), P_<double>(ctx->Lr), counter + 1, mixed, lay, mlist, counter + 2);
        FMM_LAUNCH(ctx);
    }
    if (!ctx->m2l_no_expand) {
        k_l_expand<<<std::max(g, 1), nw * 32, (size_t)nw * ctx->ncoef * 8, s>>>(
            nc, P, ctx->ncoef, P_<uint64_t>(ctx->m2l_off), ctx->m2l_off2, sexp, P_<double>(ctx->Lr),
            P_<double>(ctx->L));
        FMM_LAUNCH(ctx);
    }
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}
}  // namespace

// the reduced -> full L expansion alone (split multi-GPU flow, dist.cu): after the local and the
// remote register-kernel passes have left the summed reduced L_hat in ctx->Lr; off2 = the remote
// lists' offsets (a cell with neither a local nor a remote list gets L = 0)
fmm_status m2l_expand(fmm_ctx* ctx, const uint64_t* off2, cudaStream_t s) {
    const int64_t nc = ctx->ncell;
    const int nw = 4;
    const int g = (int)std::min<int64_t>((nc + nw - 1) / nw, (int64_t)ctx->num_sms * 16);
    k_l_expand<<<std::max(g, 1), nw * 32, (size_t)nw * ctx->ncoef * 8, s>>>(
        nc, ctx->P, ctx->ncoef, P_<uint64_t>(ctx->m2l_off), off2, ctx->m2l_sexp, P_<double>(ctx->Lr), P_<double>(ctx->L));
    FMM_LAUNCH(ctx);
    FMM_CUDA_TRY(ctx, cudaGetLastError());
    return FMM_OK;
}

// returns FMM_ERR_ARG (without launching) when no register kernel exists for (P, prec)
fmm_status m2l_fast(fmm_ctx* ctx, cudaStream_t s) {
    if (ctx->prec == FMM_F32) {
        if (ctx->m2l_variant == 0) {
            switch (ctx->P) {
                case 4: return m2l_mir_t<4>(ctx, s);
                case 6: return m2l_mir_t<6>(ctx, s);
                case 8: return m2l_mir_t<8>(ctx, s);
                case 10: return m2l_mir_t<10>(ctx, s);
                case 12: return m2l_mir_t<12>(ctx, s);
                case 16: return m2l_mir_t<16>(ctx, s);
                default: break;
            }
        }
        switch (ctx->P) {
            case 4: return m2l_fast_t<4, float>(ctx, s);
            case 6: return m2l_fast_t<6, float>(ctx, s);
            case 8: return m2l_fast_t<8, float>(ctx, s);
            case 10: return m2l_fast_t<10, float>(ctx, s);
            case 12: return m2l_mir_t<12>(ctx, s);   // no scalar P = 12, 16 kernels
            case 16: return m2l_mir_t<16>(ctx, s);
            default: break;
        }
    } else {
        switch (ctx->P) {
            case 4: return m2l_fast_t<4, double>(ctx, s);
            case 6: return m2l_fast_t<6, double>(ctx, s);
            default: break;
        }
    }
    return FMM_ERR_ARG;
}

bool m2l_fast_available(int P, int prec) {
    return prec == FMM_F32 ? (P == 4 || P == 6 || P == 8 || P == 10 || P == 12 || P == 16) : (P == 4 || P == 6);
}
