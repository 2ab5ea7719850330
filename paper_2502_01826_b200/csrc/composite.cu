// composite.cu -- TX-batched kernels on top of the shared hit lists.
//
//   K5  k_psi          psi[g][b] = sum_k c_gk basis_k(bearing mu_g -> tx_b)
//   K7  k_forward      S[b][r]  = sum_k w_k T_k psi[g_k][b]                 (SpMM)
//   K8a k_backward_rays per ray, back to front, lanes over TX:
//                      C_k = sum_b conj(lam_b) psi[g_k][b]                  (SDDMM)
//                      A_k = w_{k+1} C_{k+1} + rho_{k+1} A_{k+1}  (suffix recursion)
//                      -> per-hit scalars GW_k = Re(T_k C_k), d|rho|_k, d(phase)_k
//                      and lamT[r][b] (lambda transposed for K9)
//   K8i k_hit_keys     by-Gaussian index of the hit slots (TX independent)
//   K9  k_grad_gauss   one warp per Gaussian over its hits:
//                      fp64 mean / covariance chains (_kernels.py:387-520)
//                      summed in fp64; P[b] = sum_hits conj(lam_b) w T (lanes
//                      over TX); d_coeffs = conj(P) conj(basis) (grad.py:255);
//                      bearing chain (grad.py:167-189); Sigma -> (q, s)
//                      (grad.py:134-164).  No atomics, fixed summation order.
//
// Because the backward is linear in the upstream lambda, every sum over the
// TX batch is taken before the TX-independent geometry: per hit only GW_k
// and A_k are needed, and A_k obeys the reference's suffix recursion
// (_kernels.py:382, 522) with psi replaced by C.
#include "rfs_common.cuh"

namespace {

// ---------------------------------------------------------------- FLE basis
// e^{i m alpha} P_l^m(cos beta) with Condon-Shortley phase and its alpha /
// beta derivatives (fle.py:153-212), from the bearing vector r = tx - mu
// without trigonometry: cos(beta) = rho/|r|, sin(beta) = z/|r|,
// e^{i alpha} = (x + i y)/rho.
template <int L>
struct Fle {
    static constexpr int K = (L + 1) * (L + 1);

    __device__ static __forceinline__ void eval_full(float rx, float ry, float rz, float2* B, float2* DA, float2* DB,
                                                     const float2* co, float2* dpa, float2* dpb) {
        float d = sqrtf(rx * rx + ry * ry + rz * rz);
        bool valid = d > 1e-12f;
        float rho = sqrtf(rx * rx + ry * ry);
        float x, sig, ca, sa;
        if (valid) {
            x = rho / d;
            sig = rz / d;
            if (rho > 0.f) {
                ca = rx / rho;
                sa = ry / rho;
            } else {
                float a = atan2f(ry, rx);
                sincosf(a, &sa, &ca);
            }
        } else {
            x = 1.f; sig = 0.f; ca = 1.f; sa = 0.f;
        }
        float s = fabsf(sig);
        float sgn = (sig > 0.f) ? 1.f : ((sig < 0.f) ? -1.f : 0.f);
        float dx = -sig, ds = sgn * x;
        float p[L + 1][L + 1], dp[L + 1][L + 1];
#pragma unroll
        for (int m = 0; m <= L; ++m) {
            float c = ((m & 1) ? -1.f : 1.f);
#pragma unroll
            for (int t = 2 * m - 1; t > 1; t -= 2) c *= (float)t;
            float sm = 1.f, sm1 = 1.f;
#pragma unroll
            for (int t = 0; t < m; ++t) sm *= s;
#pragma unroll
            for (int t = 0; t < m - 1; ++t) sm1 *= s;
            p[m][m] = c * sm;
            dp[m][m] = m > 0 ? c * (float)m * sm1 * ds : 0.f;
            if (m + 1 <= L) {
                p[m + 1][m] = x * (float)(2 * m + 1) * p[m][m];
                dp[m + 1][m] = (float)(2 * m + 1) * (dx * p[m][m] + x * dp[m][m]);
            }
#pragma unroll
            for (int l = m + 2; l <= L; ++l) {
                float a = (float)(2 * l - 1), b = (float)(l + m - 1), inv = 1.f / (float)(l - m);
                p[l][m] = (x * a * p[l - 1][m] - b * p[l - 2][m]) * inv;
                dp[l][m] = (dx * a * p[l - 1][m] + x * a * dp[l - 1][m] - b * dp[l - 2][m]) * inv;
            }
        }
        float2 em[L + 1];
        em[0] = make_float2(1.f, 0.f);
#pragma unroll
        for (int m = 1; m <= L; ++m) em[m] = cmulf(em[m - 1], make_float2(ca, sa));
#pragma unroll
        for (int l = 0; l <= L; ++l) {
#pragma unroll
            for (int m = -l; m <= l; ++m) {
                int ma = m < 0 ? -m : m;
                float ratio = 1.f;
                if (m < 0) {
                    float num = 1.f, den = 1.f;
                    for (int t = 2; t <= l - ma; ++t) num *= (float)t;
                    for (int t = 2; t <= l + ma; ++t) den *= (float)t;
                    ratio = ((ma & 1) ? -1.f : 1.f) * (num / den);
                }
                float2 az = m < 0 ? make_float2(em[ma].x, -em[ma].y) : em[ma];
                int idx = l * l + l + m;
                float pv = ratio * p[l][ma];
                B[idx] = make_float2(az.x * pv, az.y * pv);
                if (DA) DA[idx] = make_float2(-(float)m * az.y * pv, (float)m * az.x * pv);
                if (DB) {
                    float dv = ratio * dp[l][ma];
                    DB[idx] = make_float2(az.x * dv, az.y * dv);
                }
                if (co) {
                    // dpsi/dalpha = sum c (i m) basis, dpsi/dbeta = sum c e^{i m a} dP
                    float2 cb = cmulf(co[idx], make_float2(az.x * pv, az.y * pv));
                    dpa->x += -(float)m * cb.y;
                    dpa->y += (float)m * cb.x;
                    float dv = ratio * dp[l][ma];
                    float2 cd = cmulf(co[idx], make_float2(az.x * dv, az.y * dv));
                    dpb->x += cd.x;
                    dpb->y += cd.y;
                }
            }
        }
    }

    __device__ static __forceinline__ void eval(float rx, float ry, float rz, float2* B, float2* DA, float2* DB) {
        eval_full(rx, ry, rz, B, DA, DB, nullptr, nullptr, nullptr);
    }
    // basis plus the bearing derivatives of psi = sum_k co_k basis_k
    __device__ static __forceinline__ void eval_psi_derivs(float rx, float ry, float rz, float2* B, const float2* co,
                                                           float2& dpa, float2& dpb) {
        dpa = make_float2(0.f, 0.f);
        dpb = make_float2(0.f, 0.f);
        eval_full(rx, ry, rz, B, nullptr, nullptr, co, &dpa, &dpb);
    }
};

// ------------------------------------------------------------------ K5: psi
template <int L>
__global__ void __launch_bounds__(256) k_psi(int n, int nb, const float* __restrict__ means,
                                             const float2* __restrict__ coeffs, const float* __restrict__ tx,
                                             float2* __restrict__ psi) {
    constexpr int K = Fle<L>::K;
    long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)n * nb) return;
    int g = (int)(idx / nb), b = (int)(idx % nb);
    float rx = tx[3 * b] - means[3 * g];
    float ry = tx[3 * b + 1] - means[3 * g + 1];
    float rz = tx[3 * b + 2] - means[3 * g + 2];
    float2 B[K];
    Fle<L>::eval(rx, ry, rz, B, nullptr, nullptr);
    float2 acc = make_float2(0.f, 0.f);
    const float2* c = coeffs + (size_t)g * K;
#pragma unroll
    for (int k = 0; k < K; ++k) acc = caddf(acc, cmulf(__ldg(&c[k]), B[k]));
    psi[idx] = acc;
}

// --------------------------------------------------------------- K7 forward
constexpr int CP_RAYS = 32;      // rays per block (output staged for coalesced [B][R] stores)
constexpr int CP_THREADS = 256;  // 8 warps, 4 rays each
constexpr int CP_BCH = 64;       // TX per block (lanes own b and b + 32)

__global__ void __launch_bounds__(CP_THREADS) k_forward(const RfsHit* __restrict__ slab, const int* __restrict__ counts,
                                                        int hcap, const float2* __restrict__ psi, int nb, int R,
                                                        float2* __restrict__ S) {
    __shared__ float2 s_out[CP_BCH][CP_RAYS + 1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int r0 = blockIdx.x * CP_RAYS, bc = blockIdx.y * CP_BCH;
    const int b0 = bc + lane, b1 = bc + 32 + lane;
    for (int rl = wid; rl < CP_RAYS; rl += CP_THREADS / 32) {
        const int r = r0 + rl;
        float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
        if (r < R) {
            const int cnt = min(counts[r], hcap);
            const RfsHit* h = slab + (size_t)r * hcap;
            for (int k = 0; k < cnt; ++k) {
                RfsHit hk = h[k];
                float2 wt = make_float2(hk.w * hk.t_re, hk.w * hk.t_im);
                const float2* row = psi + (size_t)hk.g * nb;
                if (b0 < nb) a0 = caddf(a0, cmulf(wt, __ldg(&row[b0])));
                if (b1 < nb) a1 = caddf(a1, cmulf(wt, __ldg(&row[b1])));
            }
        }
        s_out[lane][rl] = a0;
        s_out[lane + 32][rl] = a1;
    }
    __syncthreads();
    const int nbc = min(CP_BCH, nb - bc);
    for (int i = threadIdx.x; i < nbc * CP_RAYS; i += CP_THREADS) {
        int bl = i / CP_RAYS, rl = i % CP_RAYS, r = r0 + rl;
        if (r < R) S[(size_t)(bc + bl) * R + r] = s_out[bl][rl];
    }
}

// ------------------------------------------------------- K8a backward rays
constexpr int BR_RAYS = 32;
constexpr int BR_THREADS = 256;
constexpr int BR_MAXJ = 8;  // up to 256 TX per launch (lane owns b = lane + 32 j)

__global__ void __launch_bounds__(BR_THREADS) k_backward_rays(
    const RfsHit* __restrict__ slab, const int* __restrict__ counts, int hcap, const float2* __restrict__ psi,
    const float2* __restrict__ lam, const float4* __restrict__ rho32, int nb, int R, float4* __restrict__ gslab,
    float2* __restrict__ lamT) {
    extern __shared__ __align__(16) float2 s_lam[];  // [nb][BR_RAYS + 1]
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int r0 = blockIdx.x * BR_RAYS;
    for (int i = threadIdx.x; i < nb * BR_RAYS; i += BR_THREADS) {
        int b = i / BR_RAYS, rl = i % BR_RAYS, r = r0 + rl;
        s_lam[b * (BR_RAYS + 1) + rl] = r < R ? lam[(size_t)b * R + r] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    // lambda transposed to [R][nb] rows for the per-Gaussian gather of K9
    for (int i = threadIdx.x; i < nb * BR_RAYS; i += BR_THREADS) {
        int rl = i / nb, b = i % nb, r = r0 + rl;
        if (r < R) lamT[(size_t)r * nb + b] = s_lam[b * (BR_RAYS + 1) + rl];
    }
    const int nj = (nb + 31) >> 5;
    for (int rl = wid; rl < BR_RAYS; rl += BR_THREADS / 32) {
        const int r = r0 + rl;
        if (r >= R) break;
        const int cnt = min(counts[r], hcap);
        if (cnt == 0) continue;
        float2 cl[BR_MAXJ];  // conj(lambda_b) for this lane's b
#pragma unroll
        for (int j = 0; j < BR_MAXJ; ++j) {
            int b = lane + 32 * j;
            float2 l = (j < nj && b < nb) ? s_lam[b * (BR_RAYS + 1) + rl] : make_float2(0.f, 0.f);
            cl[j] = make_float2(l.x, -l.y);
        }
        const RfsHit* h = slab + (size_t)r * hcap;
        float4* gs = gslab + (size_t)r * hcap;
        // A: sum_b conj(lam_b) suffix_{k,b}; (wn, rn, cn) = w, rho, C of hit k+1
        float2 A = make_float2(0.f, 0.f);
        float wn = 0.f;
        float2 rn = make_float2(0.f, 0.f), cn = make_float2(0.f, 0.f);
        for (int k = cnt - 1; k >= 0; --k) {
            RfsHit hk = h[k];
            const float2* row = psi + (size_t)hk.g * nb;
            float2 c = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < BR_MAXJ; ++j) {
                int b = lane + 32 * j;
                if (j < nj && b < nb) c = caddf(c, cmulf(cl[j], __ldg(&row[b])));
            }
            c.x = warp_sum(c.x);
            c.y = warp_sum(c.y);
            A = caddf(make_float2(wn * cn.x, wn * cn.y), cmulf(rn, A));
            float4 rq = __ldg(&rho32[hk.g]);
            if (lane == 0) {
                float2 t = make_float2(hk.t_re, hk.t_im);
                float gw = t.x * c.x - t.y * c.y;            // Re(T C)        (_kernels.py:387-388)
                float2 ta = cmulf(t, A);
                float dmag = ta.x * rq.z - ta.y * rq.w;      // Re(T e^{jphi} A) (_kernels.py:382-383)
                float dph = -(ta.x * rq.y + ta.y * rq.x);    // -Im(T rho A)     (_kernels.py:384-385)
                float4 o = gs[k];
                gs[k] = make_float4(o.x + gw, o.y + dmag, o.z + dph, 0.f);
            }
            wn = hk.w;
            rn = make_float2(rq.x, rq.y);
            cn = c;
        }
    }
}

// ------------------------------------------- K8i by-Gaussian hit-slot index
__global__ void k_hit_keys(const RfsHit* __restrict__ slab, const int* __restrict__ counts, const uint32_t* __restrict__ ray_off,
                           int hcap, int R, uint64_t* __restrict__ keys, uint32_t* __restrict__ slots) {
    const int lane = threadIdx.x & 31;
    const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (r >= R) return;
    const int cnt = min(counts[r], hcap);
    const uint32_t base = ray_off[r];
    for (int k = lane; k < cnt; k += 32) {
        keys[base + k] = slab[(size_t)r * hcap + k].g;
        slots[base + k] = (uint32_t)((size_t)r * hcap + k);
    }
}

// g_off[g] = lower_bound(g) over the sorted Gaussian keys, g in [0, n]
__global__ void k_gauss_offsets(const uint64_t* __restrict__ keys, int h, int n, int* __restrict__ g_off) {
    int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g > n) return;
    int lo = 0, hi = h;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if ((long long)keys[mid] < g) lo = mid + 1; else hi = mid;
    }
    g_off[g] = lo;
}

// ---------------------------------------------------------------- K9
__device__ void rot_from_quat(const double q[4], double R[9]) {
    double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
}

// Sum of 32 per-lane values of 32 lanes; afterwards lane l holds the total of value l (31 shuffles).
__device__ __forceinline__ float transpose_reduce32(float v[32], int lane) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const bool upper = (lane & s) != 0;
#pragma unroll
        for (int j = 0; j < s; ++j) {
            float send = upper ? v[j] : v[j + s];
            float keep = upper ? v[j + s] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
        }
    }
    return v[0];
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

constexpr int GG_THREADS = 256;

// One warp per Gaussian.
template <int L>
__global__ void __launch_bounds__(GG_THREADS) k_grad_gauss(
    int n, int nb, const float* __restrict__ means, const float* __restrict__ quats, const float* __restrict__ log_scales,
    const float* __restrict__ raw, const float2* __restrict__ coeffs, const float* __restrict__ tx,
    const RfsGeom* __restrict__ geom, const RfsHit* __restrict__ slab, int hcap, const float4* __restrict__ gslab,
    const float2* __restrict__ lamT, const int* __restrict__ g_off, const uint32_t* __restrict__ g_slots,
    const double* __restrict__ dirs, double rx0, double rx1, double rx2, double min_t, int include_dir, int accumulate,
    float* __restrict__ d_mean, float* __restrict__ d_quat, float* __restrict__ d_log_scale, float* __restrict__ d_mag,
    float* __restrict__ d_mag_raw, float* __restrict__ d_phase, float2* __restrict__ d_coeffs, float* __restrict__ d_cov) {
    constexpr int K = Fle<L>::K;
    constexpr int NV = 2 * K;                  // real values of d_coeffs
    constexpr int NG = (NV + 31) / 32;         // transpose-reduce groups
    const int lane = threadIdx.x & 31;
    const int g = (blockIdx.x * GG_THREADS + threadIdx.x) >> 5;
    if (g >= n) return;
    const int h0 = g_off[g], h1 = g_off[g + 1];

    // ---- phase A: TX-independent geometry chains, fp64, lanes over hits
    double acc[14];
#pragma unroll
    for (int i = 0; i < 14; ++i) acc[i] = 0.0;
    if (!accumulate && h1 > h0) {
        const RfsGeom* G = geom + g;
        const double mx = rx0 - G->mu[0], my = rx1 - G->mu[1], mz = rx2 - G->mu[2];
        const double i00 = G->inv[0], i01 = G->inv[1], i02 = G->inv[2], i11 = G->inv[3], i12 = G->inv[4],
                     i22 = G->inv[5];
        const double e0 = i00 * mx + i01 * my + i02 * mz, e1 = i01 * mx + i11 * my + i12 * mz,
                     e2 = i02 * mx + i12 * my + i22 * mz;
        const double c = e0 * mx + e1 * my + e2 * mz;
        for (int h = h0 + lane; h < h1; h += 32) {
            const uint32_t s = g_slots[h];
            const int r = (int)(s / (uint32_t)hcap);
            const float w = slab[s].w;
            const float4 gs = gslab[s];
            const double dx = dirs[3 * r], dy = dirs[3 * r + 1], dz = dirs[3 * r + 2];
            const double p0 = i00 * dx + i01 * dy + i02 * dz, p1 = i01 * dx + i11 * dy + i12 * dz,
                         p2 = i02 * dx + i12 * dy + i22 * dz;
            const double a = p0 * dx + p1 * dy + p2 * dz;
            const double b = p0 * mx + p1 * my + p2 * mz;
            const double disc = b * b - a * (c - 9.0);
            const double sq = sqrt(fmax(disc, 0.0));
            const double d2 = (-b + sq) / a, d1 = (-b - sq) / a;
            const bool clamped = d1 < min_t;
            const double t_mid = 0.5 * ((clamped ? min_t : d1) + d2);
            // q = Sigma^-1 (x_mid - mu) = t_mid p + e
            const double q0 = t_mid * p0 + e0, q1 = t_mid * p1 + e1, q2 = t_mid * p2 + e2;
            const double gww = (double)gs.x * (double)w;
            double gmu[3] = {gww * q0, gww * q1, gww * q2};
            const double f = 0.5 * gww;
            const double qv[3] = {q0, q1, q2};
            const double Iv[9] = {i00, i01, i02, i01, i11, i12, i02, i12, i22};
            double cv9[9];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j) cv9[3 * i + j] = f * (qv[i] * qv[j] - Iv[3 * i + j]);
            // Midpoint chain (_kernels.py:432-507).  For an unclamped chord the
            // midpoint minimises the quadratic form along the ray, so
            // q.d = t_mid a + b = 0 and the whole chain vanishes; only clamped
            // hits carry it.
            if (clamped && disc >= RFS_TANGENT_EPS) {
                const double pv[3] = {p0, p1, p2}, ev[3] = {e0, e1, e2};
                const double s_dv = q0 * dx + q1 * dy + q2 * dz;
                const double half = -0.5 * gww * s_dv;
                const double inv2sq = 0.5 / sq;
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) {
                    double bmu = -pv[ax], cmu = -2.0 * ev[ax];
                    double dd = (2.0 * b * bmu - a * cmu) * inv2sq;
                    gmu[ax] += half * ((-bmu + dd) / a);
                }
                const double cm9 = c - 9.0;
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j) {
                        double da = -pv[i] * pv[j], db = -pv[i] * ev[j], dc = -ev[i] * ev[j];
                        double ddisc = 2.0 * b * db - cm9 * da - a * dc;
                        cv9[3 * i + j] += half * ((-db + ddisc * inv2sq) / a - d2 * da / a);
                    }
            }
            acc[0] += gmu[0];
            acc[1] += gmu[1];
            acc[2] += gmu[2];
#pragma unroll
            for (int i = 0; i < 9; ++i) acc[3 + i] += cv9[i];
            acc[12] += (double)gs.y;
            acc[13] += (double)gs.z;
        }
#pragma unroll
        for (int i = 0; i < 14; ++i) acc[i] = warp_sum_d(acc[i]);
    }

    // ---- phase B: TX-dependent terms, lanes over TX
    float vals[NG * 32];
#pragma unroll
    for (int i = 0; i < NG * 32; ++i) vals[i] = 0.f;
    float dm0 = 0.f, dm1 = 0.f, dm2 = 0.f;
    if (h1 > h0) {
        const float mxf = means[3 * g], myf = means[3 * g + 1], mzf = means[3 * g + 2];
        float2 co[K];
#pragma unroll
        for (int k = 0; k < K; ++k) co[k] = __ldg(&coeffs[(size_t)g * K + k]);
        for (int b0 = 0; b0 < nb; b0 += 32) {
            const int b = b0 + lane;
            if (b >= nb) break;
            // P[g][b] = sum over hits of conj(lam_b) w T  (grad.py:252-254 bincount of inc_pg)
            float2 P = make_float2(0.f, 0.f);
            for (int h = h0; h < h1; ++h) {
                const uint32_t s = g_slots[h];
                const int r = (int)(s / (uint32_t)hcap);
                const RfsHit hk = slab[s];
                const float2 wt = make_float2(hk.w * hk.t_re, hk.w * hk.t_im);
                const float2 l = lamT[(size_t)r * nb + b];
                P = caddf(P, cmulf(make_float2(l.x, -l.y), wt));
            }
            const float rx = tx[3 * b] - mxf, ry = tx[3 * b + 1] - myf, rz = tx[3 * b + 2] - mzf;
            float2 B[K], dpa, dpb;
            Fle<L>::eval_psi_derivs(rx, ry, rz, B, co, dpa, dpb);
#pragma unroll
            for (int k = 0; k < K; ++k) {  // conj(P) conj(basis)
                vals[2 * k] += P.x * B[k].x - P.y * B[k].y;
                vals[2 * k + 1] += -(P.x * B[k].y + P.y * B[k].x);
            }
            if (include_dir) {
                const float zeta2 = rx * rx + ry * ry + rz * rz;
                const float rho2 = rx * rx + ry * ry;
                if (sqrtf(zeta2) > 1e-12f && rho2 > 1e-18f * zeta2) {
                    const float rho = sqrtf(rho2);
                    const float ga = P.x * dpa.x - P.y * dpa.y;  // Re(p dpsi/dalpha)
                    const float gb = P.x * dpb.x - P.y * dpb.y;
                    dm0 -= ga * (-ry / rho2) + gb * (-rz * rx / (rho * zeta2));
                    dm1 -= ga * (rx / rho2) + gb * (-rz * ry / (rho * zeta2));
                    dm2 -= gb * (rho / zeta2);
                }
            }
        }
    }
    float mine[NG];
#pragma unroll
    for (int q = 0; q < NG; ++q) mine[q] = transpose_reduce32(vals + 32 * q, lane);
    dm0 = warp_sum(dm0);
    dm1 = warp_sum(dm1);
    dm2 = warp_sum(dm2);

    float* dcf = reinterpret_cast<float*>(d_coeffs + (size_t)g * K);
#pragma unroll
    for (int q = 0; q < NG; ++q) {
        const int i = 32 * q + lane;
        if (i < NV) dcf[i] = accumulate ? dcf[i] + mine[q] : mine[q];
    }
    if (accumulate) {
        if (lane == 0) {
            d_mean[3 * g + 0] += dm0;
            d_mean[3 * g + 1] += dm1;
            d_mean[3 * g + 2] += dm2;
        }
        return;
    }
    if (lane != 0) return;
    d_mean[3 * g + 0] = (float)acc[0] + dm0;
    d_mean[3 * g + 1] = (float)acc[1] + dm1;
    d_mean[3 * g + 2] = (float)acc[2] + dm2;
    d_mag[g] = (float)acc[12];
    const float sg = 1.f / (1.f + expf(-raw[g]));
    d_mag_raw[g] = (float)acc[12] * sg * (1.f - sg);
    d_phase[g] = (float)acc[13];
    const double* dcv = acc + 3;
    if (d_cov) {
#pragma unroll
        for (int i = 0; i < 9; ++i) d_cov[9 * g + i] = (float)dcv[i];
    }
    // chain_cov_to_shape (grad.py:134-164), fp64
    double q[4] = {quats[4 * g], quats[4 * g + 1], quats[4 * g + 2], quats[4 * g + 3]};
    double nrm = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    double qu[4] = {q[0] / nrm, q[1] / nrm, q[2] / nrm, q[3] / nrm};
    double R[9];
    rot_from_quat(qu, R);
    double dv[3] = {exp(2.0 * (double)log_scales[3 * g]), exp(2.0 * (double)log_scales[3 * g + 1]),
                    exp(2.0 * (double)log_scales[3 * g + 2])};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) s += R[3 * i + a] * dcv[3 * i + j] * R[3 * j + a];
        d_log_scale[3 * g + a] = (float)(2.0 * dv[a] * s);
    }
    const double w = qu[0], x = qu[1], y = qu[2], z = qu[3];
    const double dr[4][9] = {{0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0},
                             {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * w, 2 * z, 2 * w, -4 * x},
                             {-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * z, -2 * w, 2 * z, -4 * y},
                             {-4 * z, -2 * w, 2 * x, 2 * w, -4 * z, 2 * y, 2 * x, 2 * y, 0}};
    double gq[4];
#pragma unroll
    for (int qi = 0; qi < 4; ++qi) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                double s1 = 0.0, s2 = 0.0;
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    s1 += dr[qi][3 * i + j] * dv[j] * R[3 * k + j];
                    s2 += R[3 * i + j] * dv[j] * dr[qi][3 * k + j];
                }
                s += dcv[3 * i + k] * (s1 + s2);
            }
        gq[qi] = s;
    }
    double dot = gq[0] * qu[0] + gq[1] * qu[1] + gq[2] * qu[2] + gq[3] * qu[3];
#pragma unroll
    for (int qi = 0; qi < 4; ++qi) d_quat[4 * g + qi] = (float)((gq[qi] - dot * qu[qi]) / nrm);
}

template <int L>
void launch_psi(int n, int nb, const float* means, const float2* coeffs, const float* tx, float2* psi, cudaStream_t st) {
    long long tot = (long long)n * nb;
    k_psi<L><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(n, nb, means, coeffs, tx, psi);
}

}  // namespace

extern "C" {

int rfs_psi(int n, int n_tx, int degree, const float* means, const void* coeffs, const float* tx, void* psi,
            void* stream) {
    if (n <= 0 || n_tx <= 0) return RFS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const float2* c = (const float2*)coeffs;
    float2* p = (float2*)psi;
    switch (degree) {
        case 0: launch_psi<0>(n, n_tx, means, c, tx, p, st); break;
        case 1: launch_psi<1>(n, n_tx, means, c, tx, p, st); break;
        case 2: launch_psi<2>(n, n_tx, means, c, tx, p, st); break;
        case 3: launch_psi<3>(n, n_tx, means, c, tx, p, st); break;
        case 4: launch_psi<4>(n, n_tx, means, c, tx, p, st); break;
        default: return RFS_ERR_SHAPE;
    }
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_forward(const void* slab, const int* counts, int hcap, const void* psi, int n_tx, int n_rays, void* S,
                void* stream) {
    if (n_rays <= 0 || n_tx <= 0) return RFS_OK;
    dim3 grid(rfs_ceil_div(n_rays, CP_RAYS), rfs_ceil_div(n_tx, CP_BCH));
    k_forward<<<grid, CP_THREADS, 0, (cudaStream_t)stream>>>((const RfsHit*)slab, counts, hcap, (const float2*)psi,
                                                             n_tx, n_rays, (float2*)S);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_backward_rays(const void* slab, const int* counts, int hcap, const void* psi, const void* lam, const void* rho32,
                      int n_tx, int n_rays, void* gslab, void* lamT, void* stream) {
    if (n_rays <= 0 || n_tx <= 0) return RFS_OK;
    if (n_tx > 32 * BR_MAXJ) return RFS_ERR_SHAPE;
    size_t smem = (size_t)n_tx * (BR_RAYS + 1) * sizeof(float2);
    static int attr = 0;
    if (smem > 48 * 1024 && attr < (int)smem) {
        RFS_CUDA_TRY(cudaFuncSetAttribute(k_backward_rays, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = (int)smem;
    }
    k_backward_rays<<<rfs_ceil_div(n_rays, BR_RAYS), BR_THREADS, smem, (cudaStream_t)stream>>>(
        (const RfsHit*)slab, counts, hcap, (const float2*)psi, (const float2*)lam, (const float4*)rho32, n_tx, n_rays,
        (float4*)gslab, (float2*)lamT);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_hit_keys(const void* slab, const int* counts, const uint32_t* ray_off, int hcap, int n_rays, uint64_t* keys,
                 uint32_t* slots, void* stream) {
    if (n_rays <= 0) return RFS_OK;
    k_hit_keys<<<rfs_ceil_div((long long)n_rays * 32, 256), 256, 0, (cudaStream_t)stream>>>(
        (const RfsHit*)slab, counts, ray_off, hcap, n_rays, keys, slots);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_gauss_offsets(const uint64_t* keys, int n_hits, int n, int* g_off, void* stream) {
    k_gauss_offsets<<<rfs_ceil_div(n + 1, 256), 256, 0, (cudaStream_t)stream>>>(keys, n_hits, n, g_off);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_grad_gauss(int n, int n_tx, int degree, const float* means, const float* quats, const float* log_scales,
                   const float* trans_mag_raw, const void* coeffs, const float* tx, const void* geom, const void* slab,
                   int hcap, const void* gslab, const void* lamT, const int* g_off, const uint32_t* g_slots,
                   const double* dirs, const double* rx, double ress_radius, int include_direction_chain, int accumulate,
                   float* d_mean, float* d_quat, float* d_log_scale, float* d_trans_mag, float* d_trans_mag_raw,
                   float* d_trans_phase, void* d_coeffs, float* d_cov, void* stream) {
    if (n <= 0) return RFS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned grid = (unsigned)rfs_ceil_div((long long)n * 32, GG_THREADS);
#define RFS_GG(LL)                                                                                                  \
    k_grad_gauss<LL><<<grid, GG_THREADS, 0, st>>>(                                                                  \
        n, n_tx, means, quats, log_scales, trans_mag_raw, (const float2*)coeffs, tx, (const RfsGeom*)geom,          \
        (const RfsHit*)slab, hcap, (const float4*)gslab, (const float2*)lamT, g_off, g_slots, dirs, rx[0], rx[1],    \
        rx[2], ress_radius, include_direction_chain, accumulate, d_mean, d_quat, d_log_scale, d_trans_mag,           \
        d_trans_mag_raw, d_trans_phase, (float2*)d_coeffs, d_cov)
    switch (degree) {
        case 0: RFS_GG(0); break;
        case 1: RFS_GG(1); break;
        case 2: RFS_GG(2); break;
        case 3: RFS_GG(3); break;
        case 4: RFS_GG(4); break;
        default: return RFS_ERR_SHAPE;
    }
#undef RFS_GG
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // extern "C"
