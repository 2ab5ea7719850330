// composite.cu -- TX-batched kernels on top of the shared hit lists.
//
//   K5  k_psi            psi[g][b] = sum_k c_gk basis_k(bearing mu_g -> tx_b)
//   K7  k_forward        S[b][r]  = sum_k w_k T_k psi[g_k][b]          (SpMM)
//   K8a k_backward_rays  per ray, back to front: C_k = sum_b conj(lam_b) psi[g_k][b],
//                        suffix recursion for the transmittance chain, and
//                        P[g][b] += conj(lam_b) w_k T_k (vector atomics)
//   K8b k_backward_hits  per hit: fp64 mean/covariance chain (_kernels.py:387-520)
//                        scaled by the TX-reduced weight gradient, reduced
//                        per Gaussian with vector atomics
//   K9  k_epilogue       per Gaussian: d_coeffs, bearing chain, Sigma -> (q, s)
//
// Reference: forward_tiled _kernels.py:184-192, _ray_backward _kernels.py:360-522,
// backward_frame grad.py:243-258, _direction_chain grad.py:167-189,
// chain_cov_to_shape grad.py:134-164, fle_basis_with_derivs fle.py:153-212.
//
// Because the backward is linear in the upstream lambda, every sum over the
// TX batch can be taken before the TX-independent geometry: per hit only the
// scalars GW_k = Re(T_k C_k) and A_k = sum_b conj(lam_b) suffix_{k,b} are needed,
// and A_k obeys the same recursion as the reference's suffix with psi -> C.
#include "rfs_common.cuh"

namespace {

// ---------------------------------------------------------------- FLE basis
// Fourier-Legendre basis e^{i m alpha} P_l^m(cos beta) with Condon-Shortley
// phase, and its alpha / beta derivatives (fle.py:153-212), evaluated from the
// bearing vector r = tx - mu without trigonometry: cos(beta) = rho / |r|,
// sin(beta) = z / |r|, e^{i alpha} = (x + i y) / rho.
template <int L>
struct Fle {
    static constexpr int K = (L + 1) * (L + 1);

    __device__ static __forceinline__ void eval(float rx, float ry, float rz, float2* B, float2* DA, float2* DB) {
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
            }
        }
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
    const float2* __restrict__ lam, const float4* __restrict__ rho32, int nb, int R, float2* __restrict__ P,
    float4* __restrict__ gslab) {
    extern __shared__ __align__(16) float2 s_lam[];  // [nb][BR_RAYS + 1]
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int r0 = blockIdx.x * BR_RAYS;
    for (int i = threadIdx.x; i < nb * BR_RAYS; i += BR_THREADS) {
        int b = i / BR_RAYS, rl = i % BR_RAYS, r = r0 + rl;
        s_lam[b * (BR_RAYS + 1) + rl] = r < R ? lam[(size_t)b * R + r] : make_float2(0.f, 0.f);
    }
    __syncthreads();
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
        // A: running sum_b conj(lam_b) suffix_{k,b}; (wn, rn, cn) = w, rho, C of hit k+1
        float2 A = make_float2(0.f, 0.f);
        float wn = 0.f;
        float2 rn = make_float2(0.f, 0.f), cn = make_float2(0.f, 0.f);
        for (int k = cnt - 1; k >= 0; --k) {
            RfsHit hk = h[k];
            float4 rq = __ldg(&rho32[hk.g]);
            const float2* row = psi + (size_t)hk.g * nb;
            float2* prow = P + (size_t)hk.g * nb;
            float2 wt = make_float2(hk.w * hk.t_re, hk.w * hk.t_im);
            float2 c = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < BR_MAXJ; ++j) {
                int b = lane + 32 * j;
                if (j < nj && b < nb) {
                    c = caddf(c, cmulf(cl[j], __ldg(&row[b])));
                    atomicAdd(&prow[b], cmulf(cl[j], wt));  // P[g][b] += conj(lam_b) w T
                }
            }
            c.x = warp_sum(c.x);
            c.y = warp_sum(c.y);
            // A_k = w_{k+1} C_{k+1} + rho_{k+1} A_{k+1}   (A_{last} = 0)
            A = caddf(make_float2(wn * cn.x, wn * cn.y), cmulf(rn, A));
            if (lane == 0) {
                float2 t = make_float2(hk.t_re, hk.t_im);
                float gw = t.x * c.x - t.y * c.y;                    // Re(T C)
                float2 ta = cmulf(t, A);
                float dmag = ta.x * rq.z - ta.y * rq.w;              // Re(T e^{j phi} A)
                float dph = -(ta.x * rq.y + ta.y * rq.x);            // -Im(T rho A)
                float4 o = gs[k];
                gs[k] = make_float4(o.x + gw, o.y + dmag, o.z + dph, 0.f);
            }
            wn = hk.w;
            rn = make_float2(rq.x, rq.y);
            cn = c;
        }
    }
}

// ------------------------------------------------------- K8b backward hits
__device__ __forceinline__ void ray_dir64(int u, int v, int n_az, double d[3]) {
    double cell = 360.0 / (double)n_az;
    double al = ((double)u + 0.5) * cell * (RFS_PI / 180.0);
    double be = (((double)v + 0.5) * cell - 90.0) * (RFS_PI / 180.0);
    double sa, ca, sb, cb;
    sincos(al, &sa, &ca);
    sincos(be, &sb, &cb);
    d[0] = cb * ca;
    d[1] = cb * sa;
    d[2] = sb;
}

constexpr int BH_THREADS = 256;

// one warp per ray, one lane per hit
__global__ void __launch_bounds__(BH_THREADS) k_backward_hits(const RfsHit* __restrict__ slab, const int* __restrict__ counts,
                                                              int hcap, const float4* __restrict__ gslab,
                                                              const RfsGeom* __restrict__ geom, double rx0, double rx1,
                                                              double rx2, double min_t, int n_az, int n_el, int R,
                                                              float* __restrict__ gacc) {
    const int lane = threadIdx.x & 31;
    const int r = (blockIdx.x * BH_THREADS + threadIdx.x) >> 5;
    if (r >= R) return;
    const int cnt = min(counts[r], hcap);
    if (cnt == 0) return;
    const int u = r / n_el, v = r % n_el;
    double d[3];
    ray_dir64(u, v, n_az, d);
    const double dx = d[0], dy = d[1], dz = d[2];
    for (int k = lane; k < cnt; k += 32) {
        RfsHit hk = slab[(size_t)r * hcap + k];
        float4 gsk = gslab[(size_t)r * hcap + k];
        const RfsGeom* G = geom + hk.g;
        const double gw = gsk.x, w = hk.w;
        double mx = rx0 - G->mu[0], my = rx1 - G->mu[1], mz = rx2 - G->mu[2];
        double i00 = G->inv[0], i01 = G->inv[1], i02 = G->inv[2], i11 = G->inv[3], i12 = G->inv[4], i22 = G->inv[5];
        double p0 = i00 * dx + i01 * dy + i02 * dz, p1 = i01 * dx + i11 * dy + i12 * dz, p2 = i02 * dx + i12 * dy + i22 * dz;
        double e0 = i00 * mx + i01 * my + i02 * mz, e1 = i01 * mx + i11 * my + i12 * mz, e2 = i02 * mx + i12 * my + i22 * mz;
        double a = p0 * dx + p1 * dy + p2 * dz;
        double b = p0 * mx + p1 * my + p2 * mz;
        double c = e0 * mx + e1 * my + e2 * mz;
        double disc = b * b - a * (c - 9.0);
        double sq = sqrt(fmax(disc, 0.0));
        double d2 = (-b + sq) / a, d1 = (-b - sq) / a;
        bool clamped = d1 < min_t;
        double t_in = clamped ? min_t : d1;
        double t_mid = 0.5 * (t_in + d2);
        double ddx = t_mid * dx + mx, ddy = t_mid * dy + my, ddz = t_mid * dz + mz;  // x_mid - mu
        double q0 = i00 * ddx + i01 * ddy + i02 * ddz;
        double q1 = i01 * ddx + i11 * ddy + i12 * ddz;
        double q2 = i02 * ddx + i12 * ddy + i22 * ddz;
        double gmu[3] = {gw * w * q0, gw * w * q1, gw * w * q2};
        double f = gw * w * 0.5;
        double qv[3] = {q0, q1, q2};
        double Iv[9] = {i00, i01, i02, i01, i11, i12, i02, i12, i22};
        double cv9[9];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) cv9[3 * i + j] = f * (qv[i] * qv[j] - Iv[3 * i + j]);
        if (disc >= RFS_TANGENT_EPS) {
            double pv[3] = {p0, p1, p2}, ev[3] = {e0, e1, e2};
            double s_dv = q0 * dx + q1 * dy + q2 * dz;
            double half = 0.5 * (gw * (-w) * s_dv);
            double inv2sq = 0.5 / sq;
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                double bmu = -pv[ax], cmu = -2.0 * ev[ax];
                double dd = (2.0 * b * bmu - a * cmu) * inv2sq;
                double dsum = (-bmu + dd) / a;
                if (!clamped) dsum += (-bmu - dd) / a;
                gmu[ax] += half * dsum;
            }
            double cm9 = c - 9.0;
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    double da = -pv[i] * pv[j], db = -pv[i] * ev[j], dc = -ev[i] * ev[j];
                    double ddisc = 2.0 * b * db - cm9 * da - a * dc;
                    double dsum = (-db + ddisc * inv2sq) / a - d2 * da / a;
                    if (!clamped) dsum += (-db - ddisc * inv2sq) / a - d1 * da / a;
                    cv9[3 * i + j] += half * dsum;
                }
        }
        float4* acc = reinterpret_cast<float4*>(gacc + (size_t)hk.g * RFS_GACC);
        atomicAdd(acc + 0, make_float4((float)gmu[0], (float)gmu[1], (float)gmu[2], gsk.y));
        atomicAdd(acc + 1, make_float4((float)cv9[0], (float)cv9[1], (float)cv9[2], (float)cv9[3]));
        atomicAdd(acc + 2, make_float4((float)cv9[4], (float)cv9[5], (float)cv9[6], (float)cv9[7]));
        atomicAdd(acc + 3, make_float4((float)cv9[8], gsk.z, 0.f, 0.f));
    }
}

// --------------------------------------------------------------- K9 epilogue
__device__ void rot_from_quat(const double q[4], double R[9]) {
    double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
}

template <int L>
__global__ void __launch_bounds__(128) k_epilogue(
    int n, int nb, const float* __restrict__ means, const float* __restrict__ quats, const float* __restrict__ log_scales,
    const float* __restrict__ raw, const float2* __restrict__ coeffs, const float* __restrict__ tx,
    const float2* __restrict__ P, const float* __restrict__ gacc, int include_dir, int accumulate,
    float* __restrict__ d_mean, float* __restrict__ d_quat, float* __restrict__ d_log_scale, float* __restrict__ d_mag,
    float* __restrict__ d_mag_raw, float* __restrict__ d_phase, float2* __restrict__ d_coeffs, float* __restrict__ d_cov) {
    constexpr int K = Fle<L>::K;
    int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const float mx = means[3 * g], my = means[3 * g + 1], mz = means[3 * g + 2];
    float2 co[K];
#pragma unroll
    for (int k = 0; k < K; ++k) co[k] = coeffs[(size_t)g * K + k];
    float2 dc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) dc[k] = make_float2(0.f, 0.f);
    float dm0 = 0.f, dm1 = 0.f, dm2 = 0.f;
    const float2* prow = P + (size_t)g * nb;
    for (int b = 0; b < nb; ++b) {
        float2 p = prow[b];
        if (p.x == 0.f && p.y == 0.f) continue;  // Gaussian not hit under this TX
        float rx = tx[3 * b] - mx, ry = tx[3 * b + 1] - my, rz = tx[3 * b + 2] - mz;
        float2 B[K], DA[K], DB[K];
        Fle<L>::eval(rx, ry, rz, B, DA, DB);
        // d_coeffs = conj(p_acc) * conj(basis)   (grad.py:255)
#pragma unroll
        for (int k = 0; k < K; ++k) {
            dc[k].x += p.x * B[k].x - p.y * B[k].y;
            dc[k].y += -(p.x * B[k].y + p.y * B[k].x);
        }
        if (include_dir) {
            // _direction_chain (grad.py:167-189)
            float zeta2 = rx * rx + ry * ry + rz * rz;
            float rho2 = rx * rx + ry * ry;
            bool ok = (sqrtf(zeta2) > 1e-12f) && (rho2 > 1e-18f * zeta2);
            if (ok) {
                float rho = sqrtf(rho2);
                float2 dpa = make_float2(0.f, 0.f), dpb = make_float2(0.f, 0.f);
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    dpa = caddf(dpa, cmulf(co[k], DA[k]));
                    dpb = caddf(dpb, cmulf(co[k], DB[k]));
                }
                float ga = p.x * dpa.x - p.y * dpa.y;  // Re(p * dpsi/dalpha)
                float gb = p.x * dpb.x - p.y * dpb.y;
                dm0 -= ga * (-ry / rho2) + gb * (-rz * rx / (rho * zeta2));
                dm1 -= ga * (rx / rho2) + gb * (-rz * ry / (rho * zeta2));
                dm2 -= gb * (rho / zeta2);
            }
        }
    }
    if (accumulate) {
        // a later TX chunk of the same step: only the TX-dependent terms
#pragma unroll
        for (int k = 0; k < K; ++k) {
            float2 o = d_coeffs[(size_t)g * K + k];
            d_coeffs[(size_t)g * K + k] = make_float2(o.x + dc[k].x, o.y + dc[k].y);
        }
        d_mean[3 * g + 0] += dm0;
        d_mean[3 * g + 1] += dm1;
        d_mean[3 * g + 2] += dm2;
        return;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) d_coeffs[(size_t)g * K + k] = dc[k];
    const float* ga = gacc + (size_t)g * RFS_GACC;
    d_mean[3 * g + 0] = ga[0] + dm0;
    d_mean[3 * g + 1] = ga[1] + dm1;
    d_mean[3 * g + 2] = ga[2] + dm2;
    float dmag = ga[3];
    d_mag[g] = dmag;
    float sg = 1.f / (1.f + expf(-raw[g]));
    d_mag_raw[g] = dmag * sg * (1.f - sg);
    d_phase[g] = ga[13];
    double dcv[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        dcv[i] = ga[4 + i];
        if (d_cov) d_cov[9 * g + i] = ga[4 + i];
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
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) acc += R[3 * i + a] * dcv[3 * i + j] * R[3 * j + a];
        d_log_scale[3 * g + a] = (float)(2.0 * dv[a] * acc);
    }
    const double w = qu[0], x = qu[1], y = qu[2], z = qu[3];
    const double dr[4][9] = {{0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0},
                             {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * w, 2 * z, 2 * w, -4 * x},
                             {-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * z, -2 * w, 2 * z, -4 * y},
                             {-4 * z, -2 * w, 2 * x, 2 * w, -4 * z, 2 * y, 2 * x, 2 * y, 0}};
    double gq[4];
#pragma unroll
    for (int qi = 0; qi < 4; ++qi) {
        double acc = 0.0;
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
                acc += dcv[3 * i + k] * (s1 + s2);
            }
        gq[qi] = acc;
    }
    double dot = gq[0] * qu[0] + gq[1] * qu[1] + gq[2] * qu[2] + gq[3] * qu[3];
#pragma unroll
    for (int qi = 0; qi < 4; ++qi) d_quat[4 * g + qi] = (float)((gq[qi] - dot * qu[qi]) / nrm);
}

template <int L>
int launch_psi(int n, int nb, const float* means, const float2* coeffs, const float* tx, float2* psi, cudaStream_t st) {
    long long tot = (long long)n * nb;
    k_psi<L><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(n, nb, means, coeffs, tx, psi);
    return RFS_OK;
}

template <int L>
int launch_epi(int n, int nb, const float* means, const float* quats, const float* log_scales, const float* raw,
               const float2* coeffs, const float* tx, const float2* P, const float* gacc, int include_dir,
               int accumulate, float* d_mean, float* d_quat, float* d_log_scale, float* d_mag, float* d_mag_raw, float* d_phase,
               float2* d_coeffs, float* d_cov, cudaStream_t st) {
    k_epilogue<L><<<rfs_ceil_div(n, 128), 128, 0, st>>>(n, nb, means, quats, log_scales, raw, coeffs, tx, P, gacc,
                                                       include_dir, accumulate, d_mean, d_quat, d_log_scale, d_mag, d_mag_raw,
                                                       d_phase, d_coeffs, d_cov);
    return RFS_OK;
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
                      int n_tx, int n_rays, void* P, void* gslab, void* stream) {
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
        (float2*)P, (float4*)gslab);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_backward_hits(const void* slab, const int* counts, int hcap, const void* gslab, const void* geom, const double* rx,
                      double ress_radius, int n_az, int n_el, float* gacc, void* stream) {
    int R = n_az * n_el;
    if (R <= 0) return RFS_OK;
    k_backward_hits<<<rfs_ceil_div((long long)R * 32, BH_THREADS), BH_THREADS, 0, (cudaStream_t)stream>>>(
        (const RfsHit*)slab, counts, hcap, (const float4*)gslab, (const RfsGeom*)geom, rx[0], rx[1], rx[2], ress_radius,
        n_az, n_el, R, gacc);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_grad_epilogue(int n, int n_tx, int degree, const float* means, const float* quats, const float* log_scales,
                      const float* trans_mag_raw, const void* coeffs, const float* tx, const void* P, const float* gacc,
                      int include_direction_chain, int accumulate, float* d_mean, float* d_quat, float* d_log_scale,
                      float* d_trans_mag, float* d_trans_mag_raw, float* d_trans_phase, void* d_coeffs, float* d_cov,
                      void* stream) {
    if (n <= 0) return RFS_OK;
    cudaStream_t st = (cudaStream_t)stream;
#define RFS_EPI(LL)                                                                                                   \
    launch_epi<LL>(n, n_tx, means, quats, log_scales, trans_mag_raw, (const float2*)coeffs, tx, (const float2*)P, gacc, \
                   include_direction_chain, accumulate, d_mean, d_quat, d_log_scale, d_trans_mag, d_trans_mag_raw, d_trans_phase,  \
                   (float2*)d_coeffs, d_cov, st)
    switch (degree) {
        case 0: RFS_EPI(0); break;
        case 1: RFS_EPI(1); break;
        case 2: RFS_EPI(2); break;
        case 3: RFS_EPI(3); break;
        case 4: RFS_EPI(4); break;
        default: return RFS_ERR_SHAPE;
    }
#undef RFS_EPI
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // extern "C"
