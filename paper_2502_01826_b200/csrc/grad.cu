// grad.cu -- K9: per-Gaussian backward over the by-Gaussian hit index.
//
// One warp per Gaussian g, no atomics, fixed summation order (the hit slots
// of g in (ray, k) order, like the reference's bincount over slots,
// grad.py:243-254):
//   phase A (lanes over hits, fp64): mean / covariance chains of every hit
//     (_kernels.py:387-520) scaled by the TX-reduced weight gradient GW_k of
//     K8a, plus d|rho| and d(phase);
//   phase B (lanes over TX): p_acc[g][b] = sum_hits conj(lam_b) w T
//     (grad.py:252-254), d_coeffs = conj(p_acc) conj(basis) (grad.py:255) and
//     the bearing chain into d_mean (grad.py:167-189);
//   epilogue (lane 0, fp64): chain_cov_to_shape (grad.py:134-164) and
//     d_trans_mag_raw = d|rho| sigma (1 - sigma) (train.py:161-162).
#include "fle.cuh"
#include "rfs_common.cuh"

namespace {

// One warp per block: hit counts per Gaussian range from 1 to ~1e3 (Gaussians
// near the receiver), and a single-warp block releases its SM slot as soon as
// its own Gaussian is done.
constexpr int GG_THREADS = 32;
constexpr int GG_WARPS = GG_THREADS / 32;
constexpr int GG_MAXJ = 8;       // up to 256 TX per launch

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Sum of 32 per-lane values over the warp; afterwards lane l holds the total
// of value l (31 shuffles instead of 32 x 5).
__device__ __forceinline__ float transpose_reduce32(float* v, int lane) {
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

__device__ void rot_from_quat(const double q[4], double R[9]) {
    double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
}

template <int L>
__global__ void __launch_bounds__(GG_THREADS, 16) k_grad_gauss(
    int n, int nb, const float* __restrict__ means, const float* __restrict__ quats, const float* __restrict__ log_scales,
    const float* __restrict__ raw, const float2* __restrict__ coeffs, const float* __restrict__ tx,
    const RfsGeom* __restrict__ geom, const RfsHit* __restrict__ slab, int hcap, const float4* __restrict__ gslab,
    const float2* __restrict__ lamT, const int* __restrict__ g_off, const uint32_t* __restrict__ g_slots,
    const double* __restrict__ dirs, double rx0, double rx1, double rx2, double min_t, int include_dir, int accumulate,
    float* __restrict__ d_mean, float* __restrict__ d_quat, float* __restrict__ d_log_scale, float* __restrict__ d_mag,
    float* __restrict__ d_mag_raw, float* __restrict__ d_phase, float2* __restrict__ d_coeffs, float* __restrict__ d_cov) {
    constexpr int K = Fle<L>::K;
    constexpr int NV = 2 * K;             // real values of d_coeffs
    constexpr int NG = (NV + 31) / 32;    // transpose-reduce groups
    __shared__ double s_acc[GG_WARPS][14];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int g = blockIdx.x * GG_WARPS + wl;
    if (g >= n) return;
    const int h0 = g_off[g], h1 = g_off[g + 1];
    const int nj = (nb + 31) >> 5;

    // ---- phase A: TX-independent geometry chains, fp64, lanes over hits
    if (!accumulate) {
        double acc[14];
#pragma unroll
        for (int i = 0; i < 14; ++i) acc[i] = 0.0;
        if (h1 > h0) {
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
                // q.d = t_mid a + b = 0 and the chain vanishes; only clamped hits
                // carry it (the reference evaluates it to round-off).
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
        }
#pragma unroll
        for (int i = 0; i < 14; ++i) {
            double v = warp_sum_d(acc[i]);
            if (lane == 0) s_acc[wl][i] = v;
        }
    }

    // ---- phase B: TX-dependent terms, lanes over TX
    float2 P[GG_MAXJ];
#pragma unroll
    for (int j = 0; j < GG_MAXJ; ++j) P[j] = make_float2(0.f, 0.f);
    for (int hb = h0; hb < h1; hb += 32) {
        const int h = hb + lane;
        int r = 0;
        float wtr = 0.f, wti = 0.f;
        if (h < h1) {
            const uint32_t s = g_slots[h];
            r = (int)(s / (uint32_t)hcap);
            const RfsHit hk = slab[s];
            wtr = hk.w * hk.t_re;
            wti = hk.w * hk.t_im;
        }
        const int nbh = min(32, h1 - hb);
        // 4 hits per iteration: independent lambda-row loads in flight
        for (int i0 = 0; i0 < nbh; i0 += 4) {
            int ri[4];
            float2 wt[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = min(i0 + u, 31);
                ri[u] = __shfl_sync(0xffffffffu, r, i);
                const bool ok = i0 + u < nbh;
                wt[u] = make_float2(ok ? __shfl_sync(0xffffffffu, wtr, i) : 0.f,
                                    ok ? __shfl_sync(0xffffffffu, wti, i) : 0.f);
            }
#pragma unroll
            for (int j = 0; j < GG_MAXJ; ++j) {
                const int b = lane + 32 * j;
                if (j < nj && b < nb) {
                    float2 l[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) l[u] = __ldg(&lamT[(size_t)ri[u] * nb + b]);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        P[j] = caddf(P[j], cmulf(make_float2(l[u].x, -l[u].y), wt[u]));  // conj(lam) w T
                }
            }
        }
    }
    float vals[NG * 32];
#pragma unroll
    for (int i = 0; i < NG * 32; ++i) vals[i] = 0.f;
    float dm0 = 0.f, dm1 = 0.f, dm2 = 0.f;
    if (h1 > h0) {
        const float mxf = means[3 * g], myf = means[3 * g + 1], mzf = means[3 * g + 2];
        const float2* co = coeffs + (size_t)g * K;
#pragma unroll
        for (int j = 0; j < GG_MAXJ; ++j) {
            const int b = lane + 32 * j;
            if (j < nj && b < nb) {
                const float2 Pj = P[j];
                const float rx = tx[3 * b] - mxf, ry = tx[3 * b + 1] - myf, rz = tx[3 * b + 2] - mzf;
                typename Fle<L>::Tables T;
                Fle<L>::tables(rx, ry, rz, T);
                float2 dpa = make_float2(0.f, 0.f), dpb = make_float2(0.f, 0.f);
                Fle<L>::for_each(T, [&](int idx, int m, float2 bv, float2 dbv) {
                    vals[2 * idx] += Pj.x * bv.x - Pj.y * bv.y;          // Re conj(P) conj(basis)
                    vals[2 * idx + 1] += -(Pj.x * bv.y + Pj.y * bv.x);   // Im
                    if (include_dir) {
                        const float2 cc = __ldg(&co[idx]);
                        const float2 cb = cmulf(cc, bv);
                        dpa.x += -(float)m * cb.y;  // d psi / d alpha = sum c (i m) basis
                        dpa.y += (float)m * cb.x;
                        dpb = caddf(dpb, cmulf(cc, dbv));
                    }
                });
                if (include_dir) {
                    const float zeta2 = rx * rx + ry * ry + rz * rz;
                    const float rho2 = rx * rx + ry * ry;
                    if (sqrtf(zeta2) > 1e-12f && rho2 > 1e-18f * zeta2) {
                        const float rho = sqrtf(rho2);
                        const float ga = Pj.x * dpa.x - Pj.y * dpa.y;  // Re(p dpsi/dalpha)
                        const float gb = Pj.x * dpb.x - Pj.y * dpb.y;
                        dm0 -= ga * (-ry / rho2) + gb * (-rz * rx / (rho * zeta2));
                        dm1 -= ga * (rx / rho2) + gb * (-rz * ry / (rho * zeta2));
                        dm2 -= gb * (rho / zeta2);
                    }
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
    __syncwarp();
    if (lane != 0) return;
    double acc[14];
#pragma unroll
    for (int i = 0; i < 14; ++i) acc[i] = s_acc[wl][i];
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
    // rotation_derivatives (grad.py:123-131)
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

}  // namespace

extern "C" {

int rfs_grad_gauss(int n, int n_tx, int degree, const float* means, const float* quats, const float* log_scales,
                   const float* trans_mag_raw, const void* coeffs, const float* tx, const void* geom, const void* slab,
                   int hcap, const void* gslab, const void* lamT, const int* g_off, const uint32_t* g_slots,
                   const double* dirs, const double* rx, double ress_radius, int include_direction_chain, int accumulate,
                   float* d_mean, float* d_quat, float* d_log_scale, float* d_trans_mag, float* d_trans_mag_raw,
                   float* d_trans_phase, void* d_coeffs, float* d_cov, void* stream) {
    if (n <= 0) return RFS_OK;
    if (n_tx > 32 * GG_MAXJ) return RFS_ERR_SHAPE;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned grid = (unsigned)rfs_ceil_div(n, GG_WARPS);
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
