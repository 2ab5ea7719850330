// grad.cu -- K9: per-Gaussian backward over the by-Gaussian hit index.
//
// K9a k_geom_seg  (thread per hit, hits in Gaussian-sorted order, fp64):
//     mean / covariance chains of every hit (_kernels.py:387-520) scaled by
//     the TX-reduced weight gradient GW_k of K8r, plus d|rho| and d(phase);
//     each warp sums its runs of equal Gaussian id through shared memory
//     (one lane per (run, value)).  Gaussians whose hits straddle warps
//     leave per-warp partials that K9c adds in a fixed order (lanes over the
//     groups, then a fixed butterfly) -- deterministic; within a group the
//     slot order of the reference's bincount (grad.py:243-254).
// K9c k_geom_span (warp per straddling Gaussian: its group partials) + k_geom_final
//     (lane per Gaussian with hits, fp64): d_mean direct term, d_cov,
//     d|rho|, d(phase), chain_cov_to_shape (grad.py:134-164) and
//     d_trans_mag_raw = d|rho| sigma (1 - sigma) (train.py:161-162).
// K9b k_grad_tx (warp per Gaussian, lanes over TX; runs right after K8c):
//     from p_acc[g][b] (grad.py:252-254, built by K8c in fixed order),
//     d_coeffs = conj(p_acc) conj(basis) (grad.py:255) and the bearing chain
//     of d_mean (grad.py:167-189) into dm_dir, which K9c adds.
#include <algorithm>

#include "fle.cuh"
#include "rfs_common.cuh"

namespace {

constexpr int NACC = 14;         // dmu[3], dcov[9], d|rho|, d(phase)
constexpr int GB_THREADS = 128;
constexpr int GB_MAXJ = 8;       // up to 256 TX per launch
constexpr int FIX_SHORT = 16;    // straddle spans up to this many 32-hit groups: summed inline by K9c

// ------------------------------------------------------------------ K9a
__global__ void __launch_bounds__(256) k_geom_seg(
    int h, const uint32_t* __restrict__ h_dev, const uint64_t* __restrict__ sorted_g, const uint32_t* __restrict__ s_ray,
    const float* __restrict__ s_w,
    const uint32_t* __restrict__ s_slot, const float4* __restrict__ gs, const RfsGeom* __restrict__ geom, const double* __restrict__ dirs,
    const int2* __restrict__ g_rng, double rx0, double rx1, double rx2, double min_t, double* __restrict__ acc64,
    int* __restrict__ long_list, double* __restrict__ part_v) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    if (h_dev) h = min(h, (int)*h_dev);
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int wglob = p >> 5;
    if ((wglob << 5) >= h) return;  // whole warp past the device-side count
    const bool valid = p < h;
    const int g = valid ? (int)sorted_g[p] : -1;
    double v[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) v[i] = 0.0;
    if (valid) {
        const RfsGeom* G = geom + g;
        const double mx = rx0 - G->mu[0], my = rx1 - G->mu[1], mz = rx2 - G->mu[2];
        const double i00 = G->inv[0], i01 = G->inv[1], i02 = G->inv[2], i11 = G->inv[3], i12 = G->inv[4],
                     i22 = G->inv[5];
        const int r = (int)s_ray[p];
        const double w = s_w[p];
        const float4 gsv = gs[s_slot[p]];  // K8r's per-hit scalars, slab order
        const double dx = dirs[3 * r], dy = dirs[3 * r + 1], dz = dirs[3 * r + 2];
        const double e0 = i00 * mx + i01 * my + i02 * mz, e1 = i01 * mx + i11 * my + i12 * mz,
                     e2 = i02 * mx + i12 * my + i22 * mz;
        const double c = e0 * mx + e1 * my + e2 * mz;
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
        const double gww = (double)gsv.x * w;
        const double f = 0.5 * gww;
        v[0] = gww * q0;
        v[1] = gww * q1;
        v[2] = gww * q2;
        v[3] = f * (q0 * q0 - i00); v[4] = f * (q0 * q1 - i01); v[5] = f * (q0 * q2 - i02);
        v[6] = f * (q1 * q0 - i01); v[7] = f * (q1 * q1 - i11); v[8] = f * (q1 * q2 - i12);
        v[9] = f * (q2 * q0 - i02); v[10] = f * (q2 * q1 - i12); v[11] = f * (q2 * q2 - i22);
        // Midpoint chain (_kernels.py:432-507).  For an unclamped chord the
        // midpoint minimises the quadratic form along the ray, so
        // q.d = t_mid a + b = 0 and the chain vanishes; only clamped hits
        // carry it (the reference evaluates it to round-off).
        if (clamped && disc >= RFS_TANGENT_EPS) {
            const double pv[3] = {p0, p1, p2}, ev[3] = {e0, e1, e2};
            const double s_dv = q0 * dx + q1 * dy + q2 * dz;
            const double half = -0.5 * gww * s_dv;
            const double inv2sq = 0.5 / sq;
#pragma unroll 1
            for (int ax = 0; ax < 3; ++ax) {
                double bmu = -pv[ax], cmu = -2.0 * ev[ax];
                double dd = (2.0 * b * bmu - a * cmu) * inv2sq;
                v[ax] += half * ((-bmu + dd) / a);
            }
            const double cm9 = c - 9.0;
#pragma unroll 1
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    double da = -pv[i] * pv[j], db = -pv[i] * ev[j], dc = -ev[i] * ev[j];
                    double ddisc = 2.0 * b * db - cm9 * da - a * dc;
                    v[3 + 3 * i + j] += half * ((-db + ddisc * inv2sq) / a - d2 * da / a);
                }
        }
        v[12] = gsv.y;
        v[13] = (double)gsv.z + (double)gsv.w;  // d(phase) as a float pair (K8r)
    }
    // Segmented sums by Gaussian (segments are contiguous runs of lanes): the
    // lanes' values go to shared memory and task (segment k, value i) is summed
    // by one lane over the segment's hits in lane order -- fixed order,
    // deterministic, and no shuffle-bound scan.
    __shared__ double sv[256 / 32][32][NACC + 1];
    __shared__ int sg[256 / 32][32];
    __shared__ int sst[256 / 32][33];  // lane of each segment's first hit, then the end
    const int wl = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < NACC; ++i) sv[wl][lane][i] = v[i];
    sg[wl][lane] = g;
    const int gp = __shfl_up_sync(0xffffffffu, g, 1);
    const bool is_start = valid && (lane == 0 || gp != g);
    const unsigned smask = __ballot_sync(0xffffffffu, is_start);
    const int nvalid = __popc(__ballot_sync(0xffffffffu, valid));
    const int ns = __popc(smask);
    if (is_start) sst[wl][__popc(smask & ((1u << lane) - 1u))] = lane;
    if (lane == 0) sst[wl][ns] = nvalid;
    __syncwarp();
    const int wb = wglob << 5;
    for (int t = lane; t < ns * NACC; t += 32) {
        const int k = t / NACC, i = t - k * NACC;
        const int h_start = sst[wl][k];
        const int h_end = sst[wl][k + 1];
        double sum = 0.0;
        for (int q = h_start; q < h_end; ++q) sum += sv[wl][q][i];
        const int gk = sg[wl][h_start];
        const int2 rg = g_rng[gk];
        const int h0 = rg.x, h1 = rg.y;
        if (h0 >= wb && h1 - 1 <= wb + 31) {  // whole segment inside this warp
            acc64[(size_t)gk * NACC + i] = sum;
            continue;
        }
        // straddling segment: partial of this warp's first (slot 0) or last (slot 1) segment
        if (h0 < wb) part_v[(size_t)(2 * wglob) * NACC + i] = sum;
        if (h1 - 1 > wb + 31) {
            part_v[(size_t)(2 * wglob + 1) * NACC + i] = sum;
            // the warp holding a long Gaussian's first hit lists it for k_geom_span
            if (i == 0 && h0 >= wb && ((h1 - 1) >> 5) - (h0 >> 5) + 1 > FIX_SHORT) {
                const int q = atomicAdd(long_list, 1);
                long_list[1 + q] = gk;
            }
        }
    }
}

// Gaussians whose hits straddle warps: k_geom_final adds the group partials
// (slot 2w+1 of the group where the Gaussian starts, slot 2v of the later
// ones) in group order.

// chain_cov_to_shape for one Gaussian (grad.py:123-164), fp64, in closed
// form: with D = diag(e^{2s}) and Sigma = R D R^T,
//   d log_scale_a = 2 D_aa (R^T dSigma R)_aa,
//   dq_k = <dSigma, dR_k D R^T + R D dR_k^T> = sum_ij (dR_k)_ij M_ij,
//   M = (dSigma + dSigma^T) R D,
// then projected through the quaternion normalisation (grad.py:160-164) --
// the reference's triple loops (grad.py:134-158) regrouped, every array in
// registers.
__device__ __forceinline__ void cov_to_shape(const float* q4, const float* s3, const double* dcv, float* dq,
                                             float* ds) {
    const double q0 = q4[0], q1 = q4[1], q2 = q4[2], q3 = q4[3];
    const double nrm = sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
    const double qu[4] = {q0 / nrm, q1 / nrm, q2 / nrm, q3 / nrm};
    const double n2 = sqrt(qu[0] * qu[0] + qu[1] * qu[1] + qu[2] * qu[2] + qu[3] * qu[3]);
    double w = qu[0] / n2, x = qu[1] / n2, y = qu[2] / n2, z = qu[3] / n2;
    const double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                         2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                         2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
    const double dv[3] = {exp(2.0 * (double)s3[0]), exp(2.0 * (double)s3[1]), exp(2.0 * (double)s3[2])};
    // T = dSigma R (for the scales), Ssym = dSigma + dSigma^T, M = Ssym R D
    double T[9], M[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            double t = 0.0, m = 0.0;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                t += dcv[3 * i + k] * R[3 * k + j];
                m += (dcv[3 * i + k] + dcv[3 * k + i]) * R[3 * k + j];
            }
            T[3 * i + j] = t;
            M[3 * i + j] = m * dv[j];
        }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double s = R[a] * T[a] + R[3 + a] * T[3 + a] + R[6 + a] * T[6 + a];  // (R^T dSigma R)_aa
        ds[a] = (float)(2.0 * dv[a] * s);
    }
    w = qu[0]; x = qu[1]; y = qu[2]; z = qu[3];
    // rotation_derivatives (grad.py:123-131)
    const double dr[4][9] = {{0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0},
                             {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * w, 2 * z, 2 * w, -4 * x},
                             {-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * z, -2 * w, 2 * z, -4 * y},
                             {-4 * z, -2 * w, 2 * x, 2 * w, -4 * z, 2 * y, 2 * x, 2 * y, 0}};
    double gq[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        double g = 0.0;
#pragma unroll
        for (int e = 0; e < 9; ++e) g += dr[k][e] * M[e];
        gq[k] = g;
    }
    const double dot = gq[0] * qu[0] + gq[1] * qu[1] + gq[2] * qu[2] + gq[3] * qu[3];
#pragma unroll
    for (int k = 0; k < 4; ++k) dq[k] = (float)((gq[k] - dot * qu[k]) / nrm);
}

// ------------------------------------------------------------------ K9c
// k_geom_span: a block per long Gaussian (hits over more than FIX_SHORT
// 32-hit groups; k_geom_seg lists them, long_list[0] = count): its 14 sums
// from the group partials (slot 2w0+1 of the first group, slot 2v of the
// later ones), threads over the groups, then a fixed butterfly per warp and
// the 8 warp totals added in warp order (deterministic), into its acc64 row.
// A Gaussian covering thousands of rays (the 360x180 grids: up to 640
// groups) costs ceil(W/256) loads per thread.
__global__ void __launch_bounds__(256) k_geom_span(const int* __restrict__ long_list, const int2* __restrict__ g_rng,
                                                   const double* __restrict__ part_v, double* __restrict__ acc64) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    __shared__ double s_w[8][NACC];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int nl = long_list[0];
    for (int b = blockIdx.x; b < nl; b += gridDim.x) {
        const int g = long_list[1 + b];
        const int2 rg = g_rng[g];
        const int w0 = rg.x >> 5, w1 = (rg.y - 1) >> 5;
        double t[NACC];
#pragma unroll
        for (int k = 0; k < NACC; ++k) t[k] = 0.0;
        for (int v = w0 + threadIdx.x; v <= w1; v += 256) {
            const double* src = part_v + (size_t)(v == w0 ? 2 * w0 + 1 : 2 * v) * NACC;
#pragma unroll
            for (int k = 0; k < NACC; ++k) t[k] += src[k];
        }
#pragma unroll
        for (int k = 0; k < NACC; ++k) {
            double x = t[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if (lane == 0) s_w[wl][k] = x;
        }
        __syncthreads();
        if (threadIdx.x < NACC) {
            double x = s_w[0][threadIdx.x];
#pragma unroll
            for (int w = 1; w < 8; ++w) x += s_w[w][threadIdx.x];
            acc64[(size_t)g * NACC + threadIdx.x] = x;
        }
        __syncthreads();
    }
}

// k_geom_final: lane per Gaussian with live hits (order[i], i < min(cap,
// *n_used)): its 14 sums (acc64, or a short straddle's group partials), the direct d_mean term + K9b's bearing
// chain, d_cov, d|rho|, d(phase), d_trans_mag_raw and chain_cov_to_shape in
// fp64.  A grid-stride loop then zeroes the rows of the Gaussians without
// hits.  Every sum has a fixed order: deterministic.
__global__ void __launch_bounds__(128) k_geom_final(
    int cap, const uint32_t* __restrict__ n_used, const uint32_t* __restrict__ order, int n,
    const double* __restrict__ acc64, const double* __restrict__ part_v, const float* __restrict__ quats,
    const float* __restrict__ log_scales, const float* __restrict__ raw, float* __restrict__ d_mean,
    float* __restrict__ d_quat, float* __restrict__ d_log_scale, float* __restrict__ d_mag,
    float* __restrict__ d_mag_raw, float* __restrict__ d_phase, float* __restrict__ d_cov,
    const float* __restrict__ dm_dir, const int2* __restrict__ g_rng) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int m = n_used ? min(cap, (int)*n_used) : cap;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) {
        const int g = (int)order[i];
        const int2 rg = g_rng[g];
        const int w0 = rg.x >> 5, w1 = (rg.y - 1) >> 5;
        double a[NACC];
        if (w0 == w1 || w1 - w0 + 1 > FIX_SHORT) {  // one group, or summed by k_geom_span
#pragma unroll
            for (int k = 0; k < NACC; ++k) a[k] = acc64[(size_t)g * NACC + k];
        } else {  // a short straddle: the group partials in group order
#pragma unroll
            for (int k = 0; k < NACC; ++k) a[k] = part_v[(size_t)(2 * w0 + 1) * NACC + k];
            for (int v = w0 + 1; v <= w1; ++v) {
#pragma unroll
                for (int k = 0; k < NACC; ++k) a[k] += part_v[(size_t)(2 * v) * NACC + k];
            }
        }
        // direct term + the bearing chain of K9b (which ran before)
        d_mean[3 * g + 0] = (float)a[0] + (dm_dir ? dm_dir[3 * g + 0] : 0.f);
        d_mean[3 * g + 1] = (float)a[1] + (dm_dir ? dm_dir[3 * g + 1] : 0.f);
        d_mean[3 * g + 2] = (float)a[2] + (dm_dir ? dm_dir[3 * g + 2] : 0.f);
        d_mag[g] = (float)a[12];
        const float sg = 1.f / (1.f + expf(-raw[g]));
        d_mag_raw[g] = (float)a[12] * sg * (1.f - sg);
        d_phase[g] = (float)a[13];
        if (d_cov) {
#pragma unroll
            for (int k = 0; k < 9; ++k) d_cov[9 * g + k] = (float)a[3 + k];
        }
        cov_to_shape(quats + 4 * g, log_scales + 3 * g, a + 3, d_quat + 4 * g, d_log_scale + 3 * g);
    }
    // Gaussians without live hits (most): every term is zero
    for (int g = i; g < n; g += gridDim.x * blockDim.x) {
        const int2 rg = g_rng[g];
        if (rg.y != rg.x) continue;
#pragma unroll
        for (int k = 0; k < 3; ++k) d_mean[3 * g + k] = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) d_quat[4 * g + k] = 0.f;
#pragma unroll
        for (int k = 0; k < 3; ++k) d_log_scale[3 * g + k] = 0.f;
        d_mag[g] = 0.f;
        d_mag_raw[g] = 0.f;
        d_phase[g] = 0.f;
        if (d_cov) {
#pragma unroll
            for (int k = 0; k < 9; ++k) d_cov[9 * g + k] = 0.f;
        }
    }
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

// ------------------------------------------------------------------ K9b
// NJ = TX blocks of 32 per lane (compile time: no dead predicated iterations).
// Persistent warps walk the Gaussians with live hits in the index's spatial
// order (order[i], i < *n_used); the next Gaussian's p_acc row is requested
// while the current one is evaluated.  Then (unless accumulating) the
// d_coeffs rows of the Gaussians without hits (g_rng empty) are zeroed, so
// d_coeffs is complete when this kernel ends (an all-reduce bucket may
// start right behind it).
template <int L, int NJ>
__global__ void __launch_bounds__(GB_THREADS) k_grad_tx(
    int cap, const uint32_t* __restrict__ n_used, const uint32_t* __restrict__ order, int n,
    const int2* __restrict__ g_rng, int nb, const float* __restrict__ means, const float2* __restrict__ coeffs, const float* __restrict__ tx,
    const float2* __restrict__ P, int include_dir, int accumulate, float* __restrict__ dm_dir,
    float2* __restrict__ d_coeffs) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    constexpr int K = Fle<L>::K;
    constexpr int NV = 2 * K;
    constexpr int NG = (NV + 31) / 32;
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * GB_THREADS) >> 5;
    const int m = n_used ? min(cap, (int)*n_used) : cap;
    if (!accumulate) {
        for (int t = blockIdx.x * GB_THREADS + threadIdx.x; t < n; t += gridDim.x * GB_THREADS) {
            const int2 rg = g_rng[t];
            if (rg.y == rg.x)
                for (int k = 0; k < K; ++k) d_coeffs[(size_t)t * K + k] = make_float2(0.f, 0.f);
        }
    }
    int i = (blockIdx.x * GB_THREADS + threadIdx.x) >> 5;
    if (i >= m) return;
    const int nj = (nb + 31) >> 5;
    int g = (int)order[i];
    for (;;) {
        const int in = i + nw;
        int gn = 0;
        if (in < m) {
            gn = (int)order[in];
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int b = lane + 32 * j;
                if (j < nj && b < nb) asm volatile("prefetch.global.L1 [%0];" ::"l"(P + (size_t)gn * nb + b));
            }
        }
        float* dcf = reinterpret_cast<float*>(d_coeffs + (size_t)g * K);
        {  // (a used Gaussian always has hits; no branch, so the shuffles below stay warp-converged)
        float vals[NG * 32];
#pragma unroll
        for (int q = 0; q < NG * 32; ++q) vals[q] = 0.f;
        float dm0 = 0.f, dm1 = 0.f, dm2 = 0.f;
        const float mxf = means[3 * g], myf = means[3 * g + 1], mzf = means[3 * g + 2];
        const float2* co = coeffs + (size_t)g * K;
#pragma unroll 1
        for (int j = 0; j < NJ; ++j) {
            const int b = lane + 32 * j;
            if (j >= nj) break;
            if (b >= nb) continue;
            const float2 p = P[(size_t)g * nb + b];
            const float rx = tx[3 * b] - mxf, ry = tx[3 * b + 1] - myf, rz = tx[3 * b + 2] - mzf;
            typename Fle<L>::Tables T;
            Fle<L>::tables(rx, ry, rz, T);
            // grouped by order m: basis_lm = r_lm P_l^|m| E_m with E_m = e^{i m alpha}
            // (E_-m = conj E_m), so per m one complex factor serves every l:
            //   d_coeffs_lm += conj(p basis_lm) = r P_l^|m| conj(p E_m)
            //   dpsi/dalpha = sum_m (i m) E_m sum_l c_lm r P_l^|m|,
            //   dpsi/dbeta  = sum_m E_m sum_l c_lm r dP_l^|m|
            float2 q[2 * L + 1], A[2 * L + 1], Bm[2 * L + 1];
#pragma unroll
            for (int m = -L; m <= L; ++m) {
                const float2 e = m < 0 ? make_float2(T.em[-m].x, -T.em[-m].y) : T.em[m];
                const float2 pe = cmulf(p, e);
                q[m + L] = make_float2(pe.x, -pe.y);
                A[m + L] = make_float2(0.f, 0.f);
                Bm[m + L] = make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int l = 0; l <= L; ++l) {
#pragma unroll
                for (int m = -l; m <= l; ++m) {
                    const int idx = l * l + l + m, ma = m < 0 ? -m : m;
                    const float rt = Fle<L>::ratio(l, m);
                    const float pv = rt * T.p[l][ma];
                    // paired fp32 FMAs (FFMA2), the scalar form's operations
                    const float2 v2 = __ffma2_rn(make_float2(pv, pv), q[m + L],
                                                 make_float2(vals[2 * idx], vals[2 * idx + 1]));
                    vals[2 * idx] = v2.x;
                    vals[2 * idx + 1] = v2.y;
                    if (include_dir) {
                        const float2 cc = __ldg(&co[idx]);
                        const float dv = rt * T.dp[l][ma];
                        A[m + L] = __ffma2_rn(cc, make_float2(pv, pv), A[m + L]);
                        Bm[m + L] = __ffma2_rn(cc, make_float2(dv, dv), Bm[m + L]);
                    }
                }
            }
            float2 dpa = make_float2(0.f, 0.f), dpb = make_float2(0.f, 0.f);
            if (include_dir) {
#pragma unroll
                for (int m = -L; m <= L; ++m) {
                    const float2 e = m < 0 ? make_float2(T.em[-m].x, -T.em[-m].y) : T.em[m];
                    const float2 ea = cmulf(e, A[m + L]);
                    dpa.x = fmaf(-(float)m, ea.y, dpa.x);  // (i m) E_m A_m
                    dpa.y = fmaf((float)m, ea.x, dpa.y);
                    dpb = caddf(dpb, cmulf(e, Bm[m + L]));
                }
            }
            if (include_dir) {
                const float zeta2 = rx * rx + ry * ry + rz * rz;
                const float rho2 = rx * rx + ry * ry;
                if (sqrtf(zeta2) > 1e-12f && rho2 > 1e-18f * zeta2) {
                    const float rho = sqrtf(rho2);
                    const float ga = p.x * dpa.x - p.y * dpa.y;  // Re(p dpsi/dalpha)
                    const float gb = p.x * dpb.x - p.y * dpb.y;
                    dm0 -= ga * (-ry / rho2) + gb * (-rz * rx / (rho * zeta2));
                    dm1 -= ga * (rx / rho2) + gb * (-rz * ry / (rho * zeta2));
                    dm2 -= gb * (rho / zeta2);
                }
            }
        }
        float mine[NG];
#pragma unroll
        for (int q = 0; q < NG; ++q) mine[q] = transpose_reduce32(vals + 32 * q, lane);
        dm0 = warp_sum(dm0);
        dm1 = warp_sum(dm1);
        dm2 = warp_sum(dm2);
#pragma unroll
        for (int q = 0; q < NG; ++q) {
            const int t = 32 * q + lane;
            if (t < NV) dcf[t] = accumulate ? dcf[t] + mine[q] : mine[q];
        }
        if (lane == 0) {  // bearing chain of d_mean (grad.py:167-189); K9c adds the direct term
            dm_dir[3 * g + 0] = accumulate ? dm_dir[3 * g + 0] + dm0 : dm0;
            dm_dir[3 * g + 1] = accumulate ? dm_dir[3 * g + 1] + dm1 : dm1;
            dm_dir[3 * g + 2] = accumulate ? dm_dir[3 * g + 2] + dm2 : dm2;
        }
        }
        if (in >= m) break;
        i = in;
        g = gn;
    }
}

template <int L>
void launch_tx(unsigned grid, cudaStream_t st, int cap, const uint32_t* n_used, const uint32_t* order, int n,
               const int2* g_rng, int nb,
               const float* means, const float2* coeffs, const float* tx, const float2* P, int include_dir,
               int accumulate, float* dm_dir, float2* d_coeffs) {
    const int nj = (nb + 31) / 32;
#define RFS_GT(NJV)                                                                                                \
    rfs_launch(k_grad_tx<L, NJV>, grid, GB_THREADS, 0, st, cap, n_used, order, n, g_rng, nb, means, coeffs, tx, P, include_dir,     \
                                                   accumulate, dm_dir, d_coeffs)
    if (nj <= 2) RFS_GT(2); else RFS_GT(8);
#undef RFS_GT
}

}  // namespace

extern "C" {

size_t rfs_geom_part_elems(int n_hits) { return (size_t)2 * (size_t)((n_hits + 31) / 32 + 1); }

int rfs_grad_geom(int n, int n_hits, const uint32_t* h_dev, const uint64_t* sorted_g, const uint32_t* s_ray, const float* s_w,
                  const uint32_t* s_slot, const void* gs, const int* g_rng, const void* geom, const double* dirs, const double* rx,
                  double ress_radius, const float* quats, const float* log_scales, const float* trans_mag_raw,
                  int used_cap, const uint32_t* n_used, const uint32_t* order,
                  double* acc64, int* long_list, double* part_v, float* d_mean, float* d_quat, float* d_log_scale,
                  float* d_trans_mag, float* d_trans_mag_raw, float* d_trans_phase, float* d_cov, const float* dm_dir,
                  int stage, void* stream) {
    if (n <= 0) return RFS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int2* rg = (const int2*)g_rng;
    // acc64 rows / part_v slots are all written by k_geom_seg before k_geom_final
    // reads them (g_rng says which), so no clearing pass
    if (stage & 1) RFS_CUDA_TRY(rfs_fill_u32(long_list, 0u, 1, st));  // the long-Gaussian count
    if ((stage & 1) && n_hits > 0)
        rfs_launch(k_geom_seg, rfs_ceil_div(n_hits, 256), 256, 0, st, n_hits, h_dev, sorted_g, s_ray, s_w, s_slot,
                   (const float4*)gs, (const RfsGeom*)geom, dirs, rg, rx[0], rx[1], rx[2], ress_radius, acc64, long_list,
                   part_v);
    if (stage & 2) {
        if (order == nullptr) return RFS_ERR_CONTRACT;
        rfs_launch(k_geom_span, 148 * 2, 256, 0, st, (const int*)long_list, rg, (const double*)part_v, acc64);
        const long long ucap = std::max(used_cap, 1);
        const unsigned grid = (unsigned)std::max<long long>(rfs_ceil_div(ucap, 128),
                                                            std::min<long long>(rfs_ceil_div(n, 128), 148LL * 8));
        rfs_launch(k_geom_final, grid, 128, 0, st, used_cap, n_used, order, n, (const double*)acc64,
                   (const double*)part_v, quats, log_scales, trans_mag_raw, d_mean, d_quat, d_log_scale, d_trans_mag,
                   d_trans_mag_raw, d_trans_phase, d_cov, dm_dir, rg);
    }
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_grad_tx(int cap, const uint32_t* n_used, const uint32_t* order, int n, const int* g_rng, int n_tx, int degree,
                const float* means,
                const void* coeffs, const float* tx, const void* P, int include_direction_chain, int accumulate,
                float* dm_dir, void* d_coeffs, void* stream) {
    if (n <= 0) return RFS_OK;
    if (n_tx > 32 * GB_MAXJ) return RFS_ERR_SHAPE;
    if (P == nullptr || order == nullptr || g_rng == nullptr) return RFS_ERR_CONTRACT;
    cudaStream_t st = (cudaStream_t)stream;
    // persistent: 4 blocks of 4 warps per SM (128 registers per thread)
    unsigned grid = (unsigned)std::min<long long>(rfs_ceil_div((long long)std::max(cap, 1) * 32, GB_THREADS), 148LL * 4);
#define RFS_TX(LL)                                                                                                   \
    launch_tx<LL>(grid, st, cap, n_used, order, n, (const int2*)g_rng, n_tx, means, (const float2*)coeffs, tx, (const float2*)P,           \
                  include_direction_chain, accumulate, dm_dir, (float2*)d_coeffs)
    switch (degree) {
        case 0: RFS_TX(0); break;
        case 1: RFS_TX(1); break;
        case 2: RFS_TX(2); break;
        case 3: RFS_TX(3); break;
        case 4: RFS_TX(4); break;
        default: return RFS_ERR_SHAPE;
    }
#undef RFS_TX
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // extern "C"
