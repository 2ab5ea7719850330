// train.cu -- optimizer and adaptive density control on the device
// (reference train.py:85-245), so a training run never leaves HBM.
//
//   k_sgd_check   finite check of every gradient row (train.py:133-142): the
//                 first class with a bad row and its lowest index, by atomicMin
//                 on class * N + row
//   k_sgd_update  skipped when the check found a bad row (the scene is left
//                 untouched, train.py:150); else w -= lr_w dL/dw per attribute,
//                 quaternion renormalisation, the logit chain of the
//                 transmittance magnitude, and TrainState.observe (EMA of
//                 |d_mean|, last d_mean; train.py:102-105)
//   k_density_flags  per Gaussian: keep / clone / split (densify, strict
//                 thresholds, radius = trace(Sigma) / 3) or keep / remove
//                 (prune: sigmoid(raw) < floor), train.py:184-190, 234-235
//   k_density_apply  stream compaction in the reference's order -- kept
//                 Gaussians, then clones, then two children per split parent
//                 (train.py:192-222) -- from exclusive scans of the flags.
//                 Children sample N(mu, Sigma) as mu + R diag(e^s) z with z
//                 from a counter-based Philox4x32-10 keyed by (seed,
//                 iteration, parent, child): identical on every rank without
//                 communication.
#include <math.h>

#include "rfs_common.cuh"

namespace {

// ------------------------------------------------------------------ Philox
struct U4 {
    uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

__device__ __forceinline__ double u01(uint32_t a) { return ((double)a + 0.5) * (1.0 / 4294967296.0); }

// three standard normals for (seed, iteration, parent, child) by Box-Muller
__device__ void normals3(unsigned long long seed, int iteration, int parent, int child, double z[3]) {
    const U4 r = philox4x32_10(U4{(uint32_t)parent, (uint32_t)child, (uint32_t)iteration, 0u}, (uint32_t)seed,
                               (uint32_t)(seed >> 32));
    const double r1 = sqrt(-2.0 * log(u01(r.x))), t1 = RFS_TWO_PI * u01(r.y);
    const double r2 = sqrt(-2.0 * log(u01(r.z))), t2 = RFS_TWO_PI * u01(r.w);
    z[0] = r1 * cos(t1);
    z[1] = r1 * sin(t1);
    z[2] = r2 * cos(t2);
}

// ------------------------------------------------------------------ SGD
__device__ __forceinline__ bool finite_row(const float* p, int k) {
    bool ok = true;
    for (int i = 0; i < k; ++i) ok &= isfinite(p[i]);
    return ok;
}

__global__ void k_sgd_check(int n, int K, const float* __restrict__ d_mean, const float* __restrict__ d_quat,
                            const float* __restrict__ d_log_scale, const float* __restrict__ d_mag,
                            const float* __restrict__ d_phase, const float* __restrict__ d_coeffs,
                            long long* __restrict__ bad) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    // class order of _check_finite (train.py:133-142): the smallest class * n + row wins the atomicMin,
    // which is the first bad class, then its first bad row
    if (g < n) {
        int cls = -1;
        if (!finite_row(d_mean + 3 * (size_t)g, 3)) cls = 0;
        else if (!finite_row(d_quat + 4 * (size_t)g, 4)) cls = 1;
        else if (!finite_row(d_log_scale + 3 * (size_t)g, 3)) cls = 2;
        else if (!isfinite(d_mag[g])) cls = 3;
        else if (!isfinite(d_phase[g])) cls = 4;
        if (cls >= 0) atomicMin((unsigned long long*)bad, (unsigned long long)cls * (unsigned long long)n + g);
    }
    // coefficients (class 5): a flat, coalesced pass (a row of 2K floats per thread thrashes L1)
    const size_t nf = (size_t)n * 2 * K, stride = (size_t)gridDim.x * blockDim.x;
    size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    auto flag = [&](size_t i) {
        atomicMin((unsigned long long*)bad, 5ull * (unsigned long long)n + (unsigned long long)(i / (2 * K)));
    };
    if (((uintptr_t)d_coeffs & 15) == 0) {  // 16-byte loads, then the tail
        const float4* d4 = (const float4*)d_coeffs;
        for (; e < nf / 4; e += stride) {
            const float4 d = d4[e];
            if (!(isfinite(d.x) && isfinite(d.y) && isfinite(d.z) && isfinite(d.w)))
                for (int k = 0; k < 4; ++k)
                    if (!isfinite(d_coeffs[4 * e + k])) flag(4 * e + k);
        }
        e = (nf / 4) * 4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    }
    for (; e < nf; e += stride)
        if (!isfinite(d_coeffs[e])) flag(e);
}

__global__ void k_sgd_update(int n, int K, float lr_mean, float lr_rot, float lr_scale, float lr_trans, float lr_rad,
                             float decay, const float* __restrict__ d_mean, const float* __restrict__ d_quat,
                             const float* __restrict__ d_log_scale, const float* __restrict__ d_mag,
                             const float* __restrict__ d_phase, const float* __restrict__ d_coeffs,
                             float* __restrict__ means, float* __restrict__ quats, float* __restrict__ log_scales,
                             float* __restrict__ raw, float* __restrict__ phase, float* __restrict__ coeffs,
                             float* __restrict__ grad_ema, float* __restrict__ last_dmean,
                             const long long* __restrict__ bad,
                             const long long* __restrict__ prior, const float* __restrict__ lr_mean_dev) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (*bad != 0x7f7f7f7f7f7f7f7fLL) return;
    if (prior && *prior != 0x7f7f7f7f7f7f7f7fLL) return;  // an earlier step was bad: the scene stays as it was
    if (lr_mean_dev) lr_mean = *lr_mean_dev;  // the schedule's value from the device (graph-captured loops)
    // coefficients: a flat, coalesced pass over all n * 2K floats
    {
        const size_t nf = (size_t)n * 2 * K, stride = (size_t)gridDim.x * blockDim.x;
        size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
        if ((((uintptr_t)coeffs | (uintptr_t)d_coeffs) & 15) == 0) {
            float4* c4 = (float4*)coeffs;
            const float4* d4 = (const float4*)d_coeffs;
            for (; e < nf / 4; e += stride) {
                float4 c = c4[e];
                const float4 d = d4[e];
                c.x -= lr_rad * d.x;
                c.y -= lr_rad * d.y;
                c.z -= lr_rad * d.z;
                c.w -= lr_rad * d.w;
                c4[e] = c;
            }
            e = (nf / 4) * 4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x;
        }
        for (; e < nf; e += stride) coeffs[e] -= lr_rad * d_coeffs[e];
    }
    if (g >= n) return;
    float dm[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        dm[a] = d_mean[3 * g + a];
        means[3 * g + a] -= lr_mean * dm[a];
        log_scales[3 * g + a] -= lr_scale * d_log_scale[3 * g + a];
    }
    float q[4], nq = 0.f;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        q[a] = quats[4 * g + a] - lr_rot * d_quat[4 * g + a];
        nq += q[a] * q[a];
    }
    nq = sqrtf(nq);
#pragma unroll
    for (int a = 0; a < 4; ++a) quats[4 * g + a] = q[a] / nq;
    const float mag = 1.f / (1.f + expf(-raw[g]));  // from the stored logit before the step
    raw[g] -= lr_trans * d_mag[g] * mag * (1.f - mag);
    phase[g] -= lr_trans * d_phase[g];
    if (grad_ema) {  // TrainState.observe (train.py:102-105)
        grad_ema[g] = decay * grad_ema[g] + (1.f - decay) * sqrtf(dm[0] * dm[0] + dm[1] * dm[1] + dm[2] * dm[2]);
#pragma unroll
        for (int a = 0; a < 3; ++a) last_dmean[3 * g + a] = dm[a];
    }
}

// ------------------------------------------------------------------ density
// mode 0: densify (keep = !split, clone, split); mode 1: prune (keep = !remove)
__global__ void k_density_flags(int n, int mode, const float* __restrict__ grad_ema,
                                const float* __restrict__ log_scales, const float* __restrict__ raw, double thr_grad,
                                double thr_radius, double thr_prune, uint32_t* __restrict__ keep,
                                uint32_t* __restrict__ clone, uint32_t* __restrict__ split) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    uint32_t k = 1, c = 0, s = 0;
    if (mode == 0) {
        if ((double)grad_ema[g] > thr_grad) {  // strictly above (train.py:184)
            double tr = 0.0;            // trace(R diag(e^{2s}) R^T) = sum e^{2s}
            for (int a = 0; a < 3; ++a) tr += exp(2.0 * (double)log_scales[3 * g + a]);
            if (tr / 3.0 > thr_radius) {
                s = 1;
                k = 0;
            } else {
                c = 1;
            }
        }
    } else {
        const double mag = 1.0 / (1.0 + exp(-(double)raw[g]));
        if (mag < thr_prune) k = 0;  // strictly below (train.py:234)
    }
    keep[g] = k;
    clone[g] = c;
    split[g] = s;
}

__device__ __forceinline__ void copy_attrs(int K, int src, int dst, const float* quats, const float* log_scales,
                                           const float* raw, const float* phase, const float* coeffs, float* o_quats,
                                           float* o_log_scales, float* o_raw, float* o_phase, float* o_coeffs) {
    for (int a = 0; a < 4; ++a) o_quats[4 * (size_t)dst + a] = quats[4 * (size_t)src + a];
    for (int a = 0; a < 3; ++a) o_log_scales[3 * (size_t)dst + a] = log_scales[3 * (size_t)src + a];
    o_raw[dst] = raw[src];
    o_phase[dst] = phase[src];
    for (int i = 0; i < 2 * K; ++i) o_coeffs[2 * (size_t)K * dst + i] = coeffs[2 * (size_t)K * src + i];
}

__global__ void k_density_apply(int n, int K, int mode, const uint32_t* __restrict__ keep,
                                const uint32_t* __restrict__ clone, const uint32_t* __restrict__ split,
                                const uint32_t* __restrict__ keep_off, const uint32_t* __restrict__ clone_off,
                                const uint32_t* __restrict__ split_off, const uint32_t* __restrict__ totals,
                                float step, float log_split, unsigned long long seed, int iteration,
                                const float* __restrict__ means, const float* __restrict__ quats,
                                const float* __restrict__ log_scales, const float* __restrict__ raw,
                                const float* __restrict__ phase, const float* __restrict__ coeffs,
                                const float* __restrict__ grad_ema, const float* __restrict__ last_dmean,
                                float* __restrict__ o_means, float* __restrict__ o_quats,
                                float* __restrict__ o_log_scales, float* __restrict__ o_raw,
                                float* __restrict__ o_phase, float* __restrict__ o_coeffs,
                                float* __restrict__ o_ema, float* __restrict__ o_last) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const uint32_t n_keep = totals[0], n_clone = totals[1];
    const bool reset = mode == 0;  // densify resets the statistics (train.py:221); prune compacts them
    if (keep[g]) {
        const int d = (int)keep_off[g];
        for (int a = 0; a < 3; ++a) o_means[3 * (size_t)d + a] = means[3 * (size_t)g + a];
        copy_attrs(K, g, d, quats, log_scales, raw, phase, coeffs, o_quats, o_log_scales, o_raw, o_phase, o_coeffs);
        o_ema[d] = reset ? 0.f : grad_ema[g];
        for (int a = 0; a < 3; ++a) o_last[3 * (size_t)d + a] = reset ? 0.f : last_dmean[3 * (size_t)g + a];
    }
    if (clone[g]) {  // shifted one mean-rate step down the last gradient (train.py:200-201)
        const int d = (int)(n_keep + clone_off[g]);
        for (int a = 0; a < 3; ++a)
            o_means[3 * (size_t)d + a] = means[3 * (size_t)g + a] - step * last_dmean[3 * (size_t)g + a];
        copy_attrs(K, g, d, quats, log_scales, raw, phase, coeffs, o_quats, o_log_scales, o_raw, o_phase, o_coeffs);
        o_ema[d] = 0.f;
        for (int a = 0; a < 3; ++a) o_last[3 * (size_t)d + a] = 0.f;
    }
    if (split[g]) {  // two children ~ N(mu, Sigma), scales shrunk by split_factor (train.py:207-215)
        double q[4] = {quats[4 * g], quats[4 * g + 1], quats[4 * g + 2], quats[4 * g + 3]};
        const double nq = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        const double w = q[0] / nq, x = q[1] / nq, y = q[2] / nq, z = q[3] / nq;
        const double Rm[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                              2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                              2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
        const double sd[3] = {exp((double)log_scales[3 * g]), exp((double)log_scales[3 * g + 1]),
                              exp((double)log_scales[3 * g + 2])};
        for (int c = 0; c < 2; ++c) {
            const int d = (int)(n_keep + n_clone + 2 * split_off[g] + c);
            double zz[3];
            normals3(seed, iteration, g, c, zz);
            for (int a = 0; a < 3; ++a) {
                const double off = Rm[3 * a] * sd[0] * zz[0] + Rm[3 * a + 1] * sd[1] * zz[1] + Rm[3 * a + 2] * sd[2] * zz[2];
                o_means[3 * (size_t)d + a] = (float)((double)means[3 * (size_t)g + a] + off);
            }
            copy_attrs(K, g, d, quats, log_scales, raw, phase, coeffs, o_quats, o_log_scales, o_raw, o_phase,
                       o_coeffs);
            for (int a = 0; a < 3; ++a) o_log_scales[3 * (size_t)d + a] = log_scales[3 * (size_t)g + a] - log_split;
            o_ema[d] = 0.f;
            for (int a = 0; a < 3; ++a) o_last[3 * (size_t)d + a] = 0.f;
        }
    }
}

}  // namespace

extern "C" {

int rfs_sgd_step(int n, int K, const float* lrs, float ema_decay, const float* d_mean, const float* d_quat,
                 const float* d_log_scale, const float* d_trans_mag, const float* d_trans_phase, const void* d_coeffs,
                 float* means, float* quats, float* log_scales, float* trans_mag_raw, float* trans_phase,
                 void* coeffs, float* grad_ema, float* last_dmean, long long* bad, const long long* prior,
                 const float* lr_mean_dev, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    RFS_CUDA_TRY(rfs_fill_u32(bad, 0x7f7f7f7fu, 2, st));  // sentinel 0x7f7f..7f = no bad row
    if (n <= 0) return RFS_OK;
    const int grid = rfs_ceil_div(n, 256);
    rfs_launch(k_sgd_check, grid, 256, 0, st, n, K, d_mean, d_quat, d_log_scale, d_trans_mag, d_trans_phase,
                                      (const float*)d_coeffs, bad);
    rfs_launch(k_sgd_update, grid, 256, 0, st, n, K, lrs[0], lrs[1], lrs[2], lrs[3], lrs[4], ema_decay, d_mean, d_quat,
                                       d_log_scale, d_trans_mag, d_trans_phase, (const float*)d_coeffs, means, quats,
                                       log_scales, trans_mag_raw, trans_phase, (float*)coeffs, grad_ema, last_dmean,
                                       bad, prior, lr_mean_dev);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_density_flags(int n, int mode, const float* grad_ema, const float* log_scales, const float* trans_mag_raw,
                      double thr_grad, double thr_radius, double thr_prune, uint32_t* keep, uint32_t* clone,
                      uint32_t* split, void* stream) {
    if (n <= 0) return RFS_OK;
    if (mode != 0 && mode != 1) return RFS_ERR_SHAPE;
    rfs_launch(k_density_flags, rfs_ceil_div(n, 256), 256, 0, (cudaStream_t)stream, 
        n, mode, grad_ema, log_scales, trans_mag_raw, thr_grad, thr_radius, thr_prune, keep, clone, split);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_density_apply(int n, int K, int mode, const uint32_t* keep, const uint32_t* clone, const uint32_t* split,
                      const uint32_t* keep_off, const uint32_t* clone_off, const uint32_t* split_off,
                      const uint32_t* totals, float step, float log_split_factor, unsigned long long seed,
                      int iteration, const float* means, const float* quats, const float* log_scales,
                      const float* trans_mag_raw, const float* trans_phase, const void* coeffs, const float* grad_ema,
                      const float* last_dmean, float* o_means, float* o_quats, float* o_log_scales, float* o_raw,
                      float* o_phase, void* o_coeffs, float* o_ema, float* o_last, void* stream) {
    if (n <= 0) return RFS_OK;
    rfs_launch(k_density_apply, rfs_ceil_div(n, 128), 128, 0, (cudaStream_t)stream, 
        n, K, mode, keep, clone, split, keep_off, clone_off, split_off, totals, step, log_split_factor, seed,
        iteration, means, quats, log_scales, trans_mag_raw, trans_phase, (const float*)coeffs, grad_ema, last_dmean,
        o_means, o_quats, o_log_scales, o_raw, o_phase, (float*)o_coeffs, o_ema, o_last);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // extern "C"
