// loss.cu -- spectrum loss on the device, batched over frames (loss.py:65-155),
// chained into the rasterizer's upstream (upstream_to_ray, grad.py:104-120).
//
// Per frame b (power x = |S_b|^2, ground truth y, n = n_az * n_el cells):
//   L1      = mean |x - y|,                     dL1/dx = sign(x - y) / n
//   SSIM    = 1 - mean s, s = (a1 a2) / (b1 b2) with the 11x11 Gaussian window
//             (sigma 1.5, zero-padded borders, separable) and C1 = (0.01 D)^2,
//             C2 = (0.03 D)^2, D = max(max y - min y, 1e-6) (loss.py:95-128);
//             the gradient is the adjoint blur of ds/dmu, ds/dv, ds/dw
//   Fourier = sum |DFT(x) - DFT(y)|^2 / n = sum (x - y)^2 by Parseval (the
//             reference asserts that identity on every call, loss.py:131-146;
//             this takes the direct form), dF/dx = 2 (x - y)
//   total   = (1 - w_ssim - w_fourier) L1 + w_ssim SSIM + w_fourier Fourier
// and lam = 2 dL/dx S (upstream_to_ray), the complex-packed upstream of the
// backward.  The window statistics run in fp64 (E[x^2] - E[x]^2 cancels);
// every reduction uses fixed-order per-block partials (deterministic).
//
// Kernels: k_frame_range (per-frame min / max of y), k_ssim_fwd (tile of 16 x
// 32 cells + 5-cell halo in shared memory: the five blurred statistics, s and
// its three partials, per-block sums of s, |d| and d^2), k_ssim_bwd (adjoint
// blur of the partials, the blended frame gradient and lam), k_loss_final.
#include "rfs_common.cuh"

namespace {

constexpr int LW = 11, LH = 5;              // window, half width
constexpr int TU = 16, TV = 32;             // output tile (u rows, v columns)
constexpr int HU = TU + 2 * LH, HV = TV + 2 * LH;
constexpr int LT = 256;                     // threads per tile block

__constant__ double c_win[LW];

// the predicted power frame: given directly (pred) or |S|^2
__device__ __forceinline__ double power(const float2* __restrict__ S, const float* __restrict__ pred, size_t i) {
    if (pred) return (double)pred[i];
    const float2 s = S[i];
    return (double)s.x * s.x + (double)s.y * s.y;
}

// per-frame min / max of the ground truth (loss.py:108)
__global__ void __launch_bounds__(256) k_frame_range(const float* __restrict__ gt, int R, float2* __restrict__ range) {
    const int b = blockIdx.x;
    const float* y = gt + (size_t)b * R;
    float lo = INFINITY, hi = -INFINITY;
    for (int i = threadIdx.x; i < R; i += 256) {
        const float v = y[i];
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
    }
    __shared__ float sl[8], sh[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        sl[threadIdx.x >> 5] = lo;
        sh[threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) {
            lo = fminf(lo, sl[w]);
            hi = fmaxf(hi, sh[w]);
        }
        range[b] = make_float2(lo, hi);
    }
}

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < LT / 32; ++w) t += red[w];
    return t;
}

struct FwdSmem {
    double x[HU][HV], y[HU][HV];
    double h[5][HU][TV];  // v-blurred x, y, xx, yy, xy
    double red[LT / 32];
};

// grid (v tiles, u tiles, frames)
__global__ void __launch_bounds__(LT) k_ssim_fwd(const float2* __restrict__ S, const float* __restrict__ pred,
                                                 const float* __restrict__ gt,
                                                 const float2* __restrict__ range, int n_az, int n_el,
                                                 float* __restrict__ maps, double* __restrict__ part) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FwdSmem& M = *reinterpret_cast<FwdSmem*>(smem_raw);
    const int b = blockIdx.z, u0 = blockIdx.y * TU, v0 = blockIdx.x * TV;
    const size_t R = (size_t)n_az * n_el, fb = (size_t)b * R;
    const float2 rg = range[b];
    const double D = fmax((double)rg.y - (double)rg.x, 1e-6);
    const double c1 = (0.01 * D) * (0.01 * D), c2 = (0.03 * D) * (0.03 * D);
    for (int i = threadIdx.x; i < HU * HV; i += LT) {
        const int hu = i / HV, hv = i % HV, u = u0 - LH + hu, v = v0 - LH + hv;
        double xv = 0.0, yv = 0.0;
        if (u >= 0 && u < n_az && v >= 0 && v < n_el) {
            const size_t r = fb + (size_t)u * n_el + v;
            xv = power(S, pred, r);
            yv = gt[r];
        }
        M.x[hu][hv] = xv;
        M.y[hu][hv] = yv;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < HU * TV; i += LT) {  // correlate along v (axis 1)
        const int hu = i / TV, ov = i % TV;
        double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
#pragma unroll
        for (int t = 0; t < LW; ++t) {
            const double w = c_win[t], xv = M.x[hu][ov + t], yv = M.y[hu][ov + t];
            a0 += w * xv;
            a1 += w * yv;
            a2 += w * (xv * xv);
            a3 += w * (yv * yv);
            a4 += w * (xv * yv);
        }
        M.h[0][hu][ov] = a0; M.h[1][hu][ov] = a1; M.h[2][hu][ov] = a2; M.h[3][hu][ov] = a3; M.h[4][hu][ov] = a4;
    }
    __syncthreads();
    double s_sum = 0.0, l1 = 0.0, sq = 0.0;
    for (int i = threadIdx.x; i < TU * TV; i += LT) {  // correlate along u (axis 0)
        const int ou = i / TV, ov = i % TV, u = u0 + ou, v = v0 + ov;
        if (u >= n_az || v >= n_el) continue;
        double m[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int t = 0; t < LW; ++t) {
            const double w = c_win[t];
#pragma unroll
            for (int k = 0; k < 5; ++k) m[k] += w * M.h[k][ou + t][ov];
        }
        const double mx = m[0], my = m[1], vx = m[2], vy = m[3], wxy = m[4];
        const double A1 = 2.0 * mx * my + c1, A2 = 2.0 * (wxy - mx * my) + c2;
        const double B1 = mx * mx + my * my + c1, B2 = (vx - mx * mx) + (vy - my * my) + c2;
        const double s = (A1 * A2) / (B1 * B2);
        s_sum += s;
        const double ds_dmu = 2.0 * my * (A2 - A1) / (B1 * B2) - 2.0 * mx * s * (1.0 / B1 - 1.0 / B2);
        const double ds_dv = -s / B2;
        const double ds_dw = 2.0 * A1 / (B1 * B2);
        const size_t r = fb + (size_t)u * n_el + v;
        maps[r] = (float)ds_dmu;
        maps[R * gridDim.z + r] = (float)ds_dv;
        maps[2 * R * gridDim.z + r] = (float)ds_dw;
        const double d = M.x[ou + LH][ov + LH] - M.y[ou + LH][ov + LH];
        l1 += fabs(d);
        sq += d * d;
    }
    const int blk = blockIdx.y * gridDim.x + blockIdx.x, nblk = gridDim.x * gridDim.y;
    double* pb = part + ((size_t)b * nblk + blk) * 3;
    const double t0 = block_sum(s_sum, M.red);
    const double t1 = block_sum(l1, M.red);
    const double t2 = block_sum(sq, M.red);
    if (threadIdx.x == 0) {
        pb[0] = t0;
        pb[1] = t1;
        pb[2] = t2;
    }
}

struct BwdSmem {
    float m[3][HU][HV];
    double h[3][HU][TV];
};

__global__ void __launch_bounds__(LT) k_ssim_bwd(const float2* __restrict__ S, const float* __restrict__ pred,
                                                 const float* __restrict__ gt, const float* __restrict__ maps,
                                                 int n_az, int n_el, float w1, float ws, float wf,
                                                 float* __restrict__ grad, float2* __restrict__ lam) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BwdSmem& M = *reinterpret_cast<BwdSmem*>(smem_raw);
    const int b = blockIdx.z, u0 = blockIdx.y * TU, v0 = blockIdx.x * TV;
    const size_t R = (size_t)n_az * n_el, fb = (size_t)b * R, plane = R * gridDim.z;
    for (int i = threadIdx.x; i < HU * HV; i += LT) {
        const int hu = i / HV, hv = i % HV, u = u0 - LH + hu, v = v0 - LH + hv;
        const bool in = u >= 0 && u < n_az && v >= 0 && v < n_el;
        const size_t r = fb + (size_t)u * n_el + v;
#pragma unroll
        for (int k = 0; k < 3; ++k) M.m[k][hu][hv] = in ? maps[k * plane + r] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < HU * TV; i += LT) {  // adjoint of the zero-padded correlation = itself
        const int hu = i / TV, ov = i % TV;
        double a[3] = {0, 0, 0};
#pragma unroll
        for (int t = 0; t < LW; ++t) {
            const double w = c_win[t];
#pragma unroll
            for (int k = 0; k < 3; ++k) a[k] += w * (double)M.m[k][hu][ov + t];
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) M.h[k][hu][ov] = a[k];
    }
    __syncthreads();
    const double inv_n = 1.0 / (double)R;
    for (int i = threadIdx.x; i < TU * TV; i += LT) {
        const int ou = i / TV, ov = i % TV, u = u0 + ou, v = v0 + ov;
        if (u >= n_az || v >= n_el) continue;
        double a[3] = {0, 0, 0};
#pragma unroll
        for (int t = 0; t < LW; ++t) {
            const double w = c_win[t];
#pragma unroll
            for (int k = 0; k < 3; ++k) a[k] += w * M.h[k][ou + t][ov];
        }
        const size_t r = fb + (size_t)u * n_el + v;
        const double x = power(S, pred, r), y = gt[r], d = x - y;
        const double g1 = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) * inv_n;          // loss.py:65-72
        const double g2 = -(a[0] + a[1] * 2.0 * x + a[2] * y) * inv_n;                // loss.py:124-128
        const double g3 = 2.0 * d;                                                    // loss.py:146
        const double gx = (double)w1 * g1 + (double)ws * g2 + (double)wf * g3;        // loss.py:149-155
        if (grad) grad[r] = (float)gx;
        if (lam) {
            const float2 s = S[r];
            lam[r] = make_float2((float)(2.0 * gx * s.x), (float)(2.0 * gx * s.y));   // grad.py:119
        }
    }
}

// report[b] = {total, l1, ssim, fourier}
__global__ void k_loss_final(const double* __restrict__ part, int nblk, int n_frames, double n_cells, double w1,
                             double ws, double wf, double* __restrict__ report) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n_frames) return;
    double s = 0.0, l1 = 0.0, sq = 0.0;
    for (int k = 0; k < nblk; ++k) {
        const double* p = part + ((size_t)b * nblk + k) * 3;
        s += p[0];
        l1 += p[1];
        sq += p[2];
    }
    const double L1 = l1 / n_cells, SS = 1.0 - s / n_cells, FO = sq;
    report[4 * b + 0] = w1 * L1 + ws * SS + wf * FO;
    report[4 * b + 1] = L1;
    report[4 * b + 2] = SS;
    report[4 * b + 3] = FO;
}

bool g_win_ready = false;

int ensure_window() {
    if (g_win_ready) return RFS_OK;
    double w[LW], sum = 0.0;
    for (int i = 0; i < LW; ++i) {  // loss.py:75-81
        const double x = (double)(i - LH);
        w[i] = exp(-(x * x) / (2.0 * 1.5 * 1.5));
        sum += w[i];
    }
    for (int i = 0; i < LW; ++i) w[i] /= sum;
    RFS_CUDA_TRY(cudaMemcpyToSymbol(c_win, w, sizeof(w)));
    RFS_CUDA_TRY(cudaFuncSetAttribute(k_ssim_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FwdSmem)));
    RFS_CUDA_TRY(cudaFuncSetAttribute(k_ssim_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BwdSmem)));
    g_win_ready = true;
    return RFS_OK;
}

}  // namespace

extern "C" {

size_t rfs_loss_scratch_bytes(int n_frames, int n_az, int n_el) {
    const size_t R = (size_t)n_az * n_el;
    const size_t nblk = (size_t)rfs_ceil_div(n_el, TV) * rfs_ceil_div(n_az, TU);
    return 3 * R * n_frames * sizeof(float) + nblk * n_frames * 3 * sizeof(double) + n_frames * sizeof(float2) + 256;
}

int rfs_spectrum_loss(int n_frames, int n_az, int n_el, const void* S, const float* pred, const float* gt,
                      double w_ssim, double w_fourier, double* report, float* grad, void* lam, void* scratch,
                      size_t scratch_bytes, void* stream) {
    if (n_frames <= 0 || n_az <= 0 || n_el <= 0) return RFS_OK;
    if ((S == nullptr && pred == nullptr) || (lam != nullptr && S == nullptr)) return RFS_ERR_CONTRACT;
    if (scratch_bytes < rfs_loss_scratch_bytes(n_frames, n_az, n_el)) return RFS_ERR_CAPACITY;
    const int rc = ensure_window();
    if (rc != RFS_OK) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t R = (size_t)n_az * n_el;
    dim3 grid(rfs_ceil_div(n_el, TV), rfs_ceil_div(n_az, TU), n_frames);
    const int nblk = grid.x * grid.y;
    unsigned char* p = (unsigned char*)scratch;
    float* maps = (float*)p;
    p += 3 * R * n_frames * sizeof(float);
    double* part = (double*)p;
    p += (size_t)nblk * n_frames * 3 * sizeof(double);
    float2* range = (float2*)(((uintptr_t)p + 15) & ~(uintptr_t)15);
    const double w1 = 1.0 - w_ssim - w_fourier;
    k_frame_range<<<n_frames, 256, 0, st>>>(gt, (int)R, range);
    k_ssim_fwd<<<grid, LT, sizeof(FwdSmem), st>>>((const float2*)S, pred, gt, range, n_az, n_el, maps, part);
    k_ssim_bwd<<<grid, LT, sizeof(BwdSmem), st>>>((const float2*)S, pred, gt, maps, n_az, n_el, (float)w1,
                                                  (float)w_ssim, (float)w_fourier, grad, (float2*)lam);
    k_loss_final<<<rfs_ceil_div(n_frames, 128), 128, 0, st>>>(part, nblk, n_frames, (double)R, w1, w_ssim,
                                                              w_fourier, report);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // extern "C"
