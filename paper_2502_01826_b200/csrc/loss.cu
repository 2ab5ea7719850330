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
// backward.  The window statistics run in fp32 on tile-centred frames (the
// centring removes the E[x^2] - E[x]^2 cancellation), the per-cell SSIM terms
// in fp64; every reduction uses fixed-order per-block partials (deterministic).
//
// Kernels: k_frame_range (per-frame min / max of y), k_ssim_fwd (tile of 16 x
// 32 cells + 5-cell halo in shared memory: the five blurred statistics, s and
// its three partials, per-block sums of s, |d| and d^2), k_ssim_bwd (adjoint
// blur of the partials, the blended frame gradient and lam), k_loss_final.
#include "rfs_common.cuh"

namespace {

constexpr int LW = 11, LH = 5;              // window, half width
constexpr int TU = 32, TV = 32;             // output tile (u rows, v columns)
constexpr int HU = TU + 2 * LH, HV = TV + 2 * LH;
constexpr int LT = 256;                     // threads per tile block
constexpr int SEG = 4;                      // outputs per thread per pass (register sliding window)
constexpr int HVP = HV + 1, TVP = TV + 1;   // padded row pitches (conflict-free column walks)
static_assert(LT == TV * TU / SEG, "one vertical-pass item per thread");

__constant__ float c_winf[LW];

// the predicted power frame: given directly (pred) or |S|^2
__device__ __forceinline__ double power(const float2* __restrict__ S, const float* __restrict__ pred, size_t i) {
    if (pred) return (double)pred[i];
    const float2 s = S[i];
    return (double)s.x * s.x + (double)s.y * s.y;
}
// the same rounded to fp32, for the window statistics (computed in fp32): the
// correctly rounded fp32 of the fp64 power, so pred == gt gives SSIM = 1 exactly
__device__ __forceinline__ float power_f(const float2* __restrict__ S, const float* __restrict__ pred, int i) {
    if (pred) return __ldg(&pred[i]);
    const float2 s = __ldg(&S[i]);
    return (float)((double)s.x * s.x + (double)s.y * s.y);
}

// per-(frame, chunk) min / max of the ground truth (loss.py:108); the tile
// kernels reduce a frame's RCH partials themselves
constexpr int RCH = 32;
__global__ void __launch_bounds__(256) k_frame_range(const float* __restrict__ gt, int R, float2* __restrict__ range) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int b = blockIdx.y, c = blockIdx.x;
    const float* y = gt + (size_t)b * R;
    const int per = (R + RCH - 1) / RCH, i0 = c * per, i1 = min(R, i0 + per);
    float lo = INFINITY, hi = -INFINITY;
    for (int i = i0 + threadIdx.x; i < i1; i += 256) {
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
        range[b * RCH + c] = make_float2(lo, hi);
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

// Pairs of statistics are interleaved (float2) so both blur passes run as
// paired fp32 FMAs (FFMA2) on 8-byte shared-memory loads: per component the
// same fused operations in the same order as the scalar form.
struct FwdSmem {
    float2 xy[HU][HVP];            // raw frames (x, y; 0 in the padding)
    float2 h01[HU][TVP];           // v-blurred (x, y) of the centred frames
    float2 h23[HU][TVP];           // v-blurred (xx, yy)
    float h4[HU][TVP];             // v-blurred xy
    double red[LT / 32];
    float2 rng;                    // the frame's (min, max) of y
};

// The five window statistics in fp32 on frames centred by a per-tile constant
// c: with the normalised window and the zero padding written as x = 0, the
// centred frame x - c is -c in the padding, so blur(x - c) = mu_x - c and the
// (co)variances blur((x-c)^2) - blur(x-c)^2 equal vx - mu_x^2 exactly -- the
// centring removes the E[x^2] - E[x]^2 cancellation that made fp64 necessary.
// s, its partials and the sums are then evaluated in fp64 per cell.  Both
// separable passes slide an 11-value window through registers, SEG outputs
// per thread (one shared-memory load per input instead of eleven).
// grid (v tiles, u tiles, frames)
__global__ void __launch_bounds__(LT, 5) k_ssim_fwd(const float2* __restrict__ S, const float* __restrict__ pred,
                                                 const float* __restrict__ gt,
                                                 const float2* __restrict__ range, int n_az, int n_el,
                                                 float* __restrict__ maps, double* __restrict__ part) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FwdSmem& M = *reinterpret_cast<FwdSmem*>(smem_raw);
    const int b = blockIdx.z, u0 = blockIdx.y * TU, v0 = blockIdx.x * TV;
    const size_t R = (size_t)n_az * n_el, fb = (size_t)b * R;
    if (threadIdx.x < 32) {  // the frame's range: warp 0 folds the RCH = 32 chunk partials
        static_assert(RCH == 32, "one partial per lane");
        const float2 rg = range[b * RCH + threadIdx.x];
        float lo = rg.x, hi = rg.y;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (threadIdx.x == 0) M.rng = make_float2(lo, hi);
    }
    {   // halo load: the HU x HV cells in row-major order over all threads, every
        // load of the thread in flight before the stores; 32-bit frame offsets
        constexpr int NH = (HU * HV + LT - 1) / LT;
        const float2* Sb = S ? S + fb : nullptr;
        const float* pb = pred ? pred + fb : nullptr;
        const float* yb = gt + fb;
        float xv[NH], yv[NH];
#pragma unroll
        for (int k = 0; k < NH; ++k) {
            const int i = threadIdx.x + k * LT, hu = i / HV, hv = i - hu * HV;
            const int u = u0 - LH + hu, v = v0 - LH + hv;
            xv[k] = yv[k] = 0.f;
            if (hu < HU && u >= 0 && u < n_az && v >= 0 && v < n_el) {
                const int off = u * n_el + v;
                xv[k] = power_f(Sb, pb, off);
                yv[k] = __ldg(&yb[off]);
            }
        }
#pragma unroll
        for (int k = 0; k < NH; ++k) {
            const int i = threadIdx.x + k * LT, hu = i / HV, hv = i - hu * HV;
            if (hu < HU) M.xy[hu][hv] = make_float2(xv[k], yv[k]);
        }
    }
    __syncthreads();
    const double D = fmax((double)M.rng.y - (double)M.rng.x, 1e-6);
    const double c1 = (0.01 * D) * (0.01 * D), c2 = (0.03 * D) * (0.03 * D);
    const float2 cxy = M.xy[LH][LH];  // centre: the tile's first cell
    const float cx = cxy.x, cy = cxy.y;
    // correlate along v (axis 1): item = (segment, row), rows fastest -> conflict-free
    for (int it = threadIdx.x; it < (TV / SEG) * HU; it += LT) {
        const int sg = it / HU, hu = it - sg * HU, o0 = sg * SEG;
        float2 wd[SEG + LW - 1], wsq[SEG + LW - 1];
        float wxy[SEG + LW - 1];
        const float2 nc = make_float2(-cx, -cy);
#pragma unroll
        for (int j = 0; j < SEG + LW - 1; ++j) {  // the products once per input, not once per tap
            wd[j] = __fadd2_rn(M.xy[hu][o0 + j], nc);  // (x - cx, y - cy)
            wsq[j] = __fmul2_rn(wd[j], wd[j]);
            wxy[j] = wd[j].x * wd[j].y;
        }
#pragma unroll
        for (int o = 0; o < SEG; ++o) {
            float2 a01 = make_float2(0.f, 0.f), a23 = make_float2(0.f, 0.f);
            float a4 = 0.f;
#pragma unroll
            for (int t = 0; t < LW; ++t) {
                const float w = c_winf[t];
                a01 = __ffma2_rn(make_float2(w, w), wd[o + t], a01);
                a23 = __ffma2_rn(make_float2(w, w), wsq[o + t], a23);
                a4 = fmaf(w, wxy[o + t], a4);
            }
            M.h01[hu][o0 + o] = a01;
            M.h23[hu][o0 + o] = a23;
            M.h4[hu][o0 + o] = a4;
        }
    }
    __syncthreads();
    // correlate along u (axis 0): item = (segment of SEG rows, column), columns fastest
    double s_sum = 0.0, l1 = 0.0, sq = 0.0;
    {
        const int ov = threadIdx.x % TV, o0 = (threadIdx.x / TV) * SEG;  // LT = TV * TU / SEG
        const int v = v0 + ov;
        double dx[SEG];  // exact d = x - y of this thread's cells, loaded ahead of the blur
#pragma unroll
        for (int o = 0; o < SEG; ++o) {
            const int u = u0 + o0 + o;
            dx[o] = 0.0;
            if (u < n_az && v < n_el) {
                const size_t r = fb + (size_t)u * n_el + v;
                dx[o] = power(S, pred, r) - (double)gt[r];
            }
        }
        float m[5][SEG];
        {
            float2 w01[SEG + LW - 1], w23[SEG + LW - 1];
            float w4[SEG + LW - 1];
#pragma unroll
            for (int j = 0; j < SEG + LW - 1; ++j) {
                w01[j] = M.h01[o0 + j][ov];
                w23[j] = M.h23[o0 + j][ov];
                w4[j] = M.h4[o0 + j][ov];
            }
#pragma unroll
            for (int o = 0; o < SEG; ++o) {
                float2 a01 = make_float2(0.f, 0.f), a23 = make_float2(0.f, 0.f);
                float a4 = 0.f;
#pragma unroll
                for (int t = 0; t < LW; ++t) {
                    const float w = c_winf[t];
                    a01 = __ffma2_rn(make_float2(w, w), w01[o + t], a01);
                    a23 = __ffma2_rn(make_float2(w, w), w23[o + t], a23);
                    a4 = fmaf(w, w4[o + t], a4);
                }
                m[0][o] = a01.x;
                m[1][o] = a01.y;
                m[2][o] = a23.x;
                m[3][o] = a23.y;
                m[4][o] = a4;
            }
        }
#pragma unroll
        for (int o = 0; o < SEG; ++o) {
            const int u = u0 + o0 + o;
            if (u >= n_az || v >= n_el) continue;
            const double ex = m[0][o], ey = m[1][o];  // centred means
            const double mx = (double)cx + ex, my = (double)cy + ey;
            const double varx = (double)m[2][o] - ex * ex, vary = (double)m[3][o] - ey * ey;
            const double cov = (double)m[4][o] - ex * ey;
            const double A1 = 2.0 * mx * my + c1, A2 = 2.0 * cov + c2;
            const double B1 = mx * mx + my * my + c1, B2 = varx + vary + c2;
            const double inv = 1.0 / (B1 * B2);  // one division: 1/B1 = B2 inv, 1/B2 = B1 inv
            const double sv = A1 * A2 * inv;
            s_sum += sv;
            const double ds_dmu = 2.0 * my * (A2 - A1) * inv - 2.0 * mx * sv * ((B2 - B1) * inv);
            const double ds_dv = -sv * (B1 * inv);
            const double ds_dw = 2.0 * A1 * inv;
            const size_t r = fb + (size_t)u * n_el + v;
            maps[r] = (float)ds_dmu;
            maps[R * gridDim.z + r] = (float)ds_dv;
            maps[2 * R * gridDim.z + r] = (float)ds_dw;
            const double d = dx[o];
            l1 += fabs(d);
            sq += d * d;
        }
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
    float2 m01[HU][HVP];  // (ds/dmu, ds/dv) maps, interleaved for FFMA2
    float m2[HU][HVP];    // ds/dw
    float2 h01[HU][TVP];
    float h2[HU][TVP];
};

__global__ void __launch_bounds__(LT, 5) k_ssim_bwd(const float2* __restrict__ S, const float* __restrict__ pred,
                                                 const float* __restrict__ gt, const float* __restrict__ maps,
                                                 int n_az, int n_el, float w1, float ws, float wf,
                                                 float* __restrict__ grad, float2* __restrict__ lam,
                                                 float2* __restrict__ lamT) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BwdSmem& M = *reinterpret_cast<BwdSmem*>(smem_raw);
    const int b = blockIdx.z, u0 = blockIdx.y * TU, v0 = blockIdx.x * TV;
    const size_t R = (size_t)n_az * n_el, fb = (size_t)b * R, plane = R * gridDim.z;
    {   // halo load: the HU x HV cells in row-major order over all threads, every
        // load of the thread in flight before the stores; 32-bit frame offsets
        constexpr int NH = (HU * HV + LT - 1) / LT;
        const float* m0 = maps + fb;
        const float* m1 = m0 + plane;
        const float* m2 = m1 + plane;
        float mv[3][NH];
#pragma unroll
        for (int k = 0; k < NH; ++k) {
            const int i = threadIdx.x + k * LT, hu = i / HV, hv = i - hu * HV;
            const int u = u0 - LH + hu, v = v0 - LH + hv;
            const bool in = hu < HU && u >= 0 && u < n_az && v >= 0 && v < n_el;
            const int off = u * n_el + v;
            mv[0][k] = in ? __ldg(&m0[off]) : 0.f;
            mv[1][k] = in ? __ldg(&m1[off]) : 0.f;
            mv[2][k] = in ? __ldg(&m2[off]) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < NH; ++k) {
            const int i = threadIdx.x + k * LT, hu = i / HV, hv = i - hu * HV;
            if (hu < HU) {
                M.m01[hu][hv] = make_float2(mv[0][k], mv[1][k]);
                M.m2[hu][hv] = mv[2][k];
            }
        }
    }
    __syncthreads();
    // adjoint of the zero-padded correlation = the same correlation
    for (int it = threadIdx.x; it < (TV / SEG) * HU; it += LT) {
        const int sg = it / HU, hu = it - sg * HU, o0 = sg * SEG;
        float2 w01[SEG + LW - 1];
        float w2[SEG + LW - 1];
#pragma unroll
        for (int j = 0; j < SEG + LW - 1; ++j) {
            w01[j] = M.m01[hu][o0 + j];
            w2[j] = M.m2[hu][o0 + j];
        }
#pragma unroll
        for (int o = 0; o < SEG; ++o) {
            float2 a01 = make_float2(0.f, 0.f);
            float a2 = 0.f;
#pragma unroll
            for (int t = 0; t < LW; ++t) {
                const float w = c_winf[t];
                a01 = __ffma2_rn(make_float2(w, w), w01[o + t], a01);
                a2 = fmaf(w, w2[o + t], a2);
            }
            M.h01[hu][o0 + o] = a01;
            M.h2[hu][o0 + o] = a2;
        }
    }
    __syncthreads();
    const double inv_n = 1.0 / (double)R;
    const int ov = threadIdx.x % TV, o0 = (threadIdx.x / TV) * SEG;
    const int v = v0 + ov;
    float2 sv[SEG];  // this thread's cells, loaded ahead of the blur
    float xp[SEG], yv[SEG];
#pragma unroll
    for (int o = 0; o < SEG; ++o) {
        const int u = u0 + o0 + o;
        sv[o] = make_float2(0.f, 0.f);
        xp[o] = yv[o] = 0.f;
        if (u < n_az && v < n_el) {
            const size_t r = fb + (size_t)u * n_el + v;
            if (S) sv[o] = S[r];
            if (pred) xp[o] = pred[r];
            yv[o] = gt[r];
        }
    }
    float a[3][SEG];
    {
        float2 w01[SEG + LW - 1];
        float w2[SEG + LW - 1];
#pragma unroll
        for (int j = 0; j < SEG + LW - 1; ++j) {
            w01[j] = M.h01[o0 + j][ov];
            w2[j] = M.h2[o0 + j][ov];
        }
#pragma unroll
        for (int o = 0; o < SEG; ++o) {
            float2 a01 = make_float2(0.f, 0.f);
            float a2 = 0.f;
#pragma unroll
            for (int t = 0; t < LW; ++t) {
                const float w = c_winf[t];
                a01 = __ffma2_rn(make_float2(w, w), w01[o + t], a01);
                a2 = fmaf(w, w2[o + t], a2);
            }
            a[0][o] = a01.x;
            a[1][o] = a01.y;
            a[2][o] = a2;
        }
    }
#pragma unroll
    for (int o = 0; o < SEG; ++o) {
        const int u = u0 + o0 + o;
        if (u >= n_az || v >= n_el) continue;
        const size_t r = fb + (size_t)u * n_el + v;
        const double x = pred ? (double)xp[o] : (double)sv[o].x * sv[o].x + (double)sv[o].y * sv[o].y;
        const double y = yv[o], d = x - y;
        const double g1 = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) * inv_n;                   // loss.py:65-72
        const double g2 = -((double)a[0][o] + (double)a[1][o] * 2.0 * x + (double)a[2][o] * y) * inv_n;  // loss.py:124-128
        const double g3 = 2.0 * d;                                                              // loss.py:146
        const double gx = (double)w1 * g1 + (double)ws * g2 + (double)wf * g3;                  // loss.py:149-155
        if (grad) grad[r] = (float)gx;
        const float2 l = make_float2((float)(2.0 * gx * sv[o].x), (float)(2.0 * gx * sv[o].y));  // grad.py:119
        if (lam) lam[r] = l;
        if (lamT) lamT[(r - fb) * gridDim.z + b] = l;  // [R][B]: the backward's layout (a ray's TX row)
    }
}

// report[b] = {total, l1, ssim, fourier}; one warp per frame, fixed order
__global__ void k_loss_final(const double* __restrict__ part, int nblk, int n_frames, double n_cells, double w1,
                             double ws, double wf, double* __restrict__ report) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int lane = threadIdx.x & 31;
    const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (b >= n_frames) return;
    double s = 0.0, l1 = 0.0, sq = 0.0;
    for (int k = lane; k < nblk; k += 32) {
        const double* p = part + ((size_t)b * nblk + k) * 3;
        s += p[0];
        l1 += p[1];
        sq += p[2];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
    }
    if (lane) return;
    const double L1 = l1 / n_cells, SS = 1.0 - s / n_cells, FO = sq;
    report[4 * b + 0] = w1 * L1 + ws * SS + wf * FO;
    report[4 * b + 1] = L1;
    report[4 * b + 2] = SS;
    report[4 * b + 3] = FO;
}

// ------------------------------------------------------------------ scalar modes
// Single-antenna output: total = coherent sum of the frame (render_scalar,
// render.py:301-307) and scalar_loss (loss.py:158-180): mode 0 'complex'
// |total - target|^2 with upstream 2 (total - target); mode 1 'real_power'
// |10 log10 |total|^2 - dBm| with upstream sign(.) 20/ln10 total / |total|^2,
// and |total|^2 <= 1e-20 floored at -200 dBm with zero upstream.  The upstream
// of a coherent sum is the same for every ray (train.py:288): lam[b][r].
// One block per frame, fixed-order reduction.
__global__ void __launch_bounds__(256) k_scalar_loss(const float2* __restrict__ S, int R, int mode,
                                                     const float2* __restrict__ target, double* __restrict__ report,
                                                     float2* __restrict__ total_out, float2* __restrict__ lam) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int b = blockIdx.x;
    const float2* f = S + (size_t)b * R;
    double sr = 0.0, si = 0.0;
    for (int i = threadIdx.x; i < R; i += 256) {
        const float2 v = f[i];
        sr += v.x;
        si += v.y;
    }
    __shared__ double red[2][8];
    __shared__ double up[2];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sr += __shfl_xor_sync(0xffffffffu, sr, o);
        si += __shfl_xor_sync(0xffffffffu, si, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = sr;
        red[1][threadIdx.x >> 5] = si;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tr = 0.0, ti = 0.0;
        for (int w = 0; w < 8; ++w) {
            tr += red[0][w];
            ti += red[1][w];
        }
        const float2 t = target[b];
        double value, ur, ui;
        if (mode == 0) {
            const double dr = tr - t.x, di = ti - t.y;
            value = dr * dr + di * di;
            ur = 2.0 * dr;
            ui = 2.0 * di;
        } else {
            const double gt = t.x, p = tr * tr + ti * ti;
            if (p <= 1e-20) {
                value = fabs(-200.0 - gt);
                ur = ui = 0.0;
            } else {
                const double dbm = 10.0 * log10(p);
                const double sgn = dbm > gt ? 1.0 : (dbm < gt ? -1.0 : 0.0);
                const double sc = sgn * (20.0 / log(10.0)) / p;
                value = fabs(dbm - gt);
                ur = sc * tr;
                ui = sc * ti;
            }
        }
        report[4 * b + 0] = value;
        report[4 * b + 1] = value;
        report[4 * b + 2] = 0.0;
        report[4 * b + 3] = 0.0;
        if (total_out) total_out[b] = make_float2((float)tr, (float)ti);
        up[0] = ur;
        up[1] = ui;
    }
    __syncthreads();
    if (lam) {
        const float2 u = make_float2((float)up[0], (float)up[1]);
        for (int i = threadIdx.x; i < R; i += 256) lam[(size_t)b * R + i] = u;
    }
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
    float wf[LW];
    for (int i = 0; i < LW; ++i) wf[i] = (float)(w[i] / sum);
    RFS_CUDA_TRY(cudaMemcpyToSymbol(c_winf, wf, sizeof(wf)));
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
    return 3 * R * n_frames * sizeof(float) + nblk * n_frames * 3 * sizeof(double) +
           (size_t)n_frames * RCH * sizeof(float2) + 256;
}

size_t rfs_frame_range_elems(int n_frames) { return (size_t)(n_frames > 0 ? n_frames : 0) * RCH; }

int rfs_frame_range(int n_frames, int n_az, int n_el, const float* gt, void* range, void* stream) {
    if (n_frames <= 0 || n_az <= 0 || n_el <= 0) return RFS_OK;
    rfs_launch(k_frame_range, dim3(RCH, n_frames), 256, 0, (cudaStream_t)stream, gt, n_az * n_el, (float2*)range);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_spectrum_loss(int n_frames, int n_az, int n_el, const void* S, const float* pred, const float* gt,
                      double w_ssim, double w_fourier, double* report, float* grad, void* lam, void* lamT, void* scratch,
                      size_t scratch_bytes, const void* gt_range, void* stream) {
    if (n_frames <= 0 || n_az <= 0 || n_el <= 0) return RFS_OK;
    if ((S == nullptr && pred == nullptr) || ((lam != nullptr || lamT != nullptr) && S == nullptr))
        return RFS_ERR_CONTRACT;
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
    if (gt_range == nullptr)
        rfs_launch(k_frame_range, dim3(RCH, n_frames), 256, 0, st, gt, (int)R, range);
    else
        range = (float2*)gt_range;  // precomputed (rfs_frame_range, e.g. right behind the frames' H2D copy)
    rfs_launch(k_ssim_fwd, grid, LT, sizeof(FwdSmem), st, (const float2*)S, pred, gt, (const float2*)range, n_az, n_el,
               maps, part);
    rfs_launch(k_ssim_bwd, grid, LT, sizeof(BwdSmem), st, (const float2*)S, pred, gt, maps, n_az, n_el, (float)w1,
                                                  (float)w_ssim, (float)w_fourier, grad, (float2*)lam,
                                                  (float2*)lamT);
    rfs_launch(k_loss_final, rfs_ceil_div((long long)n_frames * 32, 128), 128, 0, st, part, nblk, n_frames, (double)R, w1,
                                                                                w_ssim, w_fourier, report);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_scalar_loss(int n_frames, int n_rays, int mode, const void* S, const void* target, double* report,
                    void* total, void* lam, void* stream) {
    if (n_frames <= 0 || n_rays <= 0) return RFS_OK;
    if (mode != 0 && mode != 1) return RFS_ERR_SHAPE;
    rfs_launch(k_scalar_loss, n_frames, 256, 0, (cudaStream_t)stream, (const float2*)S, n_rays, mode, (const float2*)target,
                                                              report, (float2*)total, (float2*)lam);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // extern "C"
