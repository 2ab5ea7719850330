// rfs_common.cuh -- shared device types and helpers for the sm_100a rasterizer.
//
// Data layout in HBM:
//   RfsGeom[N]      128 B fp64 record per Gaussian (projection + shape), AoS so a
//                   gather by Gaussian id is 4 aligned 32 B sectors;
//   float4 sph[N]   fp32 bounding-sphere prefilter data (mu - rx, threshold);
//   keys/vals[M]    u64 tile|depth keys and u32 Gaussian ids, sorted;
//   RfsHit[R*HCAP]  per-ray live hit slab {g, w, T} (16 B), TX-independent;
//   psi[N][B]       complex64 directional response, row = Gaussian (512 B @ B=64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define RFS_TILE 16
#define RFS_TERM_EPS2 1e-12   // _kernels.py:20
#define RFS_TANGENT_EPS 1e-10 // _kernels.py:22
#define RFS_PI 3.141592653589793
#define RFS_TWO_PI 6.283185307179586
#define RFS_RAD2DEG 57.29577951308232           // splat.py:58
#define RFS_GAUSS_NORM 0.06349363593424097      // (2pi)^-1.5, render.py:48

// status codes (include/rfsplat_b200.h)
#define RFS_OK 0
#define RFS_ERR_GEOMETRY 1
#define RFS_ERR_SHAPE 2
#define RFS_ERR_CONTRACT 3
#define RFS_ERR_NONFINITE 4
#define RFS_ERR_CUDA 5
#define RFS_ERR_CAPACITY 6

struct __align__(16) RfsGeom {
    double mu[3];    // Gaussian mean
    double inv[6];   // Sigma^-1 (i00, i01, i02, i11, i12, i22)
    double norm;     // (2pi)^-1.5 / sqrt(det Sigma)
    double cu, cv;   // grid-space centre (splat.py:233-234)
    double r2;       // splat_r2 = tile_radius^2, -1 if inactive (render.py:243)
    double lbv;      // lower bound of any hit's t_mid: depth - r3 (conservative)
    double rho_re, rho_im; // complex transmittance |rho| e^{j phase}
};
static_assert(sizeof(RfsGeom) == 128, "RfsGeom must be 128 B");

struct __align__(16) RfsHit {
    uint32_t g;  // Gaussian id
    float w;     // Gaussian density at the chord midpoint
    float t_re;  // cumulative transmittance before this hit
    float t_im;
};
static_assert(sizeof(RfsHit) == 16, "RfsHit must be 16 B");

// per-Gaussian fp32 gradient accumulator (atomic target of the backward)
// dmu[3], dcov[9], dmag, dphase  -> 14 floats, padded to 16 (64 B)
#define RFS_GACC 16

#define RFS_CUDA_TRY(expr)                                   \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) return RFS_ERR_CUDA;          \
    } while (0)

#define RFS_LAUNCH_CHECK()                                   \
    do {                                                     \
        cudaError_t _e = cudaGetLastError();                 \
        if (_e != cudaSuccess) return RFS_ERR_CUDA;          \
    } while (0)

__device__ __forceinline__ float2 cmulf(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
__device__ __forceinline__ float2 cmulf_cj(float2 a, float2 b) {
    return make_float2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ float2 caddf(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

static inline int rfs_ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }
