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
#include <utility>
#include <stdint.h>

#define RFS_TILE 16
#ifndef RFS_PCAP_EVICT
#define RFS_PCAP_EVICT 0x10000  // rfs_hits: pcap flag, as include/rfsplat_b200.h defines it
#endif
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

// ---- programmatic dependent launch (Hopper/Blackwell) ----
// Every kernel is launched with programmatic stream serialization: its CTAs
// may be scheduled while the previous kernel in the stream drains (its tail
// wave, its exit), and each kernel's first instruction is griddepcontrol.wait,
// which returns once the previous grid has completed and its memory is
// visible.  So dependent launches overlap the launch latency and the
// predecessor's tail -- also between the nodes of a captured CUDA graph --
// with unchanged semantics.
__device__ __forceinline__ void rfs_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
static inline cudaError_t rfs_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                     Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Fill n 32-bit words with v on the SMs.  Used instead of cudaMemsetAsync on
// the step path: a memset node can go through a copy engine, where it waits
// behind a concurrent bulk H2D copy (the training step's frames) and stalls
// the stream; a kernel also keeps the programmatic-launch chain unbroken.
namespace {
__global__ void __launch_bounds__(256) k_fill_u32(uint32_t* __restrict__ p, uint32_t v, size_t n) {
    rfs_pdl_wait();
    for (size_t i = (size_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256) p[i] = v;
}
}  // namespace
static inline cudaError_t rfs_fill_u32(void* p, uint32_t v, size_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const size_t blocks = (n + 255) / 256;
    return rfs_launch(k_fill_u32, dim3((unsigned)(blocks < 148 * 8 ? blocks : 148 * 8)), dim3(256), 0, st,
                      (uint32_t*)p, v, n);
}

// K6 ray patches: warp q (0..7) of a 16 x 16 tile owns a 4 (u) x 8 (v) patch.
// The patch cone (axis through the patch, half-angle covering its rays) as
// k_hits computes it; called by a full warp.  ca = (cx, cy, cz, th_p),
// cb = (cos_p, sin_p); a patch without rays gets a cone no candidate passes.
__device__ __forceinline__ void rfs_patch_cone(int tile, int q, int tiles_u, int n_az, int n_el,
                                               const double* __restrict__ dirs, float4& ca, float2& cb) {
    const int lane = threadIdx.x & 31, pu = q >> 1, pv = q & 1;
    const int u = (tile % tiles_u) * RFS_TILE + 4 * pu + (lane >> 3);
    const int v = (tile / tiles_u) * RFS_TILE + 8 * pv + (lane & 7);
    const bool valid = u < n_az && v < n_el;
    const int r = valid ? u * n_el + v : 0;
    const float fx = (float)dirs[3 * r], fy = (float)dirs[3 * r + 1], fz = (float)dirs[3 * r + 2];
    float cx = valid ? fx : 0.f, cy = valid ? fy : 0.f, cz = valid ? fz : 0.f;
    cx = warp_sum(cx);
    cy = warp_sum(cy);
    cz = warp_sum(cz);
    {
        const float inv = rsqrtf(fmaxf(cx * cx + cy * cy + cz * cz, 1e-30f));
        cx *= inv;
        cy *= inv;
        cz *= inv;
    }
    float cmin = valid ? cx * fx + cy * fy + cz * fz : 1.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cmin = fminf(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
    const float th_p = acosf(fminf(cmin, 1.f)) + 1e-4f;
    float sin_p, cos_p;
    sincosf(th_p, &sin_p, &cos_p);
    const bool any = __any_sync(0xffffffffu, valid);
    ca = any ? make_float4(cx, cy, cz, th_p) : make_float4(0.f, 0.f, 0.f, -1e30f);
    cb = any ? make_float2(cos_p, sin_p) : make_float2(1e30f, -1e30f);
}

// k_hits' cone test: may a candidate (bounding sphere sp = (mu - rx, .), cone
// record w3 = whit[4 g + 3] = (., th_g, cos th_g, sin th_g)) reach a ray of
// the patch cone (ca = (axis, th_p), cb = (cos th_p, sin th_p))?  cos(th_p +
// th_g) by angle addition, with a margin.
__device__ __forceinline__ bool rfs_cone_relevant(float4 ca, float2 cb, float4 sp, float4 w3) {
    if (ca.w + w3.y >= 3.1415f) return true;
    const float rs = rsqrtf(sp.x * sp.x + sp.y * sp.y + sp.z * sp.z);
    const float dotc = (ca.x * sp.x + ca.y * sp.y + ca.z * sp.z) * rs;
    return dotc >= cb.x * w3.z - cb.y * w3.w - 1e-5f;
}

// ---- Blackwell bulk-copy engine (cp.async.bulk, non-tensor) + mbarrier ----
// A thread copies `bytes` (multiple of 16, both addresses 16-byte aligned)
// global -> shared without staging registers; completion is counted in bytes
// on an mbarrier (complete_tx), which one thread arms with the expected total.
__device__ __forceinline__ unsigned rfs_smem_addr(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void rfs_mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(rfs_smem_addr(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void rfs_mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(rfs_smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void rfs_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            rfs_smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(rfs_smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void rfs_mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "RFS_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra RFS_WAIT_%=;\n"
        "}\n" ::"r"(rfs_smem_addr(bar)),
        "r"(phase)
        : "memory");
}
