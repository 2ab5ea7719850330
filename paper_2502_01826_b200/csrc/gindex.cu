// gindex.cu -- K8i by counting: the by-Gaussian hit index without a global radix sort.
//
// The backward sums every hit of a Gaussian in the reference's bincount slot
// order, (ray, k) ascending (grad.py:222-254).  The radix path sorts all H
// hit keys by Gaussian id (rfs_hit_keys + rfs_sort_pairs_u64 +
// rfs_gauss_offsets + rfs_gather_sorted).  Here:
//   k_gi_count     hits per Gaussian (thread per ray, atomics aggregated over
//                  the warp's rays hitting the same Gaussian);
//   (scan)         g_off = exclusive scan, g_off[n] = H;
//   k_gi_scatter   each hit's slab slot to g_off[g] + an atomic cursor: a
//                  Gaussian's hits land in its segment in arbitrary order;
//   k_gi_segsort   warp per Gaussian of <= 256 hits: slots sorted in registers
//                  (bitonic; unique, so the order is the stable sort's), then
//                  per hit its Gaussian id, ray, w and w T gathered from the
//                  slab;
//   k_gi_bitmap    a block per longer segment (listed by k_gi_segsort): a
//                  Gaussian hits a ray at most once, so a hit's sorted
//                  position is the count of the Gaussian's rays before its
//                  ray -- a bitmap over the rays plus per-word prefix counts.
// Same outputs, bitwise, as the radix path.
#include "rfs_common.cuh"

extern "C" int rfs_exclusive_scan_u32(const uint32_t* in, int n, uint32_t* out, uint32_t* total, uint32_t* temp,
                                      void* stream);

namespace {



// Thread per ray, a warp = 32 consecutive rays stepping through their k-th
// hits together: neighbouring rays hit largely the same Gaussians, so the
// counter atomics are aggregated over match_any groups (hot Gaussians have
// thousands of hits).
__global__ void __launch_bounds__(256) k_gi_count(const RfsHit* __restrict__ slab, const int* __restrict__ counts,
                                                  int hcap, int R, uint32_t* __restrict__ gcnt) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int cnt = r < R ? min(counts[r], hcap) : 0;
    const int kmax = __reduce_max_sync(0xffffffffu, (unsigned)cnt);
    unsigned lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    for (int k = 0; k < kmax; ++k) {
        const bool ok = k < cnt;
        const uint32_t g = ok ? slab[(size_t)r * hcap + k].g : 0xffffffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, g);
        if (ok && (peers & lt) == 0) atomicAdd(&gcnt[g], (uint32_t)__popc(peers));
    }
}

__global__ void __launch_bounds__(256) k_gi_scatter(const RfsHit* __restrict__ slab, const int* __restrict__ counts,
                                                    int hcap, int R, const uint32_t* __restrict__ g_off,
                                                    uint32_t* __restrict__ cur, uint32_t cap,
                                                    uint32_t* __restrict__ tmp) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int cnt = r < R ? min(counts[r], hcap) : 0;
    const int kmax = __reduce_max_sync(0xffffffffu, (unsigned)cnt);
    unsigned lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    for (int k = 0; k < kmax; ++k) {
        const bool ok = k < cnt;
        const uint32_t slot = (uint32_t)((size_t)r * hcap + k);
        const uint32_t g = ok ? slab[slot].g : 0xffffffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, g);
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (ok && (peers & lt) == 0) base = g_off[g] + atomicAdd(&cur[g], (uint32_t)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        const uint32_t pos = base + __popc(peers & lt);
        if (ok && pos < cap) tmp[pos] = slot;
    }
}

__device__ __forceinline__ void emit_sorted(uint32_t p, uint32_t g, uint32_t slot, int hcap,
                                            const RfsHit* __restrict__ slab, uint64_t* __restrict__ sorted_g,
                                            uint32_t* __restrict__ s_slot, uint32_t* __restrict__ s_ray,
                                            float* __restrict__ s_w, float2* __restrict__ s_wt) {
    const RfsHit hk = slab[slot];
    sorted_g[p] = g;
    s_slot[p] = slot;
    s_ray[p] = slot / (uint32_t)hcap;
    s_w[p] = hk.w;
    s_wt[p] = make_float2(hk.w * hk.t_re, hk.w * hk.t_im);
}

// Warp bitonic sort of a segment of L <= 32 * E unique slots, E per lane
// (element i = lane * E + e; padding 0xffffffff sorts last), then emitted.
template <int E>
__device__ __forceinline__ void warp_sort_emit(uint32_t p0, int L, uint32_t g, int hcap, const uint32_t* __restrict__ tmp,
                                               const RfsHit* __restrict__ slab, uint64_t* __restrict__ sorted_g,
                                               uint32_t* __restrict__ s_slot, uint32_t* __restrict__ s_ray,
                                               float* __restrict__ s_w, float2* __restrict__ s_wt) {
    constexpr int P = 32 * E;
    const int lane = threadIdx.x & 31;
    uint32_t a[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane * E + e;
        a[e] = i < L ? tmp[p0 + i] : 0xffffffffu;
    }
#pragma unroll
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= E) {  // partner in lane ^ (j / E), same register
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int i = lane * E + e;
                    const uint32_t y = __shfl_xor_sync(0xffffffffu, a[e], j / E);
                    const bool up = (i & k) == 0, lower = (i & j) == 0;
                    a[e] = (lower == up) ? min(a[e], y) : max(a[e], y);
                }
            } else {  // partner in this lane's registers
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    if (e & j) continue;
                    const int i = lane * E + e;
                    const bool up = (i & k) == 0;
                    const uint32_t x = a[e], y = a[e | j];
                    if ((x > y) == up) {
                        a[e] = y;
                        a[e | j] = x;
                    }
                }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane * E + e;
        if (i < L) emit_sorted(p0 + i, g, a[e], hcap, slab, sorted_g, s_slot, s_ray, s_w, s_wt);
    }
}

// warp per Gaussian: segments of up to 256 hits sorted in registers, longer
// ones listed for k_gi_bitmap
__global__ void __launch_bounds__(256) k_gi_segsort(int n, const uint32_t* __restrict__ g_off, uint32_t cap, int hcap,
                                                    const uint32_t* __restrict__ tmp, const RfsHit* __restrict__ slab,
                                                    uint64_t* __restrict__ sorted_g, uint32_t* __restrict__ s_slot,
                                                    uint32_t* __restrict__ s_ray, float* __restrict__ s_w,
                                                    float2* __restrict__ s_wt, uint32_t* __restrict__ long_list,
                                                    int* __restrict__ n_long) {
    const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (g >= n) return;
    const uint32_t p0 = min(g_off[g], cap), p1 = min(g_off[g + 1], cap);
    const int L = (int)(p1 - p0);
    if (L == 0) return;
    const uint32_t gg = (uint32_t)g;
    if (L <= 32)
        warp_sort_emit<1>(p0, L, gg, hcap, tmp, slab, sorted_g, s_slot, s_ray, s_w, s_wt);
    else if (L <= 64)
        warp_sort_emit<2>(p0, L, gg, hcap, tmp, slab, sorted_g, s_slot, s_ray, s_w, s_wt);
    else if (L <= 128)
        warp_sort_emit<4>(p0, L, gg, hcap, tmp, slab, sorted_g, s_slot, s_ray, s_w, s_wt);
    else if (L <= 256)
        warp_sort_emit<8>(p0, L, gg, hcap, tmp, slab, sorted_g, s_slot, s_ray, s_w, s_wt);
    else if ((threadIdx.x & 31) == 0)
        long_list[atomicAdd(n_long, 1)] = gg;
}

// Segments of more than 256 hits, a block each (grid-stride over the list): a
// Gaussian hits a ray at most once, so the slot order is the ray order, and
// a hit's sorted position is the number of the Gaussian's rays before its
// ray -- a bitmap over the rays it spans plus a prefix count per word.
constexpr int GI_BM_NT = 256;
constexpr int GI_BM_WORDS = 2048;  // >= 360 * 180 / 32
__global__ void __launch_bounds__(GI_BM_NT) k_gi_bitmap(const uint32_t* __restrict__ long_list,
                                                        const int* __restrict__ n_long,
                                                        const uint32_t* __restrict__ g_off, uint32_t cap, int hcap,
                                                        const uint32_t* __restrict__ tmp,
                                                        const RfsHit* __restrict__ slab,
                                                        uint64_t* __restrict__ sorted_g, uint32_t* __restrict__ s_slot,
                                                        uint32_t* __restrict__ s_ray, float* __restrict__ s_w,
                                                        float2* __restrict__ s_wt) {
    __shared__ uint32_t bits[GI_BM_WORDS], wpre[GI_BM_WORDS];
    __shared__ uint32_t wsum[GI_BM_NT / 32];
    __shared__ int w_lo, w_hi;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nl = *n_long;
    for (int e = blockIdx.x; e < nl; e += gridDim.x) {
        const uint32_t g = long_list[e];
        const uint32_t p0 = min(g_off[g], cap), p1 = min(g_off[g + 1], cap);
        if (tid == 0) {
            w_lo = GI_BM_WORDS;
            w_hi = -1;
        }
        __syncthreads();
        int lo = GI_BM_WORDS, hi = -1;
        for (uint32_t p = p0 + tid; p < p1; p += GI_BM_NT) {
            const int w = (int)((tmp[p] / (uint32_t)hcap) >> 5);
            lo = min(lo, w);
            hi = max(hi, w);
        }
        atomicMin(&w_lo, lo);
        atomicMax(&w_hi, hi);
        __syncthreads();
        const int W0 = w_lo, NWd = w_hi - w_lo + 1;
        for (int w = tid; w < NWd; w += GI_BM_NT) bits[w] = 0u;
        __syncthreads();
        for (uint32_t p = p0 + tid; p < p1; p += GI_BM_NT) {
            const uint32_t r = tmp[p] / (uint32_t)hcap;
            atomicOr(&bits[(int)(r >> 5) - W0], 1u << (r & 31));
        }
        __syncthreads();
        // exclusive prefix of the set bits per word: thread-contiguous runs
        const int per = (NWd + GI_BM_NT - 1) / GI_BM_NT;
        const int a0 = min(tid * per, NWd), a1 = min(a0 + per, NWd);
        uint32_t c = 0;
        for (int w = a0; w < a1; ++w) c += __popc(bits[w]);
        uint32_t x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[wid] = x;
        __syncthreads();
        uint32_t run = x - c;
        for (int w = 0; w < wid; ++w) run += wsum[w];
        for (int w = a0; w < a1; ++w) {
            wpre[w] = run;
            run += __popc(bits[w]);
        }
        __syncthreads();
        for (uint32_t p = p0 + tid; p < p1; p += GI_BM_NT) {
            const uint32_t slot = tmp[p], r = slot / (uint32_t)hcap;
            const int w = (int)(r >> 5) - W0;
            const uint32_t pos = wpre[w] + __popc(bits[w] & ((1u << (r & 31)) - 1u));
            emit_sorted(p0 + pos, g, slot, hcap, slab, sorted_g, s_slot, s_ray, s_w, s_wt);
        }
        __syncthreads();
    }
}

}  // namespace

extern "C" {

int rfs_gauss_index(const void* slab, const int* counts, int hcap, int n_rays, int n, int cap, uint32_t* scratch,
                    uint32_t* scan_temp, int* g_off, uint64_t* sorted_g, uint32_t* s_slot, uint32_t* s_ray, float* s_w,
                    void* s_wt, void* stream) {
    if (n <= 0 || n_rays <= 0 || hcap <= 0 || cap < 0) return RFS_ERR_SHAPE;
    if ((n_rays + 31) / 32 > GI_BM_WORDS) return RFS_ERR_SHAPE;
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t* gcnt = scratch;          // n
    uint32_t* cur = scratch + n;       // n
    uint32_t* long_list = cur + n;     // n
    int* n_long = (int*)(long_list + n);
    uint32_t* tmp = (uint32_t*)(n_long + 2);  // cap: the unsorted segments
    RFS_CUDA_TRY(cudaMemsetAsync(scratch, 0, sizeof(uint32_t) * (2 * (size_t)n), st));
    RFS_CUDA_TRY(cudaMemsetAsync(n_long, 0, 2 * sizeof(int), st));
    const int grid_r = rfs_ceil_div(n_rays, 256);
    k_gi_count<<<grid_r, 256, 0, st>>>((const RfsHit*)slab, counts, hcap, n_rays, gcnt);
    RFS_LAUNCH_CHECK();
    int rc = rfs_exclusive_scan_u32(gcnt, n, (uint32_t*)g_off, (uint32_t*)g_off + n, scan_temp, stream);
    if (rc != RFS_OK) return rc;
    if (cap == 0) return RFS_OK;
    k_gi_scatter<<<grid_r, 256, 0, st>>>((const RfsHit*)slab, counts, hcap, n_rays, (const uint32_t*)g_off, cur,
                                         (uint32_t)cap, tmp);
    RFS_LAUNCH_CHECK();
    k_gi_segsort<<<rfs_ceil_div(n * 32, 256), 256, 0, st>>>(n, (const uint32_t*)g_off, (uint32_t)cap, hcap, tmp,
                                                            (const RfsHit*)slab, sorted_g, s_slot, s_ray, s_w,
                                                            (float2*)s_wt, long_list, n_long);
    RFS_LAUNCH_CHECK();
    k_gi_bitmap<<<4 * 148, GI_BM_NT, 0, st>>>(long_list, n_long, (const uint32_t*)g_off, (uint32_t)cap, hcap, tmp,
                                              (const RfsHit*)slab, sorted_g, s_slot, s_ray, s_w, (float2*)s_wt);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

// u32 elements: 3 n (counts, cursors, long list) + 2 counters + cap (unsorted segments)
size_t rfs_gauss_index_scratch_elems(int n, int cap) {
    return 3 * (size_t)(n > 0 ? n : 0) + 2 + (size_t)(cap > 0 ? cap : 0);
}

}  // extern "C"
