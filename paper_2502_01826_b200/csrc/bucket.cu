// bucket.cu -- K2b-K4b by tile buckets: the tile-key sort without a global radix sort.
//
// The reference orders every (tile, Gaussian) incidence with a stable argsort
// of tile << 32 | depth bits (splat.py:337), i.e. by (tile, depth, expansion
// position), then takes each tile's range (splat.py:340-343).  A 360 x 180
// grid has at most 23 x 12 = 276 tiles, so the tile part is a stable counting
// sort and only the depth part needs sorting, tile by tile:
//   k_tile_count   incidences per (256-Gaussian block, tile);
//   k_tile_blockscan / k_tile_offsets
//                  each block's base inside a tile's bucket (blocks in
//                  order), the tile totals and offsets (= the ranges);
//   k_fill_stable  each incidence to its tile's bucket at base + its rank
//                  among the block's Gaussians hitting that tile (one warp
//                  ballot per tile; a Gaussian hits a tile at most once):
//                  buckets hold their incidences in expansion order;
//   k_seg_sort     one block per tile: stable LSD radix sort of the 31-bit
//                  depth codes in shared memory (4 digit passes), then the
//                  sorted compact keys, Gaussian ids and the emission bounds
//                  lb[i] = min_{j >= i} lbv[g_j] of K4b.
// Same outputs, bitwise, as K2b + K3 + K4 + K4b (rfs_bin_fill, the radix
// sort, rfs_tile_ranges, rfs_lower_bounds).  Three k_seg_sort classes: lists
// up to 4096 (512 threads) and 12288 (1024 threads) in shared memory, longer
// ones with the same passes over global (L2-resident) ping-pong buffers.
#include <cooperative_groups.h>

#include "rfs_common.cuh"

namespace {

constexpr int BK_MAX_TILES = 512;   // >= 23 x 12 (rfs_project caps the grid at 360 x 180)
constexpr int BK_BLK = 256;         // Gaussians per fill block
constexpr int BK_SEG_SMALL = 4096;  // tile lists sorted by 512-thread blocks
constexpr int BK_SEG_MAX = 12288;   // longest tile list sorted in one block's shared memory (1024 threads)
constexpr int BK_CL = 4;            // cluster of CTAs sorting one longer list in distributed shared memory
constexpr int BK_SEG_CLUSTER = BK_CL * BK_SEG_MAX;  // longest tile list sorted by a cluster

struct __align__(16) Rect {  // project.cu's splat rectangle
    short s1_lo, s1_hi, s2_hi, tv_lo, tv_hi, pad0, pad1, pad2;
};

// incidences of Gaussian g in expand_tile_rects order (_kernels.py:545-558):
// rows tv ascending, then the s1 run, then the wrapped s2 run
template <typename F>
__device__ __forceinline__ void for_each_tile(const Rect& r, int tiles_u, F&& f) {
    if (r.tv_hi < r.tv_lo) return;
    int k = 0;
    for (int tv = r.tv_lo; tv <= r.tv_hi; ++tv) {
        const int row = tv * tiles_u;
        for (int tu = r.s1_lo; tu <= r.s1_hi; ++tu) f(row + tu, k++);
        for (int tu = 0; tu <= r.s2_hi; ++tu) f(row + tu, k++);
    }
}

// bits lo..hi (inclusive) of a word; empty if hi < lo (tiles_u <= 23 < 32)
__device__ __forceinline__ uint32_t bit_range(int lo, int hi) {
    return hi < lo ? 0u : ((2u << hi) - 1u) & ~((1u << lo) - 1u);
}

// hit[t][w] = mask of warp w's lanes whose Gaussian's rectangle contains tile
// t: per tile row, each lane's row of column bits, transposed across the warp
// (32 x 32 bit transpose by shuffles), lane tu then holds column tu's mask
__device__ __forceinline__ void block_hit_masks(const Rect& r, int tiles_u, int n_tiles,
                                                uint32_t (*hit)[BK_BLK / 32]) {
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t cols = bit_range(r.s1_lo, r.s1_hi) | bit_range(0, r.s2_hi);
    const int tiles_v = n_tiles / tiles_u;
    for (int tv = 0; tv < tiles_v; ++tv) {
        uint32_t x = (tv >= r.tv_lo && tv <= r.tv_hi) ? cols : 0u;
#pragma unroll
        for (int j = 16; j > 0; j >>= 1) {
            const uint32_t m = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu
                             : j == 2 ? 0x33333333u : 0x55555555u;
            const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
            x = (lane & j) == 0 ? (x & m) | ((y & m) << j) : (x & ~m) | ((y & ~m) >> j);
        }
        if (lane < tiles_u) hit[tv * tiles_u + lane][wid] = x;
    }
}

// per (tile, block) incidence counts, tile-major: tab[t * nb + b]
// (shared-memory atomics: a count does not depend on the order)
__global__ void __launch_bounds__(BK_BLK) k_tile_count(int n, const Rect* __restrict__ rects, int tiles_u,
                                                       int n_tiles, int nb, uint32_t* __restrict__ tab) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    __shared__ uint32_t h[BK_MAX_TILES];
    for (int t = threadIdx.x; t < n_tiles; t += BK_BLK) h[t] = 0;
    __syncthreads();
    const int g = blockIdx.x * BK_BLK + threadIdx.x;
    if (g < n) {
        const Rect r = rects[g];
        for_each_tile(r, tiles_u, [&](int t, int) { atomicAdd(&h[t], 1u); });
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n_tiles; t += BK_BLK) tab[(size_t)t * nb + blockIdx.x] = h[t];
}

// warp per tile: exclusive scan of its blocks' counts in place, total -> tot[t]
__global__ void __launch_bounds__(128) k_tile_blockscan(int nb, int n_tiles, uint32_t* __restrict__ tab,
                                                        uint32_t* __restrict__ tot) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int t = (blockIdx.x * 128 + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (t >= n_tiles) return;
    uint32_t* row = tab + (size_t)t * nb;
    uint32_t carry = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
        const int b = b0 + lane;
        const uint32_t c = b < nb ? row[b] : 0u;
        uint32_t x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (b < nb) row[b] = carry + x - c;
        carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) tot[t] = carry;
}

// single block: tile offsets = the ranges (clamped to the capacity)
__global__ void __launch_bounds__(BK_MAX_TILES) k_tile_offsets(int n_tiles, const uint32_t* __restrict__ tot,
                                                               uint32_t cap, int2* __restrict__ ranges,
                                                               uint32_t* __restrict__ off_out,
                                                               int* __restrict__ status) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    __shared__ uint32_t wsum[BK_MAX_TILES / 32];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const uint32_t c = t < n_tiles ? tot[t] : 0u;
    uint32_t v = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) wsum[wid] = v;
    __syncthreads();
    uint32_t off = v - c;
    for (int w = 0; w < wid; ++w) off += wsum[w];
    if (t >= n_tiles) return;
    ranges[t] = make_int2((int)min(off, cap), (int)min(off + c, cap));
    off_out[t] = off;
}

__global__ void __launch_bounds__(BK_BLK) k_fill_stable(int n, const Rect* __restrict__ rects,
                                                        const uint32_t* __restrict__ code, int tiles_u, int n_tiles,
                                                        int nb, uint32_t cap, const uint32_t* __restrict__ tab,
                                                        const uint32_t* __restrict__ toff,
                                                        uint32_t* __restrict__ bcodes, uint32_t* __restrict__ bvals) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    constexpr int NW = BK_BLK / 32;
    __shared__ uint32_t hit[BK_MAX_TILES][NW];
    __shared__ uint32_t base[BK_MAX_TILES][NW];  // slot of warp w's first incidence in tile t
    const int g = blockIdx.x * BK_BLK + threadIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    Rect r;
    r.s1_lo = 0;
    r.s1_hi = r.s2_hi = -1;
    r.tv_lo = 1;
    r.tv_hi = 0;
    if (g < n) r = rects[g];
    block_hit_masks(r, tiles_u, n_tiles, hit);
    __syncthreads();
    for (int t = threadIdx.x; t < n_tiles; t += BK_BLK) {
        uint32_t b = toff[t] + tab[(size_t)t * nb + blockIdx.x];
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            base[t][w] = b;
            b += __popc(hit[t][w]);
        }
    }
    __syncthreads();
    if (g >= n) return;
    const uint32_t c = code[g];
    const unsigned below = (1u << lane) - 1u;
    for_each_tile(r, tiles_u, [&](int t, int) {
        const uint32_t slot = base[t][wid] + __popc(hit[t][wid] & below);
        if (slot < cap) {
            bcodes[slot] = c;
            bvals[slot] = (uint32_t)g;
        }
    });
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// exclusive scan of a 256-entry digit table by the first 8 warps (named barrier 1)
__device__ __forceinline__ uint32_t scan256_excl(uint32_t c, uint32_t* wsc) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsc[wid] = x;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    x -= c;
    for (int w = 0; w < wid; ++w) x += wsc[w];
    asm volatile("bar.sync 1, 256;" ::: "memory");  // wsc reusable
    return x;
}

// One block per tile with a list of (lo, CAP] entries: stable LSD radix sort
// of the bucket's depth codes in shared memory (bits 0-7, 8-15, 16-23,
// 24-30).  A round covers NT * ITEMS items, warp w a contiguous run of
// 32 * ITEMS of them taken 32 at a time, so a warp's digit ranks come from
// match_any plus its running per-digit counts, and the round's per-digit
// offsets from a scan over the warps -- order within a digit is kept.
// CAP == 0: lists longer than every shared-memory class -- the same passes
// with the ping-pong buffers in global memory (the bucket itself and an
// alternate pair), L2-resident.
template <int CAP, int NT>
__global__ void __launch_bounds__(NT) k_seg_sort(const int2* __restrict__ ranges, int lo, uint32_t* __restrict__ bcodes,
                                                 uint32_t* __restrict__ bvals, uint32_t* __restrict__ altc,
                                                 uint32_t* __restrict__ altv, const RfsGeom* __restrict__ geom,
                                                 uint64_t* __restrict__ ckeys, uint32_t* __restrict__ vals,
                                                 double* __restrict__ lb) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    constexpr int NW = NT / 32, ITEMS = 8, ROUND = NT * ITEMS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tile = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int2 rg = ranges[tile];
    const int L = rg.y - rg.x;
    if (L <= lo || (CAP > 0 && L > CAP)) return;  // another launch's class (block-uniform)
    uint32_t *k0, *v0, *k1, *v1;
    if (CAP > 0) {  // ping-pong codes / ids in shared memory, 4 x CAP
        k0 = reinterpret_cast<uint32_t*>(smem_raw);
        v0 = k0 + CAP;
        k1 = v0 + CAP;
        v1 = k1 + CAP;
    } else {
        k0 = bcodes + rg.x;
        v0 = bvals + rg.x;
        k1 = altc + rg.x;
        v1 = altv + rg.x;
    }
    __shared__ uint32_t dbase[256], rtot[256], wsc[8];
    __shared__ uint16_t wcnt[NW][256];
    __shared__ double wmin[NW];
    if (CAP > 0) {
        for (int i = tid; i < L; i += NT) {
            k0[i] = bcodes[rg.x + i];
            v0[i] = bvals[rg.x + i];
        }
    }
    const unsigned lt = lanemask_lt();
    const bool multi = L > ROUND;
    uint32_t *sk = k0, *sv = v0, *dk = k1, *dv = v1;
    __syncthreads();
    for (int sh = 0; sh < 31; sh += 8) {
        if (multi) {  // digit totals up front when the list takes several rounds
            for (int d = tid; d < 256; d += NT) rtot[d] = 0;
            __syncthreads();
            for (int i = tid; i < L; i += NT) {
                const uint32_t d = (sk[i] >> sh) & 255u;
                const unsigned peers = __match_any_sync(__activemask(), d);
                if ((peers & lt) == 0) atomicAdd(&rtot[d], (uint32_t)__popc(peers));
            }
            __syncthreads();
            if (tid < 256) dbase[tid] = scan256_excl(rtot[tid], wsc);
            __syncthreads();
        }
        for (int r0 = 0; r0 < L; r0 += ROUND) {
            for (int e = tid; e < NW * 256; e += NT) (&wcnt[0][0])[e] = 0;
            __syncthreads();
            uint32_t key[ITEMS], val[ITEMS], dig[ITEMS], rk[ITEMS];
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) {
                const int i = r0 + wid * 32 * ITEMS + j * 32 + lane;
                const bool ok = i < L;
                key[j] = ok ? sk[i] : 0u;
                val[j] = ok ? sv[i] : 0u;
                dig[j] = ok ? (key[j] >> sh) & 255u : 256u;
                const unsigned peers = __match_any_sync(0xffffffffu, dig[j]);
                const uint32_t cur = ok ? wcnt[wid][dig[j]] : 0u;
                rk[j] = cur + __popc(peers & lt);
                __syncwarp();
                if (ok && (peers & lt) == 0) wcnt[wid][dig[j]] = (uint16_t)(cur + __popc(peers));
                __syncwarp();
            }
            __syncthreads();
            if (tid < 256) {  // per digit: exclusive scan over the warps of this round
                uint32_t run = 0;
#pragma unroll 4
                for (int w = 0; w < NW; ++w) {
                    const uint32_t x = wcnt[w][tid];
                    wcnt[w][tid] = (uint16_t)run;
                    run += x;
                }
                if (!multi) dbase[tid] = scan256_excl(run, wsc);
                rtot[tid] = run;
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) {
                if (dig[j] < 256u) {
                    const uint32_t dst = dbase[dig[j]] + wcnt[wid][dig[j]] + rk[j];
                    dk[dst] = key[j];
                    dv[dst] = val[j];
                }
            }
            __syncthreads();
            if (multi && tid < 256) dbase[tid] += rtot[tid];
        }
        uint32_t* t = sk;
        sk = dk;
        dk = t;
        t = sv;
        sv = dv;
        dv = t;
        __syncthreads();
    }
    // sorted compact keys (tile << 31 | depth code), Gaussian ids, lbv -> the
    // now free ping-pong buffer (as doubles; in global mode lb itself)
    const uint64_t th = (uint64_t)tile << 31;
    double* sl = CAP > 0 ? reinterpret_cast<double*>(dk) : lb + rg.x;  // dk + dv: 8 B x CAP
    for (int i = tid; i < L; i += NT) {
        const uint32_t g = sv[i];
        ckeys[rg.x + i] = th | sk[i];
        vals[rg.x + i] = g;
        sl[i] = geom[g].lbv;
    }
    __syncthreads();
    // lb[i] = min_{j >= i} lbv_j: each thread a contiguous run, runs combined
    // right to left across the block
    const int E = (L + NT - 1) / NT;
    const int i0 = tid * E, i1 = min(i0 + E, L);
    double run = INFINITY;
    for (int i = i1 - 1; i >= i0; --i) run = fmin(run, sl[i]);
    double v = run;  // inclusive suffix min within the warp (towards higher lanes)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_down_sync(0xffffffffu, v, o);
        if (lane + o < 32) v = fmin(v, y);
    }
    if (lane == 0) wmin[wid] = v;
    __syncthreads();
    double carry = __shfl_down_sync(0xffffffffu, v, 1);
    if (lane == 31) carry = INFINITY;
    for (int w = wid + 1; w < NW; ++w) carry = fmin(carry, wmin[w]);
    for (int i = i1 - 1; i >= i0; --i) {  // (global mode: each thread rewrites its own run)
        carry = fmin(carry, sl[i]);
        lb[rg.x + i] = carry;
    }
}

// Tile lists of (BK_SEG_MAX, BK_CL * BK_SEG_MAX] entries (0.5M-1M-Gaussian
// scenes): a thread-block cluster of BK_CL CTAs sorts one list in distributed
// shared memory.  CTA c owns the contiguous slice [c S, (c + 1) S) of the
// list (S = ceil(L / BK_CL) <= 12288, one round of 1024 x 12 items).  Per
// 8-bit pass each CTA ranks its slice stably in registers (match_any +
// per-warp counts, as k_seg_sort), scatters it locally into digit order, reads
// the other CTAs' digit counts over DSMEM to find where digit d of its slice
// starts in the whole list ((all digits < d) + (digit d of slices < c)), and
// copies each digit run to the CTA(s) owning that range -- contiguous runs,
// so the DSMEM stores coalesce; cluster barriers separate the passes.  The
// emission bounds' suffix minimum crosses slices the same way.  Bitwise the
// outputs of the single-block classes and of the radix path.
__global__ void __launch_bounds__(1024) k_seg_sort_cluster(const int2* __restrict__ ranges, int lo,
                                                           const uint32_t* __restrict__ bcodes,
                                                           const uint32_t* __restrict__ bvals,
                                                           const RfsGeom* __restrict__ geom,
                                                           uint64_t* __restrict__ ckeys, uint32_t* __restrict__ vals,
                                                           double* __restrict__ lb) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    namespace cg = cooperative_groups;
    constexpr int NT = 1024, NW = NT / 32, ITEMS = 12, CAPL = BK_SEG_MAX;
    static_assert(NT * ITEMS >= CAPL, "a slice is one round");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int tile = blockIdx.x / BK_CL, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int2 rg = ranges[tile];
    const int L = rg.y - rg.x;
    if (L <= lo || L > BK_CL * CAPL) return;  // another launch's class (uniform over the cluster)
    const int S = (L + BK_CL - 1) / BK_CL;
    const int s0 = rank * S, Ls = max(0, min(L, s0 + S) - s0);
    uint32_t* k0 = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* v0 = k0 + CAPL;
    uint32_t* k1 = v0 + CAPL;
    uint32_t* v1 = k1 + CAPL;
    __shared__ uint32_t cnt[256], loff[256], gbase[256], wsc[8];
    __shared__ uint16_t wcnt[NW][256];
    __shared__ double wmin[NW];
    __shared__ double smin;
    for (int i = tid; i < Ls; i += NT) {
        k0[i] = bcodes[rg.x + s0 + i];
        v0[i] = bvals[rg.x + s0 + i];
    }
    const unsigned lt = lanemask_lt();
    uint32_t *sk = k0, *sv = v0, *dk = k1, *dv = v1;
    __syncthreads();
    for (int sh = 0; sh < 31; sh += 8) {
        // 1. stable ranks of the slice in registers
        for (int e = tid; e < NW * 256; e += NT) (&wcnt[0][0])[e] = 0;
        __syncthreads();
        uint32_t key[ITEMS], val[ITEMS], dig[ITEMS], rk[ITEMS];
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const int i = wid * 32 * ITEMS + j * 32 + lane;
            const bool ok = i < Ls;
            key[j] = ok ? sk[i] : 0u;
            val[j] = ok ? sv[i] : 0u;
            dig[j] = ok ? (key[j] >> sh) & 255u : 256u;
            const unsigned peers = __match_any_sync(0xffffffffu, dig[j]);
            const uint32_t cur = ok ? wcnt[wid][dig[j]] : 0u;
            rk[j] = cur + __popc(peers & lt);
            __syncwarp();
            if (ok && (peers & lt) == 0) wcnt[wid][dig[j]] = (uint16_t)(cur + __popc(peers));
            __syncwarp();
        }
        __syncthreads();
        if (tid < 256) {  // per digit: exclusive scan over the warps, the slice count, its local start
            uint32_t run = 0;
#pragma unroll 4
            for (int w = 0; w < NW; ++w) {
                const uint32_t x = wcnt[w][tid];
                wcnt[w][tid] = (uint16_t)run;
                run += x;
            }
            cnt[tid] = run;
            loff[tid] = scan256_excl(run, wsc);
        }
        __syncthreads();
        // 2. the slice in digit order, in place (every element is in registers)
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            if (dig[j] < 256u) {
                const uint32_t dst = loff[dig[j]] + wcnt[wid][dig[j]] + rk[j];
                sk[dst] = key[j];
                sv[dst] = val[j];
            }
        }
        cluster.sync();  // every slice's digit counts are final (and its digit-ordered copy)
        // 3. where digit d of this slice starts in the whole list
        if (tid < 256) {
            uint32_t all = 0, before = 0;
#pragma unroll
            for (int c = 0; c < BK_CL; ++c) {
                const uint32_t x = cluster.map_shared_rank(cnt, c)[tid];
                all += x;
                if (c < rank) before += x;
            }
            gbase[tid] = scan256_excl(all, wsc) + before;
        }
        __syncthreads();
        // 4. digit runs to their owners: consecutive elements -> consecutive destinations
        for (int i = tid; i < Ls; i += NT) {
            const uint32_t k = sk[i], d = (k >> sh) & 255u;
            const uint32_t dst = gbase[d] + ((uint32_t)i - loff[d]);
            const int owner = (int)(dst / (uint32_t)S);
            const uint32_t off = dst - (uint32_t)owner * (uint32_t)S;
            cluster.map_shared_rank(dk, owner)[off] = k;
            cluster.map_shared_rank(dv, owner)[off] = sv[i];
        }
        cluster.sync();  // every element of the pass has landed; counts read
        uint32_t* t = sk;
        sk = dk;
        dk = t;
        t = sv;
        sv = dv;
        dv = t;
    }
    // sorted compact keys (tile << 31 | depth code), Gaussian ids, lbv of this slice
    const uint64_t th = (uint64_t)tile << 31;
    double* sl = reinterpret_cast<double*>(dk);  // dk + dv: 8 B x CAPL
    for (int i = tid; i < Ls; i += NT) {
        const uint32_t g = sv[i];
        ckeys[rg.x + s0 + i] = th | sk[i];
        vals[rg.x + s0 + i] = g;
        sl[i] = geom[g].lbv;
    }
    __syncthreads();
    // lb[i] = min_{j >= i} lbv_j: runs within the slice as k_seg_sort, then
    // the minimum of the later slices (DSMEM) folded in
    const int E = (Ls + NT - 1) / NT;
    const int i0 = tid * E, i1 = min(i0 + E, Ls);
    double run = INFINITY;
    for (int i = i1 - 1; i >= i0; --i) run = fmin(run, sl[i]);
    double v = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_down_sync(0xffffffffu, v, o);
        if (lane + o < 32) v = fmin(v, y);
    }
    if (lane == 0) wmin[wid] = v;
    __syncthreads();
    if (tid == 0) {
        double m = INFINITY;
        for (int w = 0; w < NW; ++w) m = fmin(m, wmin[w]);
        smin = m;
    }
    cluster.sync();  // every slice's minimum is published
    double later = INFINITY;
    for (int c = rank + 1; c < BK_CL; ++c) later = fmin(later, *cluster.map_shared_rank(&smin, c));
    double carry = __shfl_down_sync(0xffffffffu, v, 1);
    if (lane == 31) carry = INFINITY;
    for (int w = wid + 1; w < NW; ++w) carry = fmin(carry, wmin[w]);
    carry = fmin(carry, later);
    for (int i = i1 - 1; i >= i0; --i) {
        carry = fmin(carry, sl[i]);
        lb[rg.x + s0 + i] = carry;
    }
    cluster.sync();  // no CTA leaves while another may still read its shared memory
}

int launch_seg_sort_cluster(int n_tiles, const int* ranges, int lo, const uint32_t* bcodes, const uint32_t* bvals,
                            const void* geom, uint64_t* ckeys, uint32_t* vals, double* lb, cudaStream_t st) {
    static bool attr = false;
    const size_t smem = (size_t)BK_SEG_MAX * 16;
    if (!attr) {
        RFS_CUDA_TRY(cudaFuncSetAttribute(k_seg_sort_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(n_tiles * BK_CL));
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = BK_CL;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 2;
    RFS_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_seg_sort_cluster, (const int2*)ranges, lo, bcodes, bvals,
                                    (const RfsGeom*)geom, ckeys, vals, lb));
    return RFS_OK;
}

template <int CAP, int NT>
int launch_seg_sort(int n_tiles, const int* ranges, int lo, uint32_t* bcodes, uint32_t* bvals, uint32_t* altc,
                    uint32_t* altv, const void* geom, uint64_t* ckeys, uint32_t* vals, double* lb, cudaStream_t st) {
    static bool attr = false;
    const size_t smem = (size_t)CAP * 16;
    if (!attr && smem > 0) {
        RFS_CUDA_TRY(cudaFuncSetAttribute(k_seg_sort<CAP, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    rfs_launch(k_seg_sort<CAP, NT>, n_tiles, NT, smem, st, (const int2*)ranges, lo, bcodes, bvals, altc, altv,
                                                   (const RfsGeom*)geom, ckeys, vals, lb);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // namespace

extern "C" {

size_t rfs_bin_bucket_temp_bytes(int n, int n_az, int n_el, int cap) {
    const int n_tiles = ((n_az + RFS_TILE - 1) / RFS_TILE) * ((n_el + RFS_TILE - 1) / RFS_TILE);
    const size_t nb = (size_t)rfs_ceil_div(n > 0 ? n : 1, BK_BLK);
    // block table, tile totals, tile offsets, alternate codes / ids for long lists
    return sizeof(uint32_t) * (nb * (size_t)n_tiles + 2 * (size_t)n_tiles + 2 * (size_t)(cap > 0 ? cap : 0));
}

int rfs_bin_bucket(int n, const void* rects, const uint32_t* depth_code, int n_az, int n_el, int cap, const void* geom,
                   uint32_t* bcodes, uint32_t* bvals, void* temp, uint64_t* ckeys, uint32_t* vals, int* ranges,
                   double* lb, int* status, void* stream) {
    const int tiles_u = (n_az + RFS_TILE - 1) / RFS_TILE, tiles_v = (n_el + RFS_TILE - 1) / RFS_TILE;
    const int n_tiles = tiles_u * tiles_v;
    if (n_tiles > BK_MAX_TILES || cap < 0 || n < 0) return RFS_ERR_SHAPE;
    cudaStream_t st = (cudaStream_t)stream;
    const int nb = rfs_ceil_div(n > 0 ? n : 1, BK_BLK);
    uint32_t* tab = (uint32_t*)temp;  // [n_tiles][nb]
    uint32_t* tot = tab + (size_t)nb * n_tiles;
    uint32_t* toff = tot + n_tiles;
    uint32_t* altc = toff + n_tiles;
    uint32_t* altv = altc + (cap > 0 ? cap : 0);
    if (n > 0) {
        rfs_launch(k_tile_count, nb, BK_BLK, 0, st, n, (const Rect*)rects, tiles_u, n_tiles, nb, tab);
        RFS_LAUNCH_CHECK();
    } else {
        RFS_CUDA_TRY(rfs_fill_u32(tab, 0u, (size_t)n_tiles, st));
    }
    rfs_launch(k_tile_blockscan, rfs_ceil_div(n_tiles * 32, 128), 128, 0, st, nb, n_tiles, tab, tot);
    RFS_LAUNCH_CHECK();
    rfs_launch(k_tile_offsets, 1, BK_MAX_TILES, 0, st, n_tiles, tot, (uint32_t)cap, (int2*)ranges, toff, status);
    RFS_LAUNCH_CHECK();
    if (n <= 0 || cap <= 0) return RFS_OK;
    rfs_launch(k_fill_stable, nb, BK_BLK, 0, st, n, (const Rect*)rects, depth_code, tiles_u, n_tiles, nb, (uint32_t)cap, tab,
                                         toff, bcodes, bvals);
    RFS_LAUNCH_CHECK();
    int rc = launch_seg_sort<BK_SEG_SMALL, 512>(n_tiles, ranges, 0, bcodes, bvals, altc, altv, geom, ckeys, vals, lb,
                                                st);
    if (rc != RFS_OK) return rc;
    rc = launch_seg_sort<BK_SEG_MAX, 1024>(n_tiles, ranges, BK_SEG_SMALL, bcodes, bvals, altc, altv, geom, ckeys,
                                           vals, lb, st);
    if (rc != RFS_OK) return rc;
    rc = launch_seg_sort_cluster(n_tiles, ranges, BK_SEG_MAX, bcodes, bvals, geom, ckeys, vals, lb, st);
    if (rc != RFS_OK) return rc;
    return launch_seg_sort<0, 1024>(n_tiles, ranges, BK_SEG_CLUSTER, bcodes, bvals, altc, altv, geom, ckeys, vals, lb,
                                    st);
}

}  // extern "C"
