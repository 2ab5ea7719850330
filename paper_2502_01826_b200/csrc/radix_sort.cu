// radix_sort.cu -- K3: hand-written stable LSD radix sort of (u64 key, u32 value)
// pairs, plus a cub::DeviceRadixSort entry point for comparison.
//
// Replaces np.argsort(keys, kind="stable") of splat.py:337.  Keys are the
// compact tile keys of project.cu (tile << 31 | float32 depth bits), so a
// 276-tile grid needs 40 key bits = 5 passes of 8 bits.
//
// Each pass is ONE kernel ("onesweep"): a block ranks a 1024-4096-key tile with
// warp-level match_any multisplit, publishes its per-digit counts through a
// decoupled look-back chain, scatters block-locally through shared memory and
// writes runs of equal digits with coalesced stores.  Block tiles are claimed
// with an atomic counter, so every predecessor a block waits on is resident.
// Stability: ranks follow (warp, item, lane) order = input order.
#include <cub/device/device_radix_sort.cuh>

#include "rfs_common.cuh"

namespace {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
// keys per block = RS_THREADS * ITEMS (ITEMS a template parameter)
constexpr int RS_BITS = 8;
constexpr int RS_RADIX = 1 << RS_BITS;
constexpr int RS_MAX_PASSES = 8;
constexpr uint32_t LB_AGG = 1u << 30;
constexpr uint32_t LB_INC = 2u << 30;
constexpr uint32_t LB_MASK = (1u << 30) - 1;
constexpr int HIST_THREADS = 256;
constexpr int HIST_ITEMS = 16;

// one read: digit histograms of every pass at once
__global__ void __launch_bounds__(HIST_THREADS) k_hist(const uint64_t* __restrict__ keys, int m,
                                                      const uint32_t* __restrict__ m_dev, int passes,
                                                      uint32_t* __restrict__ hist) {
    if (m_dev) m = min(m, (int)*m_dev);
    if ((long long)blockIdx.x * HIST_THREADS * HIST_ITEMS >= m) return;
    __shared__ uint32_t sh[RS_MAX_PASSES][RS_RADIX];
    for (int i = threadIdx.x; i < passes * RS_RADIX; i += HIST_THREADS) sh[i / RS_RADIX][i % RS_RADIX] = 0;
    __syncthreads();
    long long base = (long long)blockIdx.x * HIST_THREADS * HIST_ITEMS;
#pragma unroll 4
    for (int it = 0; it < HIST_ITEMS; ++it) {
        long long j = base + (long long)it * HIST_THREADS + threadIdx.x;
        if (j < m) {
            uint64_t k = keys[j];
            for (int p = 0; p < passes; ++p) atomicAdd(&sh[p][(k >> (p * RS_BITS)) & (RS_RADIX - 1)], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * RS_RADIX; i += HIST_THREADS) {
        uint32_t v = sh[i / RS_RADIX][i % RS_RADIX];
        if (v) atomicAdd(&hist[i], v);
    }
}

// exclusive scan of each pass's 256-bin histogram (one block, one warp per pass)
__global__ void k_hist_scan(uint32_t* __restrict__ hist, int passes) {
    int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (wid >= passes) return;
    uint32_t* h = hist + wid * RS_RADIX;
    uint32_t carry = 0;
    for (int c = 0; c < RS_RADIX; c += 32) {
        uint32_t v = h[c + lane];
        uint32_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        h[c + lane] = carry + inc - v;
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
}

template <int ITEMS>
struct OnesweepSmem {
    static constexpr int TILE = RS_THREADS * ITEMS;
    uint64_t keys[TILE];
    uint32_t vals[TILE];
    uint32_t warp_hist[RS_WARPS][RS_RADIX];
    uint32_t digit_excl[RS_RADIX];  // block-local exclusive start of each digit
    uint32_t global_base[RS_RADIX]; // global start of this block's run of each digit
    uint32_t scan_tmp[RS_WARPS + 1];
    int tile_id;
};

template <int RS_ITEMS>
__global__ void __launch_bounds__(RS_THREADS) k_onesweep(const uint64_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                                                        uint64_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, int m,
                                                        int shift, const uint32_t* __restrict__ digit_start,
                                                        uint32_t* __restrict__ lookback, int* __restrict__ tile_counter,
                                                        const uint32_t* __restrict__ m_dev) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int RS_TILE = RS_THREADS * RS_ITEMS;
    OnesweepSmem<RS_ITEMS>& S = *reinterpret_cast<OnesweepSmem<RS_ITEMS>*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) S.tile_id = atomicAdd(tile_counter, 1);
    for (int i = tid; i < RS_WARPS * RS_RADIX; i += RS_THREADS) (&S.warp_hist[0][0])[i] = 0;
    __syncthreads();
    const int tile = S.tile_id;
    const long long tile_base = (long long)tile * RS_TILE;
    if (m_dev) m = min(m, (int)*m_dev);
    // tiles past the device-side count: no data, and every later tile (the
    // only ones that would look back at this one) is empty too
    if (tile_base >= m && tile > 0) return;
    const int tile_n = (int)min((long long)RS_TILE, (long long)m - tile_base);

    // warp-striped load: warp w owns keys [w*512, w*512+512) of the tile
    uint64_t k[RS_ITEMS];
    uint32_t v[RS_ITEMS];
    uint32_t rank[RS_ITEMS];
    const int wbase = wid * 32 * RS_ITEMS;
#pragma unroll
    for (int i = 0; i < RS_ITEMS; ++i) {
        int j = wbase + i * 32 + lane;
        if (j < tile_n) {
            k[i] = keys_in[tile_base + j];
            v[i] = vals_in[tile_base + j];
        } else {
            k[i] = 0;
            v[i] = 0;
        }
    }
    // warp multisplit ranking in (item, lane) order
    const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < RS_ITEMS; ++i) {
        int j = wbase + i * 32 + lane;
        bool valid = j < tile_n;
        uint32_t d = valid ? (uint32_t)((k[i] >> shift) & (RS_RADIX - 1)) : (uint32_t)RS_RADIX;  // sentinel
        uint32_t peers = __match_any_sync(0xffffffffu, d);
        int leader = __ffs(peers) - 1;
        uint32_t cnt = 0;
        if (valid && lane == leader) {
            cnt = S.warp_hist[wid][d];
            S.warp_hist[wid][d] = cnt + __popc(peers);
        }
        cnt = __shfl_sync(0xffffffffu, cnt, leader);
        rank[i] = cnt + __popc(peers & lt_mask);
        __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive prefix across warps, block count
    uint32_t bcount;
    {
        int d = tid;  // RS_THREADS == RS_RADIX
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) {
            uint32_t t = S.warp_hist[w][d];
            S.warp_hist[w][d] = run;
            run += t;
        }
        bcount = run;
    }
    // block-wide exclusive scan of the digit counts
    {
        uint32_t inc = bcount;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) S.scan_tmp[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            uint32_t t = lane < RS_WARPS ? S.scan_tmp[lane] : 0;
            uint32_t ti = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t u = __shfl_up_sync(0xffffffffu, ti, o);
                if (lane >= o) ti += u;
            }
            if (lane < RS_WARPS) S.scan_tmp[lane] = ti - t;
        }
        __syncthreads();
        S.digit_excl[tid] = S.scan_tmp[wid] + inc - bcount;
    }
    // decoupled look-back over previous tiles, digit = tid
    {
        const int d = tid;
        volatile uint32_t* lbv = lookback;
        uint32_t* my = lookback + (size_t)tile * RS_RADIX + d;
        uint32_t excl = 0;
        if (tile == 0) {
            atomicExch(my, LB_INC | bcount);
        } else {
            atomicExch(my, LB_AGG | bcount);
            int j = tile - 1;
            while (true) {
                uint32_t w;
                do {
                    w = lbv[(size_t)j * RS_RADIX + d];
                } while ((w & ~LB_MASK) == 0);
                excl += w & LB_MASK;
                if ((w & ~LB_MASK) == LB_INC) break;
                --j;
            }
            atomicExch(my, LB_INC | (excl + bcount));
        }
        S.global_base[d] = digit_start[d] + excl;
    }
    __syncthreads();
    // block-local scatter into digit order
#pragma unroll
    for (int i = 0; i < RS_ITEMS; ++i) {
        int j = wbase + i * 32 + lane;
        if (j < tile_n) {
            uint32_t d = (uint32_t)((k[i] >> shift) & (RS_RADIX - 1));
            uint32_t p = S.digit_excl[d] + S.warp_hist[wid][d] + rank[i];
            S.keys[p] = k[i];
            S.vals[p] = v[i];
        }
    }
    __syncthreads();
    // coalesced write-out of digit runs
    for (int j = tid; j < tile_n; j += RS_THREADS) {
        uint64_t kk = S.keys[j];
        uint32_t d = (uint32_t)((kk >> shift) & (RS_RADIX - 1));
        uint32_t o = S.global_base[d] + (uint32_t)j - S.digit_excl[d];
        keys_out[o] = kk;
        vals_out[o] = S.vals[j];
    }
}

inline int num_passes(int end_bit) { return (end_bit + RS_BITS - 1) / RS_BITS; }
inline int items_for(int m) {
    // measured on B200 (483k and 1.15M keys): 16 items per thread beats 4 / 8
    // -- a pass is bound by the look-back chain, which smaller tiles lengthen
    return m >= 0 ? 16 : 4;
}
inline int num_tiles(int m) { return rfs_ceil_div(m > 0 ? m : 1, RS_THREADS * items_for(m)); }

template <int ITEMS>
int run_passes(uint64_t* kin, uint32_t* vin, uint64_t* kout, uint32_t* vout, int m, int passes, const uint32_t* hist,
               uint32_t* lb, int* ctr, const uint32_t* m_dev, cudaStream_t st) {
    static bool attr_set = false;
    const size_t smem = sizeof(OnesweepSmem<ITEMS>);
    if (!attr_set) {
        RFS_CUDA_TRY(cudaFuncSetAttribute(k_onesweep<ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set = true;
    }
    const int nt = num_tiles(m);
    for (int p = 0; p < passes; ++p) {
        k_onesweep<ITEMS><<<nt, RS_THREADS, smem, st>>>(kin, vin, kout, vout, m, p * RS_BITS, hist + p * RS_RADIX,
                                                        lb + (size_t)p * nt * RS_RADIX, ctr + p, m_dev);
        uint64_t* tk = kin; kin = kout; kout = tk;
        uint32_t* tv = vin; vin = vout; vout = tv;
    }
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // namespace

extern "C" {

// Temp bytes for rfs_sort_pairs_u64: histograms + tile counters + look-back words.
size_t rfs_sort_temp_bytes(int m, int end_bit) {
    int p = num_passes(end_bit);
    size_t hist = (size_t)RS_MAX_PASSES * RS_RADIX * sizeof(uint32_t);
    size_t ctr = 64 * sizeof(int);
    size_t lb = (size_t)p * num_tiles(m) * RS_RADIX * sizeof(uint32_t);
    return hist + ctr + lb;
}

// Stable LSD radix sort of (keys, vals) on bits [0, end_bit); m is the
// capacity (grid size) and, when m_dev is given, the device-side count
// min(*m_dev, m) is sorted (no host read needed).  Ping-pongs
// between (keys, vals) and (keys_alt, vals_alt); *result_in_alt tells the
// caller which pair holds the sorted output.
int rfs_sort_pairs_u64(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt, int m, int end_bit,
                       void* temp, size_t temp_bytes, int* result_in_alt, const uint32_t* m_dev, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    *result_in_alt = 0;
    if (m <= 1) return RFS_OK;
    if ((unsigned)m >= LB_MASK || end_bit < 1 || end_bit > 64) return RFS_ERR_CAPACITY;
    int passes = num_passes(end_bit);
    if (passes > RS_MAX_PASSES) return RFS_ERR_CAPACITY;
    if (temp_bytes < rfs_sort_temp_bytes(m, end_bit)) return RFS_ERR_CAPACITY;
    unsigned char* t = (unsigned char*)temp;
    uint32_t* hist = (uint32_t*)t;
    int* ctr = (int*)(t + (size_t)RS_MAX_PASSES * RS_RADIX * sizeof(uint32_t));
    uint32_t* lb = (uint32_t*)((unsigned char*)ctr + 64 * sizeof(int));
    int nt = num_tiles(m);
    RFS_CUDA_TRY(cudaMemsetAsync(temp, 0, rfs_sort_temp_bytes(m, end_bit), st));
    k_hist<<<rfs_ceil_div(m, HIST_THREADS * HIST_ITEMS), HIST_THREADS, 0, st>>>(keys, m, m_dev, passes, hist);
    k_hist_scan<<<1, 32 * RS_MAX_PASSES, 0, st>>>(hist, passes);
    int rc;
    switch (items_for(m)) {
        case 16: rc = run_passes<16>(keys, vals, keys_alt, vals_alt, m, passes, hist, lb, ctr, m_dev, st); break;
        case 8: rc = run_passes<8>(keys, vals, keys_alt, vals_alt, m, passes, hist, lb, ctr, m_dev, st); break;
        default: rc = run_passes<4>(keys, vals, keys_alt, vals_alt, m, passes, hist, lb, ctr, m_dev, st); break;
    }
    if (rc != RFS_OK) return rc;
    *result_in_alt = (passes & 1);
    return RFS_OK;
}

// cub::DeviceRadixSort::SortPairs on the same buffers, for benchmarking K3.
size_t rfs_sort_cub_temp_bytes(int m, int end_bit) {
    size_t bytes = 0;
    cub::DoubleBuffer<uint64_t> dk(nullptr, nullptr);
    cub::DoubleBuffer<uint32_t> dv(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dv, m, 0, end_bit);
    return bytes;
}

int rfs_sort_pairs_u64_cub(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt, int m, int end_bit,
                           void* temp, size_t temp_bytes, int* result_in_alt, void* stream) {
    cub::DoubleBuffer<uint64_t> dk(keys, keys_alt);
    cub::DoubleBuffer<uint32_t> dv(vals, vals_alt);
    size_t bytes = temp_bytes;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, bytes, dk, dv, m, 0, end_bit, (cudaStream_t)stream);
    if (e != cudaSuccess) return RFS_ERR_CUDA;
    *result_in_alt = dk.selector;
    return RFS_OK;
}

}  // extern "C"
