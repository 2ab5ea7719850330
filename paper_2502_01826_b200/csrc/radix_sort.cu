// radix_sort.cu -- K3: hand-written stable LSD radix sort of (u64 key, u32 value)
// pairs, plus a cub::DeviceRadixSort entry point for comparison.
//
// Replaces np.argsort(keys, kind="stable") of splat.py:337.  Keys are the
// compact tile keys of project.cu (tile << 31 | float32 depth bits), so a
// 276-tile grid needs 40 key bits = 5 passes of 8 bits.
//
// Each pass is ONE kernel ("onesweep"): a block ranks a 4096-key tile with
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
constexpr int RS_ITEMS = 16;                    // keys per thread: 4096 keys per block
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;
constexpr int RS_MAX_BITS = 11;                 // digit width per pass: 8..11 bits
constexpr int RS_MAX_RADIX = 1 << RS_MAX_BITS;
constexpr int RS_MAX_PASSES = 8;
constexpr uint32_t LB_AGG = 1u << 30;
constexpr uint32_t LB_INC = 2u << 30;
constexpr uint32_t LB_MASK = (1u << 30) - 1;
constexpr int HIST_THREADS = 256;
constexpr int HIST_ITEMS = 16;

// Digit width: 8 bits.  Measured on B200 (483k 40-bit tile keys, 1.15M
// 17-bit Gaussian ids): 10- / 9-bit digits save a pass but each pass costs
// ~1.6x (DPT look-backs per thread, larger shared footprint), a net loss at
// these sizes; the wider kernels stay instantiable through RS_DIGIT_BITS.
#ifndef RS_DIGIT_BITS
#define RS_DIGIT_BITS 8
#endif
inline int bits_for(int) { return RS_DIGIT_BITS; }
inline int passes_for(int end_bit) { return (end_bit + bits_for(end_bit) - 1) / bits_for(end_bit); }

// one read: digit histograms of every pass at once
template <int BITS>
__global__ void __launch_bounds__(HIST_THREADS) k_hist(const uint64_t* __restrict__ keys, int m,
                                                      const uint32_t* __restrict__ m_dev, int passes,
                                                      uint32_t* __restrict__ hist) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    constexpr int RADIX = 1 << BITS;
    if (m_dev) m = min(m, (int)*m_dev);
    if ((long long)blockIdx.x * HIST_THREADS * HIST_ITEMS >= m) return;
    extern __shared__ uint32_t sh[];  // [passes][RADIX]
    for (int i = threadIdx.x; i < passes * RADIX; i += HIST_THREADS) sh[i] = 0;
    __syncthreads();
    long long base = (long long)blockIdx.x * HIST_THREADS * HIST_ITEMS;
#pragma unroll 4
    for (int it = 0; it < HIST_ITEMS; ++it) {
        long long j = base + (long long)it * HIST_THREADS + threadIdx.x;
        if (j < m) {
            uint64_t k = keys[j];
            for (int p = 0; p < passes; ++p) atomicAdd(&sh[p * RADIX + ((k >> (p * BITS)) & (RADIX - 1))], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * RADIX; i += HIST_THREADS) {
        uint32_t v = sh[i];
        if (v) atomicAdd(&hist[i], v);
    }
}

// exclusive scan of each pass's histogram (one block, one warp per pass)
__global__ void k_hist_scan(uint32_t* __restrict__ hist, int passes, int radix) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (wid >= passes) return;
    uint32_t* h = hist + wid * radix;
    uint32_t carry = 0;
    for (int c = 0; c < radix; c += 32) {
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

template <int BITS>
struct OnesweepSmem {
    static constexpr int RADIX = 1 << BITS;
    uint64_t keys[RS_TILE];
    uint32_t vals[RS_TILE];
    uint32_t warp_hist[RS_WARPS][RADIX];
    uint32_t digit_excl[RADIX];  // block-local exclusive start of each digit
    uint32_t global_base[RADIX]; // global start of this block's run of each digit
    uint32_t scan_tmp[RS_WARPS + 1];
    int tile_id;
};

// One LSD pass of BITS-bit digits.  Thread t owns digits t*DPT .. t*DPT+DPT-1
// for the per-digit phases (cross-warp prefix, block scan, look-back).
template <int BITS>
#ifndef RFS_OS_MINB
#define RFS_OS_MINB 3  // 80 registers, no spill: 3 blocks per SM (+0.8 % on the step)
#endif
__global__ void __launch_bounds__(RS_THREADS, RFS_OS_MINB) k_onesweep(const uint64_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                                                        uint64_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, int m,
                                                        int shift, const uint32_t* __restrict__ digit_start,
                                                        uint32_t* __restrict__ lookback, int* __restrict__ tile_counter,
                                                        const uint32_t* __restrict__ m_dev) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    constexpr int RADIX = 1 << BITS, DPT = RADIX / RS_THREADS;
    static_assert(DPT >= 1, "at least one digit per thread");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    OnesweepSmem<BITS>& S = *reinterpret_cast<OnesweepSmem<BITS>*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) S.tile_id = atomicAdd(tile_counter, 1);
    for (int i = tid; i < RS_WARPS * RADIX; i += RS_THREADS) (&S.warp_hist[0][0])[i] = 0;
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
        uint32_t d = valid ? (uint32_t)((k[i] >> shift) & (RADIX - 1)) : (uint32_t)RADIX;  // sentinel
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
    uint32_t bcount[DPT], tsum = 0;
#pragma unroll
    for (int q = 0; q < DPT; ++q) {
        const int d = tid * DPT + q;
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w) {
            uint32_t t = S.warp_hist[w][d];
            S.warp_hist[w][d] = run;
            run += t;
        }
        bcount[q] = run;
        tsum += run;
    }
    // block-wide exclusive scan of the digit counts (thread sums, then within the thread)
    {
        uint32_t inc = tsum;
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
        uint32_t ex = S.scan_tmp[wid] + inc - tsum;
#pragma unroll
        for (int q = 0; q < DPT; ++q) {
            S.digit_excl[tid * DPT + q] = ex;
            ex += bcount[q];
        }
    }
    // decoupled look-back over previous tiles, DPT digits per thread
#pragma unroll
    for (int q = 0; q < DPT; ++q) {
        const int d = tid * DPT + q;
        volatile uint32_t* lbv = lookback;
        uint32_t* my = lookback + (size_t)tile * RADIX + d;
        uint32_t excl = 0;
        if (tile == 0) {
            atomicExch(my, LB_INC | bcount[q]);
        } else {
            atomicExch(my, LB_AGG | bcount[q]);
            int j = tile - 1;
            while (true) {
                uint32_t w;
                do {
                    w = lbv[(size_t)j * RADIX + d];
                } while ((w & ~LB_MASK) == 0);
                excl += w & LB_MASK;
                if ((w & ~LB_MASK) == LB_INC) break;
                --j;
            }
            atomicExch(my, LB_INC | (excl + bcount[q]));
        }
        S.global_base[d] = digit_start[d] + excl;
    }
    __syncthreads();
    // block-local scatter into digit order
#pragma unroll
    for (int i = 0; i < RS_ITEMS; ++i) {
        int j = wbase + i * 32 + lane;
        if (j < tile_n) {
            uint32_t d = (uint32_t)((k[i] >> shift) & (RADIX - 1));
            uint32_t p = S.digit_excl[d] + S.warp_hist[wid][d] + rank[i];
            S.keys[p] = k[i];
            S.vals[p] = v[i];
        }
    }
    __syncthreads();
    // coalesced write-out of digit runs
    for (int j = tid; j < tile_n; j += RS_THREADS) {
        uint64_t kk = S.keys[j];
        uint32_t d = (uint32_t)((kk >> shift) & (RADIX - 1));
        uint32_t o = S.global_base[d] + (uint32_t)j - S.digit_excl[d];
        keys_out[o] = kk;
        vals_out[o] = S.vals[j];
    }
}

inline int num_tiles(int m) { return rfs_ceil_div(m > 0 ? m : 1, RS_TILE); }

template <int BITS>
int run_sort(uint64_t* kin, uint32_t* vin, uint64_t* kout, uint32_t* vout, int m, int passes, uint32_t* hist,
             uint32_t* lb, int* ctr, const uint32_t* m_dev, cudaStream_t st) {
    constexpr int RADIX = 1 << BITS;
    static bool attr_set = false;
    const size_t smem = sizeof(OnesweepSmem<BITS>);
    if (!attr_set) {
        RFS_CUDA_TRY(cudaFuncSetAttribute(k_onesweep<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        RFS_CUDA_TRY(cudaFuncSetAttribute(k_hist<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(RS_MAX_PASSES * RADIX * sizeof(uint32_t))));
        attr_set = true;
    }
    rfs_launch(k_hist<BITS>, rfs_ceil_div(m, HIST_THREADS * HIST_ITEMS), HIST_THREADS, passes * RADIX * sizeof(uint32_t), st, 
        kin, m, m_dev, passes, hist);
    rfs_launch(k_hist_scan, 1, 32 * RS_MAX_PASSES, 0, st, hist, passes, RADIX);
    const int nt = num_tiles(m);
    for (int p = 0; p < passes; ++p) {
        rfs_launch(k_onesweep<BITS>, nt, RS_THREADS, smem, st, kin, vin, kout, vout, m, p * BITS, hist + p * RADIX,
                                                       lb + (size_t)p * nt * RADIX, ctr + p, m_dev);
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
    const int p = passes_for(end_bit), radix = 1 << bits_for(end_bit);
    size_t hist = (size_t)RS_MAX_PASSES * RS_MAX_RADIX * sizeof(uint32_t);
    size_t ctr = 64 * sizeof(int);
    size_t lb = (size_t)p * num_tiles(m) * radix * sizeof(uint32_t);
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
    const int passes = passes_for(end_bit);
    if (passes > RS_MAX_PASSES) return RFS_ERR_CAPACITY;
    if (temp_bytes < rfs_sort_temp_bytes(m, end_bit)) return RFS_ERR_CAPACITY;
    unsigned char* t = (unsigned char*)temp;
    uint32_t* hist = (uint32_t*)t;
    int* ctr = (int*)(t + (size_t)RS_MAX_PASSES * RS_MAX_RADIX * sizeof(uint32_t));
    uint32_t* lb = (uint32_t*)((unsigned char*)ctr + 64 * sizeof(int));
    RFS_CUDA_TRY(rfs_fill_u32(temp, 0u, rfs_sort_temp_bytes(m, end_bit) / 4, st));
    int rc;
    switch (bits_for(end_bit)) {
        case 8: rc = run_sort<8>(keys, vals, keys_alt, vals_alt, m, passes, hist, lb, ctr, m_dev, st); break;
        case 9: rc = run_sort<9>(keys, vals, keys_alt, vals_alt, m, passes, hist, lb, ctr, m_dev, st); break;
        case 10: rc = run_sort<10>(keys, vals, keys_alt, vals_alt, m, passes, hist, lb, ctr, m_dev, st); break;
        default: rc = run_sort<11>(keys, vals, keys_alt, vals_alt, m, passes, hist, lb, ctr, m_dev, st); break;
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
