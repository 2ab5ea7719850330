// composite.cu -- TX-batched kernels on top of the shared hit lists.
//
//   K5  k_psi          psi[g][b] = sum_k c_gk basis_k(bearing mu_g -> tx_b)
//   K7  k_forward      S[b][r]  = sum_k w_k T_k psi[g_k][b]                 (SpMM)
//   K8i k_hit_keys / k_gather_sorted / k_gauss_offsets
//                      by-Gaussian index of the live hits (TX independent):
//                      hits sorted by Gaussian id (stable, so (ray, k) order
//                      within a Gaussian = the reference's bincount slot
//                      order), per sorted hit its ray, w and w T, the inverse
//                      map slot -> sorted position, and per-Gaussian offsets
//   (K8a, the TX-batched backward sweep, is in backward.cu)
#include "fle.cuh"
#include "rfs_common.cuh"

namespace {

// ------------------------------------------------------------------ K5: psi
// A warp per group of PSI_G consecutive Gaussians: one coalesced load of their
// `used` marks (nullable: all), then, Gaussian by Gaussian (warp-uniform),
// lanes over the TX.  Only ~30 % of the Gaussians have live hits at config 2;
// a thread per (Gaussian, TX) spent most of its blocks on an early exit.  The
// rows of unused Gaussians are never read by K7 / K8c and are left unwritten.
#ifndef PSI_G
#define PSI_G 8  // Gaussians per warp: 8 -> 26 us, 16 -> 31, 32 -> 35 (more warps in flight)
#endif
template <int L>
__global__ void __launch_bounds__(256) k_psi(int n, int nb, const float* __restrict__ means,
                                             const float2* __restrict__ coeffs, const float* __restrict__ tx,
                                             const uint32_t* __restrict__ used, float2* __restrict__ psi) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int lane = threadIdx.x & 31;
    const int g0 = (blockIdx.x * 8 + (threadIdx.x >> 5)) * PSI_G;
    if (g0 >= n) return;
    const int g_l = g0 + lane;
    unsigned todo = __ballot_sync(0xffffffffu, lane < PSI_G && g_l < n && (!used || used[g_l] != 0u));
    while (todo) {
        const int g = g0 + __ffs(todo) - 1;
        todo &= todo - 1;
        const float mx = means[3 * g], my = means[3 * g + 1], mz = means[3 * g + 2];
        const float2* c = coeffs + (size_t)g * Fle<L>::K;
#pragma unroll 2
        for (int b = lane; b < nb; b += 32)
            psi[(size_t)g * nb + b] = Fle<L>::psi(tx[3 * b] - mx, tx[3 * b + 1] - my, tx[3 * b + 2] - mz, c);
    }
}

// --------------------------------------------------------------- K7 forward
constexpr int CP_RAYS = 32;      // rays per block (output staged for coalesced [B][R] stores)
constexpr int CP_THREADS = 256;  // 8 warps, 4 rays each
constexpr int CP_BCH = 64;       // TX per block (lanes own b and b + 32)

__global__ void __launch_bounds__(CP_THREADS) k_forward(const RfsHit* __restrict__ slab, const int* __restrict__ counts,
                                                        int hcap, const float2* __restrict__ psi, int nb, int R,
                                                        float2* __restrict__ S) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    __shared__ float2 s_out[CP_BCH][CP_RAYS + 1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int r0 = blockIdx.x * CP_RAYS, bc = blockIdx.y * CP_BCH;
    const int b0 = bc + lane, b1 = bc + 32 + lane;
    for (int rl = wid; rl < CP_RAYS; rl += CP_THREADS / 32) {
        const int r = r0 + rl;
        float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
        if (r < R) {
            const int cnt = min(counts[r], hcap);
            const RfsHit* h = slab + (size_t)r * hcap;
            for (int k = 0; k < cnt; ++k) {
                RfsHit hk = h[k];
                float2 wt = make_float2(hk.w * hk.t_re, hk.w * hk.t_im);
                const float2* row = psi + (size_t)hk.g * nb;
                if (b0 < nb) a0 = caddf(a0, cmulf(wt, __ldg(&row[b0])));
                if (b1 < nb) a1 = caddf(a1, cmulf(wt, __ldg(&row[b1])));
            }
        }
        s_out[lane][rl] = a0;
        s_out[lane + 32][rl] = a1;
    }
    __syncthreads();
    const int nbc = min(CP_BCH, nb - bc);
    for (int i = threadIdx.x; i < nbc * CP_RAYS; i += CP_THREADS) {
        int bl = i / CP_RAYS, rl = i % CP_RAYS, r = r0 + rl;
        if (r < R) S[(size_t)(bc + bl) * R + r] = s_out[bl][rl];
    }
}

// Even TX count: lanes own TX pairs (one 16-byte psi vector per hit).  A
// block covers a column of FP_V rays (neighbouring rays cross mostly the
// same Gaussians, so their psi rows are L1 hits); warp w owns rays
// v0 + w + 8 j, j < FV_RPW.  Per 32-hit chunk every lane loads one hit
// record, forms w T and the hit's psi row offset once and parks them in a
// per-warp shared-memory slot; the hit loop reads each record with one
// broadcast LDS.128 and issues, per hit, one address IMAD, one 16-byte psi
// load and 4 FFMA2 (paired fp32 FMAs).  Latency is covered by software pipelining: the next
// group of FV_U psi vectors is in flight while the current group is summed,
// and the next chunk's (or next ray's) hit records while the current chunk
// is composited.  psi row offsets are 32-bit float4 counts (N B / 2 < 2^32).
#ifndef RFS_FV_U
#define RFS_FV_U 4
#endif
constexpr int FV_U = RFS_FV_U;
constexpr int FP_V = 32, FP_RAYS = FP_V;
constexpr int FV_RPW = FP_RAYS / (CP_THREADS / 32);  // rays per warp
#ifndef RFS_FV_MINB
#define RFS_FV_MINB 5  // 48 registers (a small spill): 5 blocks per SM measured fastest (51 vs 53 us at 1..4)
#endif
__global__ void __launch_bounds__(CP_THREADS, RFS_FV_MINB) k_forward_v(const RfsHit* __restrict__ slab,
                                                          const int* __restrict__ counts, int hcap,
                                                          const float4* __restrict__ psi, int nb, int n_az, int n_el,
                                                          float2* __restrict__ S) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    __shared__ float2 s_out[CP_BCH][FP_RAYS + 1];
    __shared__ float4 s_hit[CP_THREADS / 32][32 + 2 * FV_U];  // (row offset bits, w T re, -w T im, w T im)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int pv_blocks = (n_el + FP_V - 1) / FP_V;
    const int u = blockIdx.x / pv_blocks, v0 = (blockIdx.x % pv_blocks) * FP_V;
    const int bc = blockIdx.y * CP_BCH;
    const int R = n_az * n_el;
    const uint32_t nq = (uint32_t)(nb >> 1);
    const bool on = 2 * lane + bc < nb;
    // this lane's float4 column; lanes past the batch re-read column 0 (never stored)
    const float4* __restrict__ pl = psi + (on ? (bc >> 1) + lane : 0);
    asm("mov.b64 %0, %0;" : "+l"(pl));  // opaque: per-hit address = one wide IMAD on this base
    float4* sh = s_hit[wid];
    if (lane < 2 * FV_U) sh[32 + lane] = make_float4(0.f, 0.f, 0.f, 0.f);  // padding: offset 0, w T = 0
    int my_cnt = 0;  // lane j < FV_RPW: live hits of the warp's ray j
    if (lane < FV_RPW) {
        const int v = v0 + wid + (CP_THREADS / 32) * lane;
        if (u < n_az && v < n_el) my_cnt = min(counts[u * n_el + v], hcap);
    }
    auto load_rec = [&](int j, int k, int cnt) -> float4 {  // staged form of hit k of ray j (zero past cnt)
        float4 e = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < cnt) {
            const RfsHit hl = slab[(size_t)(u * n_el + v0 + wid + (CP_THREADS / 32) * j) * hcap + k];
            const float wi = hl.w * hl.t_im;
            e = make_float4(__uint_as_float(hl.g * nq), hl.w * hl.t_re, -wi, wi);
        }
        return e;
    };
    float4 rec = load_rec(0, lane, __shfl_sync(0xffffffffu, my_cnt, 0));
#pragma unroll 1
    for (int j = 0; j < FV_RPW; ++j) {
        const int cnt = __shfl_sync(0xffffffffu, my_cnt, j);
        const int cnt_n = __shfl_sync(0xffffffffu, my_cnt, (j + 1) % FV_RPW);
        float2 a01 = make_float2(0.f, 0.f), a23 = make_float2(0.f, 0.f);
        if (cnt == 0 && j + 1 < FV_RPW) rec = load_rec(j + 1, lane, cnt_n);
        for (int kc = 0; kc < cnt; kc += 32) {
            __syncwarp();
            sh[lane] = rec;
            __syncwarp();
            if (kc + 32 < cnt) rec = load_rec(j, kc + 32 + lane, cnt);
            else if (j + 1 < FV_RPW) rec = load_rec(j + 1, lane, cnt_n);
            const int n_in = min(32, cnt - kc);
            // ping-pong register buffers (A: even groups, B: odd groups); entries
            // past n_in read offset 0 with w T = 0
            float4 ea[FV_U], pa[FV_U], eb[FV_U], pb[FV_U];
            auto fetch = [&](float4(&e)[FV_U], float4(&p)[FV_U], int i0) {
#pragma unroll
                for (int k = 0; k < FV_U; ++k) {
                    e[k] = sh[i0 + k];
                    p[k] = __ldg(pl + __float_as_uint(e[k].x));
                }
            };
            // acc += (w T) psi for the lane's two TX, as paired fp32 FMAs (FFMA2:
            // the same fused operations per component, half the instructions)
            auto madd = [&](const float4(&e)[FV_U], const float4(&p)[FV_U]) {
#pragma unroll
                for (int k = 0; k < FV_U; ++k) {
                    const float2 wr = make_float2(e[k].y, e[k].y), wi = make_float2(e[k].z, e[k].w);  // (-wi, wi)
                    a01 = __ffma2_rn(wr, make_float2(p[k].x, p[k].y), a01);
                    a01 = __ffma2_rn(wi, make_float2(p[k].y, p[k].x), a01);
                    a23 = __ffma2_rn(wr, make_float2(p[k].z, p[k].w), a23);
                    a23 = __ffma2_rn(wi, make_float2(p[k].w, p[k].z), a23);
                }
            };
            fetch(ea, pa, 0);
            for (int i0 = 0;;) {
                fetch(eb, pb, i0 + FV_U);
                madd(ea, pa);
                i0 += FV_U;
                if (i0 >= n_in) break;
                fetch(ea, pa, i0 + FV_U);
                madd(eb, pb);
                i0 += FV_U;
                if (i0 >= n_in) break;
            }
        }
        const int rl = wid + (CP_THREADS / 32) * j;
        s_out[2 * lane][rl] = a01;
        s_out[2 * lane + 1][rl] = a23;
    }
    __syncthreads();
    const int nbc = min(CP_BCH, nb - bc);
    for (int i = threadIdx.x; i < nbc * FP_RAYS; i += CP_THREADS) {
        const int bl = i / FP_RAYS, rl = i % FP_RAYS;
        const int v = v0 + rl;
        if (u < n_az && v < n_el) S[(size_t)(bc + bl) * R + u * n_el + v] = s_out[bl][rl];
    }
}

// ------------------------------------------- K8i by-Gaussian hit index
// The hits are ordered by the compact id of their Gaussian among the
// Gaussians with a live hit (cid, an exclusive scan of K6's used marks: the
// Gaussian-id order in fewer key bits) and, stably, by (ray, k) within it --
// the reference's bincount slot order, so every per-Gaussian sum keeps its
// order.  (A spatial rank -- Gaussians sorted by the Morton code of their
// projected centre -- was measured: the lambda-row gathers of K8c went from
// 0.5 % to 4 % L1 hits, -4 us, while ranking cost +50 us.)

// order[cid[g]] = g for the Gaussians with a live hit (entries at cid >= cap
// are dropped: the caller checks the count and rebuilds)
__global__ void k_used_list(int n, const uint32_t* __restrict__ used, const uint32_t* __restrict__ cid, int cap,
                            uint32_t* __restrict__ order) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n || !used[g]) return;
    const uint32_t c = cid[g];
    if (c < (uint32_t)cap) order[c] = (uint32_t)g;
}

// keys[c] = rank[g] = cid[g] (or the Gaussian id when rank is NULL), vals[c] = slab
// slot r*hcap + k, c = ray_off[r] + k
__global__ void k_hit_keys(const RfsHit* __restrict__ slab, const int* __restrict__ counts,
                           const uint32_t* __restrict__ ray_off, int hcap, int R, const uint32_t* __restrict__ rank,
                           uint64_t* __restrict__ keys, uint32_t* __restrict__ slots) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int lane = threadIdx.x & 31;
    const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (r >= R) return;
    const int cnt = min(counts[r], hcap);
    const uint32_t base = ray_off[r];
    for (int k = lane; k < cnt; k += 32) {
        const uint32_t g = slab[(size_t)r * hcap + k].g;
        keys[base + k] = rank ? rank[g] : g;
        slots[base + k] = (uint32_t)((size_t)r * hcap + k);
    }
}

// per sorted hit p: its ray, w, w T; inverse map slot -> p (nullable); with
// keys (compact-id sort), the keys are replaced by the Gaussian ids
__global__ void k_gather_sorted(const uint32_t* __restrict__ sorted_slots, int h, const uint32_t* __restrict__ h_dev,
                                int hcap,
                                const RfsHit* __restrict__ slab, uint32_t* __restrict__ s_ray,
                                float* __restrict__ s_w, float2* __restrict__ s_wt, uint32_t* __restrict__ inv_slot,
                                uint64_t* __restrict__ keys) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    if (h_dev) h = min(h, (int)*h_dev);
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= h) return;
    const uint32_t s = sorted_slots[p];
    const RfsHit hk = slab[s];
    s_ray[p] = s / (uint32_t)hcap;
    s_w[p] = hk.w;
    s_wt[p] = make_float2(hk.w * hk.t_re, hk.w * hk.t_im);
    if (inv_slot) inv_slot[s] = (uint32_t)p;
    if (keys) keys[p] = hk.g;
}

// g_rng[g] = [first, end) of g's run of sorted hits ((0, 0) for a Gaussian
// without hits: the array is cleared first); sorted_g = Gaussian id per hit
__global__ void k_gauss_ranges(const uint64_t* __restrict__ sorted_g, int h, const uint32_t* __restrict__ h_dev,
                               int2* __restrict__ g_rng) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    if (h_dev) h = min(h, (int)*h_dev);
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= h) return;
    const uint64_t g = sorted_g[p];
    if (p == 0 || sorted_g[p - 1] != g) g_rng[g].x = p;
    if (p == h - 1 || sorted_g[p + 1] != g) g_rng[g].y = p + 1;
}

template <int L>
void launch_psi(int n, int nb, const float* means, const float2* coeffs, const float* tx, const uint32_t* used,
                float2* psi, cudaStream_t st) {
    rfs_launch(k_psi<L>, rfs_ceil_div(n, 8 * PSI_G), 256, 0, st, n, nb, means, coeffs, tx, used, psi);
}

}  // namespace

extern "C" {

int rfs_psi(int n, int n_tx, int degree, const float* means, const void* coeffs, const float* tx, const uint32_t* used,
            void* psi, void* stream) {
    if (n <= 0 || n_tx <= 0) return RFS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const float2* c = (const float2*)coeffs;
    float2* p = (float2*)psi;
    switch (degree) {
        case 0: launch_psi<0>(n, n_tx, means, c, tx, used, p, st); break;
        case 1: launch_psi<1>(n, n_tx, means, c, tx, used, p, st); break;
        case 2: launch_psi<2>(n, n_tx, means, c, tx, used, p, st); break;
        case 3: launch_psi<3>(n, n_tx, means, c, tx, used, p, st); break;
        case 4: launch_psi<4>(n, n_tx, means, c, tx, used, p, st); break;
        default: return RFS_ERR_SHAPE;
    }
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_forward(const void* slab, const int* counts, int hcap, const void* psi, int n_tx, int n_az, int n_el, void* S,
                void* stream) {
    const int n_rays = n_az * n_el;
    if (n_rays <= 0 || n_tx <= 0) return RFS_OK;
    dim3 grid(rfs_ceil_div(n_rays, CP_RAYS), rfs_ceil_div(n_tx, CP_BCH));
    if (n_tx % 2 == 0) {
        dim3 gv(n_az * rfs_ceil_div(n_el, FP_V), rfs_ceil_div(n_tx, CP_BCH));
        rfs_launch(k_forward_v, gv, CP_THREADS, 0, (cudaStream_t)stream, (const RfsHit*)slab, counts, hcap,
                                                                 (const float4*)psi, n_tx, n_az, n_el, (float2*)S);
    } else
        rfs_launch(k_forward, grid, CP_THREADS, 0, (cudaStream_t)stream, (const RfsHit*)slab, counts, hcap,
                                                                 (const float2*)psi, n_tx, n_rays, (float2*)S);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_used_list(int n, const uint32_t* used, const uint32_t* cid, int cap, uint32_t* order, void* stream) {
    if (n <= 0) return RFS_OK;
    rfs_launch(k_used_list, rfs_ceil_div(n, 256), 256, 0, (cudaStream_t)stream, n, used, cid, cap, order);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_hit_keys(const void* slab, const int* counts, const uint32_t* ray_off, int hcap, int n_rays,
                 const uint32_t* rank, uint64_t* keys, uint32_t* slots, void* stream) {
    if (n_rays <= 0) return RFS_OK;
    rfs_launch(k_hit_keys, rfs_ceil_div((long long)n_rays * 32, 256), 256, 0, (cudaStream_t)stream, 
        (const RfsHit*)slab, counts, ray_off, hcap, n_rays, rank, keys, slots);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_gather_sorted(const uint32_t* sorted_slots, int n_hits, const uint32_t* h_dev, int hcap, const void* slab,
                      uint32_t* s_ray,
                      float* s_w, void* s_wt, uint32_t* inv_slot, uint64_t* keys, void* stream) {
    if (n_hits <= 0) return RFS_OK;
    rfs_launch(k_gather_sorted, rfs_ceil_div(n_hits, 256), 256, 0, (cudaStream_t)stream, 
        sorted_slots, n_hits, h_dev, hcap, (const RfsHit*)slab, s_ray, s_w, (float2*)s_wt, inv_slot, keys);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_gauss_ranges(const uint64_t* sorted_g, int n_hits, const uint32_t* h_dev, int n, int* g_rng, void* stream) {
    if (n <= 0) return RFS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    RFS_CUDA_TRY(rfs_fill_u32(g_rng, 0u, 2 * (size_t)n, st));
    if (n_hits > 0)
        rfs_launch(k_gauss_ranges, rfs_ceil_div(n_hits, 256), 256, 0, st, sorted_g, n_hits, h_dev, (int2*)g_rng);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // extern "C"
