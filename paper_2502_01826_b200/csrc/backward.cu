// backward.cu -- K8a: TX-batched reverse sweep over the shared hit lists.
//
// Restates the complex part of _ray_backward (_kernels.py:360-387, 522) for a
// batch of transmitters.  Because the backward is linear in the upstream
// lambda, every sum over the TX batch is taken before the TX-independent
// geometry, so per hit only two TX-reduced quantities are needed:
//   C_k = sum_b conj(lam_b) psi[g_k][b]                          (SDDMM)
//   A_k = sum_b conj(lam_b) suffix_{k,b}
//       = w_{k+1} C_{k+1} + rho_{k+1} A_{k+1}                    (the reference's
//         suffix recursion with psi replaced by C, _kernels.py:522)
// giving the per-hit scalars GW_k = Re(T_k C_k) (_kernels.py:387-388),
// d|rho|_k = Re(T_k e^{j phi} A_k) and d(phase)_k = -Im(T_k rho A_k)
// (_kernels.py:382-385), written at the hit's Gaussian-sorted position for the
// fixed-order per-Gaussian reduction of grad.cu.  Optionally accumulates
// p_acc[g][b] += conj(lam_b) w_k T_k (inc_pg + bincount, grad.py:252-254) with
// vector atomics, and writes lambda transposed for the deterministic gather.
//
// Mapping: one warp sweeps two rays at once (16 lanes per ray); a lane owns
// TX pairs (2l, 2l+1) + 32 j, so psi rows are read as contiguous 8-byte pairs
// and the per-hit TX reduction is a 4-step half-warp butterfly.  Hit records
// are loaded 16 at a time lane-parallel and broadcast with width-16 shuffles;
// the next hit's psi row is prefetched while the current one is reduced.
#include "rfs_common.cuh"

namespace {

constexpr int BR_RAYS = 32;      // rays per block (lambda staged in shared memory)
constexpr int BR_THREADS = 256;  // 8 warps x 2 rays x 2 rounds
constexpr int BR_MAXJ = 8;       // up to 256 TX per launch

template <int NJ>
__device__ __forceinline__ void load_row(const float2* __restrict__ psi, uint32_t g, int nb, int hl,
                                         float2 (&p)[NJ][2]) {
    const float2* row = psi + (size_t)g * nb;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const int b = 2 * hl + 32 * j;
        p[j][0] = b < nb ? __ldg(&row[b]) : make_float2(0.f, 0.f);
        p[j][1] = b + 1 < nb ? __ldg(&row[b + 1]) : make_float2(0.f, 0.f);
    }
}

// NJ = ceil(n_tx / 32) (compile time: no dead predicated iterations)
template <int NJ>
__global__ void __launch_bounds__(BR_THREADS) k_backward_rays(
    const RfsHit* __restrict__ slab, const int* __restrict__ counts, int hcap, const float2* __restrict__ psi,
    const float2* __restrict__ lam, const float4* __restrict__ rho32, int nb, int R,
    const uint32_t* __restrict__ inv_slot, float4* __restrict__ s_gs, float2* __restrict__ lamT,
    float2* __restrict__ P) {
    extern __shared__ __align__(16) float2 s_lam[];  // [nb][BR_RAYS + 1]
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int half = lane >> 4, hl = lane & 15;
    const int r0 = blockIdx.x * BR_RAYS;
    for (int i = threadIdx.x; i < nb * BR_RAYS; i += BR_THREADS) {
        int b = i / BR_RAYS, rl = i % BR_RAYS, r = r0 + rl;
        s_lam[b * (BR_RAYS + 1) + rl] = r < R ? lam[(size_t)b * R + r] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    if (lamT) {  // lambda transposed to [R][nb] rows for the deterministic p_acc gather
        for (int i = threadIdx.x; i < nb * BR_RAYS; i += BR_THREADS) {
            int rl = i / nb, b = i % nb, r = r0 + rl;
            if (r < R) lamT[(size_t)r * nb + b] = s_lam[b * (BR_RAYS + 1) + rl];
        }
    }
    for (int pr = wid; pr < BR_RAYS / 2; pr += BR_THREADS / 32) {
        const int rl = 2 * pr + half, r = r0 + rl;
        const int cnt = r < R ? min(counts[r], hcap) : 0;
        const int cmax = max(cnt, __shfl_xor_sync(0xffffffffu, cnt, 16));
        if (cmax == 0) continue;
        float2 cl[NJ][2];  // conj(lambda_b) of this lane's TX
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int b = 2 * hl + e + 32 * j;
                const float2 l = b < nb ? s_lam[b * (BR_RAYS + 1) + rl] : make_float2(0.f, 0.f);
                cl[j][e] = make_float2(l.x, -l.y);
            }
        const RfsHit* hrow = slab + (size_t)r * hcap;
        const uint32_t* irow = inv_slot + (size_t)r * hcap;
        // suffix recursion state in fp64 (a Gaussian every ray crosses first makes
        // d(phase) a sum of ~1e3 cancelling terms)
        double Ar = 0.0, Ai = 0.0, wn = 0.0, rnr = 0.0, rni = 0.0, cnr = 0.0, cni = 0.0;
        RfsHit hc;
        hc.g = 0; hc.w = 0.f; hc.t_re = 0.f; hc.t_im = 0.f;
        float4 rq = make_float4(0.f, 0.f, 0.f, 0.f);
        uint32_t pos = 0;
        float2 pv[NJ][2], pn[NJ][2];
        for (int k = cmax - 1; k >= 0; --k) {
            const int ks = k & 15;
            if (k == cmax - 1 || ks == 15) {
                // lane-parallel load of this ray's hits [k - ks, k - ks + 16)
                const int kk = (k - ks) + hl;
                if (kk < cnt) {
                    hc = hrow[kk];
                    rq = __ldg(&rho32[hc.g]);
                    pos = irow[kk];
                }
                const uint32_t g0 = __shfl_sync(0xffffffffu, hc.g, ks, 16);
                load_row<NJ>(psi, g0, nb, hl, pn);
            }
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                pv[j][0] = pn[j][0];
                pv[j][1] = pn[j][1];
            }
            const bool act = k < cnt;
            const float w = __shfl_sync(0xffffffffu, hc.w, ks, 16);
            const float tre = __shfl_sync(0xffffffffu, hc.t_re, ks, 16);
            const float tim = __shfl_sync(0xffffffffu, hc.t_im, ks, 16);
            const uint32_t g = __shfl_sync(0xffffffffu, hc.g, ks, 16);
            const float rqx = __shfl_sync(0xffffffffu, rq.x, ks, 16);
            const float rqy = __shfl_sync(0xffffffffu, rq.y, ks, 16);
            // prefetch the next (lower) hit's psi row within the loaded chunk
            const uint32_t gp = __shfl_sync(0xffffffffu, hc.g, ks > 0 ? ks - 1 : 0, 16);
            if (ks > 0) load_row<NJ>(psi, gp, nb, hl, pn);
            const float2 wt = make_float2(w * tre, w * tim);
            float2 c = make_float2(0.f, 0.f);
            if (act) {
#pragma unroll
                for (int j = 0; j < NJ; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        c = caddf(c, cmulf(cl[j][e], pv[j][e]));
                        const int b = 2 * hl + e + 32 * j;
                        if (P && b < nb) atomicAdd(&P[(size_t)g * nb + b], cmulf(cl[j][e], wt));
                    }
            }
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) {
                c.x += __shfl_xor_sync(0xffffffffu, c.x, o);
                c.y += __shfl_xor_sync(0xffffffffu, c.y, o);
            }
            if (act) {
                const double cr = c.x, ci = c.y;
                const double nr = wn * cnr + (rnr * Ar - rni * Ai);
                const double ni = wn * cni + (rnr * Ai + rni * Ar);
                Ar = nr;
                Ai = ni;
                if (hl == ks) {  // the lane holding hit k writes its scalars
                    const double tr = tre, ti = tim;
                    const double gw = tr * cr - ti * ci;               // Re(T C)
                    const double tar = tr * Ar - ti * Ai, tai = tr * Ai + ti * Ar;
                    const double dmag = tar * rq.z - tai * rq.w;       // Re(T e^{j phi} A)
                    const double dph = -(tar * rq.y + tai * rq.x);     // -Im(T rho A)
                    // fire-and-forget vector reduction: one writer per launch and
                    // TX chunks are stream-ordered, so the result is deterministic
                    atomicAdd(&s_gs[pos], make_float4((float)gw, (float)dmag, (float)dph, 0.f));
                }
                wn = w;
                rnr = rqx;
                rni = rqy;
                cnr = cr;
                cni = ci;
            }
        }
    }
}

}  // namespace

extern "C" {

int rfs_backward_rays(const void* slab, const int* counts, int hcap, const void* psi, const void* lam, const void* rho32,
                      int n_tx, int n_rays, const uint32_t* inv_slot, void* s_gs, void* lamT, void* P, void* stream) {
    if (n_rays <= 0 || n_tx <= 0) return RFS_OK;
    if (n_tx > 32 * BR_MAXJ) return RFS_ERR_SHAPE;
    size_t smem = (size_t)n_tx * (BR_RAYS + 1) * sizeof(float2);
    const int nj = (n_tx + 31) / 32;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned grid = (unsigned)rfs_ceil_div(n_rays, BR_RAYS);
#define RFS_BR(NJV)                                                                                                 \
    do {                                                                                                            \
        static int attr = 0;                                                                                        \
        if (smem > 48 * 1024 && attr < (int)smem) {                                                                 \
            RFS_CUDA_TRY(                                                                                           \
                cudaFuncSetAttribute(k_backward_rays<NJV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
            attr = (int)smem;                                                                                       \
        }                                                                                                           \
        k_backward_rays<NJV><<<grid, BR_THREADS, smem, st>>>(                                                       \
            (const RfsHit*)slab, counts, hcap, (const float2*)psi, (const float2*)lam, (const float4*)rho32, n_tx,  \
            n_rays, inv_slot, (float4*)s_gs, (float2*)lamT, (float2*)P);                                            \
    } while (0)
    if (nj == 1) RFS_BR(1);
    else if (nj == 2) RFS_BR(2);
    else if (nj <= 4) RFS_BR(4);
    else RFS_BR(8);
#undef RFS_BR
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // extern "C"
