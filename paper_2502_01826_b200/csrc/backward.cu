// backward.cu -- K8: TX-batched backward over the shared hit lists, atomic-free.
//
// Restates the complex part of _ray_backward (_kernels.py:360-387, 522) and
// the p_acc bincount (grad.py:252-254) for a batch of transmitters.  The
// backward is linear in the upstream lambda, so every sum over the TX batch
// is taken before the TX-independent geometry; per live hit k (ray r,
// Gaussian g) only two TX-reduced complex scalars are needed:
//   C_k = sum_b conj(lam_b[r]) psi[g][b]                              (SDDMM)
//   A_k = sum_b conj(lam_b[r]) suffix_{k,b}
//       = w_{k+1} C_{k+1} + rho_{k+1} A_{k+1}   (the reference's suffix
//         recursion, _kernels.py:522, with psi replaced by C)
// and per Gaussian the TX-dependent row
//   p_acc[g][b] = sum_{hits k of g} conj(lam_b[r_k]) w_k T_k          (SpMM^T)
// Three kernels, none with atomics, every sum in a fixed order:
//   K8t k_lam_transpose  lam [B][R] -> lamT [R][B] (a ray's TX row contiguous)
//   K8c k_bwd_gauss      hits in Gaussian-sorted order, one warp per chunk of
//                        BG_CHUNK hits, lanes over TX: C_k for every hit and
//                        p_acc rows accumulated in registers -- the
//                        Gaussian's psi row is loaded once per segment, the
//                        lambda rows of its rays are gathered four hits at a
//                        time.  Gaussians straddling chunks leave per-chunk
//                        partial rows that
//   K8f k_bwd_pfix       adds (a block per straddling Gaussian, fixed order).
//   K8r k_bwd_rays       one thread per ray, hits back to front: the suffix
//                        recursion in fp64, then GW_k = Re(T_k C_k) (_kernels.py:387-388),
//                        d|rho|_k = Re(T_k e^{j phi} A_k), d(phase)_k =
//                        -Im(T_k rho A_k) (_kernels.py:382-385), stored at
//                        the hit's sorted position for K9a.
#include "rfs_common.cuh"

namespace {

// ------------------------------------------------------------ K8t transpose
__global__ void __launch_bounds__(256) k_lam_transpose(const float2* __restrict__ lam, int nb, int R,
                                                       float2* __restrict__ lamT) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    __shared__ float2 t[32][33];
    const int r0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int i = ty; i < 32; i += 8) {
        const int b = b0 + i, r = r0 + tx;
        t[i][tx] = (b < nb && r < R) ? lam[(size_t)b * R + r] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    for (int i = ty; i < 32; i += 8) {
        const int r = r0 + i, b = b0 + tx;
        if (r < R && b < nb) lamT[(size_t)r * nb + b] = t[tx][i];
    }
}

// ------------------------------------------------------------ K8c by Gaussian
constexpr int BG_CHUNK = 128;   // sorted hits per warp
constexpr int BG_WARPS = 4;     // warps per block
constexpr int BG_MAXJ = 8;      // lanes own b = lane + 32 j: up to 256 TX per launch
constexpr int BG_U = 4;         // hits in flight per warp

// Sum of 8 per-lane values over the warp in 9 shuffles (instead of 40):
// afterwards value i is held by lanes 4i .. 4i+3.
__device__ __forceinline__ float reduce8(float (&v)[8], int lane) {
#pragma unroll
    for (int s = 16, h = 4; s >= 4; s >>= 1, h >>= 1) {
        const bool upper = (lane & s) != 0;
#pragma unroll
        for (int j = 0; j < h; ++j) {
            const float send = upper ? v[j] : v[j + h];
            const float keep = upper ? v[j + h] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
        }
    }
    float x = v[0];
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    return x;
}

// Generic TX count: lanes own b = lane + 32 j (float2 loads).
template <int NJ>
__global__ void __launch_bounds__(BG_WARPS * 32) k_bwd_gauss(
    int h_tot, const uint32_t* __restrict__ h_dev, int nb, const uint64_t* __restrict__ sorted_g,
    const uint32_t* __restrict__ s_slot, int hshift, const float2* __restrict__ s_wt, const int2* __restrict__ g_rng,
    const float2* __restrict__ psi, const float2* __restrict__ lamT, int accumulate, float2* __restrict__ C,
    float2* __restrict__ P, float2* __restrict__ part, int* __restrict__ strad) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    if (h_dev) h_tot = min(h_tot, (int)*h_dev);
    __shared__ uint32_t sh_g[BG_WARPS][BG_CHUNK];
    __shared__ uint32_t sh_r[BG_WARPS][BG_CHUNK];
    __shared__ float2 sh_wt[BG_WARPS][BG_CHUNK];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int wglob = blockIdx.x * BG_WARPS + wl;
    const int c0 = wglob * BG_CHUNK;
    if (c0 >= h_tot) return;
    const int c1 = min(c0 + BG_CHUNK, h_tot);
    for (int i = lane; i < c1 - c0; i += 32) {
        sh_g[wl][i] = (uint32_t)sorted_g[c0 + i];
        sh_r[wl][i] = s_slot[c0 + i];
        sh_wt[wl][i] = s_wt[c0 + i];
    }
    __syncwarp();
    int h = c0;
    while (h < c1) {
        const int g = (int)sh_g[wl][h - c0];
        const int2 rg = g_rng[g];
        const int hs = rg.x, he = rg.y;
        const int send = min(he, c1);
        float2 ps[NJ], pa[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int b = lane + 32 * j;
            ps[j] = b < nb ? __ldg(&psi[(size_t)g * nb + b]) : make_float2(0.f, 0.f);
            pa[j] = make_float2(0.f, 0.f);
        }
        for (int hh = h; hh < send; hh += BG_U) {
            float2 l[BG_U][NJ];
            float2 wt[BG_U];
#pragma unroll
            for (int u = 0; u < BG_U; ++u) {
                const bool ok = hh + u < send;
                const int r = ok ? (int)(sh_r[wl][hh + u - c0] >> hshift) : 0;
                wt[u] = ok ? sh_wt[wl][hh + u - c0] : make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    const int b = lane + 32 * j;
                    l[u][j] = (ok && b < nb) ? __ldg(&lamT[(size_t)r * nb + b]) : make_float2(0.f, 0.f);
                }
            }
            float v[8];
#pragma unroll
            for (int u = 0; u < BG_U; ++u) {
                float2 c = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    c = caddf(c, cmulf_cj(l[u][j], ps[j]));         // conj(lam) psi
                    pa[j] = caddf(pa[j], cmulf_cj(l[u][j], wt[u]));  // conj(lam) w T
                }
                v[2 * u] = c.x;
                v[2 * u + 1] = c.y;
            }
            const float x = reduce8(v, lane);
            // lanes 4i hold value i = 2u + component of hit hh + u
            if ((lane & 3) == 0) {
                const int i = lane >> 2, u = i >> 1;
                if (hh + u < send) {
                    float* cf = reinterpret_cast<float*>(C + sh_r[wl][hh + u - c0]) + (i & 1);
                    *cf = accumulate ? *cf + x : x;
                }
            }
        }
        // flush p_acc for g: whole row if g's hits lie inside this chunk,
        // else this chunk's partial (slot 2w: first segment, 2w+1: last)
        float2* dst;
        if (hs >= c0 && he <= c1) {
            dst = P + (size_t)g * nb;
        } else {
            dst = part + (size_t)(hs < c0 ? 2 * wglob : 2 * wglob + 1) * nb;
        }
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int b = lane + 32 * j;
            if (b < nb) dst[b] = pa[j];
        }
        if (hs < c0 && he > c1) {  // g covers the whole chunk: first and last segment
            float2* d2 = part + (size_t)(2 * wglob + 1) * nb;
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int b = lane + 32 * j;
                if (b < nb) d2[b] = pa[j];
            }
        }
        if (lane == 0 && hs >= c0 && he > c1) {  // g starts here and straddles: list it for k_bwd_pfix
            const int q = atomicAdd(strad, 1);
            strad[1 + q] = g;
        }
        h = send;
    }
}

// B a multiple of 64: lanes own TX pairs b = 2 lane + 64 j + {0, 1}, so a
// lambda / psi / p_acc row is one 16-byte vector per lane and NP = B / 64
// vectors per row.  Staging: per sorted hit one float4 (lambda-row offset of
// its ray, slab slot, w T) in shared memory, read back with one broadcast
// LDS.128 per hit; per hit then one wide IMAD, NP 16-byte lambda loads and
// 16 NP FFMA (8 for C, 8 for p_acc).  Segments (runs of one Gaussian) are
// found from a ballot mask of the staged chunk, chunk-straddling from the
// neighbouring keys; the next segment's psi row is prefetched while the
// current one is reduced.
#ifndef RFS_BG_MINB
#define RFS_BG_MINB 8
#endif
template <int NP>
__global__ void __launch_bounds__(BG_WARPS * 32, RFS_BG_MINB) k_bwd_gauss_v(
    int h_tot, const uint32_t* __restrict__ h_dev, int nb, const uint64_t* __restrict__ sorted_g,
    const uint32_t* __restrict__ s_slot, int hshift, const float2* __restrict__ s_wt, const float4* __restrict__ psi,
    const float4* __restrict__ lamT, int accumulate, float2* __restrict__ C, float4* __restrict__ P,
    float4* __restrict__ part, const int2* __restrict__ g_rng, int* __restrict__ cnt) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    if (h_dev) h_tot = min(h_tot, (int)*h_dev);
    __shared__ uint32_t sh_g[BG_WARPS][BG_CHUNK + 1];
    __shared__ float4 sh_e[BG_WARPS][BG_CHUNK];  // (lambda row offset, slot, w T re, w T im)
    __shared__ uint32_t sh_m[BG_WARPS][BG_CHUNK / 32];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int wglob = blockIdx.x * BG_WARPS + wl;
    const int c0 = wglob * BG_CHUNK;
    if (c0 >= h_tot) return;
    const int n = min(BG_CHUNK, h_tot - c0);
    const uint32_t nq = (uint32_t)(nb >> 1);  // float4 per row
    const float4* __restrict__ ll = lamT + lane;
    asm("mov.b64 %0, %0;" : "+l"(ll));  // opaque: per-hit address = one wide IMAD on this base
    for (int i = lane; i < n; i += 32) {
        sh_g[wl][i] = (uint32_t)sorted_g[c0 + i];
        const uint32_t sl = s_slot[c0 + i];
        const float2 wt = s_wt[c0 + i];
        sh_e[wl][i] = make_float4(__uint_as_float((sl >> hshift) * nq), __uint_as_float(sl), wt.x, wt.y);
    }
    __syncwarp();
    const bool first_out = c0 > 0 && (uint32_t)sorted_g[c0 - 1] == sh_g[wl][0];
    const bool last_out = c0 + n < h_tot && (uint32_t)sorted_g[c0 + n] == sh_g[wl][n - 1];
#pragma unroll
    for (int q = 0; q < BG_CHUNK / 32; ++q) {
        const int i = 32 * q + lane;
        const bool st = i < n && (i == 0 || sh_g[wl][i] != sh_g[wl][i - 1]);
        const uint32_t m = __ballot_sync(0xffffffffu, st);
        if (lane == 0) sh_m[wl][q] = m;
    }
    if (lane == 0) sh_g[wl][n] = 0xffffffffu;
    __syncwarp();
    // next segment start after position s (or n)
    auto next_start = [&](int s) -> int {
        for (int q = (s + 1) >> 5; q < BG_CHUNK / 32; ++q) {
            const int sh = (s + 1) - 32 * q;
            uint32_t m = sh_m[wl][q];
            if (sh > 0) m &= 0xffffffffu << sh;
            if (m) return min(32 * q + __ffs(m) - 1, n);
        }
        return n;
    };
    // per hit: conj(lam) psi summed over this lane's TX (cr, ci) and p_acc += conj(lam) w T,
    // as paired fp32 FMAs (FFMA2) with a broadcast lambda component -- per
    // component the same fused operations in the same order as the scalar
    // form (negations folded into qn = (q.y, -q.x, q.w, -q.z), the segment's
    // psi row, and (wi, -wr), the hit's), half the FMA instructions
    auto hit_terms = [&](const float4 (&a)[NP], const float4 (&q)[NP], const float4 (&qn)[NP], float wr, float wi,
                         float4 (&pa)[NP], float& cr, float& ci) {
        float2 c = make_float2(0.f, 0.f);
        const float2 w1 = make_float2(wr, wi), w2 = make_float2(wi, -wr);
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const float2 ax = make_float2(a[j].x, a[j].x), ay = make_float2(a[j].y, a[j].y);
            const float2 az = make_float2(a[j].z, a[j].z), aw = make_float2(a[j].w, a[j].w);
            c = __ffma2_rn(ax, make_float2(q[j].x, q[j].y), c);
            c = __ffma2_rn(ay, make_float2(qn[j].x, qn[j].y), c);
            c = __ffma2_rn(az, make_float2(q[j].z, q[j].w), c);
            c = __ffma2_rn(aw, make_float2(qn[j].z, qn[j].w), c);
            float2 p01 = make_float2(pa[j].x, pa[j].y), p23 = make_float2(pa[j].z, pa[j].w);
            p01 = __ffma2_rn(ax, w1, p01);
            p01 = __ffma2_rn(ay, w2, p01);
            p23 = __ffma2_rn(az, w1, p23);
            p23 = __ffma2_rn(aw, w2, p23);
            pa[j] = make_float4(p01.x, p01.y, p23.x, p23.y);
        }
        cr = c.x;
        ci = c.y;
    };
    float4 ps[NP], pn[NP], qn[NP];
    {
        const int g = (int)sh_g[wl][0];
#pragma unroll
        for (int j = 0; j < NP; ++j) pn[j] = __ldg(&psi[(size_t)g * nq + lane + 32 * j]);
    }
    int s0 = 0;
    while (s0 < n) {
        const int e = next_start(s0);
        const int g = (int)sh_g[wl][s0];
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            ps[j] = pn[j];
            qn[j] = make_float4(pn[j].y, -pn[j].x, pn[j].w, -pn[j].z);
        }
        if (e < n) {
            const int gn = (int)sh_g[wl][e];
#pragma unroll
            for (int j = 0; j < NP; ++j) pn[j] = __ldg(&psi[(size_t)gn * nq + lane + 32 * j]);
        }
        float4 pa[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) pa[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        // full groups of BG_U hits (one transposed 8-value reduction each),
        // then the segment's 1-3 remaining hits one at a time: most segments
        // in a chunk are short, so padding them to BG_U would waste ~2x
        int i0 = s0;
        for (; i0 + BG_U <= e; i0 += BG_U) {
            float4 l[BG_U][NP], eu[BG_U];
#pragma unroll
            for (int u = 0; u < BG_U; ++u) {
                eu[u] = sh_e[wl][i0 + u];
                const float4* row = ll + __float_as_uint(eu[u].x);
#pragma unroll
                for (int j = 0; j < NP; ++j) l[u][j] = __ldg(row + 32 * j);
            }
            float v[8];
#pragma unroll
            for (int u = 0; u < BG_U; ++u) hit_terms(l[u], ps, qn, eu[u].z, eu[u].w, pa, v[2 * u], v[2 * u + 1]);
            const float x = reduce8(v, lane);
            if ((lane & 3) == 0) {  // lanes 4i hold value i = 2u + component of hit i0 + u
                const int i = lane >> 2, u = i >> 1;
                float* cf = reinterpret_cast<float*>(C + __float_as_uint(sh_e[wl][i0 + u].y)) + (i & 1);
                *cf = accumulate ? *cf + x : x;
            }
        }
        for (; i0 < e; ++i0) {
            const float4 eu = sh_e[wl][i0];
            const float4* row = ll + __float_as_uint(eu.x);
            float4 l[NP];
#pragma unroll
            for (int j = 0; j < NP; ++j) l[j] = __ldg(row + 32 * j);
            float cr, ci;
            hit_terms(l, ps, qn, eu.z, eu.w, pa, cr, ci);
            cr = warp_sum(cr);
            ci = warp_sum(ci);
            if (lane == 0) {
                float2* cp = C + __float_as_uint(eu.y);
                *cp = accumulate ? make_float2(cp->x + cr, cp->y + ci) : make_float2(cr, ci);
            }
        }
        // flush p_acc: whole row, or this chunk's partial (2w: first segment, 2w+1: last)
        const bool fo = s0 == 0 && first_out, lo = e == n && last_out;
        float4* dst = fo ? part + (size_t)(2 * wglob) * nq : (lo ? part + (size_t)(2 * wglob + 1) * nq
                                                                 : P + (size_t)g * nq);
#pragma unroll
        for (int j = 0; j < NP; ++j) dst[lane + 32 * j] = pa[j];
        if (fo && lo) {
#pragma unroll
            for (int j = 0; j < NP; ++j) part[(size_t)(2 * wglob + 1) * nq + lane + 32 * j] = pa[j];
        }
        s0 = e;
    }
    // Gaussians straddling chunks: the last chunk to finish (counted on cnt[g])
    // adds the chunk partials in chunk order -- deterministic, no fix-up launch
    if (!first_out && !last_out) return;
    __threadfence();
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        if (k == 0 ? !first_out : !last_out) continue;
        const int gk = (int)sh_g[wl][k == 0 ? 0 : n - 1];
        if (k == 1 && first_out && gk == (int)sh_g[wl][0]) break;  // one Gaussian spans the chunk: counted once
        const int2 rg = g_rng[gk];
        const int w0 = rg.x / BG_CHUNK, w1 = (rg.y - 1) / BG_CHUNK;
        int last = 0;
        if (lane == 0) last = atomicAdd(&cnt[gk], 1) == w1 - w0;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (!last) continue;
        __threadfence();
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const int q = lane + 32 * j;
            float4 acc = __ldcg(&part[(size_t)(2 * w0 + 1) * nq + q]);
            for (int w = w0 + 1; w <= w1; ++w) {
                const float4 t = __ldcg(&part[(size_t)(2 * w) * nq + q]);
                acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
            }
            P[(size_t)gk * nq + q] = acc;
        }
    }
}

// Gaussians whose hits straddle chunks (listed by k_bwd_gauss, strad[0] =
// count): a block per Gaussian sums its chunk partials (slot 2w0+1 of the
// first chunk, slot 2v of the later ones).  Threads = (TX b, phase): phase p
// adds the chunks w0 + p, w0 + p + PH, ... in order, then the PH phase sums
// are added in phase order -- a fixed order (deterministic) with chains of
// W / PH partials instead of W (a Gaussian crossed by thousands of rays at
// 360x180 spans ~160 chunks).
__global__ void __launch_bounds__(256) k_bwd_pfix(int nb, const int* __restrict__ strad,
                                                  const int2* __restrict__ g_rng, const float2* __restrict__ part,
                                                  float2* __restrict__ P) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    __shared__ float2 s_ph[256];
    const int ph_n = max(1, 256 / nb);  // phases (nb <= 256)
    const int t = threadIdx.x, b = t % nb, ph = t / nb;
    const bool act = ph < ph_n;
    const int nl = strad[0];
    for (int i = blockIdx.x; i < nl; i += gridDim.x) {
        const int g = strad[1 + i];
        const int2 rg = g_rng[g];
        const int w0 = rg.x / BG_CHUNK, w1 = (rg.y - 1) / BG_CHUNK;
        float2 acc = make_float2(0.f, 0.f);
        if (act) {
            for (int v = w0 + ph; v <= w1; v += ph_n)
                acc = caddf(acc, part[(size_t)(v == w0 ? 2 * w0 + 1 : 2 * v) * nb + b]);
            s_ph[t] = acc;
        }
        __syncthreads();
        if (t < nb) {
            float2 sum = s_ph[t];
            for (int p = 1; p < ph_n; ++p) sum = caddf(sum, s_ph[p * nb + t]);
            P[(size_t)g * nb + t] = sum;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ K8r ray recursion
// Thread per ray, hits walked back to front in fp64 (the reference's suffix
// recursion, _kernels.py:522): A_{cnt-1} = 0, A_{k-1} = w_k C_k + rho_k A_k.
// The loads of a hit do not depend on A, so they run ahead of the short
// complex FMA chain; the 32 rays of a warp are neighbours (consecutive v),
// so their rho gathers share L1 lines.
// Precision: rho in fp64 from the geometry record (the reference's value),
// and d(phase) -- a sum of strongly cancelling terms for Gaussians crossed by
// many rays -- is stored as a float pair (hi, lo) for the fp64 sums of K9a.
__global__ void __launch_bounds__(128) k_bwd_rays(const RfsHit* __restrict__ slab, const int* __restrict__ counts,
                                                  int hcap, int R, const float4* __restrict__ rho32,
                                                  const RfsGeom* __restrict__ geom, const float2* __restrict__ C,
                                                  float4* __restrict__ gs) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    const int cnt = min(counts[r], hcap);
    const size_t base = (size_t)r * hcap;
    double Ar = 0.0, Ai = 0.0;
#pragma unroll 4
    for (int k = cnt - 1; k >= 0; --k) {
        const RfsHit hk = slab[base + k];
        const float2 ck = C[base + k];
        const float4 rq = __ldg(&rho32[hk.g]);
        const double rr = __ldg(&geom[hk.g].rho_re), ri = __ldg(&geom[hk.g].rho_im);
        const double tr = hk.t_re, ti = hk.t_im;
        const double gw = tr * (double)ck.x - ti * (double)ck.y;  // Re(T C)          (_kernels.py:387-388)
        const double tar = tr * Ar - ti * Ai, tai = tr * Ai + ti * Ar;
        const double dmag = tar * rq.z - tai * rq.w;             // Re(T e^{jphi} A) (_kernels.py:382-383)
        const double dph = -(tar * ri + tai * rr);               // -Im(T rho A)     (_kernels.py:384-385)
        const float dph_hi = (float)dph;
        gs[base + k] = make_float4((float)gw, (float)dmag, dph_hi, (float)(dph - (double)dph_hi));
        const double wcr = (double)hk.w * (double)ck.x, wci = (double)hk.w * (double)ck.y;
        const double nr = wcr + (rr * Ar - ri * Ai);
        const double ni = wci + (rr * Ai + ri * Ar);
        Ar = nr;
        Ai = ni;
    }
}

}  // namespace

extern "C" {

int rfs_lam_transpose(const void* lam, int n_tx, int n_rays, void* lamT, void* stream) {
    if (n_rays <= 0 || n_tx <= 0) return RFS_OK;
    dim3 grid(rfs_ceil_div(n_rays, 32), rfs_ceil_div(n_tx, 32));
    rfs_launch(k_lam_transpose, grid, 256, 0, (cudaStream_t)stream, (const float2*)lam, n_tx, n_rays, (float2*)lamT);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

size_t rfs_bwd_part_elems(int n_hits, int n_tx) {
    return (size_t)2 * (size_t)((n_hits + BG_CHUNK - 1) / BG_CHUNK + 1) * (size_t)(n_tx > 0 ? n_tx : 1);
}

int rfs_bwd_gauss(int n, int n_hits, const uint32_t* h_dev, int n_tx, const uint64_t* sorted_g, const uint32_t* s_slot,
                  int hcap,
                  const void* s_wt, const int* g_rng, const void* psi, const void* lamT, int accumulate, void* C,
                  void* P, void* part, int* cnt, void* stream) {
    if (n <= 0 || n_hits <= 0 || n_tx <= 0) return RFS_OK;
    if (n_tx > 32 * BG_MAXJ) return RFS_ERR_SHAPE;
    if (hcap <= 0 || (hcap & (hcap - 1))) return RFS_ERR_SHAPE;
    const int hshift = __builtin_ctz((unsigned)hcap);
    cudaStream_t st = (cudaStream_t)stream;
    const int nwarps = rfs_ceil_div(n_hits, BG_CHUNK);
    const unsigned grid = (unsigned)rfs_ceil_div(nwarps, BG_WARPS);
    if (n_tx % 64 == 0) {
        RFS_CUDA_TRY(rfs_fill_u32(cnt, 0u, (size_t)n, st));
#define RFS_BV(NPV)                                                                                              \
    rfs_launch(k_bwd_gauss_v<NPV>, grid, BG_WARPS * 32, 0, st, n_hits, h_dev, n_tx, sorted_g, s_slot, hshift,                   \
                                                       (const float2*)s_wt, (const float4*)psi,                  \
                                                       (const float4*)lamT, accumulate, (float2*)C, (float4*)P,  \
                                                       (float4*)part, (const int2*)g_rng, cnt)
        switch (n_tx / 64) {
            case 1: RFS_BV(1); break;
            case 2: RFS_BV(2); break;
            case 3: RFS_BV(3); break;
            default: RFS_BV(4); break;
        }
#undef RFS_BV
    } else {
        const int nj = (n_tx + 31) / 32;
        RFS_CUDA_TRY(rfs_fill_u32(cnt, 0u, 1, st));  // the straddler list's count
#define RFS_BG(NJV)                                                                                              \
    rfs_launch(k_bwd_gauss<NJV>, grid, BG_WARPS * 32, 0, st, n_hits, h_dev, n_tx, sorted_g, s_slot, hshift,             \
                                                     (const float2*)s_wt,                                        \
                                                     (const int2*)g_rng, (const float2*)psi, (const float2*)lamT, accumulate, \
                                                     (float2*)C, (float2*)P, (float2*)part, cnt)
        if (nj == 1) RFS_BG(1);
        else if (nj == 2) RFS_BG(2);
        else if (nj <= 4) RFS_BG(4);
        else RFS_BG(8);
#undef RFS_BG
        rfs_launch(k_bwd_pfix, 148 * 4, 256, 0, st, n_tx, (const int*)cnt, (const int2*)g_rng, (const float2*)part,
                   (float2*)P);
    }
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_bwd_rays(const void* slab, const int* counts, int hcap, int n_rays, const void* rho32, const void* geom,
                 const void* C, void* gs, void* stream) {
    if (n_rays <= 0) return RFS_OK;
    rfs_launch(k_bwd_rays, rfs_ceil_div(n_rays, 128), 128, 0, (cudaStream_t)stream, 
        (const RfsHit*)slab, counts, hcap, n_rays, (const float4*)rho32, (const RfsGeom*)geom, (const float2*)C,
        (float4*)gs);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // extern "C"
