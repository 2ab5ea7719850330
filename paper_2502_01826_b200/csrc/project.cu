// project.cu -- K1 projection, K2 tile binning (count, warp-scan, fill),
// K4 tile ranges and the per-incidence emission bound.
//
// Compiled with -fmad=false: the tile index must be bit-exact with the
// reference, so every fp64 expression that feeds a floor() or the depth key
// is evaluated with the same roundings as numpy (no FMA contraction).
#include "rfs_common.cuh"

namespace {

struct __align__(16) Rect {
    short s1_lo, s1_hi, s2_hi, tv_lo, tv_hi, pad0, pad1, pad2;
};

__device__ __forceinline__ long long floordiv_ll(long long a, long long b) {
    long long q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
    return q;
}
__device__ __forceinline__ double clampd(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }
// numpy float remainder: sign follows the divisor (npy_divmod)
__device__ __forceinline__ double py_fmod(double a, double b) {
    double m = fmod(a, b);
    if (m != 0.0) {
        if ((b < 0.0) != (m < 0.0)) m += b;
    } else {
        m = copysign(0.0, b);
    }
    return m;
}

// Tile rectangle of one splat: splat.py:308-328 (integer logic restated).
__device__ Rect splat_rect(double cu, double cv, double radius, int n_az, int n_el, int tiles_u) {
    Rect r;
    double flo = floor(cv - radius), fhi = floor(cv + radius);
    long long v_lo = (long long)flo, v_hi = (long long)fhi;
    v_lo = v_lo < 0 ? 0 : (v_lo > n_el - 1 ? n_el - 1 : v_lo);
    v_hi = v_hi < -1 ? -1 : (v_hi > n_el - 1 ? n_el - 1 : v_hi);
    bool off_grid = (fhi < 0.0) || (flo > (double)(n_el - 1));
    long long tv_lo = floordiv_ll(v_lo, RFS_TILE);
    long long tv_hi = off_grid ? -1 : floordiv_ll(v_hi, RFS_TILE);
    long long u_lo = (long long)floor(cu - radius), u_hi = (long long)floor(cu + radius);
    bool span_all = (u_hi - u_lo + 1) >= n_az;
    long long a = u_lo - floordiv_ll(u_lo, n_az) * n_az;
    long long b = a + (u_hi - u_lo);
    bool wrap = b > n_az - 1;
    long long s1_lo = floordiv_ll(a, RFS_TILE);
    long long s1_hi = wrap ? tiles_u - 1 : floordiv_ll(b < n_az - 1 ? b : n_az - 1, RFS_TILE);
    long long s2_hi = wrap ? floordiv_ll(b - n_az, RFS_TILE) : -1;
    bool full = span_all || (wrap && (s2_hi >= s1_lo));
    if (full) { s1_lo = 0; s1_hi = tiles_u - 1; s2_hi = -1; }
    r.s1_lo = (short)s1_lo; r.s1_hi = (short)s1_hi; r.s2_hi = (short)s2_hi;
    r.tv_lo = (short)tv_lo; r.tv_hi = (short)tv_hi;
    r.pad0 = r.pad1 = r.pad2 = 0;
    return r;
}

// K1: one thread per Gaussian.  prepare_context's shape part (render.py:220-227,
// scene.py:118-161), project_scene (splat.py:212-268) and the count pass of
// expand_tile_rects (_kernels.py:532-541), all fp64.
#ifndef RFS_PJ_MINB
#define RFS_PJ_MINB 3  // 80 registers (spills a little): one wave of the grid, 20 -> 17 us
#endif
__global__ void __launch_bounds__(256, RFS_PJ_MINB) k_project(
    int n, const float* __restrict__ means, const float* __restrict__ quats,
    const float* __restrict__ log_scales, const float* __restrict__ raw, const float* __restrict__ phase,
    double rx0, double rx1, double rx2, double ress, int n_az, int n_el, int tiles_u,
    RfsGeom* __restrict__ geom, float4* __restrict__ sph, float4* __restrict__ whit, uint32_t* __restrict__ code,
    Rect* __restrict__ rects, uint32_t* __restrict__ counts, float4* __restrict__ rho32,
    double* __restrict__ proj, int* __restrict__ err) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    double mx = (double)means[3 * g], my = (double)means[3 * g + 1], mz = (double)means[3 * g + 2];
    double qw = quats[4 * g], qx = quats[4 * g + 1], qy = quats[4 * g + 2], qz = quats[4 * g + 3];
    double s0 = log_scales[3 * g], s1 = log_scales[3 * g + 1], s2 = log_scales[3 * g + 2];

    // rotation from the normalized quaternion (scene.py:118-142)
    double qn = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    double w = qw / qn, x = qx / qn, y = qy / qn, z = qz / qn;
    double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                   2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                   2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
    double e0 = exp(2.0 * s0), e1 = exp(2.0 * s1), e2 = exp(2.0 * s2);
    double ie[3] = {1.0 / e0, 1.0 / e1, 1.0 / e2};
    // Sigma^-1 = R diag(e^{-2s}) R^T: symmetric by construction (reference
    // inverts then symmetrizes, render.py:221-222; agreement ~1e-16 rel)
    double I[6];
    {
        int ij[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            int i = ij[k][0], j = ij[k][1];
            I[k] = R[3 * i] * ie[0] * R[3 * j] + R[3 * i + 1] * ie[1] * R[3 * j + 1] + R[3 * i + 2] * ie[2] * R[3 * j + 2];
        }
    }
    RfsGeom G;
    G.mu[0] = mx; G.mu[1] = my; G.mu[2] = mz;
#pragma unroll
    for (int k = 0; k < 6; ++k) G.inv[k] = I[k];
    G.norm = RFS_GAUSS_NORM * exp(-(s0 + s1 + s2)); // (2pi)^-1.5 / sqrt(det Sigma)
    double mag = 1.0 / (1.0 + exp(-(double)raw[g]));
    double ph = (double)phase[g];
    double sp, cp;
    sincos(ph, &sp, &cp);
    G.rho_re = mag * cp;
    G.rho_im = mag * sp;
    rho32[g] = make_float4((float)G.rho_re, (float)G.rho_im, (float)cp, (float)sp);

    // projection onto the grid (splat.py:223-234)
    double ox = mx - rx0, oy = my - rx1, oz = mz - rx2;
    double depth = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(ox, ox), __dmul_rn(oy, oy)), __dmul_rn(oz, oz)));
    if (depth < 1e-9) atomicOr(err, 1 << RFS_ERR_GEOMETRY);
    bool active = depth >= ress;
    double cell = 360.0 / (double)n_az;
    double cover_all = (double)(n_az + n_el);
    double alpha = py_fmod(atan2(oy, ox), RFS_TWO_PI);
    double beta = RFS_PI / 2.0 - acos(clampd(oz / depth, -1.0, 1.0));
    double cu = alpha * RFS_RAD2DEG / cell;
    double cv = (beta * RFS_RAD2DEG + 90.0) / cell;
    G.cu = cu;
    G.cv = cv;

    // conservative incidence radius (splat.py:256-267); lambda_max = max e^{2s}
    double lam3 = fmax(fmax(e0, e1), e2);
    double r3 = 3.0 * sqrt(lam3);
    bool inside = depth <= r3;
    double rho2 = ox * ox + oy * oy;
    double pd = 1e-12 * depth;
    bool polar = rho2 <= pd * pd;
    double theta = asin(clampd(r3 / depth, 0.0, 1.0));
    double ca = cos(beta - theta), cb = cos(beta + theta);
    double cos_lo = ca < cb ? ca : cb;
    double st = sin(theta);
    bool pole_touch = cos_lo <= st;
    double az_extent = asin(clampd(st / (pole_touch ? 1.0 : cos_lo), 0.0, 1.0));
    double extent = pole_touch ? RFS_PI : (theta > az_extent ? theta : az_extent);
    double tr = extent * RFS_RAD2DEG / cell + 2.0;
    if (tr > cover_all) tr = cover_all;
    if (inside || polar) tr = cover_all;
    G.r2 = active ? tr * tr : -1.0;
    // any hit's chord midpoint lies inside the 3-sigma ball, so
    // t_mid >= depth - r3; widen by 1e-9 relative to absorb round-off
    G.lbv = (depth - r3) - 1e-9 * (depth + r3);
    geom[g] = G;

    // fp32 bounding-sphere prefilter: accept if |(mu-rx) x d|^2 <= thr.
    // Margin 1e-6 |mu-rx| + 1e-6 relative covers fp32 rounding of the cross
    // product (~6 ulp) with a 2x safety factor; see DESIGN.md §4 (K6).
    double om = depth;
    double thr = (r3 + 1e-6 * om) * (1.0 + 1e-6);
    thr = thr * thr;
    sph[g] = make_float4((float)ox, (float)oy, (float)oz, __double2float_ru(thr));

    // fp32 whitened ellipsoid prefilter (K6).  With L = diag(e^-s) R^T
    // (L^T L = Sigma^-1), q = L d and p = L (rx - mu), the reference
    // discriminant is disc = 9|q|^2 - |q x p|^2, so a hit needs
    // |q x p| <= 3|q|.  The fp32 error of |q x p| is bounded by
    // ~10 aniso u |q||p| (u = 2^-24, aniso = e^{smax-smin}); the margin below
    // is 4x that plus slack, so the test never rejects an fp64 hit.
    {
        double es[3] = {exp(-s0), exp(-s1), exp(-s2)};
        double L[9];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int j = 0; j < 3; ++j) L[3 * a + j] = es[a] * R[3 * j + a];
        double mm[3] = {rx0 - mx, rx1 - my, rx2 - mz};
        double p[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) p[a] = L[3 * a] * mm[0] + L[3 * a + 1] * mm[1] + L[3 * a + 2] * mm[2];
        double pn = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
        double smax = fmax(fmax(s0, s1), s2), smin = fmin(fmin(s0, s1), s2);
        double aniso = exp(smax - smin);
        double margin = 4e-6 * aniso * (pn + 1.0) + 1e-5;
        double thw = (3.0 + margin) * (3.0 + margin);
        whit[4 * g + 0] = make_float4((float)L[0], (float)L[1], (float)L[2], (float)L[3]);
        whit[4 * g + 1] = make_float4((float)L[4], (float)L[5], (float)L[6], (float)L[7]);
        whit[4 * g + 2] = make_float4((float)L[8], (float)p[0], (float)p[1], (float)p[2]);
        // .y: half-angle of the bounding-sphere cone seen from rx, asin(r3/depth)
        // (pi when rx is inside the ball), for the per-warp cone cull in K6;
        // its axis is sph.xyz normalised.
        // .z/.w: cos / sin of that angle (rounded so cos(th_p + th) is not overestimated)
        double th = inside ? RFS_PI : asin(fmin(r3 / depth, 1.0)) + 1e-6;
        whit[4 * g + 3] = make_float4(__double2float_ru(thw), __double2float_ru(th), __double2float_rd(cos(th)),
                                      __double2float_ru(sin(th)));
    }

    float fd = __double2float_rn(depth);
    code[g] = __float_as_uint(fd);

    Rect rc = splat_rect(cu, cv, tr, n_az, n_el, tiles_u);
    uint32_t cnt = 0;
    if (active) {
        long long nv = (long long)rc.tv_hi - rc.tv_lo + 1;
        if (nv > 0) {
            long long nu = (long long)rc.s1_hi - rc.s1_lo + 1;
            if (rc.s2_hi >= 0) nu += rc.s2_hi + 1;
            cnt = (uint32_t)(nv * nu);
        }
    }
    if (!active) rc.tv_hi = -1;
    rects[g] = rc;
    counts[g] = cnt;

    if (proj) {
        // linearized radius of J Sigma J^T (splat.py:236-254), API parity only
        double Sg[9];
        double ev[3] = {e0, e1, e2};
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int k = 0; k < 3; ++k)
                Sg[3 * i + k] = R[3 * i] * ev[0] * R[3 * k] + R[3 * i + 1] * ev[1] * R[3 * k + 1] + R[3 * i + 2] * ev[2] * R[3 * k + 2];
        double r2s = rho2 + oz * oz;
        double rho_s = sqrt(polar ? 1.0 : rho2);
        double scale = RFS_RAD2DEG / cell;
        double rc2 = rho2 < 1e-300 ? 1e-300 : rho2;
        double J[6] = {-oy / rc2 * scale, ox / rc2 * scale, 0.0,
                       -oz * ox / (rho_s * r2s) * scale, -oz * oy / (rho_s * r2s) * scale, rho_s / r2s * scale};
        double c2[4];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int l = 0; l < 2; ++l) {
                double acc = 0.0;
                for (int j = 0; j < 3; ++j)
                    for (int k = 0; k < 3; ++k) acc += J[3 * i + j] * Sg[3 * j + k] * J[3 * l + k];
                c2[2 * i + l] = acc;
            }
        double half_tr = 0.5 * (c2[0] + c2[3]);
        double det2 = c2[0] * c2[3] - c2[1] * c2[2];
        double dsc = half_tr * half_tr - det2;
        double lmax = half_tr + sqrt(dsc > 0.0 ? dsc : 0.0);
        double rpx = polar ? cover_all : 3.0 * sqrt(lmax > 0.0 ? lmax : 0.0);
        proj[6 * g + 0] = cu;
        proj[6 * g + 1] = cv;
        proj[6 * g + 2] = rpx;
        proj[6 * g + 3] = tr;
        proj[6 * g + 4] = depth;
        proj[6 * g + 5] = active ? 1.0 : 0.0;
    }
}

// ---- K2: exclusive scan of per-Gaussian splat counts (warp-shuffle scan) ----
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// block-wide exclusive scan of one value per thread; returns the block total
__device__ uint32_t block_excl_scan(uint32_t v, uint32_t& excl) {
    __shared__ uint32_t warp_tot[32];
    __shared__ uint32_t block_tot;
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t inc = warp_incl_scan(v);
    if (lane == 31) warp_tot[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int nw = blockDim.x >> 5;
        uint32_t t = lane < nw ? warp_tot[lane] : 0;
        uint32_t ti = warp_incl_scan(t);
        if (lane < nw) warp_tot[lane] = ti - t;
        if (lane == nw - 1) block_tot = ti;
    }
    __syncthreads();
    excl = warp_tot[wid] + inc - v;
    uint32_t total = block_tot;
    __syncthreads();
    return total;
}

// Single-pass exclusive scan (chained, decoupled look-back): blocks claim
// 4096-element tiles in order through an atomic counter, publish their
// aggregate, then look back over predecessors' published aggregates /
// inclusive prefixes (status word: 2 flag bits << 32 | value).
constexpr unsigned long long SC_AGG = 1ull << 32, SC_INC = 2ull << 32;
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_onepass(const uint32_t* __restrict__ in, int n,
                                                              uint32_t* __restrict__ out, uint32_t* __restrict__ total_out,
                                                              unsigned int* __restrict__ counter,
                                                              unsigned long long* __restrict__ status) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    __shared__ int tile_s;
    __shared__ uint32_t prefix_s;
    if (threadIdx.x == 0) tile_s = (int)atomicAdd(counter, 1u);
    __syncthreads();
    const int tile = tile_s;
    const long long base = (long long)tile * SCAN_TILE + (long long)threadIdx.x * SCAN_ITEMS;
    uint32_t v[SCAN_ITEMS];
    uint32_t sum = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        const long long j = base + i;
        v[i] = j < n ? in[j] : 0u;
        sum += v[i];
    }
    uint32_t ex;
    const uint32_t agg = block_excl_scan(sum, ex);
    if (threadIdx.x == 0) {
        volatile unsigned long long* st = status;
        uint32_t prefix = 0;
        if (tile == 0) {
            atomicExch(&status[0], SC_INC | agg);
        } else {
            atomicExch(&status[tile], SC_AGG | agg);
            for (int j = tile - 1; j >= 0; --j) {
                unsigned long long w;
                do {
                    w = st[j];
                } while ((w >> 32) == 0);
                prefix += (uint32_t)w;
                if ((w >> 32) == 2) break;
            }
            atomicExch(&status[tile], SC_INC | (unsigned long long)(prefix + agg));
        }
        prefix_s = prefix;
        if ((long long)(tile + 1) * SCAN_TILE >= n) *total_out = prefix + agg;
    }
    __syncthreads();
    ex += prefix_s;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        const long long j = base + i;
        if (j < n) out[j] = ex;
        ex += v[i];
    }
}

// K2b: fill (compact key, Gaussian id) pairs in expand_tile_rects order
// (_kernels.py:545-558): per splat, tv ascending, s1 tiles then s2 tiles.
// Compact key = tile << 31 | depth_code (the code's sign bit is always 0),
// so the radix sort needs 31 + ceil(log2 tiles) bits.
// Writes only positions < cap (the caller's capacity); the caller compares the
// scan total M with cap after the fact and redoes the binning if it overflowed.
__global__ void __launch_bounds__(256) k_fill(int n, const Rect* __restrict__ rects, const uint32_t* __restrict__ code,
                                              const uint32_t* __restrict__ offs, int tiles_u, uint32_t cap,
                                              uint64_t* __restrict__ ckeys, uint32_t* __restrict__ vals) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    Rect r = rects[g];
    if (r.tv_hi < r.tv_lo) return;
    uint32_t pos = offs[g];
    uint64_t c = code[g];
    for (int tv = r.tv_lo; tv <= r.tv_hi; ++tv) {
        int row = tv * tiles_u;
        for (int tu = r.s1_lo; tu <= r.s1_hi; ++tu) {
            if (pos >= cap) return;
            ckeys[pos] = ((uint64_t)(row + tu) << 31) | c;
            vals[pos] = (uint32_t)g;
            ++pos;
        }
        for (int tu = 0; tu <= r.s2_hi; ++tu) {
            if (pos >= cap) return;
            ckeys[pos] = ((uint64_t)(row + tu) << 31) | c;
            vals[pos] = (uint32_t)g;
            ++pos;
        }
    }
}

// K4: per-tile [start, end) = searchsorted left/right (splat.py:340-343)
// thread per sorted incidence i in [0, m]: where the tile id steps from
// prev to cur, i starts tiles prev+1..cur and ends tiles prev..cur-1
// (searchsorted left / right, splat.py:340-343); tiles with no incidence
// get an empty range at the right place.
// m_dev (nullable): the device-side count, clamped to m (then the capacity)
__global__ void k_ranges(const uint64_t* __restrict__ ckeys, int m, const uint32_t* __restrict__ m_dev, int n_tiles,
                         int2* __restrict__ ranges) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (m_dev) m = min(m, (int)*m_dev);
    if (i > m) return;
    const long long prev = i > 0 ? (long long)(ckeys[i - 1] >> 31) : -1;
    const long long cur = i < m ? (long long)(ckeys[i] >> 31) : (long long)n_tiles;
    for (long long t = prev + 1; t <= cur; ++t) {
        if (t < n_tiles) ranges[t].x = i;
        if (t >= 1) ranges[t - 1].y = i;
    }
}

// Restore reference keys (tile << 32 | code) for TileIndex.keys.
__global__ void k_expand_keys(const uint64_t* __restrict__ ckeys, int m, uint64_t* __restrict__ keys) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    uint64_t c = ckeys[i];
    keys[i] = ((c >> 31) << 32) | (c & 0x7fffffffull);
}

// K4b: emission bound lb[i] = min_{j >= i in tile} lbv[g_j] (reverse
// segmented min-scan, one block per tile).  Used by the exact streaming
// re-sort in K6: a pending hit with t_mid < lb[i] precedes every hit that
// candidates i.. can still produce.  Each warp owns a contiguous stretch of
// the tile list: it writes its stretch's suffix minima (32 at a time, from
// the end), then, once every stretch's minimum is known, folds in the minimum
// of the later stretches -- no block barrier inside the loops.
constexpr int LB_THREADS = 1024;
__global__ void __launch_bounds__(LB_THREADS) k_lower_bounds(const int2* __restrict__ ranges, const uint32_t* __restrict__ vals,
                                                              const RfsGeom* __restrict__ geom, double* __restrict__ lb) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    constexpr int NW = LB_THREADS / 32;
    __shared__ double smin[NW];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int2 rg = ranges[blockIdx.x];
    const int L = rg.y - rg.x;
    const int per = (L + NW - 1) / NW;
    const int s0 = rg.x + min(wid * per, L), s1 = rg.x + min(wid * per + per, L);
    double carry = INFINITY;
    for (int k0 = s1 - 32; k0 > s0 - 32; k0 -= 32) {
        const int i = k0 + lane;
        double v = i >= s0 ? geom[vals[i]].lbv : INFINITY;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_down_sync(0xffffffffu, v, o);
            if (lane + o < 32) v = fmin(v, y);
        }
        v = fmin(v, carry);
        if (i >= s0) lb[i] = v;
        carry = __shfl_sync(0xffffffffu, v, 0);
    }
    if (lane == 0) smin[wid] = carry;
    __syncthreads();
    double later = INFINITY;
    for (int w = wid + 1; w < NW; ++w) later = fmin(later, smin[w]);
    if (later == INFINITY) return;
    for (int i = s0 + lane; i < s1; i += 32) lb[i] = fmin(lb[i], later);
}

}  // namespace

// ------------------------------------------------------------------ C ABI
extern "C" {

int rfs_project(int n, const float* means, const float* quats, const float* log_scales, const float* trans_mag_raw,
                const float* trans_phase, const double* rx, double ress_radius, int n_az, int n_el,
                void* geom, void* sph, void* whit, uint32_t* depth_code, void* rects, uint32_t* counts, void* rho32,
                double* proj_out, int* err_flags, void* stream) {
    if (n < 0 || n_az < 1 || n_az > 360 || n_el < 1 || n_el > 180) return RFS_ERR_SHAPE;
    if (n == 0) return RFS_OK;
    int tiles_u = (n_az + RFS_TILE - 1) / RFS_TILE;
    cudaStream_t st = (cudaStream_t)stream;
    rfs_launch(k_project, rfs_ceil_div(n, 256), 256, 0, st, 
        n, means, quats, log_scales, trans_mag_raw, trans_phase, rx[0], rx[1], rx[2], ress_radius, n_az, n_el,
        tiles_u, (RfsGeom*)geom, (float4*)sph, (float4*)whit, depth_code, (Rect*)rects, counts, (float4*)rho32, proj_out, err_flags);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

// temp (u32 elements): a claim counter and one 64-bit status word per tile
size_t rfs_scan_temp_elems(int n) { return 2 + 2 * ((size_t)rfs_ceil_div(n > 0 ? n : 1, SCAN_TILE) + 1); }

int rfs_exclusive_scan_u32(const uint32_t* in, int n, uint32_t* out, uint32_t* total, uint32_t* temp, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) {
        RFS_CUDA_TRY(rfs_fill_u32(total, 0u, 1, st));
        return RFS_OK;
    }
    const int nb = rfs_ceil_div(n, SCAN_TILE);
    RFS_CUDA_TRY(rfs_fill_u32(temp, 0u, rfs_scan_temp_elems(n), st));
    rfs_launch(k_scan_onepass, nb, SCAN_THREADS, 0, st, in, n, out, total, (unsigned int*)temp,
                                                (unsigned long long*)(temp + 2));
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_bin_fill(int n, const void* rects, const uint32_t* depth_code, const uint32_t* offsets, int n_az, int cap,
                 uint64_t* ckeys, uint32_t* vals, void* stream) {
    if (n <= 0 || cap <= 0) return RFS_OK;
    int tiles_u = (n_az + RFS_TILE - 1) / RFS_TILE;
    rfs_launch(k_fill, rfs_ceil_div(n, 256), 256, 0, (cudaStream_t)stream, n, (const Rect*)rects, depth_code, offsets, tiles_u,
                                                                    (uint32_t)cap, ckeys, vals);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_tile_ranges(const uint64_t* ckeys, int m, const uint32_t* m_dev, int n_tiles, int* ranges, void* stream) {
    rfs_launch(k_ranges, rfs_ceil_div(m + 1, 256), 256, 0, (cudaStream_t)stream, ckeys, m, m_dev, n_tiles, (int2*)ranges);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_expand_keys(const uint64_t* ckeys, int m, uint64_t* keys, void* stream) {
    if (m <= 0) return RFS_OK;
    rfs_launch(k_expand_keys, rfs_ceil_div(m, 256), 256, 0, (cudaStream_t)stream, ckeys, m, keys);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_lower_bounds(const int* ranges, int n_tiles, const uint32_t* vals, const void* geom, double* lb, void* stream) {
    if (n_tiles <= 0) return RFS_OK;
    rfs_launch(k_lower_bounds, n_tiles, LB_THREADS, 0, (cudaStream_t)stream, (const int2*)ranges, vals, (const RfsGeom*)geom, lb);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // extern "C"
