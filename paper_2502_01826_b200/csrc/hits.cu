// hits.cu -- K6: per-ray live hit lists, shared by every transmitter of a batch.
//
// Restates _collect_hits (_kernels.py:27-112) + the live-hit walk of
// forward_tiled / count_hits_tiled (_kernels.py:176-191, 237-247): per ray,
// every candidate of the ray's tile is tested (disc prefilter, 3-sigma
// quadratic), hits are ordered by (t_mid, Gaussian id), and the cumulative
// complex transmittance T is carried until |T|^2 < 1e-12.  The hit set, the
// order and T do not depend on the transmitter, so this
// runs once per step and the TX batch composites from its output.
//
// Exact streaming re-sort: candidates arrive in tile-key
// (depth) order; a hit's t_mid is >= depth - r3 of its Gaussian, so a pending
// hit whose t_mid is below lb[i] = min_{j>=i} (depth_j - r3_j) precedes every
// hit the remaining candidates can produce and is emitted immediately.  The
// emitted sequence equals the reference's sorted list, so rays stop scanning
// as soon as they terminate.  Pending hits live in a per-thread ring buffer in
// shared memory; a ray that overflows it is redone by k_hits_slow with a
// global-memory buffer sized to its tile.
//
// Arithmetic: an fp32 bounding-sphere test rejects most candidates; survivors
// get the reference's fp64 disc prefilter and fp64 quadratic, so hit sets and
// orderings match the fp64 oracle.  T is carried in fp64.
#include "rfs_common.cuh"

namespace {

constexpr int HT_THREADS = 128;  // half a 16x16 tile: 8 u-columns x 16 v-rows
constexpr int HT_BATCH = 128;    // candidates staged per iteration
constexpr int HT_PCAP = 32;      // pending ring capacity per ray (power of 2)

struct RayState {
    double d[3];
    float d32[3];
    double tre, tim;
    int live;
    bool done;
};

// Exact hit test of candidate geometry G against a ray; returns true and
// (t_mid, w) on a hit.  Same expressions as _kernels.py:45-91.
__device__ __forceinline__ bool exact_hit(const RfsGeom* __restrict__ Gp, const double d[3], double u, double v,
                                          double n_az, double rx0, double rx1, double rx2, double min_t,
                                          double& t_mid, float& w_out) {
    double r2 = __ldg(&Gp->r2);
    if (r2 < 0.0) return false;
    double du = fabs(u - __ldg(&Gp->cu));
    if (n_az - du < du) du = n_az - du;
    double dv = v - __ldg(&Gp->cv);
    if (du * du + dv * dv > r2) return false;
    double mx = rx0 - __ldg(&Gp->mu[0]), my = rx1 - __ldg(&Gp->mu[1]), mz = rx2 - __ldg(&Gp->mu[2]);
    double i00 = __ldg(&Gp->inv[0]), i01 = __ldg(&Gp->inv[1]), i02 = __ldg(&Gp->inv[2]);
    double i11 = __ldg(&Gp->inv[3]), i12 = __ldg(&Gp->inv[4]), i22 = __ldg(&Gp->inv[5]);
    double dx = d[0], dy = d[1], dz = d[2];
    double sx = i00 * dx + i01 * dy + i02 * dz;
    double sy = i01 * dx + i11 * dy + i12 * dz;
    double sz = i02 * dx + i12 * dy + i22 * dz;
    double a = sx * dx + sy * dy + sz * dz;
    double b = sx * mx + sy * my + sz * mz;
    double c = (i00 * mx + i01 * my + i02 * mz) * mx + (i01 * mx + i11 * my + i12 * mz) * my +
               (i02 * mx + i12 * my + i22 * mz) * mz;
    double disc = b * b - a * (c - 9.0);
    if (disc < 0.0) return false;
    double sq = sqrt(disc);
    double d2 = (-b + sq) / a;
    if (d2 < min_t) return false;
    double d1 = (-b - sq) / a;
    double t_in = d1 < min_t ? min_t : d1;
    t_mid = 0.5 * (t_in + d2);
    double ex = t_mid * dx + mx, ey = t_mid * dy + my, ez = t_mid * dz + mz;
    double qf = (i00 * ex + i01 * ey + i02 * ez) * ex + (i01 * ex + i11 * ey + i12 * ez) * ey +
                (i02 * ex + i12 * ey + i22 * ez) * ez;
    w_out = (float)(__ldg(&Gp->norm) * exp(-0.5 * qf));
    return true;
}

__device__ __forceinline__ bool sphere_pass(float4 s, const float d[3]) {
    float cx = s.y * d[2] - s.z * d[1];
    float cy = s.z * d[0] - s.x * d[2];
    float cz = s.x * d[1] - s.y * d[0];
    return cx * cx + cy * cy + cz * cz <= s.w;
}

// Emit one hit in sorted order: terminate, record, advance T (_kernels.py:186-191).
__device__ __forceinline__ void emit_hit(RayState& st, uint32_t g, float w, const RfsGeom* __restrict__ geom,
                                         RfsHit* __restrict__ slab_ray, int hcap, bool& hcap_over) {
    if (st.tre * st.tre + st.tim * st.tim < RFS_TERM_EPS2) {
        st.done = true;
        return;
    }
    if (st.live < hcap) {
        RfsHit h;
        h.g = g;
        h.w = w;
        h.t_re = (float)st.tre;
        h.t_im = (float)st.tim;
        slab_ray[st.live] = h;
    } else {
        hcap_over = true;
    }
    st.live += 1;
    double rr = __ldg(&geom[g].rho_re), ri = __ldg(&geom[g].rho_im);
    double nr = st.tre * rr - st.tim * ri;
    double ni = st.tre * ri + st.tim * rr;
    st.tre = nr;
    st.tim = ni;
}

__device__ __forceinline__ void ray_dir(int u, int v, int n_az, double d[3]) {
    double cell = 360.0 / (double)n_az;
    double al = ((double)u + 0.5) * cell * (RFS_PI / 180.0);
    double be = (((double)v + 0.5) * cell - 90.0) * (RFS_PI / 180.0);
    double sa, ca, sb, cb;
    sincos(al, &sa, &ca);
    sincos(be, &sb, &cb);
    d[0] = cb * ca;
    d[1] = cb * sa;
    d[2] = sb;
}

struct HitsSmem {
    double pt[HT_PCAP][HT_THREADS];
    uint32_t pg[HT_PCAP][HT_THREADS];
    float pw[HT_PCAP][HT_THREADS];
    float4 sph[HT_BATCH];
    double lb[HT_BATCH];
    uint32_t g[HT_BATCH];
};

__global__ void __launch_bounds__(HT_THREADS) k_hits(
    const int2* __restrict__ ranges, const uint32_t* __restrict__ vals, const double* __restrict__ lb,
    const float4* __restrict__ sph, const RfsGeom* __restrict__ geom, double rx0, double rx1, double rx2,
    double min_t, int n_az, int n_el, int tiles_u, int hcap, RfsHit* __restrict__ slab, int* __restrict__ counts,
    int* __restrict__ slow_list, int* __restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    HitsSmem& S = *reinterpret_cast<HitsSmem*>(smem_raw);
    const int tile = blockIdx.x >> 1, half = blockIdx.x & 1;
    const int tid = threadIdx.x;
    const int u = (tile % tiles_u) * RFS_TILE + half * 8 + (tid >> 4);
    const int v = (tile / tiles_u) * RFS_TILE + (tid & 15);
    const bool valid = u < n_az && v < n_el;
    const int r = valid ? u * n_el + v : 0;
    RayState st;
    st.tre = 1.0;
    st.tim = 0.0;
    st.live = 0;
    st.done = !valid;
    ray_dir(valid ? u : 0, valid ? v : 0, n_az, st.d);
    st.d32[0] = (float)st.d[0];
    st.d32[1] = (float)st.d[1];
    st.d32[2] = (float)st.d[2];
    const double du_f = (double)u, dv_f = (double)v, naz = (double)n_az;
    RfsHit* slab_ray = slab + (size_t)r * hcap;
    bool hcap_over = false, pend_over = false;
    int head = 0, npend = 0;
    const int2 rg = ranges[tile];

    for (int base = rg.x; base < rg.y; base += HT_BATCH) {
        const int nb = min(HT_BATCH, rg.y - base);
        __syncthreads();
        for (int j = tid; j < nb; j += HT_THREADS) {
            uint32_t g = vals[base + j];
            S.g[j] = g;
            S.sph[j] = __ldg(&sph[g]);
            S.lb[j] = lb[base + j];
        }
        __syncthreads();
        if (!st.done) {
            for (int j = 0; j < nb; ++j) {
                const double lbj = S.lb[j];
                while (npend > 0) {
                    int hslot = head & (HT_PCAP - 1);
                    if (!(S.pt[hslot][tid] < lbj)) break;
                    emit_hit(st, S.pg[hslot][tid], S.pw[hslot][tid], geom, slab_ray, hcap, hcap_over);
                    ++head;
                    --npend;
                    if (st.done) break;
                }
                if (st.done) break;
                if (!sphere_pass(S.sph[j], st.d32)) continue;
                const uint32_t g = S.g[j];
                double t_mid;
                float w;
                if (!exact_hit(geom + g, st.d, du_f, dv_f, naz, rx0, rx1, rx2, min_t, t_mid, w)) continue;
                if (npend == HT_PCAP) {
                    pend_over = true;
                    st.done = true;
                    break;
                }
                // sorted insertion by (t_mid, g) into the ring
                int k = npend;
                while (k > 0) {
                    int ps = (head + k - 1) & (HT_PCAP - 1);
                    double pt = S.pt[ps][tid];
                    if (pt > t_mid || (pt == t_mid && S.pg[ps][tid] > g)) {
                        int qs = (head + k) & (HT_PCAP - 1);
                        S.pt[qs][tid] = pt;
                        S.pg[qs][tid] = S.pg[ps][tid];
                        S.pw[qs][tid] = S.pw[ps][tid];
                        --k;
                    } else {
                        break;
                    }
                }
                int qs = (head + k) & (HT_PCAP - 1);
                S.pt[qs][tid] = t_mid;
                S.pg[qs][tid] = g;
                S.pw[qs][tid] = w;
                ++npend;
            }
        }
        if (__syncthreads_and(st.done)) break;
    }
    // drain: every candidate seen, pending hits are final
    while (!st.done && npend > 0) {
        int hslot = head & (HT_PCAP - 1);
        emit_hit(st, S.pg[hslot][tid], S.pw[hslot][tid], geom, slab_ray, hcap, hcap_over);
        ++head;
        --npend;
    }
    if (!valid) return;
    if (pend_over) {
        int idx = atomicAdd(&stats[0], 1);
        slow_list[idx] = r;
        return;
    }
    counts[r] = st.live;
    if (hcap_over) atomicAdd(&stats[1], 1);
    atomicMax(&stats[2], st.live);
    atomicAdd(&stats[3], st.live);
}

// Slow path for rays whose pending buffer overflowed: one thread per ray,
// pending list in global scratch of capacity `pcap` (>= the largest tile
// list, so it cannot overflow).  Same emission rule and arithmetic.
__global__ void k_hits_slow(const int* __restrict__ rays, int n_rays, const int2* __restrict__ ranges,
                            const uint32_t* __restrict__ vals, const double* __restrict__ lb,
                            const float4* __restrict__ sph, const RfsGeom* __restrict__ geom, double rx0, double rx1,
                            double rx2, double min_t, int n_az, int n_el, int tiles_u, int hcap,
                            RfsHit* __restrict__ slab, int* __restrict__ counts, double* __restrict__ pt,
                            uint32_t* __restrict__ pg, float* __restrict__ pw, int pcap, int* __restrict__ stats) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rays) return;
    const int r = rays[i];
    const int u = r / n_el, v = r % n_el;
    const int tile = (v / RFS_TILE) * tiles_u + (u / RFS_TILE);
    RayState st;
    st.tre = 1.0;
    st.tim = 0.0;
    st.live = 0;
    st.done = false;
    ray_dir(u, v, n_az, st.d);
    st.d32[0] = (float)st.d[0];
    st.d32[1] = (float)st.d[1];
    st.d32[2] = (float)st.d[2];
    RfsHit* slab_ray = slab + (size_t)r * hcap;
    double* my_t = pt + (size_t)i * pcap;
    uint32_t* my_g = pg + (size_t)i * pcap;
    float* my_w = pw + (size_t)i * pcap;
    bool hcap_over = false;
    int head = 0, npend = 0;
    const int2 rg = ranges[tile];
    for (int j = rg.x; j < rg.y && !st.done; ++j) {
        const double lbj = lb[j];
        while (npend > 0 && my_t[head] < lbj) {
            emit_hit(st, my_g[head], my_w[head], geom, slab_ray, hcap, hcap_over);
            ++head;
            --npend;
            if (st.done) break;
        }
        if (st.done) break;
        const uint32_t g = vals[j];
        if (!sphere_pass(__ldg(&sph[g]), st.d32)) continue;
        double t_mid;
        float w;
        if (!exact_hit(geom + g, st.d, (double)u, (double)v, (double)n_az, rx0, rx1, rx2, min_t, t_mid, w)) continue;
        // linear layout [head, head + npend); compact when the tail hits pcap
        if (head + npend == pcap) {
            for (int k = 0; k < npend; ++k) {
                my_t[k] = my_t[head + k];
                my_g[k] = my_g[head + k];
                my_w[k] = my_w[head + k];
            }
            head = 0;
        }
        int k = head + npend;
        while (k > head && (my_t[k - 1] > t_mid || (my_t[k - 1] == t_mid && my_g[k - 1] > g))) {
            my_t[k] = my_t[k - 1];
            my_g[k] = my_g[k - 1];
            my_w[k] = my_w[k - 1];
            --k;
        }
        my_t[k] = t_mid;
        my_g[k] = g;
        my_w[k] = w;
        ++npend;
    }
    while (!st.done && npend > 0) {
        emit_hit(st, my_g[head], my_w[head], geom, slab_ray, hcap, hcap_over);
        ++head;
        --npend;
    }
    counts[r] = st.live;
    if (hcap_over) atomicAdd(&stats[1], 1);
    atomicMax(&stats[2], st.live);
    atomicAdd(&stats[3], st.live);
}

__global__ void k_max_range(const int2* __restrict__ ranges, int n_tiles, int* __restrict__ out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_tiles) atomicMax(out, ranges[t].y - ranges[t].x);
}

}  // namespace

extern "C" {

// stats: [0] rays sent to the slow path, [1] rays whose live count exceeded
// hcap, [2] max live count, [3] total live hits, [4] largest tile list.
int rfs_hits(const int* ranges, int n_tiles, const uint32_t* vals, const double* lb, const void* sph, const void* geom,
             const double* rx, double ress_radius, int n_az, int n_el, int hcap, void* slab, int* counts,
             int* slow_list, int* stats, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    int tiles_u = (n_az + RFS_TILE - 1) / RFS_TILE;
    static bool attr = false;
    size_t smem = sizeof(HitsSmem);
    if (!attr) {
        RFS_CUDA_TRY(cudaFuncSetAttribute(k_hits, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    RFS_CUDA_TRY(cudaMemsetAsync(stats, 0, 8 * sizeof(int), st));
    RFS_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int) * (size_t)n_az * n_el, st));
    if (n_tiles <= 0) return RFS_OK;
    k_hits<<<n_tiles * 2, HT_THREADS, smem, st>>>((const int2*)ranges, vals, lb, (const float4*)sph,
                                                   (const RfsGeom*)geom, rx[0], rx[1], rx[2], ress_radius, n_az, n_el,
                                                   tiles_u, hcap, (RfsHit*)slab, counts, slow_list, stats);
    k_max_range<<<rfs_ceil_div(n_tiles, 256), 256, 0, st>>>((const int2*)ranges, n_tiles, stats + 4);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_hits_slow(const int* rays, int n_rays, const int* ranges, const uint32_t* vals, const double* lb,
                  const void* sph, const void* geom, const double* rx, double ress_radius, int n_az, int n_el,
                  int hcap, void* slab, int* counts, double* pend_t, uint32_t* pend_g, float* pend_w, int pcap,
                  int* stats, void* stream) {
    if (n_rays <= 0) return RFS_OK;
    int tiles_u = (n_az + RFS_TILE - 1) / RFS_TILE;
    k_hits_slow<<<rfs_ceil_div(n_rays, 64), 64, 0, (cudaStream_t)stream>>>(
        rays, n_rays, (const int2*)ranges, vals, lb, (const float4*)sph, (const RfsGeom*)geom, rx[0], rx[1], rx[2],
        ress_radius, n_az, n_el, tiles_u, hcap, (RfsHit*)slab, counts, pend_t, pend_g, pend_w, pcap, stats);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // extern "C"
