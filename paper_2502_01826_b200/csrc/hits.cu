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
// Exact streaming re-sort: one thread per ray walks its
// tile's depth-ordered candidate list; a
// hit's chord midpoint lies in the Gaussian's 3-sigma ball, so
// t_mid >= depth - r3, and a pending hit whose t_mid is below
// lb[i] = min_{j>=i} (depth_j - r3_j) precedes every hit the remaining
// candidates can produce: it is final and is emitted, and a ray stops
// scanning as soon as it terminates.  Pending (t_mid, g, w) entries live in a
// per-thread ring in shared memory; a full ring keeps the PCAP smallest and
// remembers the smallest hit it dropped -- a ray that terminates before that
// hit is due is exact as is, one that would need it is redone by k_hits_slow
// with a global buffer sized to its tile (exact, rarely taken).
//   Per warp (a 4 x 8 ray patch), chunks of CH candidates: stage the fp32
//   filter data in warp-private shared memory and have the bulk-copy engine
//   bring the fp64 records of the cone-relevant ones (cp.async.bulk, one per
//   record, completion counted on a warp mbarrier); every lane tests the
//   chunk against its ray;
//   survivors run the fp64 test and are inserted in (t_mid, g) order; pending
//   hits below the next chunk's bound are emitted.
//
// Arithmetic: the fp32 tests carry proven margins (project.cu) so they never
// reject an fp64 hit; the fp64 test follows the reference's operation order
// with no FMA contraction (explicit __d*_rn), so exact ties order like the
// reference; T *= rho is the reference's complex product without contraction.
// Ray directions come from a table built with the reference's formula
// (render.py:103-117).
#include "rfs_common.cuh"

namespace {

constexpr double DINF = 1.0e300;

#define DM(a, b) __dmul_rn((a), (b))
#define DA(a, b) __dadd_rn((a), (b))
#define DS(a, b) __dsub_rn((a), (b))

// Reference quadratic + midpoint density (_kernels.py:45-91): true, t_mid, w on a hit.
__device__ __forceinline__ bool exact_hit(const RfsGeom* __restrict__ G, double dx, double dy, double dz, double u,
                                          double v, double n_az, double rx0, double rx1, double rx2, double min_t,
                                          double& t_mid, float& w_out) {
    double r2 = __ldg(&G->r2);
    if (r2 < 0.0) return false;
    double du = fabs(DS(u, __ldg(&G->cu)));
    if (DS(n_az, du) < du) du = DS(n_az, du);
    double dv = DS(v, __ldg(&G->cv));
    if (DA(DM(du, du), DM(dv, dv)) > r2) return false;
    double mx = DS(rx0, __ldg(&G->mu[0])), my = DS(rx1, __ldg(&G->mu[1])), mz = DS(rx2, __ldg(&G->mu[2]));
    double i00 = __ldg(&G->inv[0]), i01 = __ldg(&G->inv[1]), i02 = __ldg(&G->inv[2]);
    double i11 = __ldg(&G->inv[3]), i12 = __ldg(&G->inv[4]), i22 = __ldg(&G->inv[5]);
    double sx = DA(DA(DM(i00, dx), DM(i01, dy)), DM(i02, dz));
    double sy = DA(DA(DM(i01, dx), DM(i11, dy)), DM(i12, dz));
    double sz = DA(DA(DM(i02, dx), DM(i12, dy)), DM(i22, dz));
    double a = DA(DA(DM(sx, dx), DM(sy, dy)), DM(sz, dz));
    double b = DA(DA(DM(sx, mx), DM(sy, my)), DM(sz, mz));
    double c = DA(DA(DM(DA(DA(DM(i00, mx), DM(i01, my)), DM(i02, mz)), mx),
                     DM(DA(DA(DM(i01, mx), DM(i11, my)), DM(i12, mz)), my)),
                  DM(DA(DA(DM(i02, mx), DM(i12, my)), DM(i22, mz)), mz));
    double disc = DS(DM(b, b), DM(a, DS(c, 9.0)));
    if (disc < 0.0) return false;
    double sq = __dsqrt_rn(disc);
    double d2 = __ddiv_rn(DA(-b, sq), a);
    if (d2 < min_t) return false;
    double d1 = __ddiv_rn(DS(-b, sq), a);
    double t_in = d1 < min_t ? min_t : d1;
    t_mid = DM(0.5, DA(t_in, d2));
    double ex = DA(DM(t_mid, dx), mx), ey = DA(DM(t_mid, dy), my), ez = DA(DM(t_mid, dz), mz);
    double qf = DA(DA(DM(DA(DA(DM(i00, ex), DM(i01, ey)), DM(i02, ez)), ex),
                      DM(DA(DA(DM(i01, ex), DM(i11, ey)), DM(i12, ez)), ey)),
                   DM(DA(DA(DM(i02, ex), DM(i12, ey)), DM(i22, ez)), ez));
    // same arithmetic as exact_hit_s (fp32 exp of the fp64 exponent), so the
    // slow path and the ring path produce bitwise identical hit lists
    w_out = (float)__ldg(&G->norm) * expf((float)DM(-0.5, qf));
    return true;
}

__device__ __forceinline__ bool sphere_pass(float4 s, float d0, float d1, float d2) {
    float cx = s.y * d2 - s.z * d1;
    float cy = s.z * d0 - s.x * d2;
    float cz = s.x * d1 - s.y * d0;
    return cx * cx + cy * cy + cz * cz <= s.w;
}

// L rows: (a.x a.y a.z) (a.w b.x b.y) (b.z b.w c.x); p = (c.y c.z c.w); threshold e.x
__device__ __forceinline__ bool whitened_pass(float4 a, float4 b, float4 c, float thr, float d0, float d1, float d2) {
    float q0 = a.x * d0 + a.y * d1 + a.z * d2;
    float q1 = a.w * d0 + b.x * d1 + b.y * d2;
    float q2 = b.z * d0 + b.w * d1 + c.x * d2;
    float x0 = q1 * c.w - q2 * c.z;
    float x1 = q2 * c.y - q0 * c.w;
    float x2 = q0 * c.z - q1 * c.y;
    return x0 * x0 + x1 * x1 + x2 * x2 <= thr * (q0 * q0 + q1 * q1 + q2 * q2);
}

struct Ray {
    double dx, dy, dz;
    float fx, fy, fz;
    double tre, tim;
    int live;
    bool done;
    bool hcap_over;
};

// T *= rho (_kernels.py:191), complex128 product without contraction
__device__ __forceinline__ void advance_t(double& tre, double& tim, double rr, double ri) {
    const double nr = DS(DM(tre, rr), DM(tim, ri));
    const double ni = DA(DM(tre, ri), DM(tim, rr));
    tre = nr;
    tim = ni;
}

__device__ __forceinline__ bool terminated(double tre, double tim) {
    return DA(DM(tre, tre), DM(tim, tim)) < RFS_TERM_EPS2;  // _kernels.py:186-187
}

// Emit one hit in sorted order: terminate, record, advance T (_kernels.py:186-191).
__device__ __forceinline__ void emit_hit(Ray& st, uint32_t g, float w, const RfsGeom* __restrict__ geom,
                                         RfsHit* __restrict__ slab_ray, int hcap, uint32_t* __restrict__ used,
                                         int* __restrict__ stats) {
    if (terminated(st.tre, st.tim)) {
        st.done = true;
        return;
    }
    if (used) used[g] = 1u;  // Gaussian has a live hit: its psi row is needed (counted by k_count_used)
    if (st.live < hcap) {
        RfsHit h;
        h.g = g;
        h.w = w;
        h.t_re = (float)st.tre;
        h.t_im = (float)st.tim;
        slab_ray[st.live] = h;
    } else {
        st.hcap_over = true;
    }
    st.live += 1;
    const RfsGeom* G = geom + g;
    advance_t(st.tre, st.tim, __ldg(&G->rho_re), __ldg(&G->rho_im));
}

// Reference quadratic on a shared-memory copy of the first 13 doubles of an
// RfsGeom record (mu[3], inv[6], norm, cu, cv, r2); same arithmetic as exact_hit.
__device__ __forceinline__ bool exact_hit_s(const double* __restrict__ G, double dx, double dy, double dz, double u,
                                            double v, double n_az, double rx0, double rx1, double rx2, double min_t,
                                            double& t_mid, float& w_out) {
    double r2 = G[12];
    if (r2 < 0.0) return false;
    double du = fabs(DS(u, G[10]));
    if (DS(n_az, du) < du) du = DS(n_az, du);
    double dv = DS(v, G[11]);
    if (DA(DM(du, du), DM(dv, dv)) > r2) return false;
    double mx = DS(rx0, G[0]), my = DS(rx1, G[1]), mz = DS(rx2, G[2]);
    double i00 = G[3], i01 = G[4], i02 = G[5], i11 = G[6], i12 = G[7], i22 = G[8];
    double sx = DA(DA(DM(i00, dx), DM(i01, dy)), DM(i02, dz));
    double sy = DA(DA(DM(i01, dx), DM(i11, dy)), DM(i12, dz));
    double sz = DA(DA(DM(i02, dx), DM(i12, dy)), DM(i22, dz));
    double a = DA(DA(DM(sx, dx), DM(sy, dy)), DM(sz, dz));
    double b = DA(DA(DM(sx, mx), DM(sy, my)), DM(sz, mz));
    double c = DA(DA(DM(DA(DA(DM(i00, mx), DM(i01, my)), DM(i02, mz)), mx),
                     DM(DA(DA(DM(i01, mx), DM(i11, my)), DM(i12, mz)), my)),
                  DM(DA(DA(DM(i02, mx), DM(i12, my)), DM(i22, mz)), mz));
    double disc = DS(DM(b, b), DM(a, DS(c, 9.0)));
    if (disc < 0.0) return false;
    double sq = __dsqrt_rn(disc);
    double d2 = __ddiv_rn(DA(-b, sq), a);
    if (d2 < min_t) return false;
    double d1 = __ddiv_rn(DS(-b, sq), a);
    double t_in = d1 < min_t ? min_t : d1;
    t_mid = DM(0.5, DA(t_in, d2));
    double ex = DA(DM(t_mid, dx), mx), ey = DA(DM(t_mid, dy), my), ez = DA(DM(t_mid, dz), mz);
    double qf = DA(DA(DM(DA(DA(DM(i00, ex), DM(i01, ey)), DM(i02, ez)), ex),
                      DM(DA(DA(DM(i01, ex), DM(i11, ey)), DM(i12, ez)), ey)),
                   DM(DA(DA(DM(i02, ex), DM(i12, ey)), DM(i22, ez)), ez));
    // w is stored in fp32: an fp32 exp of the fp64 exponent is within ~2 ulp
    w_out = (float)G[9] * expf((float)DM(-0.5, qf));
    return true;
}

constexpr int GD = 13;   // doubles of an RfsGeom record used by the exact test
constexpr int GDS = 14;  // their shared-memory row (112 B: one bulk copy of the record head)


template <int CH>
struct WarpStage {
    float4 sph[CH];
    float4 wh[CH][4];
    uint32_t g[CH];
    double gd[CH][GDS];  // fp64 records of the chunk's cone-relevant candidates (by slot)
    uint64_t bar;        // completion of the chunk's record copies (bulk-copy engine)
};

template <int PCAP, int NT, int CH>
struct HitsSmem {
    double pt[PCAP][NT];
    uint32_t pg[PCAP][NT];
    float pw[PCAP][NT];
    WarpStage<CH> ws[NT / 32];
};

// Streaming K6 (dense scenes): see the file comment.  EVICT: a full ring keeps
// its PCAP smallest hits (else the ray goes to the slow path at once) --
// switched on by the host once a scene sends many rays to the slow path.
template <int PCAP, int NT, int CH, bool EVICT>
__global__ void __launch_bounds__(NT) k_hits(
    const int2* __restrict__ ranges, const uint32_t* __restrict__ vals, const double* __restrict__ lb,
    const float4* __restrict__ sph, const float4* __restrict__ whit, const RfsGeom* __restrict__ geom,
    const double* __restrict__ dirs, double rx0, double rx1, double rx2, double min_t, int n_az, int n_el,
    int tiles_u, int hcap, RfsHit* __restrict__ slab, int* __restrict__ counts, int* __restrict__ slow_list,
    int* __restrict__ stats, uint32_t* __restrict__ used, int tile_lo) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    extern __shared__ __align__(16) unsigned char smem_raw[];
    HitsSmem<PCAP, NT, CH>& S = *reinterpret_cast<HitsSmem<PCAP, NT, CH>*>(smem_raw);
    constexpr int PARTS = 256 / NT;
    const int tile = tile_lo + (int)blockIdx.x / PARTS, part = blockIdx.x % PARTS;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // each warp owns a 4 (u) x 8 (v) patch of the 16 x 16 tile
    const int q = part * (NT / 32) + wid, pu = q >> 1, pv = q & 1;
    const int u = (tile % tiles_u) * RFS_TILE + 4 * pu + (lane >> 3);
    const int v = (tile / tiles_u) * RFS_TILE + 8 * pv + (lane & 7);
    const bool valid = u < n_az && v < n_el;
    const int r = valid ? u * n_el + v : 0;
    Ray st;
    st.dx = dirs[3 * r];
    st.dy = dirs[3 * r + 1];
    st.dz = dirs[3 * r + 2];
    st.fx = (float)st.dx;
    st.fy = (float)st.dy;
    st.fz = (float)st.dz;
    st.tre = 1.0;
    st.tim = 0.0;
    st.live = 0;
    st.done = !valid;
    st.hcap_over = false;
    const double uf = (double)u, vf = (double)v, naz = (double)n_az;
    RfsHit* slab_ray = slab + (size_t)r * hcap;
    bool pend_over = false;
    int head = 0, npend = 0, max_pend = 0;
    int n_sph = 0, n_wh = 0;
    double head_t = DINF;
    // a full ring keeps the PCAP smallest (t_mid, g) pending hits: the evicted
    // or refused ones are represented by their minimum (ev_t, ev_g); the ray
    // only fails (-> slow path) if it would have to emit that hit
    double ev_t = DINF;
    uint32_t ev_g = 0xffffffffu;
    const int2 rg = ranges[tile];
    const int c_lo = rg.x, c_hi = rg.y;
    WarpStage<CH>& W = S.ws[wid];
    if (lane == 0) rfs_mbar_init(&W.bar, 1);
    __syncwarp();
    unsigned bar_phase = 0;

    // Warp cone: axis c through the patch, half-angle th_p covering its rays.
    // A ray can only hit a Gaussian whose bounding-sphere cone (axis mu - rx,
    // half-angle th_g = asin(r3/depth)) contains it, so a candidate is
    // relevant to the warp only if angle(c, mu - rx) <= th_p + th_g.
    float4 ca;
    float2 cb;
    rfs_patch_cone(tile, q, tiles_u, n_az, n_el, dirs, ca, cb);

    // register prefetch of the next chunk's filter data (lane j loads candidate base + j)
    uint32_t pf_g = 0;
    float4 pf_s = make_float4(0.f, 0.f, 0.f, 0.f), pf_w[4];
    double pf_lb = DINF;
    // candidate ids run one chunk further ahead than their records, so the
    // record gathers never wait on the id load (in-order issue)
    uint32_t nx_g = c_lo + lane < c_hi ? vals[c_lo + lane] : 0u;
    auto prefetch = [&](int b0) {
        if (b0 + lane < c_hi) {
            pf_g = nx_g;
            pf_s = __ldg(&sph[pf_g]);
#pragma unroll
            for (int k = 0; k < 4; ++k) pf_w[k] = __ldg(&whit[4 * pf_g + k]);
        }
        if (b0 + CH + lane < c_hi) nx_g = vals[b0 + CH + lane];
        const int nxt = min(b0 + CH, c_hi);  // bound of every candidate after this chunk
        pf_lb = nxt < c_hi ? lb[nxt] : DINF;
    };
    prefetch(c_lo);
    // emit every pending hit below `bound` (in (t_mid, g) order)
    auto emit_until = [&](double bound) {
        while (!st.done && head_t < bound) {
            emit_hit(st, S.pg[head][tid], S.pw[head][tid], geom, slab_ray, hcap, used, stats);
            head = (head + 1) & (PCAP - 1);
            --npend;
            head_t = npend > 0 ? S.pt[head][tid] : DINF;
        }
        if constexpr (EVICT) {
            if (!st.done && ev_t < bound) {  // a dropped hit is due: redo the ray on the slow path
                pend_over = true;
                st.done = true;
            }
        }
    };

    for (int base = c_lo; base < c_hi; base += CH) {
        if (__all_sync(0xffffffffu, st.done)) break;
        const int nb = min(CH, c_hi - base);
        // 1. stage the prefetched chunk, cone-cull it for the warp, start loading the next one
        bool rel = false;
        if (lane < nb) {
            W.g[lane] = pf_g;
            W.sph[lane] = pf_s;
#pragma unroll
            for (int k = 0; k < 4; ++k) W.wh[lane][k] = pf_w[k];
            rel = rfs_cone_relevant(ca, cb, pf_s, pf_w[3]);
        }
        const unsigned relmask = __ballot_sync(0xffffffffu, rel);
        const double lb_next = pf_lb;
        __syncwarp();
        // fp64 records of the cone-relevant candidates -> shared memory by the
        // bulk-copy engine (lane j requests its own candidate's 112 bytes):
        // they land while the fp32 filters run
        if (relmask) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after the last chunk's reads
            if (lane == 0) rfs_mbar_arrive_expect_tx(&W.bar, (unsigned)__popc(relmask) * (GDS * 8u));
            if (rel) rfs_bulk_g2s(W.gd[lane], geom + pf_g, GDS * 8u, &W.bar);
        }
        if (base + CH < c_hi) prefetch(base + CH);
        // 2. survivor mask from shared memory
        unsigned mask = 0;
        if (!st.done) {
            unsigned rm = relmask;
            while (rm) {
                const int j = __ffs(rm) - 1;
                rm &= rm - 1;
                if (sphere_pass(W.sph[j], st.fx, st.fy, st.fz)) {
                    ++n_sph;
                    if (whitened_pass(W.wh[j][0], W.wh[j][1], W.wh[j][2], W.wh[j][3].x, st.fx, st.fy, st.fz)) {
                        mask |= 1u << j;
                        ++n_wh;
                    }
                }
            }
        }
        // 3a. the records' copies have landed
        if (relmask) {
            rfs_mbar_wait(&W.bar, bar_phase);
            bar_phase ^= 1u;
        }
        if (!st.done) {
            // 3b. exact fp64 test and sorted insertion by (t_mid, g)
            while (mask) {
                const int j = __ffs(mask) - 1;
                mask &= mask - 1;
                const uint32_t g = W.g[j];
                double t_mid;
                float w;
                if (!exact_hit_s(W.gd[j], st.dx, st.dy, st.dz, uf, vf, naz, rx0, rx1, rx2, min_t, t_mid, w)) continue;
                if constexpr (EVICT) {
                    if (ev_t < t_mid || (ev_t == t_mid && ev_g < g)) continue;  // after a dropped hit: dropped too
                    if (npend == PCAP) {  // full: keep the PCAP smallest, remember the smallest dropped
                        const int tl = (head + PCAP - 1) & (PCAP - 1);
                        const double tt = S.pt[tl][tid];
                        const uint32_t tg = S.pg[tl][tid];
                        if (tt > t_mid || (tt == t_mid && tg > g)) {
                            ev_t = tt;  // the tail is the largest pending entry, and below every earlier drop
                            ev_g = tg;
                            --npend;
                        } else {
                            ev_t = t_mid;
                            ev_g = g;
                            continue;
                        }
                    }
                } else if (npend == PCAP) {
                    pend_over = true;
                    st.done = true;
                    break;
                }
                int k = npend;
                int ps = (head + k - 1) & (PCAP - 1);
                while (k > 0) {
                    const double pt = S.pt[ps][tid];
                    if (!(pt > t_mid || (pt == t_mid && S.pg[ps][tid] > g))) break;
                    const int qs = (ps + 1) & (PCAP - 1);
                    S.pt[qs][tid] = pt;
                    S.pg[qs][tid] = S.pg[ps][tid];
                    S.pw[qs][tid] = S.pw[ps][tid];
                    --k;
                    ps = (ps - 1) & (PCAP - 1);
                }
                // emit_hit reads rho from the record later: bring its line into L1 now
                asm volatile("prefetch.global.L1 [%0];" ::"l"(&geom[g].rho_re));
                const int qs = (ps + 1) & (PCAP - 1);
                S.pt[qs][tid] = t_mid;
                S.pg[qs][tid] = g;
                S.pw[qs][tid] = w;
                ++npend;
                max_pend = max(max_pend, npend);
                head_t = fmin(head_t, t_mid);
            }
            // 4. emit every pending hit that precedes all later candidates
            emit_until(lb_next);
        }
        __syncwarp();
    }
    // drain (also covers rays whose tile list ended with pending hits)
    while (!st.done && npend > 0) {
        emit_hit(st, S.pg[head][tid], S.pw[head][tid], geom, slab_ray, hcap, used, stats);
        head = (head + 1) & (PCAP - 1);
        --npend;
    }
    if constexpr (EVICT) {
        if (!st.done && ev_t < DINF) pend_over = true;  // it needed a dropped hit
    }
    if (!valid) return;
    atomicMax(&stats[5], max_pend);
    atomicAdd(&stats[6], n_sph);
    atomicAdd(&stats[7], n_wh);
    if (pend_over) {  // the slow path redoes the whole ray
        const int idx = atomicAdd(&stats[0], 1);
        slow_list[idx] = r;
        return;
    }
    counts[r] = min(st.live, hcap);  // stored hits; live > hcap is flagged in stats[1]
    if (st.hcap_over) atomicAdd(&stats[1], 1);
    atomicMax(&stats[2], st.live);
    atomicAdd(&stats[3], min(st.live, hcap));
}

// Slow path for rays whose pending ring overflowed: one thread per ray,
// pending list in global scratch of capacity `pcap` (>= the largest tile
// list, so it cannot overflow).  Same emission rule and arithmetic.
__global__ void k_hits_slow(const int* __restrict__ rays, int n_rays, const int2* __restrict__ ranges,
                            const uint32_t* __restrict__ vals, const double* __restrict__ lb,
                            const float4* __restrict__ sph, const float4* __restrict__ whit,
                            const RfsGeom* __restrict__ geom, const double* __restrict__ dirs, double rx0, double rx1,
                            double rx2, double min_t, int n_az, int n_el, int tiles_u, int hcap,
                            RfsHit* __restrict__ slab, int* __restrict__ counts, double* __restrict__ pt,
                            uint32_t* __restrict__ pg, float* __restrict__ pw, int pcap, int* __restrict__ stats,
                            uint32_t* __restrict__ used) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_rays) return;
    const int r = rays[i];
    const int u = r / n_el, v = r % n_el;
    const int tile = (v / RFS_TILE) * tiles_u + (u / RFS_TILE);
    Ray st;
    st.dx = dirs[3 * r];
    st.dy = dirs[3 * r + 1];
    st.dz = dirs[3 * r + 2];
    st.fx = (float)st.dx;
    st.fy = (float)st.dy;
    st.fz = (float)st.dz;
    st.tre = 1.0;
    st.tim = 0.0;
    st.live = 0;
    st.done = false;
    st.hcap_over = false;
    RfsHit* slab_ray = slab + (size_t)r * hcap;
    double* my_t = pt + (size_t)i * pcap;
    uint32_t* my_g = pg + (size_t)i * pcap;
    float* my_w = pw + (size_t)i * pcap;
    int head = 0, npend = 0;
    const int2 rg = ranges[tile];
    for (int j = rg.x; j < rg.y && !st.done; ++j) {
        const double lbj = lb[j];
        while (npend > 0 && my_t[head] < lbj) {
            emit_hit(st, my_g[head], my_w[head], geom, slab_ray, hcap, used, stats);
            ++head;
            --npend;
            if (st.done) break;
        }
        if (st.done) break;
        const uint32_t g = vals[j];
        if (!sphere_pass(__ldg(&sph[g]), st.fx, st.fy, st.fz)) continue;
        if (!whitened_pass(__ldg(&whit[4 * g]), __ldg(&whit[4 * g + 1]), __ldg(&whit[4 * g + 2]),
                           __ldg(&whit[4 * g + 3]).x, st.fx, st.fy, st.fz))
            continue;
        double t_mid;
        float w;
        if (!exact_hit(geom + g, st.dx, st.dy, st.dz, (double)u, (double)v, (double)n_az, rx0, rx1, rx2, min_t,
                       t_mid, w))
            continue;
        // linear layout [head, head + npend): total inserts <= tile length <= pcap
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
        emit_hit(st, my_g[head], my_w[head], geom, slab_ray, hcap, used, stats);
        ++head;
        --npend;
    }
    counts[r] = min(st.live, hcap);  // stored hits; live > hcap is flagged in stats[1]
    if (st.hcap_over) atomicAdd(&stats[1], 1);
    atomicMax(&stats[2], st.live);
    atomicAdd(&stats[3], min(st.live, hcap));
}

// stats[8] = number of Gaussians with a live hit (the by-Gaussian index sizes
// its compact keys from it); stats[8] is zeroed by the caller
__global__ void __launch_bounds__(256) k_count_used(const uint32_t* __restrict__ used, int n, int* __restrict__ stats) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    int c = 0;
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x) c += used[g] != 0u;
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&stats[8], c);
}

__global__ void k_max_range(const int2* __restrict__ ranges, int n_tiles, int* __restrict__ out) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_tiles) atomicMax(out, ranges[t].y - ranges[t].x);
}

// Ray directions through cell centres, render.py:103-117, same operation
// order as numpy (deg2rad(x) = x * (pi/180)); used only when the host does
// not supply the table.
__global__ void k_ray_dirs(int n_az, int n_el, double* __restrict__ dirs) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_az * n_el) return;
    int u = r / n_el, v = r % n_el;
    double cell = 360.0 / (double)n_az;
    double al = DM(DM(DA((double)u, 0.5), cell), RFS_PI / 180.0);
    double be = DM(DS(DM(DA((double)v, 0.5), cell), 90.0), RFS_PI / 180.0);
    dirs[3 * r] = DM(cos(be), cos(al));
    dirs[3 * r + 1] = DM(cos(be), sin(al));
    dirs[3 * r + 2] = sin(be);
}

template <int PCAP, int NT, int CH, bool EVICT>
int launch_hits(int tile_lo, int tile_hi, const int* ranges, const uint32_t* vals, const double* lb, const void* sph,
                const void* whit, const void* geom, const double* dirs, const double* rx, double min_t, int n_az,
                int n_el, int tiles_u, int hcap, void* slab, int* counts, int* slow_list, int* stats, uint32_t* used,
                cudaStream_t st) {
    static bool attr = false;
    size_t smem = sizeof(HitsSmem<PCAP, NT, CH>);
    if (!attr) {
        RFS_CUDA_TRY(
            cudaFuncSetAttribute(k_hits<PCAP, NT, CH, EVICT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        // the whole grid must be resident at once (a late-starting tile extends
        // the kernel): ask for the largest shared-memory carveout
        RFS_CUDA_TRY(cudaFuncSetAttribute(k_hits<PCAP, NT, CH, EVICT>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                          (int)cudaSharedmemCarveoutMaxShared));
        attr = true;
    }
    rfs_launch(k_hits<PCAP, NT, CH, EVICT>, (tile_hi - tile_lo) * (256 / NT), NT, smem, st, 
        (const int2*)ranges, vals, lb, (const float4*)sph, (const float4*)whit, (const RfsGeom*)geom, dirs, rx[0],
        rx[1], rx[2], min_t, n_az, n_el, tiles_u, hcap, (RfsHit*)slab, counts, slow_list, stats, used, tile_lo);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // namespace

extern "C" {

int rfs_ray_dirs(int n_az, int n_el, double* dirs, void* stream) {
    int R = n_az * n_el;
    if (R <= 0) return RFS_OK;
    rfs_launch(k_ray_dirs, rfs_ceil_div(R, 256), 256, 0, (cudaStream_t)stream, n_az, n_el, dirs);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_hits(const int* ranges, int n_tiles, const uint32_t* vals, const double* lb, const void* sph, const void* whit,
             const void* geom, const double* dirs, const double* rx, double ress_radius, int n_az, int n_el, int hcap,
             int pcap, void* slab, int* counts, int* slow_list, int* stats, uint32_t* used, int n, int tile_lo,
             int tile_hi, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (used && n > 0) RFS_CUDA_TRY(rfs_fill_u32(used, 0u, (size_t)n, st));
    const int tiles_u = (n_az + RFS_TILE - 1) / RFS_TILE;
    const int R = n_az * n_el;
    RFS_CUDA_TRY(rfs_fill_u32(stats, 0u, 16, st));
    RFS_CUDA_TRY(rfs_fill_u32(counts, 0u, (size_t)R, st));
    if (n_tiles <= 0) return RFS_OK;
    if (tile_hi < 0) tile_hi = n_tiles;  // default: every tile
    if (tile_lo < 0 || tile_lo > tile_hi || tile_hi > n_tiles) return RFS_ERR_SHAPE;
    // 64-thread blocks: 7 per SM, so 68 of a 360x180 grid's 1104 blocks start
    // late; 128-thread blocks (all resident) measured no faster -- the kernel
    // is set by the longest warps' chains, not by the late starts
    int rc = RFS_OK;
    if (tile_hi > tile_lo) {
#define RFS_LH(P, T, C, E) launch_hits<P, T, C, E>(tile_lo, tile_hi, ranges, vals, lb, sph, whit, geom, dirs, rx, \
                                                  ress_radius, n_az, n_el, tiles_u, hcap, slab, counts, slow_list, \
                                                  stats, used, st)
        const bool evict = (pcap & RFS_PCAP_EVICT) != 0;
        const int pc = pcap & ~RFS_PCAP_EVICT;
        if (pc <= 16) rc = evict ? RFS_LH(16, 64, 32, true) : RFS_LH(16, 64, 32, false);
        else if (pc <= 32) rc = evict ? RFS_LH(32, 64, 32, true) : RFS_LH(32, 64, 32, false);
        else rc = evict ? RFS_LH(64, 32, 16, true) : RFS_LH(64, 32, 16, false);
#undef RFS_LH
    }
    if (rc != RFS_OK) return rc;
    rfs_launch(k_max_range, rfs_ceil_div(n_tiles, 256), 256, 0, st, (const int2*)ranges, n_tiles, stats + 4);
    if (used && n > 0) rfs_launch(k_count_used, min(rfs_ceil_div(n, 256), 148 * 4), 256, 0, st, used, n, stats);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_hits_slow(const int* rays, int n_rays, const int* ranges, const uint32_t* vals, const double* lb,
                  const void* sph, const void* whit, const void* geom, const double* dirs, const double* rx,
                  double ress_radius, int n_az, int n_el, int hcap, void* slab, int* counts, double* pend_t,
                  uint32_t* pend_g, float* pend_w, int pcap, int* stats, uint32_t* used, int n, void* stream) {
    if (n_rays <= 0) return RFS_OK;
    int tiles_u = (n_az + RFS_TILE - 1) / RFS_TILE;
    rfs_launch(k_hits_slow, rfs_ceil_div(n_rays, 64), 64, 0, (cudaStream_t)stream, 
        rays, n_rays, (const int2*)ranges, vals, lb, (const float4*)sph, (const float4*)whit, (const RfsGeom*)geom,
        dirs, rx[0], rx[1], rx[2], ress_radius, n_az, n_el, tiles_u, hcap, (RfsHit*)slab, counts, pend_t, pend_g,
        pend_w, pcap, stats, used);
    if (used && n > 0) {  // the slow path marks more Gaussians: recount
        RFS_CUDA_TRY(rfs_fill_u32(stats + 8, 0u, 1, (cudaStream_t)stream));
        rfs_launch(k_count_used, min(rfs_ceil_div(n, 256), 148 * 4), 256, 0, (cudaStream_t)stream, used, n, stats);
    }
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // extern "C"
