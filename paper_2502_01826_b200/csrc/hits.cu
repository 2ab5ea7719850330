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
// (depth) order; a hit's chord midpoint lies in the Gaussian's 3-sigma ball,
// so t_mid >= depth - r3, and a pending hit whose t_mid is below
// lb[i] = min_{j>=i} (depth_j - r3_j) precedes every hit the remaining
// candidates can produce: it is final and is emitted, and a ray stops
// scanning as soon as it terminates.  Pending (t_mid, g, w) entries live in a
// per-thread ring in shared memory; a ray that overflows it is redone by
// k_hits_slow with a global buffer sized to its tile (exact, rarely taken).
//
// Execution: one thread per ray, 64-thread blocks (a 4 x 16 quarter tile, so
// the whole grid is resident at once).  Each warp streams its tile's
// candidate list on its own in chunks of CH:
//   1. stage the chunk's fp32 filter data (bounding sphere, whitened ellipsoid)
//      in warp-private shared memory (coalesced gathers, __syncwarp only);
//   2. every lane tests all CH candidates against its ray from shared memory
//      (no divergent global latency), building a survivor mask;
//   3. survivors run the reference's fp64 disc prefilter + quadratic and are
//      inserted in (t_mid, g) order;
//   4. pending hits below the next chunk's bound are emitted.
// Emitting once per chunk instead of per candidate does not change the order:
// every hit of the chunk is >= its first candidate's bound.
//
// Arithmetic: the fp32 tests carry proven margins (project.cu) so they never
// reject an fp64 hit; the fp64 test follows the reference's operation order
// with no FMA contraction (explicit __d*_rn), so exact ties order like the
// reference.  Ray directions come from a table built with the reference's
// formula (render.py:103-117).  T is carried in fp64.
#include "rfs_common.cuh"

namespace {

constexpr double DINF = 1.0e300;

// diagnostics: per-warp start / end %globaltimer of k_hits (null = off)
__device__ unsigned long long* g_k6_timing = nullptr;

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

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

// Emit one hit in sorted order: terminate, record, advance T (_kernels.py:186-191).
__device__ __forceinline__ void emit_hit(Ray& st, uint32_t g, float w, const RfsGeom* __restrict__ geom,
                                         RfsHit* __restrict__ slab_ray, int hcap, uint8_t* __restrict__ used) {
    if (st.tre * st.tre + st.tim * st.tim < RFS_TERM_EPS2) {
        st.done = true;
        return;
    }
    if (used) used[g] = 1;  // Gaussian has a live hit: its psi row is needed
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
    double rr = __ldg(&G->rho_re), ri = __ldg(&G->rho_im);
    double nr = st.tre * rr - st.tim * ri;
    double ni = st.tre * ri + st.tim * rr;
    st.tre = nr;
    st.tim = ni;
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
constexpr int GDS = 14;  // their shared-memory row: 7 x 16-byte cp.async pieces

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}

// Long tile lists set K6's critical path (tools/k6_timing.py: the warps of the
// longest lists take ~2x the mean).  Lists longer than split_min are split at
// mid: piece A streams [start, mid) exactly as an unsplit list (emitting every
// hit that precedes all of B's candidates, t_mid < lb[mid]) and parks its
// still-pending hits and its T; piece B streams [mid, end) concurrently into a
// sorted list of its own, without T or termination; k_hits_merge then merges
// the two (t_mid, g)-sorted lists and walks them with T and the termination
// rule -- the same hit sequence as one pass, since the reference itself sorts
// all hits of a ray and walks them (_kernels.py:27-112, 184-191).
constexpr int KS_ACAP = 64;  // A's parked hits (>= the largest pending ring)
struct KSplit {
    int split_min;  // lists longer than this are split (<= 0: never)
    int bcap;       // capacity of a ray's B list
    int* flag;      // per ray: 1 = A parked it (merge), 2 = the slow path owns it
    double *a_tre, *a_tim;
    int *a_live, *a_n;
    double* a_t;
    uint32_t* a_g;
    float* a_w;
    int* b_n;
    double* b_t;
    uint32_t* b_g;
    float* b_w;
};

// Per-patch candidate lists (k_patch_lists): a tile list filtered by the
// warp cone of each of its 8 ray patches (4 x 8 rays), with the emission
// bounds recomputed over each filtered list.  K6 then streams only the
// cone-relevant candidates (~15 % of the tile list at config 2): the same
// hits (the cone test never rejects a hit), far fewer chunks per warp.
struct KPatch {
    const uint32_t* vals;  // [8 * M]: tile t's patch p list at 8 * start(t) + p * len(t); null: off
    const double* lb;      // same layout: min over the list's later entries of lbv
    const int* cnt;        // [n_tiles * 8]
};

template <int CH>
struct WarpStage {
    float4 sph[CH];
    float4 wh[CH][4];
    uint32_t g[CH];
    double gd[CH][GDS];  // fp64 records of the chunk's cone-relevant candidates (by slot)
    double lbs[CH];      // patch mode: emission bound after candidate j (lb of candidate j + 1)
};

template <int PCAP, int NT, int CH>
struct HitsSmem {
    double pt[PCAP][NT];
    uint32_t pg[PCAP][NT];
    float pw[PCAP][NT];
    WarpStage<CH> ws[NT / 32];
};

template <int PCAP, int NT, int CH>
__global__ void __launch_bounds__(NT) k_hits(
    const int2* __restrict__ ranges, const uint32_t* __restrict__ vals, const double* __restrict__ lb,
    const float4* __restrict__ sph, const float4* __restrict__ whit, const RfsGeom* __restrict__ geom,
    const double* __restrict__ dirs, double rx0, double rx1, double rx2, double min_t, int n_az, int n_el,
    int tiles_u, int hcap, RfsHit* __restrict__ slab, int* __restrict__ counts, int* __restrict__ slow_list,
    int* __restrict__ stats, uint8_t* __restrict__ used, KSplit ks, KPatch kp) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    HitsSmem<PCAP, NT, CH>& S = *reinterpret_cast<HitsSmem<PCAP, NT, CH>*>(smem_raw);
    constexpr int PARTS = 256 / NT;
    // split lists: a tile's piece-B blocks follow its piece-A blocks, so both
    // pieces of a tile are resident together
    const int per_tile = ks.split_min > 0 ? 2 * PARTS : PARTS;
    const int tile = blockIdx.x / per_tile, wblk = blockIdx.x % per_tile, part = wblk % PARTS;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // each warp owns a 4 (u) x 8 (v) patch of the 16 x 16 tile
    const int q = part * (NT / 32) + wid, pu = q >> 1, pv = q & 1;
    const int u = (tile % tiles_u) * RFS_TILE + 4 * pu + (lane >> 3);
    const int v = (tile / tiles_u) * RFS_TILE + 8 * pv + (lane & 7);
    const bool valid = u < n_az && v < n_el;
    const int r = valid ? u * n_el + v : 0;
    const unsigned long long t_start = g_k6_timing ? gtimer() : 0ull;
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
    unsigned d_chunks = 0, d_rel = 0, d_nu = 0, d_mx = 0;  // diagnostics (g_k6_timing)
    double head_t = DINF;
    const int2 rg = ranges[tile];
    const int Lt = rg.y - rg.x;
    const bool pmode = kp.vals != nullptr;  // this warp's filtered patch list
    const bool split = !pmode && ks.split_min > 0 && Lt > ks.split_min;
    const bool second = wblk >= PARTS;  // piece B of a split list
    if (second && !split) return;         // block-uniform
    const int mid = split ? rg.x + Lt / 2 : rg.y;
    const uint32_t* vl = vals;
    const double* lbp = lb;
    int c_lo, c_hi, c_end;
    if (pmode) {
        const size_t pb = 8 * (size_t)rg.x + (size_t)q * (size_t)Lt;
        vl = kp.vals + pb;
        lbp = kp.lb + pb;
        c_lo = 0;
        c_hi = c_end = kp.cnt[tile * 8 + q];
    } else {
        c_lo = second ? mid : rg.x;
        c_hi = second ? rg.y : mid;
        c_end = rg.y;
    }
    int b_n = 0;
    WarpStage<CH>& W = S.ws[wid];

    // Warp cone: axis c through the patch, half-angle th_p covering its rays.
    // A ray can only hit a Gaussian whose bounding-sphere cone (axis mu - rx,
    // half-angle th_g = asin(r3/depth)) contains it, so a candidate is
    // relevant to the warp only if angle(c, mu - rx) <= th_p + th_g.
    float cx = valid ? st.fx : 0.f, cy = valid ? st.fy : 0.f, cz = valid ? st.fz : 0.f;
    cx = warp_sum(cx);
    cy = warp_sum(cy);
    cz = warp_sum(cz);
    {
        const float inv = rsqrtf(fmaxf(cx * cx + cy * cy + cz * cz, 1e-30f));
        cx *= inv;
        cy *= inv;
        cz *= inv;
    }
    float cmin = valid ? cx * st.fx + cy * st.fy + cz * st.fz : 1.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cmin = fminf(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
    const float th_p = acosf(fminf(cmin, 1.f)) + 1e-4f;
    float sin_p, cos_p;
    sincosf(th_p, &sin_p, &cos_p);

    // register prefetch of the next chunk's filter data (lane j loads candidate base + j)
    uint32_t pf_g = 0;
    float4 pf_s = make_float4(0.f, 0.f, 0.f, 0.f), pf_w[4];
    double pf_lb = DINF, pf_lbs = DINF;
    // candidate ids run one chunk further ahead than their records, so the
    // record gathers never wait on the id load (in-order issue)
    uint32_t nx_g = c_lo + lane < c_hi ? vl[c_lo + lane] : 0u;
    auto prefetch = [&](int b0) {
        if (b0 + lane < c_hi) {
            pf_g = nx_g;
            pf_s = __ldg(&sph[pf_g]);
#pragma unroll
            for (int k = 0; k < 4; ++k) pf_w[k] = __ldg(&whit[4 * pf_g + k]);
        }
        if (b0 + CH + lane < c_hi) nx_g = vl[b0 + CH + lane];
        // bound of every candidate after this chunk -- for piece A's last chunk
        // that is B's first candidate, mid
        const int nxt = min(b0 + CH, c_hi);
        pf_lb = nxt < c_end ? lbp[nxt] : DINF;
        if (pmode) pf_lbs = b0 + lane + 1 < c_end ? lbp[b0 + lane + 1] : DINF;
    };
    prefetch(c_lo);
    // emit every pending hit below `bound` (in (t_mid, g) order)
    auto emit_until = [&](double bound) {
        while (!st.done && head_t < bound) {
            if (second) {  // piece B: into its own sorted list, no T / termination
                if (b_n == ks.bcap) {
                    pend_over = true;
                    st.done = true;
                    break;
                }
                const size_t o = (size_t)r * ks.bcap + b_n++;
                ks.b_t[o] = S.pt[head][tid];
                ks.b_g[o] = S.pg[head][tid];
                ks.b_w[o] = S.pw[head][tid];
            } else {
                emit_hit(st, S.pg[head][tid], S.pw[head][tid], geom, slab_ray, hcap, used);
            }
            head = (head + 1) & (PCAP - 1);
            --npend;
            head_t = npend > 0 ? S.pt[head][tid] : DINF;
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
            if (pmode) W.lbs[lane] = pf_lbs;
#pragma unroll
            for (int k = 0; k < 4; ++k) W.wh[lane][k] = pf_w[k];
            const float ang = th_p + pf_w[3].y;
            if (pmode || ang >= 3.1415f) {  // patch lists are cone-filtered already
                rel = true;
            } else {
                // cos(th_p + th_g) by angle addition (cos/sin th_g precomputed in K1)
                const float m2 = pf_s.x * pf_s.x + pf_s.y * pf_s.y + pf_s.z * pf_s.z;
                const float dotc = (cx * pf_s.x + cy * pf_s.y + cz * pf_s.z) * rsqrtf(m2);
                rel = dotc >= cos_p * pf_w[3].z - sin_p * pf_w[3].w - 1e-5f;
            }
        }
        const unsigned relmask = __ballot_sync(0xffffffffu, rel);
        if (g_k6_timing) {
            d_chunks += 1;
            d_rel += __popc(relmask);
        }
        const double lb_next = pf_lb;
        __syncwarp();
        // fp64 records of the cone-relevant candidates -> shared memory,
        // asynchronously (cp.async; lane j copies its own candidate's): they
        // land while the fp32 filters run
        if (rel) {
            const char* src = reinterpret_cast<const char*>(geom + pf_g);
#pragma unroll
            for (int part = 0; part < GDS / 2; ++part) cp_async16(&W.gd[lane][2 * part], src + 16 * part);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
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
        // 3a. the records' copies have landed (own copies, then the warp's)
        if (g_k6_timing) {
            d_nu += __popc(__reduce_or_sync(0xffffffffu, mask));
            d_mx += __reduce_max_sync(0xffffffffu, (unsigned)__popc(mask));
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        if (!st.done) {
            // 3b. exact fp64 test and sorted insertion by (t_mid, g)
            while (mask) {
                const int j = __ffs(mask) - 1;
                mask &= mask - 1;
                const uint32_t g = W.g[j];
                double t_mid;
                float w;
                if (!exact_hit_s(W.gd[j], st.dx, st.dy, st.dz, uf, vf, naz, rx0, rx1, rx2, min_t, t_mid, w)) continue;
                if (npend == PCAP) {
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
                // patch lists are dense: emit as soon as a hit precedes every
                // later candidate (this lane has tested all candidates <= j),
                // which keeps the pending ring short
                if (pmode) {
                    emit_until(W.lbs[j]);
                    if (st.done) break;
                }
            }
            // 4. emit every pending hit that precedes all later candidates
            emit_until(lb_next);
        }
        __syncwarp();
    }
    // drain (also covers rays whose tile list ended with pending hits); a
    // split list's piece A parks its pending hits and T for k_hits_merge
    const bool park = split && !second && !st.done;
    if (second) {
        while (!st.done && npend > 0) {
            if (b_n == ks.bcap) {
                pend_over = true;
                st.done = true;
                break;
            }
            const size_t o = (size_t)r * ks.bcap + b_n++;
            ks.b_t[o] = S.pt[head][tid];
            ks.b_g[o] = S.pg[head][tid];
            ks.b_w[o] = S.pw[head][tid];
            head = (head + 1) & (PCAP - 1);
            --npend;
        }
    } else if (park) {
        for (int i = 0; i < npend; ++i) {
            const int sl = (head + i) & (PCAP - 1);
            const size_t o = (size_t)r * KS_ACAP + i;
            ks.a_t[o] = S.pt[sl][tid];
            ks.a_g[o] = S.pg[sl][tid];
            ks.a_w[o] = S.pw[sl][tid];
        }
    } else {
        while (!st.done && npend > 0) {
            emit_hit(st, S.pg[head][tid], S.pw[head][tid], geom, slab_ray, hcap, used);
            head = (head + 1) & (PCAP - 1);
            --npend;
        }
    }
    if (g_k6_timing) {
        const unsigned live_max = __reduce_max_sync(0xffffffffu, (unsigned)st.live);
        if (lane == 0) {
            unsigned long long* o = g_k6_timing + 8 * ((blockIdx.x * NT + tid) >> 5);
            o[0] = t_start;
            o[1] = gtimer();
            o[2] = (unsigned long long)(c_hi - c_lo);
            o[3] = d_chunks;
            o[4] = d_rel;
            o[5] = d_mx;
            o[6] = d_nu;
            o[7] = live_max;
        }
    }
    if (!valid) return;
    atomicMax(&stats[5], max_pend);
    atomicAdd(&stats[6], n_sph);
    atomicAdd(&stats[7], n_wh);
    // split-ray handshake on flag[r]: 0 open, 1 parked by A (merge), 2 owned
    // by the slow path, 3 terminated within A (B's hits are irrelevant)
    if (pend_over) {  // the slow path redoes the whole ray
        bool to_slow = true;
        if (split) {
            const int old = second ? atomicCAS(&ks.flag[r], 0, 2) : atomicExch(&ks.flag[r], 2);
            if (second && old == 1) atomicExch(&ks.flag[r], 2);
            to_slow = second ? (old == 0 || old == 1) : old != 2;
        }
        if (to_slow) {
            int idx = atomicAdd(&stats[0], 1);
            slow_list[idx] = r;
        }
        return;
    }
    if (second) {
        ks.b_n[r] = b_n;
        return;
    }
    if (park) {
        ks.a_n[r] = npend;
        ks.a_tre[r] = st.tre;
        ks.a_tim[r] = st.tim;
        ks.a_live[r] = st.live;
        atomicCAS(&ks.flag[r], 0, 1);  // unless B already handed the ray to the slow path
        return;
    }
    if (split && atomicCAS(&ks.flag[r], 0, 3) == 2) return;  // B overflowed first: the slow path redoes it
    counts[r] = min(st.live, hcap);  // stored hits; live > hcap is flagged in stats[1]
    if (st.hcap_over) atomicAdd(&stats[1], 1);
    atomicMax(&stats[2], st.live);
    atomicAdd(&stats[3], min(st.live, hcap));
}

// K6a: the per-patch candidate lists of KPatch.  Block per tile, warp w
// computes patch w's cone exactly as k_hits does; every candidate is tested
// against the 8 cones, compacted per patch in list order (ballots + warp
// prefix), then each patch's emission bounds are the suffix minima of lbv
// over its own list.
constexpr int PL_NT = 1024;  // k_patch_lists threads: one tile list round of 1024 candidates
__global__ void __launch_bounds__(PL_NT, 2) k_patch_lists(const int2* __restrict__ ranges, const uint32_t* __restrict__ vals,
                                                       const float4* __restrict__ sph, const float4* __restrict__ whit,
                                                       const RfsGeom* __restrict__ geom, const double* __restrict__ dirs,
                                                       int n_az, int n_el, int tiles_u, uint32_t* __restrict__ pvals,
                                                       double* __restrict__ plb, int* __restrict__ pcnt) {
    constexpr int NW = PL_NT / 32;
    __shared__ float4 ca[8];  // cx, cy, cz, th_p of patch p (a patch without rays never passes)
    __shared__ float2 cb[8];  // cos_p, sin_p
    __shared__ int run[8];
    __shared__ unsigned wb[NW][8];  // [warp][patch] ballots of the current round
    __shared__ int wpre[NW][8];     // [warp][patch] first position of the warp's entries
    const int tile = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (wid < 8) {  // warp q: the cone of patch q, as k_hits computes it
        float4 a;
        float2 c;
        rfs_patch_cone(tile, wid, tiles_u, n_az, n_el, dirs, a, c);
        if (lane == 0) {
            ca[wid] = a;
            cb[wid] = c;
            run[wid] = 0;
        }
    }
    __syncthreads();
    const int2 rg = ranges[tile];
    const size_t L = (size_t)(rg.y - rg.x), tb = 8 * (size_t)rg.x;
    unsigned lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    for (int b0 = rg.x; b0 < rg.y; b0 += PL_NT) {
        const int i = b0 + tid;
        uint32_t g = 0, pm = 0;
        double lbv = 0.0;
        if (i < rg.y) {
            g = vals[i];
            const float4 sp = __ldg(&sph[g]);
            const float4 w3 = __ldg(&whit[4 * g + 3]);
            lbv = __ldg(&geom[g].lbv);
            pm = rfs_patch_mask(ca, cb, sp, w3);
        }
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            const unsigned m = __ballot_sync(0xffffffffu, (pm >> p) & 1u);
            if (lane == 0) wb[wid][p] = m;
        }
        __syncthreads();
        if (tid < 8) {  // per patch: each warp's first position this round
            int acc = run[tid];
            for (int w = 0; w < NW; ++w) {
                wpre[w][tid] = acc;
                acc += __popc(wb[w][tid]);
            }
            run[tid] = acc;
        }
        __syncthreads();
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            if (!((pm >> p) & 1u)) continue;
            const uint32_t pos = wpre[wid][p] + __popc(wb[wid][p] & lt);
            pvals[tb + (size_t)p * L + pos] = g;
            plb[tb + (size_t)p * L + pos] = lbv;  // raw lbv; suffix minima below
        }
        __syncthreads();
    }
    // warps 0-7: suffix minima of lbv over patch list p (contiguous, in place)
    if (wid >= 8) return;
    const int cnt = run[wid];
    if (lane == 0) pcnt[tile * 8 + wid] = cnt;
    double* pl = plb + tb + (size_t)wid * L;
    double carry = INFINITY;
    for (int k0 = ((cnt - 1) >> 5) << 5; k0 >= 0; k0 -= 32) {
        const int k = k0 + lane;
        double v = k < cnt ? pl[k] : INFINITY;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_down_sync(0xffffffffu, v, o);
            if (lane + o < 32) v = fmin(v, y);
        }
        v = fmin(v, carry);
        if (k < cnt) pl[k] = v;
        carry = __shfl_sync(0xffffffffu, v, 0);
    }
}

// Merge of a split list's two pieces (see KSplit): thread per ray parked by A.
__global__ void k_hits_merge(int R, int hcap, KSplit ks, const RfsGeom* __restrict__ geom,
                             RfsHit* __restrict__ slab, int* __restrict__ counts, int* __restrict__ stats,
                             uint8_t* __restrict__ used) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R || ks.flag[r] != 1) return;
    Ray st;
    st.tre = ks.a_tre[r];
    st.tim = ks.a_tim[r];
    st.live = ks.a_live[r];
    st.done = false;
    st.hcap_over = st.live > hcap;
    RfsHit* slab_ray = slab + (size_t)r * hcap;
    const int na = ks.a_n[r], nbb = ks.b_n[r];
    const double* at = ks.a_t + (size_t)r * KS_ACAP;
    const uint32_t* ag = ks.a_g + (size_t)r * KS_ACAP;
    const float* aw = ks.a_w + (size_t)r * KS_ACAP;
    const double* bt = ks.b_t + (size_t)r * ks.bcap;
    const uint32_t* bg = ks.b_g + (size_t)r * ks.bcap;
    const float* bw = ks.b_w + (size_t)r * ks.bcap;
    int i = 0, j = 0;
    while (!st.done && (i < na || j < nbb)) {
        const bool from_a = i < na && (j >= nbb || at[i] < bt[j] || (at[i] == bt[j] && ag[i] < bg[j]));
        if (from_a) {
            emit_hit(st, ag[i], aw[i], geom, slab_ray, hcap, used);
            ++i;
        } else {
            emit_hit(st, bg[j], bw[j], geom, slab_ray, hcap, used);
            ++j;
        }
    }
    counts[r] = min(st.live, hcap);
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
                            uint8_t* __restrict__ used) {
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
            emit_hit(st, my_g[head], my_w[head], geom, slab_ray, hcap, used);
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
        emit_hit(st, my_g[head], my_w[head], geom, slab_ray, hcap, used);
        ++head;
        --npend;
    }
    counts[r] = min(st.live, hcap);  // stored hits; live > hcap is flagged in stats[1]
    if (st.hcap_over) atomicAdd(&stats[1], 1);
    atomicMax(&stats[2], st.live);
    atomicAdd(&stats[3], min(st.live, hcap));
}

__global__ void k_max_range(const int2* __restrict__ ranges, int n_tiles, int* __restrict__ out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_tiles) atomicMax(out, ranges[t].y - ranges[t].x);
}

// Ray directions through cell centres, render.py:103-117, same operation
// order as numpy (deg2rad(x) = x * (pi/180)); used only when the host does
// not supply the table.
__global__ void k_ray_dirs(int n_az, int n_el, double* __restrict__ dirs) {
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

template <int PCAP, int NT, int CH>
int launch_hits(int n_tiles, const int* ranges, const uint32_t* vals, const double* lb, const void* sph,
                const void* whit, const void* geom, const double* dirs, const double* rx, double min_t, int n_az,
                int n_el, int tiles_u, int hcap, void* slab, int* counts, int* slow_list, int* stats, uint8_t* used,
                const KSplit& ks, const KPatch& kp, cudaStream_t st) {
    static bool attr = false;
    size_t smem = sizeof(HitsSmem<PCAP, NT, CH>);
    if (!attr) {
        RFS_CUDA_TRY(
            cudaFuncSetAttribute(k_hits<PCAP, NT, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        // the whole grid must be resident at once (a late-starting tile extends
        // the kernel): ask for the largest shared-memory carveout
        RFS_CUDA_TRY(cudaFuncSetAttribute(k_hits<PCAP, NT, CH>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                          (int)cudaSharedmemCarveoutMaxShared));
        attr = true;
    }
    const int per_tile = (256 / NT) * (ks.split_min > 0 ? 2 : 1);
    k_hits<PCAP, NT, CH><<<n_tiles * per_tile, NT, smem, st>>>(
        (const int2*)ranges, vals, lb, (const float4*)sph, (const float4*)whit, (const RfsGeom*)geom, dirs, rx[0],
        rx[1], rx[2], min_t, n_az, n_el, tiles_u, hcap, (RfsHit*)slab, counts, slow_list, stats, used, ks, kp);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // namespace

extern "C" {

// diagnostics (not part of the rasterizer path): per-warp timing of k_hits into
// buf (u64[8 * warps]: start, end, candidates, chunks, cone survivors, sum over
// chunks of the most exact tests on one lane, union size, max live); NULL: off
int rfs_debug_k6_timing(unsigned long long* buf) {
    RFS_CUDA_TRY(cudaMemcpyToSymbol(g_k6_timing, &buf, sizeof(buf)));
    return RFS_OK;
}

int rfs_ray_dirs(int n_az, int n_el, double* dirs, void* stream) {
    int R = n_az * n_el;
    if (R <= 0) return RFS_OK;
    k_ray_dirs<<<rfs_ceil_div(R, 256), 256, 0, (cudaStream_t)stream>>>(n_az, n_el, dirs);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

// pcap selects the pending-ring template: 16 entries (64-thread blocks, 9
// blocks/SM), 32 entries (64-thread blocks) or 64 entries (32-thread blocks)
// for dense scenes.
size_t rfs_hits_split_bytes(int n_rays, int bcap) {
    const size_t R = (size_t)(n_rays > 0 ? n_rays : 0), B = (size_t)(bcap > 0 ? bcap : 0);
    // per ray: flag, a_n, a_live, b_n (int); a_tre, a_tim (double); A's and B's lists (16 B per entry)
    return R * (4 * sizeof(int) + 2 * sizeof(double)) + R * (KS_ACAP + B) * 16;
}

size_t rfs_hits_patch_bytes(int m_cap, int n_tiles) {
    const size_t M = (size_t)(m_cap > 0 ? m_cap : 0), T = (size_t)(n_tiles > 0 ? n_tiles : 0);
    return 8 * M * sizeof(double) + 8 * M * sizeof(uint32_t) + 8 * T * sizeof(int) + 64;
}

int rfs_hits(const int* ranges, int n_tiles, const uint32_t* vals, const double* lb, const void* sph, const void* whit,
             const void* geom, const double* dirs, const double* rx, double ress_radius, int n_az, int n_el, int hcap,
             int pcap, void* slab, int* counts, int* slow_list, int* stats, uint8_t* used, int n, int split_min,
             int bcap, void* split_ws, int m_cap, void* patch_ws, int patch_built, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (used && n > 0) RFS_CUDA_TRY(cudaMemsetAsync(used, 0, (size_t)n, st));
    int tiles_u = (n_az + RFS_TILE - 1) / RFS_TILE;
    const int R = n_az * n_el;
    RFS_CUDA_TRY(cudaMemsetAsync(stats, 0, 8 * sizeof(int), st));
    RFS_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int) * (size_t)R, st));
    if (n_tiles <= 0) return RFS_OK;
    KSplit ks{};
    ks.split_min = (split_ws && bcap > 0) ? split_min : 0;
    if (ks.split_min > 0) {
        // carve the workspace: 8-byte arrays first, then 4-byte ones
        char* p = (char*)split_ws;
        auto take = [&](size_t bytes) {
            char* q = p;
            p += bytes;
            return q;
        };
        const size_t Rz = (size_t)R, A = (size_t)KS_ACAP * Rz, B = (size_t)bcap * Rz;
        ks.bcap = bcap;
        ks.a_tre = (double*)take(Rz * 8);
        ks.a_tim = (double*)take(Rz * 8);
        ks.a_t = (double*)take(A * 8);
        ks.b_t = (double*)take(B * 8);
        ks.flag = (int*)take(Rz * 4);
        ks.a_n = (int*)take(Rz * 4);
        ks.a_live = (int*)take(Rz * 4);
        ks.b_n = (int*)take(Rz * 4);
        ks.a_g = (uint32_t*)take(A * 4);
        ks.b_g = (uint32_t*)take(B * 4);
        ks.a_w = (float*)take(A * 4);
        ks.b_w = (float*)take(B * 4);
        RFS_CUDA_TRY(cudaMemsetAsync(ks.flag, 0, Rz * 4, st));
    }
    KPatch kp{};
    if (patch_ws && ks.split_min <= 0 && m_cap > 0) {
        double* plb = (double*)patch_ws;
        uint32_t* pv = (uint32_t*)(plb + 8 * (size_t)m_cap);
        int* pc = (int*)(pv + 8 * (size_t)m_cap);
        if (!patch_built) {  // else rfs_bin_bucket wrote them
            k_patch_lists<<<n_tiles, PL_NT, 0, st>>>((const int2*)ranges, vals, (const float4*)sph,
                                                     (const float4*)whit, (const RfsGeom*)geom, dirs, n_az, n_el,
                                                     tiles_u, pv, plb, pc);
            RFS_LAUNCH_CHECK();
        }
        kp.vals = pv;
        kp.lb = plb;
        kp.cnt = pc;
    }
    int rc;
    // 64-thread blocks: 7 per SM, so 68 of a 360x180 grid's 1104 blocks start
    // late (~90 us); 128-thread blocks (all resident) measured no faster -- the
    // kernel is set by the longest warps' chains, not by the late starts
    // (tools/k6_timing.py: warp duration mean 124 us, max 238 us at 100k)
    if (pcap <= 16)
        rc = launch_hits<16, 64, 32>(n_tiles, ranges, vals, lb, sph, whit, geom, dirs, rx, ress_radius, n_az, n_el,
                                     tiles_u, hcap, slab, counts, slow_list, stats, used, ks, kp, st);
    else if (pcap <= 32)
        rc = launch_hits<32, 64, 32>(n_tiles, ranges, vals, lb, sph, whit, geom, dirs, rx, ress_radius, n_az, n_el,
                                     tiles_u, hcap, slab, counts, slow_list, stats, used, ks, kp, st);
    else
        rc = launch_hits<64, 32, 16>(n_tiles, ranges, vals, lb, sph, whit, geom, dirs, rx, ress_radius, n_az, n_el,
                                     tiles_u, hcap, slab, counts, slow_list, stats, used, ks, kp, st);
    if (rc != RFS_OK) return rc;
    if (ks.split_min > 0) {
        k_hits_merge<<<rfs_ceil_div(R, 128), 128, 0, st>>>(R, hcap, ks, (const RfsGeom*)geom, (RfsHit*)slab, counts,
                                                            stats, used);
        RFS_LAUNCH_CHECK();
    }
    k_max_range<<<rfs_ceil_div(n_tiles, 256), 256, 0, st>>>((const int2*)ranges, n_tiles, stats + 4);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_hits_slow(const int* rays, int n_rays, const int* ranges, const uint32_t* vals, const double* lb,
                  const void* sph, const void* whit, const void* geom, const double* dirs, const double* rx,
                  double ress_radius, int n_az, int n_el, int hcap, void* slab, int* counts, double* pend_t,
                  uint32_t* pend_g, float* pend_w, int pcap, int* stats, uint8_t* used, void* stream) {
    if (n_rays <= 0) return RFS_OK;
    int tiles_u = (n_az + RFS_TILE - 1) / RFS_TILE;
    k_hits_slow<<<rfs_ceil_div(n_rays, 64), 64, 0, (cudaStream_t)stream>>>(
        rays, n_rays, (const int2*)ranges, vals, lb, (const float4*)sph, (const float4*)whit, (const RfsGeom*)geom,
        dirs, rx[0], rx[1], rx[2], ress_radius, n_az, n_el, tiles_u, hcap, (RfsHit*)slab, counts, pend_t, pend_g,
        pend_w, pcap, stats, used);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // extern "C"
