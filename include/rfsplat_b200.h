/*
 * rfsplat_b200.h -- C ABI of the B200 (sm_100a) RF-splatting rasterizer.
 *
 * Drop-in boundary for the reference package `rfsplat` (pkg/src/rfsplat/).
 * The reference has no native library: its hot path is numba-compiled Python
 * called through plain functions over caller-allocated numpy arrays
 * (_kernels.py:140-559).  The FFI a maintainer would bind (ctypes, see
 * INTEGRATION.md) is this header: plain device pointers, sizes and a
 * cudaStream_t passed as void*, integer status codes, no torch types.
 *
 * Ownership: the caller allocates every buffer (the Python host layer uses
 * the torch caching allocator); the library never frees caller memory.
 * All entry points are stream-ordered and asynchronous unless noted.
 *
 * Status codes map onto rfsplat.errors (errors.py:4-40):
 *   0 OK, 1 GeometryError, 2 ShapeError, 3 ContractViolationError,
 *   4 NonFiniteGradientError, 5 CUDA failure, 6 capacity exceeded (retry
 *   with larger scratch).
 *
 * Layouts (N Gaussians, B transmitters, R = n_az * n_el rays, r = u*n_el+v):
 *   means f32[N*3], quats f32[N*4] (w,x,y,z), log_scales f32[N*3],
 *   trans_mag_raw f32[N], trans_phase f32[N], coeffs complex64[N*K]
 *   (K = (L+1)^2, index l*l+l+m), rx f64[3] (host), tx f32[B*3],
 *   S / grad_S complex64[B*R], psi complex64[N*B], dirs f64[R*3].
 * Opaque records: geom 128 B/Gaussian, sph 16 B/Gaussian, whit 64 B/Gaussian,
 *   rects 16 B/Gaussian, rho32 16 B/Gaussian, hit slab 16 B/(ray*hcap),
 *   gslab 16 B/(ray*hcap).
 */
#ifndef RFSPLAT_B200_H
#define RFSPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RFS_GEOM_BYTES 128
#define RFS_SPH_BYTES 16
#define RFS_WHIT_BYTES 64
#define RFS_RECT_BYTES 16
#define RFS_RHO_BYTES 16
#define RFS_HIT_BYTES 16
#define RFS_GSLAB_BYTES 16

/* K1: per-Gaussian shape, transmittance, projection and tile counts.
 * Replaces scene.covariances (scene.py:157-161), prepare_context's inverse /
 * normalizer / rho (render.py:220-227), project_scene (splat.py:212-268),
 * the rectangle math of _tiles_from_arrays (splat.py:308-328) and the count
 * pass of expand_tile_rects (_kernels.py:532-541).  proj_out (nullable,
 * f64[N*6]) receives SceneProjection (center_u, center_v, radius_px,
 * tile_radius, depth, active).  err_flags bit 1 set => GeometryError. */
int rfs_project(int n, const float* means, const float* quats, const float* log_scales, const float* trans_mag_raw,
                const float* trans_phase, const double* rx, double ress_radius, int n_az, int n_el, void* geom,
                void* sph, void* whit, uint32_t* depth_code, void* rects, uint32_t* counts, void* rho32,
                double* proj_out, int* err_flags, void* stream);

/* K2: exclusive warp-shuffle scan of per-Gaussian splat counts -> offsets;
 * *total (device) = M.  Replaces the implicit cumulative positions of
 * expand_tile_rects (_kernels.py:533-545).  temp: rfs_scan_temp_elems(n) u32. */
size_t rfs_scan_temp_elems(int n);
int rfs_exclusive_scan_u32(const uint32_t* in, int n, uint32_t* out, uint32_t* total, uint32_t* temp, void* stream);

/* K2b: fill (compact key, Gaussian id) pairs in the reference expansion
 * order (_kernels.py:545-558).  Compact key = tile << 31 | float32 depth
 * bits; rfs_expand_keys restores the reference key tile << 32 | bits.
 * Only positions < cap are written (compare M with cap afterwards). */
int rfs_bin_fill(int n, const void* rects, const uint32_t* depth_code, const uint32_t* offsets, int n_az, int cap,
                 uint64_t* ckeys, uint32_t* vals, void* stream);
int rfs_expand_keys(const uint64_t* ckeys, int m, uint64_t* keys, void* stream);

/* K3: stable LSD radix sort of (u64 key, u32 value) on bits [0, end_bit).
 * Replaces np.argsort(keys, kind="stable") (splat.py:337).  Hand-written
 * onesweep passes; the _cub variant calls cub::DeviceRadixSort::SortPairs for
 * comparison.  *result_in_alt (host) = 1 if the sorted data is in *_alt.
 * m_dev (nullable, hand-written sort only): device-side count; m is then the
 * capacity and min(*m_dev, m) keys are sorted without a host read. */
size_t rfs_sort_temp_bytes(int m, int end_bit);
int rfs_sort_pairs_u64(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt, int m, int end_bit,
                       void* temp, size_t temp_bytes, int* result_in_alt, const uint32_t* m_dev, void* stream);
size_t rfs_sort_cub_temp_bytes(int m, int end_bit);
int rfs_sort_pairs_u64_cub(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt, int m, int end_bit,
                           void* temp, size_t temp_bytes, int* result_in_alt, void* stream);

/* K4: per-tile [start, end) ranges = searchsorted left/right of each tile id
 * (splat.py:340-343); ranges is int32[n_tiles*2]. */
int rfs_tile_ranges(const uint64_t* ckeys, int m, const uint32_t* m_dev, int n_tiles, int* ranges, void* stream);

/* K2b + K3 + K4 + K4b by tile buckets (bucket.cu): a stable counting sort
 * by tile (per-block tile counts, offsets = the ranges, clamped to cap; a fill
 * that keeps expansion order inside each tile's bucket), then one stable
 * radix sort of the depth codes per tile (shared memory up to 12288 entries,
 * L2-resident global buffers beyond), which writes the sorted compact keys,
 * Gaussian ids and emission bounds -- bitwise the outputs of rfs_bin_fill +
 * rfs_sort_pairs_u64 + rfs_tile_ranges + rfs_lower_bounds (splat.py:337-343).
 * bcodes / bvals u32[cap] and temp (rfs_bin_bucket_temp_bytes) are scratch;
 * status is reserved.  Grids up to 512 tiles. */
size_t rfs_bin_bucket_temp_bytes(int n, int n_az, int n_el, int cap);
int rfs_bin_bucket(int n, const void* rects, const uint32_t* depth_code, int n_az, int n_el, int cap, const void* geom,
                   uint32_t* bcodes, uint32_t* bvals, void* temp, uint64_t* ckeys, uint32_t* vals, int* ranges,
                   double* lb, int* status, void* stream);

/* K4b: per-incidence emission bound for the exact streaming re-sort:
 * lb[i] = min_{j >= i, same tile} (depth_j - r3_j). */
int rfs_lower_bounds(const int* ranges, int n_tiles, const uint32_t* vals, const void* geom, double* lb, void* stream);

/* Ray directions through the cell centres (render.py:103-117); the Python
 * host layer uploads a numpy-built table instead (bitwise the reference's). */
int rfs_ray_dirs(int n_az, int n_el, double* dirs, void* stream);

/* K6: TX-independent live hit lists.  Replaces _collect_hits + the live walk
 * of forward_tiled / count_hits_tiled (_kernels.py:27-112, 140-192, 237-292).
 * Writes hits of ray r to slab[r*hcap ...], counts[r] = live count.
 * stats (device int[8]): [0] rays needing rfs_hits_slow (listed in slow_list), [1] rays
 * with live > hcap (caller must retry with larger hcap), [2] max live,
 * [3] total live hits, [4] longest tile list, [5] see below, [8] Gaussians
 * with a live hit (stats is int[16]).
 * used (nullable u32[n], zeroed here): 1 for every Gaussian with a live hit.
 * The exact streaming re-sort with early termination (hits.cu); pcap
 * selects the pending ring (<= 16 -> 16 entries per ray, <= 32 -> 32, else
 * 64), and pcap | RFS_PCAP_EVICT makes a full ring keep its smallest hits
 * (a ray then needs the slow path only if it must emit a dropped hit);
 * stats[5] = the largest pending set, stats[6] / [7] = fp32 sphere /
 * whitened-ellipsoid passes (diagnostics).  Only the rays of tiles
 * [tile_lo, tile_hi) are traced (tile_hi < 0: all tiles); the others get no
 * hits -- the tile shard of a rank in the strong-scaling mode. */
#define RFS_PCAP_EVICT 0x10000
int rfs_hits(const int* ranges, int n_tiles, const uint32_t* vals, const double* lb, const void* sph, const void* whit,
             const void* geom, const double* dirs, const double* rx, double ress_radius, int n_az, int n_el, int hcap,
             int pcap, void* slab, int* counts, int* slow_list, int* stats, uint32_t* used, int n, int tile_lo,
             int tile_hi, void* stream);
int rfs_hits_slow(const int* rays, int n_rays, const int* ranges, const uint32_t* vals, const double* lb,
                  const void* sph, const void* whit, const void* geom, const double* dirs, const double* rx,
                  double ress_radius, int n_az, int n_el, int hcap, void* slab, int* counts, double* pend_t,
                  uint32_t* pend_g, float* pend_w, int pcap, int* stats, uint32_t* used, int n, void* stream);

/* K5: psi[g][b] = sum_k coeffs[g][k] * basis_k(bearing of tx_b from mu_g);
 * with used (nullable, rfs_hits' u8 marks) only rows of Gaussians with live
 * hits -- the only rows K7 / K8 read -- are computed.
 * Replaces render.py:229-238 + fle.fle_basis_with_derivs (fle.py:153-212). */
int rfs_psi(int n, int n_tx, int degree, const float* means, const void* coeffs, const float* tx, const uint32_t* used,
            void* psi, void* stream);


/* K7: S[b][r] = sum over live hits of w * T * psi[g][b].  Replaces the
 * composite of forward_tiled (_kernels.py:184-192) for a TX batch. */
int rfs_forward(const void* slab, const int* counts, int hcap, const void* psi, int n_tx, int n_az, int n_el, void* S,
                void* stream);

/* K8i: by-Gaussian index of the live hits (TX independent).
 * rfs_used_list: order[cid[g]] = g for every g with used[g] (cid = the
 * exclusive scan of rfs_hits' used marks: the compact id among the Gaussians
 * with a live hit; entries at cid >= cap are dropped -- the caller checks
 * the count and rebuilds).
 * rfs_hit_keys: keys[ray_off[r]+k] = rank[g] (rank = cid, nullable: the
 * Gaussian id), slots[...] = r*hcap + k (ray_off = exclusive scan of counts);
 * sort the pairs with rfs_sort_pairs_u64 (stable: (ray, k) order within a
 * Gaussian, the slot order of the reference's bincount, grad.py:243-254);
 * rfs_gather_sorted: per sorted hit p its ray s_ray[p], w s_w[p], w T
 * s_wt[p] (complex64) and, if inv_slot is not NULL, inv_slot[slot] = p
 * (u32[R*hcap]); with keys (nullable: a compact-id sort) the sorted keys are
 * replaced by the Gaussian ids;
 * rfs_gauss_ranges: g_rng (int32[2N]) = [first, end) of each Gaussian's run
 * of sorted hits, (0, 0) for Gaussians without hits.
 * Entry points taking (n_hits, h_dev) treat n_hits as the capacity and, when
 * h_dev (device u32) is given, process min(*h_dev, n_hits) hits -- the hit
 * index and the backward then need no host read of the hit count. */
int rfs_used_list(int n, const uint32_t* used, const uint32_t* cid, int cap, uint32_t* order, void* stream);
int rfs_hit_keys(const void* slab, const int* counts, const uint32_t* ray_off, int hcap, int n_rays,
                 const uint32_t* rank, uint64_t* keys, uint32_t* slots, void* stream);
int rfs_gather_sorted(const uint32_t* sorted_slots, int n_hits, const uint32_t* h_dev, int hcap, const void* slab,
                      uint32_t* s_ray, float* s_w, void* s_wt, uint32_t* inv_slot, uint64_t* keys, void* stream);
int rfs_gauss_ranges(const uint64_t* sorted_g, int n_hits, const uint32_t* h_dev, int n, int* g_rng, void* stream);


/* K8: TX-batched backward over the shared hit lists, atomic-free and
 * deterministic (every sum in a fixed order).  Replaces the complex part of
 * _ray_backward (_kernels.py:360-387, 522) and the p_acc bincount
 * (grad.py:252-254) for a batch of transmitters.
 * rfs_lam_transpose: lam complex64[B*R] -> lamT complex64[R*B].
 * rfs_bwd_gauss: over the Gaussian-sorted hits (s_slot = slab slot r*hcap+k
 *   of each sorted hit, hcap a power of two), C[slot] = sum_b
 *   conj(lam_b[ray]) psi[g][b] (complex64[R*hcap]; accumulate = 1 adds a
 *   further TX chunk) and P[g][b] = p_acc (complex64[N*B]; rows of Gaussians
 *   without hits are left unwritten).  part: complex64[rfs_bwd_part_elems(H,
 *   B)] and cnt (i32[N + 1]) scratch.  B a multiple of 64 takes the 16-byte-vector
 *   path, whose chunks complete straddling Gaussians themselves (last chunk
 *   to finish sums the partials in chunk order).
 * rfs_bwd_rays: per ray the suffix recursion A_k = w_{k+1} C_{k+1} +
 *   rho_{k+1} A_{k+1} (rho fp64 from geom) and the per-hit scalars
 *   {Re(T C), d|rho|, d(phase) hi, lo}
 *   (float4[R*hcap], slab order) in gs.
 * n_tx <= 256 per rfs_bwd_gauss call. */
int rfs_lam_transpose(const void* lam, int n_tx, int n_rays, void* lamT, void* stream);
size_t rfs_bwd_part_elems(int n_hits, int n_tx);
int rfs_bwd_gauss(int n, int n_hits, const uint32_t* h_dev, int n_tx, const uint64_t* sorted_g, const uint32_t* s_slot,
                  int hcap,
                  const void* s_wt, const int* g_rng, const void* psi, const void* lamT, int accumulate, void* C,
                  void* P, void* part, int* cnt, void* stream);
int rfs_bwd_rays(const void* slab, const int* counts, int hcap, int n_rays, const void* rho32, const void* geom,
                 const void* C, void* gs, void* stream);

/* K9a/K9c: per-Gaussian TX-independent chains in fp64 with a fixed
 * summation order (deterministic): thread per sorted hit with a warp
 * segmented scan, per-warp partials added in warp order for Gaussians whose
 * hits straddle warps, then per Gaussian: mean / covariance chains
 * (_kernels.py:387-520), d|rho|, d(phase), chain_cov_to_shape
 * (grad.py:134-164) and d_trans_mag_raw = d|rho| sigma(1-sigma)
 * (train.py:161-162).  Writes d_mean (direct term), d_quat, d_log_scale,
 * d_trans_mag, d_trans_mag_raw, d_trans_phase, d_cov (nullable); d_mean =
 * direct term + dm_dir (the bearing chain of rfs_grad_tx, nullable; read
 * only for Gaussians with hits).
 * Stage 2 walks the Gaussians with live hits, order[i] for i < min(used_cap,
 * *n_used) (rfs_used_list; n_used nullable), and zeroes every output row
 * of the others.
 * Scratch: acc64 f64[N*14], long_list i32[rfs_geom_part_elems(H)] ([0] =
 * count of the Gaussians whose hits span more than 16 groups of 32, then
 * their ids; stage 1 fills it, stage 2 sums them a block each),
 * part_v f64[14*rfs_geom_part_elems(H)].  stage (bit mask): 1 = the per-hit
 * sums (K9a), 2 = the per-Gaussian chains (K9c) -- so only K9c has to wait
 * for rfs_grad_tx's dm_dir when that runs on another stream. */
size_t rfs_geom_part_elems(int n_hits);
int rfs_grad_geom(int n, int n_hits, const uint32_t* h_dev, const uint64_t* sorted_g, const uint32_t* s_ray, const float* s_w,
                  const uint32_t* s_slot, const void* gs, const int* g_rng, const void* geom, const double* dirs, const double* rx,
                  double ress_radius, const float* quats, const float* log_scales, const float* trans_mag_raw,
                  int used_cap, const uint32_t* n_used, const uint32_t* order,
                  double* acc64, int* long_list, double* part_v, float* d_mean, float* d_quat, float* d_log_scale,
                  float* d_trans_mag, float* d_trans_mag_raw, float* d_trans_phase, float* d_cov, const float* dm_dir,
                  int stage, void* stream);

/* K9b: per-Gaussian TX-dependent terms: d_coeffs = conj(p_acc) conj(basis)
 * (grad.py:255) and the bearing chain of d_mean (grad.py:167-189) into dm_dir
 * (f32[N*3]), from P of rfs_bwd_gauss, for the Gaussians with live hits:
 * order[i], i < min(cap, *n_used) (rfs_used_list; n_used
 * nullable); the d_coeffs rows of the other Gaussians (g_rng of
 * rfs_gauss_ranges empty) are zeroed.  accumulate = 1 adds a further TX
 * chunk's terms (and leaves the zero rows alone).  Run before rfs_grad_geom's
 * stage 2, which adds dm_dir to d_mean. */
int rfs_grad_tx(int cap, const uint32_t* n_used, const uint32_t* order, int n, const int* g_rng, int n_tx, int degree,
                const float* means,
                const void* coeffs, const float* tx, const void* P, int include_direction_chain, int accumulate,
                float* dm_dir, void* d_coeffs, void* stream);

/* Spectrum loss (loss.py:65-155) for n_frames frames [B][n_az*n_el], chained
 * into the rasterizer's upstream (upstream_to_ray, grad.py:104-120).  The
 * predicted power is pred (f32, nullable) or |S|^2 (S complex64, nullable);
 * gt is the ground-truth power (f32).  report (f64[B*4], device) = {total,
 * L1, SSIM, Fourier} per frame; grad (f32[B*R], nullable) = dL/dP; lam
 * (complex64[B*R], nullable, needs S) = 2 dL/dP S; lamT (complex64[R*B],
 * nullable, needs S) the same values ray-major -- the layout rfs_bwd_gauss
 * reads, so the training step needs no transpose.  L1 = mean|d|; SSIM = 1 -
 * mean of the 11x11 sigma-1.5 zero-padded windowed SSIM with C1, C2 from the
 * ground-truth range; Fourier = sum d^2 (= the mean squared DFT difference by
 * Parseval).  Deterministic.  scratch: rfs_loss_scratch_bytes bytes. */
size_t rfs_loss_scratch_bytes(int n_frames, int n_az, int n_el);
int rfs_spectrum_loss(int n_frames, int n_az, int n_el, const void* S, const float* pred, const float* gt,
                      double w_ssim, double w_fourier, double* report, float* grad, void* lam, void* lamT, void* scratch,
                      size_t scratch_bytes, const void* gt_range, void* stream);
/* The per-frame (min, max) partials of the ground truth (SSIM's dynamic range,
 * loss.py:108): float2[rfs_frame_range_elems(B)]; rfs_spectrum_loss computes
 * them itself when gt_range is NULL, or takes them precomputed -- e.g. on the
 * copy stream right behind the frames' H2D copy, off the critical path. */
size_t rfs_frame_range_elems(int n_frames);
int rfs_frame_range(int n_frames, int n_az, int n_el, const float* gt, void* range, void* stream);

/* Scalar (single-antenna) modes: total_b = sum_r S[b][r] (render_scalar,
 * render.py:301-307) and scalar_loss (loss.py:158-180) per frame; mode 0
 * 'complex' (target complex64[B], CSI), mode 1 'real_power' (target[b].x =
 * ground-truth dBm, RSSI).  report f64[B*4] = {value, value, 0, 0}; total
 * (complex64[B], nullable); lam (complex64[B*R], nullable) = the constant
 * per-frame upstream of the coherent sum (train.py:288). */
int rfs_scalar_loss(int n_frames, int n_rays, int mode, const void* S, const void* target, double* report,
                    void* total, void* lam, void* stream);

/* Optimizer and density control (train.py:85-245), in place on the device.
 * rfs_sgd_step: lrs (host float[5]) = {lr_mean(iteration), lr_rotation,
 *   lr_scale, lr_transmittance, lr_radiance}; w -= lr_w dL/dw, quaternions
 *   renormalised, the magnitude gradient chained onto the logit
 *   (train.py:145-162); grad_ema / last_dmean (nullable) get
 *   TrainState.observe (train.py:102-105).  *bad (device i64) = class * N + row
 *   of the first non-finite gradient row (class order of train.py:133-142),
 *   0x7f7f7f7f7f7f7f7f if none -- in which case nothing is updated; prior
 *   (nullable, device i64): the first bad value of earlier steps -- a value
 *   other than the sentinel skips the update too (a training loop that checks
 *   only at its sync points leaves the scene as of its last good step);
 *   lr_mean_dev (nullable, device f32): replaces lrs[0] -- a graph-captured
 *   training iteration reads the schedule's value for its iteration there.
 * rfs_density_flags: mode 0 densify (keep = !split, clone, split: grad_ema >
 *   thr_grad, radius = trace(Sigma)/3 > thr_radius splits), mode 1 prune
 *   (keep = sigmoid(raw) >= thr_prune); u32 flags per Gaussian.
 * rfs_density_apply: with exclusive scans of the flags (keep_off, clone_off,
 *   split_off) and totals = {n_keep, n_clone}, writes the new arrays in the
 *   reference order (kept, clones, two children per split parent); clones are
 *   shifted by -step * last_dmean, children sample mu + R diag(e^s) z with a
 *   Philox4x32-10 stream keyed by (seed, iteration, parent, child) and scales
 *   reduced by log_split_factor; state arrays are reset (densify) or
 *   compacted (prune). */
int rfs_sgd_step(int n, int K, const float* lrs, float ema_decay, const float* d_mean, const float* d_quat,
                 const float* d_log_scale, const float* d_trans_mag, const float* d_trans_phase, const void* d_coeffs,
                 float* means, float* quats, float* log_scales, float* trans_mag_raw, float* trans_phase,
                 void* coeffs, float* grad_ema, float* last_dmean, long long* bad,
                 const long long* prior, const float* lr_mean_dev, void* stream);
int rfs_density_flags(int n, int mode, const float* grad_ema, const float* log_scales, const float* trans_mag_raw,
                      double thr_grad, double thr_radius, double thr_prune, uint32_t* keep, uint32_t* clone,
                      uint32_t* split, void* stream);
int rfs_density_apply(int n, int K, int mode, const uint32_t* keep, const uint32_t* clone, const uint32_t* split,
                      const uint32_t* keep_off, const uint32_t* clone_off, const uint32_t* split_off,
                      const uint32_t* totals, float step, float log_split_factor, unsigned long long seed,
                      int iteration, const float* means, const float* quats, const float* log_scales,
                      const float* trans_mag_raw, const float* trans_phase, const void* coeffs, const float* grad_ema,
                      const float* last_dmean, float* o_means, float* o_quats, float* o_log_scales, float* o_raw,
                      float* o_phase, void* o_coeffs, float* o_ema, float* o_last, void* stream);

/* Synthetic datasets on the GPU (oracle.py:100-177: multipath_signal,
 * spectrum_oracle, rssi_oracle, csi_oracle) for a batch of n_samples TX
 * (tx f64[S*3], device).  paths: n_paths records of rfs_datagen_path_bytes()
 * bytes {f64 reflector[3], amplitude, extra_phase; i32 direct, pad} (device).
 * rfs_spectrum_dataset: gain (complex128[S*P]) / cell (i32[2*S*P]) are
 * scratch, power32 (f32[S*n_az*n_el], nullable) / power64 (f64, nullable) the
 * frames |coherent sum of gain x Gaussian beam|^2.  rfs_scalar_dataset:
 * mode 0 rssi (f64[S] dBm), mode 1 csi (complex128[S*n_sub] at f_c + k
 * spacing).  status (device i32): bit 0 = zero-length path, bit 1 = arrival
 * point on the receiver (the reference's GeometryError). */
size_t rfs_datagen_path_bytes(void);
int rfs_spectrum_dataset(int n_samples, const double* tx, int n_paths, const void* paths, const double* rx,
                         double f_c, int n_az, int n_el, double sigma_beam, int rolloff, void* gain, int* cell,
                         float* power32, double* power64, int* status, void* stream);
int rfs_scalar_dataset(int n_samples, const double* tx, int n_paths, const void* paths, const double* rx,
                       double f_c, int mode, int n_sub, double spacing, int rolloff, double* rssi, void* csi,
                       int* status, void* stream);

/* Library / build identification. */
int rfs_version(void);
int rfs_device_arch(void); /* compute capability the library was built for, e.g. 100 */

#ifdef __cplusplus
}
#endif
#endif /* RFSPLAT_B200_H */
