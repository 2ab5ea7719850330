// datagen.cu -- GPU synthetic datasets: the reference's multipath oracles.
//
// Restates oracle.py:100-153 (multipath_signal, spectrum_oracle, _gain,
// _arrival_bearing) and oracle.py:156-177 (rssi_oracle, csi_oracle) for a
// batch of transmitters, so a training set is produced where it is consumed
// (HBM) instead of by a Python loop over samples and paths.
//
//   k_path_gain   thread per (sample s, path p): path length (direct or
//                 two-leg bounce, oracle.py:86-99), complex gain
//                 A e^{j (2 pi f d / c + theta)} (A / d with rolloff), and the
//                 arrival cell of the last leg (splat.to_spherical / to_grid,
//                 splat.py:121-148), all in fp64 with the reference's
//                 operation order;
//   k_spectrum    thread per (sample, cell): coherent sum over the paths of
//                 gain x circular Gaussian beam kernel
//                 exp(-(du^2 + dv^2) / (2 sigma^2)) with periodic du
//                 (sigma <= 0: a delta at the arrival cell), power |sum|^2;
//   k_scalar      thread per (sample, subcarrier): the coherent sum itself
//                 (rssi: 10 log10 |s|^2 floored at -200 dBm; csi: the
//                 complex response at f_c + k spacing).
#include "rfs_common.cuh"

namespace {

constexpr double SPEED_OF_LIGHT = 3.0e8;  // oracle.py:46

struct PathRec {  // one propagation path (oracle.PathSpec)
    double refl[3];
    double amplitude;
    double extra_phase;
    int direct;  // reflector is None
    int pad;
};

__device__ __forceinline__ double norm3(double x, double y, double z) { return sqrt(x * x + y * y + z * z); }

// oracle.path_length (oracle.py:86-99); <= 0 flags the reference's GeometryError
__device__ double path_len(const PathRec& p, const double* tx, const double* rx) {
    if (p.direct) return norm3(tx[0] - rx[0], tx[1] - rx[1], tx[2] - rx[2]);
    return norm3(tx[0] - p.refl[0], tx[1] - p.refl[1], tx[2] - p.refl[2]) +
           norm3(p.refl[0] - rx[0], p.refl[1] - rx[1], p.refl[2] - rx[2]);
}

__global__ void k_path_gain(int n_s, int n_p, const double* __restrict__ tx, const PathRec* __restrict__ paths,
                            double rx0, double rx1, double rx2, double f_c, int rolloff, int n_az, int n_el,
                            double2* __restrict__ gain, int2* __restrict__ cell, int* __restrict__ status) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_s * n_p) return;
    const int s = i / n_p, pi = i - s * n_p;
    const PathRec p = paths[pi];
    const double t[3] = {tx[3 * s], tx[3 * s + 1], tx[3 * s + 2]};
    const double r[3] = {rx0, rx1, rx2};
    const double d = path_len(p, t, r);
    if (!(d > 0.0)) {
        atomicOr(status, 1);
        return;
    }
    const double amp = rolloff ? p.amplitude / d : p.amplitude;
    const double phase = 2.0 * RFS_PI * f_c * (d / SPEED_OF_LIGHT) + p.extra_phase;
    double sn, cs;
    sincos(phase, &sn, &cs);
    gain[i] = make_double2(amp * cs, amp * sn);
    if (cell) {  // arrival bearing of the last leg (oracle.py:113-117)
        const double* src = p.direct ? t : p.refl;
        const double ox = src[0] - rx0, oy = src[1] - rx1, oz = src[2] - rx2;
        const double dist = norm3(ox, oy, oz);
        if (dist == 0.0) {
            atomicOr(status, 2);
            return;
        }
        double alpha = fmod(atan2(oy, ox), 2.0 * RFS_PI);  // Python % (floor mod) for a divisor > 0
        if (alpha < 0.0) alpha += 2.0 * RFS_PI;
        const double beta = RFS_PI / 2.0 - acos(fmin(fmax(oz / dist, -1.0), 1.0));
        const double cellw = 360.0 / (double)n_az;
        int u = (int)floor(alpha * RFS_RAD2DEG / cellw);
        u = min(max(u, 0), n_az - 1);
        int v = (int)floor((beta * RFS_RAD2DEG + 90.0) / cellw);
        v = min(max(v, 0), n_el - 1);
        cell[i] = make_int2(u, v);
    }
}

__global__ void k_spectrum(int n_s, int n_p, int n_az, int n_el, double sigma_cells,
                           const double2* __restrict__ gain, const int2* __restrict__ cell,
                           float* __restrict__ power32, double* __restrict__ power64) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int R = n_az * n_el;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int s = blockIdx.y;
    if (r >= R) return;
    const int u = r / n_el, v = r - u * n_el;
    double fr = 0.0, fi = 0.0;
    const double two_s2 = 2.0 * (sigma_cells * sigma_cells);
    for (int p = 0; p < n_p; ++p) {
        const double2 g = gain[(size_t)s * n_p + p];
        const int2 c = cell[(size_t)s * n_p + p];
        if (sigma_cells <= 0.0) {
            if (c.x == u && c.y == v) {
                fr += g.x;
                fi += g.y;
            }
            continue;
        }
        int du = abs(u - c.x);
        du = min(du, n_az - du);
        const int dv = v - c.y;
        const double k = exp(-(double)(du * du + dv * dv) / two_s2);
        fr += g.x * k;
        fi += g.y * k;
    }
    const double a = hypot(fr, fi);  // np.abs(field) ** 2
    const double pw = a * a;
    if (power32) power32[(size_t)s * R + r] = (float)pw;
    if (power64) power64[(size_t)s * R + r] = pw;
}

// mode 0 rssi: out64[s] = 10 log10 |sum|^2 (-200 below 1e-20); mode 1 csi:
// out_c[s][k] = sum at f_c + k spacing (gains computed per subcarrier)
__global__ void k_scalar(int n_s, int n_p, int n_sub, int mode, const double* __restrict__ tx,
                         const PathRec* __restrict__ paths, double rx0, double rx1, double rx2, double f_c,
                         double spacing, int rolloff, double* __restrict__ rssi, double2* __restrict__ csi,
                         int* __restrict__ status) {
    rfs_pdl_wait();  // programmatic dependent launch: the previous kernel's writes are visible
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_s * n_sub) return;
    const int s = i / n_sub, k = i - s * n_sub;
    const double f = f_c + (double)k * spacing;
    const double t[3] = {tx[3 * s], tx[3 * s + 1], tx[3 * s + 2]};
    const double r[3] = {rx0, rx1, rx2};
    double re = 0.0, im = 0.0;
    for (int pi = 0; pi < n_p; ++pi) {
        const PathRec p = paths[pi];
        const double d = path_len(p, t, r);
        if (!(d > 0.0)) {
            atomicOr(status, 1);
            return;
        }
        const double amp = rolloff ? p.amplitude / d : p.amplitude;
        double sn, cs;
        sincos(2.0 * RFS_PI * f * (d / SPEED_OF_LIGHT) + p.extra_phase, &sn, &cs);
        re += amp * cs;
        im += amp * sn;
    }
    if (mode == 0) {
        const double a = hypot(re, im);
        const double pw = a * a;
        rssi[s] = pw <= 1e-20 ? -200.0 : 10.0 * log10(pw);
    } else {
        csi[i] = make_double2(re, im);
    }
}

}  // namespace

extern "C" {

size_t rfs_datagen_path_bytes(void) { return sizeof(PathRec); }

int rfs_spectrum_dataset(int n_samples, const double* tx, int n_paths, const void* paths, const double* rx,
                         double f_c, int n_az, int n_el, double sigma_beam, int rolloff, void* gain, int* cell,
                         float* power32, double* power64, int* status, void* stream) {
    if (n_samples <= 0) return RFS_OK;
    if (n_paths <= 0 || n_az <= 0 || n_el <= 0) return RFS_ERR_SHAPE;
    cudaStream_t st = (cudaStream_t)stream;
    RFS_CUDA_TRY(rfs_fill_u32(status, 0u, 1, st));
    const int np = n_samples * n_paths;
    rfs_launch(k_path_gain, rfs_ceil_div(np, 128), 128, 0, st, n_samples, n_paths, tx, (const PathRec*)paths, rx[0], rx[1],
                                                       rx[2], f_c, rolloff, n_az, n_el, (double2*)gain, (int2*)cell,
                                                       status);
    const double sigma_cells = sigma_beam / (360.0 / (double)n_az);
    dim3 grid(rfs_ceil_div(n_az * n_el, 256), n_samples);
    rfs_launch(k_spectrum, grid, 256, 0, st, n_samples, n_paths, n_az, n_el, sigma_cells, (const double2*)gain,
                                     (const int2*)cell, power32, power64);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

int rfs_scalar_dataset(int n_samples, const double* tx, int n_paths, const void* paths, const double* rx,
                       double f_c, int mode, int n_sub, double spacing, int rolloff, double* rssi, void* csi,
                       int* status, void* stream) {
    if (n_samples <= 0) return RFS_OK;
    if (n_paths <= 0 || (mode != 0 && mode != 1) || (mode == 1 && n_sub <= 0)) return RFS_ERR_SHAPE;
    cudaStream_t st = (cudaStream_t)stream;
    RFS_CUDA_TRY(rfs_fill_u32(status, 0u, 1, st));
    const int ns = mode == 0 ? 1 : n_sub;
    rfs_launch(k_scalar, rfs_ceil_div(n_samples * ns, 128), 128, 0, st, n_samples, n_paths, ns, mode, tx,
                                                                 (const PathRec*)paths, rx[0], rx[1], rx[2], f_c,
                                                                 spacing, rolloff, rssi, (double2*)csi, status);
    RFS_LAUNCH_CHECK();
    return RFS_OK;
}

}  // extern "C"
