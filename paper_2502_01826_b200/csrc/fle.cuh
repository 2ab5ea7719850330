// fle.cuh -- Fourier-Legendre directional basis on the device.
//
// e^{i m alpha} P_l^m(cos beta) with the Condon-Shortley phase, flat index
// l*l + l + m (fle.py:46-50), and its alpha / beta derivatives
// (fle_basis_with_derivs, fle.py:153-212).  Evaluated in fp32 from the
// bearing vector r = tx - mu without trigonometry: cos(beta) = rho/|r|,
// sin(beta) = z/|r|, e^{i alpha} = (x + i y)/rho -- the same angles as the
// reference's atan2 / arccos route (render.py:229-236), better conditioned.
#pragma once
#include "rfs_common.cuh"

template <int L>
struct Fle {
    static constexpr int K = (L + 1) * (L + 1);

    struct Tables {
        float p[L + 1][L + 1], dp[L + 1][L + 1];
        float2 em[L + 1];
    };

    __device__ static __forceinline__ void tables(float rx, float ry, float rz, Tables& T) {
        const float d2 = rx * rx + ry * ry + rz * rz;
        const float rho2 = rx * rx + ry * ry;
        bool valid = d2 > 1e-24f;  // render.py:231 (bearing_valid: |r| > 1e-12)
        float x, sig, ca, sa;
        if (valid) {
            const float id = rsqrtf(d2);
            sig = rz * id;
            if (rho2 > 0.f) {
                const float ir = rsqrtf(rho2);
                x = rho2 * ir * id;
                ca = rx * ir;
                sa = ry * ir;
            } else {
                x = 0.f;
                float a = atan2f(ry, rx);
                sincosf(a, &sa, &ca);
            }
        } else {
            x = 1.f; sig = 0.f; ca = 1.f; sa = 0.f;
        }
        float s = fabsf(sig);
        float sgn = (sig > 0.f) ? 1.f : ((sig < 0.f) ? -1.f : 0.f);
        float dx = -sig, ds = sgn * x;
#pragma unroll
        for (int m = 0; m <= L; ++m) {
            float c = ((m & 1) ? -1.f : 1.f);
#pragma unroll
            for (int t = 2 * m - 1; t > 1; t -= 2) c *= (float)t;
            float sm = 1.f, sm1 = 1.f;
#pragma unroll
            for (int t = 0; t < m; ++t) sm *= s;
#pragma unroll
            for (int t = 0; t < m - 1; ++t) sm1 *= s;
            T.p[m][m] = c * sm;
            T.dp[m][m] = m > 0 ? c * (float)m * sm1 * ds : 0.f;
            if (m + 1 <= L) {
                T.p[m + 1][m] = x * (float)(2 * m + 1) * T.p[m][m];
                T.dp[m + 1][m] = (float)(2 * m + 1) * (dx * T.p[m][m] + x * T.dp[m][m]);
            }
#pragma unroll
            for (int l = m + 2; l <= L; ++l) {
                float a = (float)(2 * l - 1), b = (float)(l + m - 1), inv = 1.f / (float)(l - m);
                T.p[l][m] = (x * a * T.p[l - 1][m] - b * T.p[l - 2][m]) * inv;
                T.dp[l][m] = (dx * a * T.p[l - 1][m] + x * a * T.dp[l - 1][m] - b * T.dp[l - 2][m]) * inv;
            }
        }
        T.em[0] = make_float2(1.f, 0.f);
#pragma unroll
        for (int m = 1; m <= L; ++m) T.em[m] = cmulf(T.em[m - 1], make_float2(ca, sa));
    }

    // (-1)^m (l-m)!/(l+m)! for negative orders (fle.py:99-100, 121-124)
    __device__ static __forceinline__ float ratio(int l, int m) {
        if (m >= 0) return 1.f;
        int ma = -m;
        float num = 1.f, den = 1.f;
        for (int t = 2; t <= l - ma; ++t) num *= (float)t;
        for (int t = 2; t <= l + ma; ++t) den *= (float)t;
        return ((ma & 1) ? -1.f : 1.f) * (num / den);
    }

    // Calls f(idx, m, basis, dbasis/dbeta) for every basis function.
    template <class F>
    __device__ static __forceinline__ void for_each(const Tables& T, F&& f) {
#pragma unroll
        for (int l = 0; l <= L; ++l) {
#pragma unroll
            for (int m = -l; m <= l; ++m) {
                const int ma = m < 0 ? -m : m;
                const float rt = ratio(l, m);
                const float2 az = m < 0 ? make_float2(T.em[ma].x, -T.em[ma].y) : T.em[ma];
                const float pv = rt * T.p[l][ma], dv = rt * T.dp[l][ma];
                f(l * l + l + m, m, make_float2(az.x * pv, az.y * pv), make_float2(az.x * dv, az.y * dv));
            }
        }
    }

    // psi = sum_k c_k basis_k (render.py:238)
    __device__ static __forceinline__ float2 psi(float rx, float ry, float rz, const float2* __restrict__ c) {
        Tables T;
        tables(rx, ry, rz, T);
        // acc += c_k b_k as paired fp32 FMAs (FFMA2): (re, im) += c.x (b.x, b.y) + c.y (-b.y, b.x)
        float2 acc = make_float2(0.f, 0.f);
        for_each(T, [&](int idx, int, float2 b, float2) {
            const float2 ck = __ldg(&c[idx]);
            acc = __ffma2_rn(make_float2(ck.x, ck.x), b, acc);
            acc = __ffma2_rn(make_float2(ck.y, ck.y), make_float2(-b.y, b.x), acc);
        });
        return acc;
    }
};
