// hit.cuh -- the per-(ray, record) device functions shared by K5/K6 (render.cu) and the
// backward kernel (backward.cu): pixel ray, record colour, exact hit + Eq. 8 + Eq. 9.
// Product code; nothing here is shared with oracle/.
#pragma once

#include <math.h>

#include "snp_internal.cuh"

namespace snp {
namespace {

struct Ray {
    float dhx, dhy, dhz, dlx, dly, dlz;   // unit direction, hi + lo
    float t_near, t_far;
};

__device__ __forceinline__ Ray make_ray(const DevCam &cam, int x, int y) {
    // d = normalize(R_wc ((x+.5-cx)/fx, (y+.5-cy)/fy, 1)) in FP64 (R6), split into hi + lo
    const double u = ((double)x + 0.5 - (double)cam.cx) * cam.ifx;
    const double v = ((double)y + 0.5 - (double)cam.cy) * cam.ify;
    double r[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        r[i] = (double)cam.R[3 * i] * u + (double)cam.R[3 * i + 1] * v + (double)cam.R[3 * i + 2];
    const double inv = rsqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    Ray ray;
    const double d0 = r[0] * inv, d1 = r[1] * inv, d2 = r[2] * inv;
    ray.dhx = (float)d0; ray.dlx = (float)(d0 - (double)ray.dhx);
    ray.dhy = (float)d1; ray.dly = (float)(d1 - (double)ray.dhy);
    ray.dhz = (float)d2; ray.dlz = (float)(d2 - (double)ray.dhz);
    ray.t_near = cam.t_near;
    ray.t_far = cam.t_far;
    return ray;
}

// Colour of primitive id for this pixel, as (_, r, g, b) like the record's kRecConicRgb
// slot.  kRay = false: the record's colour (SH at normalize(mu - C), per primitive and
// view, R14).  kRay = true: the SH of the scene's coefficients at the
// pixel's own unit ray direction, c = max(0, sum_lm Y_lm(d) sh_lm + 0.5) (R15);
// fp32 suffices, colour enters the pixel linearly.
template <bool kRay>
__device__ __forceinline__ float4 hit_rgb(const float4 *rec, const float *sh_all, int degree, uint32_t id,
                                          const Ray &r) {
    if (!kRay) return __ldg(rec + kRecConicRgb);
    const float4 *sh4 = reinterpret_cast<const float4 *>(sh_all + (size_t)48 * id);
    const float x = r.dhx, y = r.dhy, z = r.dhz;
    const float xx = x * x, yy = y * y, zz = z * z;
    float Y[16];
    Y[0] = 0.28209479177387814f;
    Y[1] = -0.4886025119029199f * y;
    Y[2] = 0.4886025119029199f * z;
    Y[3] = -0.4886025119029199f * x;
    Y[4] = 1.0925484305920792f * (x * y);
    Y[5] = -1.0925484305920792f * (y * z);
    Y[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
    Y[7] = -1.0925484305920792f * (x * z);
    Y[8] = 0.5462742152960396f * (xx - yy);
    Y[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
    Y[10] = 2.890611442640554f * (x * y) * z;
    Y[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
    Y[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    Y[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
    Y[14] = 1.445305721320277f * z * (xx - yy);
    Y[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
    const int nc = (degree + 1) * (degree + 1);
    float acc[3] = {0.5f, 0.5f, 0.5f};
#pragma unroll
    for (int q = 0; q < 12; ++q) {       // coefficients 4q/3 .. : 4 floats per load, RGB innermost
        const float4 t = __ldg(sh4 + q);
        const float v[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int f = 4 * q + u, i = f / 3, c = f % 3;
            if (i < nc) acc[c] = fmaf(Y[i], v[u], acc[c]);
        }
    }
    return make_float4(0.f, fmaxf(acc[0], 0.f), fmaxf(acc[1], 0.f), fmaxf(acc[2], 0.f));
}

// MUFU sin/cos take the argument through one FMUL by 1/(2 pi): for |phase| <= 60 rad
// (|omega W1| <= 17 rad per unit radius, |omega b1| <= 30) that rounding costs <= 4e-6 rad,
// i.e. <= 4e-6 * |W2 dt| per hidden unit -- well inside the 1e-4 pixel tolerance.
// sinc uses its Taylor polynomial below |x| = 0.25 where sin(x)/x loses relative accuracy.
// MUFU reciprocal (rcp.approx: ~1 ulp), no special-case handling: callers divide by
// values bounded away from 0 and infinity.
__device__ __forceinline__ float rcp_fast(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float sinc_f(float x) {
    const float x2 = x * x;
    // 1 - x^2/6 + x^4/120; the dropped x^6/5040 term is < 5e-8 below |x| = 0.25
    const float poly = fmaf(x2, fmaf(x2, 8.3333333e-03f, -1.6666667e-01f), 1.0f);
    const float s = __sinf(x) * rcp_fast(x);
    return fabsf(x) < 0.25f ? poly : s;
}

// Exact hit + kernel for one (ray, record) of N hidden units.  Returns false on a miss.
template <int N>
__device__ __forceinline__ bool exact_hit(const float4 *__restrict__ rec, const Ray &r, float &t_hi, float &t_lo,
                                          float &kap) {
    const float4 mh = rec[kRecMh];
    const float4 ml = rec[kRecMl];
    const float4 w0 = rec[kRecWh0];
    const float4 w1 = rec[kRecWh1];
    // closest-approach parameter and compensated offset p = t_c d - m (|p| ~ s, not ~ distance)
    const float tc = fmaf(r.dhz, mh.z, fmaf(r.dhy, mh.y, r.dhx * mh.x));
    const float px = fmaf(tc, r.dhx, -mh.x) + fmaf(tc, r.dlx, -ml.x);
    const float py = fmaf(tc, r.dhy, -mh.y) + fmaf(tc, r.dly, -ml.y);
    const float pz = fmaf(tc, r.dhz, -mh.z) + fmaf(tc, r.dlz, -ml.z);
    // unit-sphere frame: a = Wh d, b = Wh p;  |b + tau a|^2 = 1
    const float ax = fmaf(w0.y, r.dhz, fmaf(w0.x, r.dhy, ml.w * r.dhx));
    const float ay = fmaf(w1.x, r.dhz, fmaf(w0.w, r.dhy, w0.z * r.dhx));
    const float az = fmaf(w1.w, r.dhz, fmaf(w1.z, r.dhy, w1.y * r.dhx));
    const float bx = fmaf(w0.y, pz, fmaf(w0.x, py, ml.w * px));
    const float by = fmaf(w1.x, pz, fmaf(w0.w, py, w0.z * px));
    const float bz = fmaf(w1.w, pz, fmaf(w1.z, py, w1.y * px));
    // roots about the ray's closest approach to the centre in the unit-sphere metric,
    // tau* = -(a.b)/|a|^2, from the perpendicular offset b_perp = b + tau* a (one FMA
    // per component): 1 - |b_perp|^2 is O(1) accurate even for needle- or sheet-like
    // ellipsoids, where B^2 - AC cancels catastrophically in fp32
    const float A = fmaf(az, az, fmaf(ay, ay, ax * ax));
    const float B = fmaf(az, bz, fmaf(ay, by, ax * bx));
    const float iA = rcp_fast(A);
    const float ts = -B * iA;
    const float qx = fmaf(ts, ax, bx), qy = fmaf(ts, ay, by), qz = fmaf(ts, az, bz);
    const float q1 = 1.0f - fmaf(qz, qz, fmaf(qy, qy, qx * qx));
    if (!(q1 > 0.0f)) return false;
    const float hq = q1 * iA;
    const float hc = hq * rsqrtf(hq);   // half chord
    const float t0 = ts - hc, t1 = ts + hc;
    const float lo_lim = r.t_near - tc, hi_lim = r.t_far - tc;
    const bool clipped = !(t0 > lo_lim);
    const float tlo = clipped ? lo_lim : t0;
    const float thi = t1 < hi_lim ? t1 : hi_lim;
    if (!(thi > tlo)) return false;
    const float dt = thi - tlo;
    const float tm = 0.5f * (tlo + thi);
    const float hdt = 0.5f * dt;
    float acc = 0.f;
    float W2[N];
#pragma unroll
    for (int j = 0; j < N / 4; ++j) {
        const float4 w = rec[rec_w2(N) + j];
        W2[4 * j] = w.x; W2[4 * j + 1] = w.y; W2[4 * j + 2] = w.z; W2[4 * j + 3] = w.w;
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const float4 u = rec[kRecUnits + k];
        const float h = fmaf(u.z, r.dhz, fmaf(u.y, r.dhy, u.x * r.dhx));
        const float g = fmaf(u.z, pz, fmaf(u.y, py, fmaf(u.x, px, u.w)));
        const float phi = fmaf(h, tm, g);
        acc = fmaf(W2[k], __cosf(phi) * sinc_f(h * hdt), acc);
    }
    const float I = dt * (acc + mh.w);
    kap = 1.0f - __expf(-fmaxf(I, 0.0f));
    if (clipped) {
        t_hi = r.t_near;
        t_lo = 0.f;
    } else {  // TwoSum(tc, t0): t_in = t_hi + t_lo exactly
        const float s = tc + t0;
        const float bb = s - tc;
        t_hi = s;
        t_lo = (tc - (s - bb)) + (t0 - bb);
    }
    return true;
}

__device__ __forceinline__ bool before(float ah, float al, uint32_t aid, float bh, float bl, uint32_t bid) {
    return ah < bh || (ah == bh && (al < bl || (al == bl && aid < bid)));
}

}  // namespace
}  // namespace snp
