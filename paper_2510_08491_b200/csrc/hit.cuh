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

// dL/dI and dL/dc of one composited hit (K5 grad mode; K7s from recorded hits -- the same
// arithmetic in both): out = sum_j T_j k_j c_j + T_end bg, so the light behind the hit is
// U = F - (colour accumulated up to and including it); dL/dk = G_rgb . (T c - U / (1 - k))
// + G_a T_end / (1 - k), dL/dI = (1 - k) dL/dk for I > 0 (Eq. 9), dL/dc = T k G_rgb on
// unclamped channels.  G = dL/d(out), F = out, Tb = T before the hit, rgb in .yzw.
__device__ __forceinline__ void hit_out_grads(const float4 &G, const float4 &F, float Tb, float kap, const float4 &rgb,
                                              float cr, float cg, float cb, float &gI, float gc[3]) {
    const float iom = rcp_fast(fmaxf(1.0f - kap, 1e-20f));
    float dk = G.w * (1.0f - F.w) * iom;
    dk = fmaf(G.x, fmaf(-(F.x - cr), iom, Tb * rgb.y), dk);
    dk = fmaf(G.y, fmaf(-(F.y - cg), iom, Tb * rgb.z), dk);
    dk = fmaf(G.z, fmaf(-(F.z - cb), iom, Tb * rgb.w), dk);
    const float w = Tb * kap;
    gI = kap > 0.f ? dk * (1.0f - kap) : 0.f;
    gc[0] = rgb.y > 0.f ? w * G.x : 0.f;
    gc[1] = rgb.z > 0.f ? w * G.y : 0.f;
    gc[2] = rgb.w > 0.f ? w * G.z : 0.f;
}
__device__ __forceinline__ float sinc_f(float x) {
    const float x2 = x * x;
    // 1 - x^2/6 + x^4/120; the dropped x^6/5040 term is < 5e-8 below |x| = 0.25
    const float poly = fmaf(x2, fmaf(x2, 8.3333333e-03f, -1.6666667e-01f), 1.0f);
    const float s = __sinf(x) * rcp_fast(x);
    return fabsf(x) < 0.25f ? poly : s;
}

// ---- rare FP64 branch for grazing rays (R23)
// The chord of a ray that grazes an ellipsoid is hc = sqrt(Q / |a|^2), Q = 1 - |b_perp|^2.
// In fp32, Q carries an absolute error of a few 1e-7 (the record's fp32 whitening matrix,
// the rounding of |b_perp|^2), i.e. a relative chord error ~ 2e-7 / Q, which a dense
// primitive turns into a kappa error ~ I exp(-I) x 2e-7 / Q: 2e-4 at Q = 1e-4, I = 1.
// Below kGrazeQ the roots are recomputed in FP64 from the primitive's own parameters
// (mu, q, s), which bounds that error by ~4e-6 at the threshold and
// ~1e-13 below it; the integral then runs in fp32 on the accurate segment as usual.
constexpr float kGrazeQ = 4e-3f;
// K5 (fp32 only): a hit whose kappa may be off by more than kGrazeK0 carries an error
// exponent e; it is blended in fp32 only while T 2^e <= 2, i.e. while its share of the
// pixel, T dkappa |c - behind| <= T kGrazeK0 2^e x 2 (colours <= 2), stays <= 6e-5
constexpr float kGrazeK0 = 1.5e-5f;
struct Prec64 {
    const float *centers, *rotations, *scales;   // scene parameters [n][3], [n][4], [n][3]
    float cx, cy, cz;                             // camera centre
};

// Segment [t0, t1] of ray C + t d inside the ellipsoid of primitive id, clipped to
// [t_near, t_far], in FP64; returned relative to tc (the fp32 path's origin of tau).
// Returns false on a miss.
__device__ __forceinline__ bool roots_f64(const Prec64 &g, uint32_t id, const Ray &r, float tc, float &tlo_rel,
                                       float &thi_rel, int &clipped, double &t_in) {
    const double d[3] = {(double)r.dhx + (double)r.dlx, (double)r.dhy + (double)r.dly,
                         (double)r.dhz + (double)r.dlz};
    const float *q4 = g.rotations + 4 * (size_t)id;
    const float *s3 = g.scales + 3 * (size_t)id;
    const float *m3 = g.centers + 3 * (size_t)id;
    double w = q4[0], x = q4[1], y = q4[2], z = q4[3];
    const double qn = 1.0 / sqrt(w * w + x * x + y * y + z * z);   // (R8: normalised on read)
    w *= qn; x *= qn; y *= qn; z *= qn;
    // columns of R(q) (w, x, y, z); Wh = diag(1/s) R^T has them as rows
    const double R[9] = {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y),
                         2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
                         2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)};
    const double o[3] = {(double)g.cx - (double)m3[0], (double)g.cy - (double)m3[1], (double)g.cz - (double)m3[2]};
    double a[3], b[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double is = 1.0 / (double)s3[k];
        a[k] = (R[k] * d[0] + R[3 + k] * d[1] + R[6 + k] * d[2]) * is;
        b[k] = (R[k] * o[0] + R[3 + k] * o[1] + R[6 + k] * o[2]) * is;
    }
    const double A = a[0] * a[0] + a[1] * a[1] + a[2] * a[2];
    const double ts = -(a[0] * b[0] + a[1] * b[1] + a[2] * b[2]) / A;
    const double p0 = b[0] + ts * a[0], p1 = b[1] + ts * a[1], p2 = b[2] + ts * a[2];
    const double Q = 1.0 - (p0 * p0 + p1 * p1 + p2 * p2);
    if (!(Q > 0.0)) return false;
    const double hc = sqrt(Q / A);
    const double t0 = ts - hc, t1 = ts + hc;
    const double lo = t0 > (double)r.t_near ? t0 : (double)r.t_near;
    const double hi = t1 < (double)r.t_far ? t1 : (double)r.t_far;
    if (!(hi > lo)) return false;
    clipped = !(t0 > (double)r.t_near);
    t_in = lo;
    tlo_rel = (float)(lo - (double)tc);
    thi_rel = (float)(hi - (double)tc);
    return true;
}

// Exact hit + kernel for one (ray, record) of N hidden units, primitive id.  Returns
// false on a miss.  Grazing rays (|Q| < kGrazeQ): kGraze = kGrazeInline takes the FP64
// branch in place (K6, K7); kGraze = kGrazeDefer (K5) stays in fp32 and reports, in
// *graze / *gexp, how far the chord's rounding could move kappa: K5 blends the hit or
// hands the pixel to K6 (no FP64 code or registers in K5's hot loop).
enum { kGrazeInline = 0, kGrazeDefer = 1 };
template <int N, int kGraze>
__device__ __forceinline__ bool exact_hit(const float4 *__restrict__ rec, const Ray &r, float &t_hi, float &t_lo,
                                          float &kap, const Prec64 *g, uint32_t id, bool *graze = nullptr,
                                          int *gexp = nullptr) {
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
    float tlo, thi, hc = 0.f;
    bool clipped;
    double t_in64 = 0.0;
    bool f64 = false;
    if (kGraze == kGrazeInline && q1 < kGrazeQ && q1 > -kGrazeQ) {   // grazing (or a near miss): FP64 roots
        int cl = 0;
        if (!roots_f64(*g, id, r, tc, tlo, thi, cl, t_in64)) return false;
        clipped = cl != 0;
        f64 = true;
    } else {
        if (!(q1 > 0.0f)) return false;
        const float hq = q1 * iA;
        hc = hq * rsqrtf(hq);   // half chord
        const float t0 = ts - hc, t1 = ts + hc;
        const float lo_lim = r.t_near - tc, hi_lim = r.t_far - tc;
        clipped = !(t0 > lo_lim);
        tlo = clipped ? lo_lim : t0;
        thi = t1 < hi_lim ? t1 : hi_lim;
        if (!(thi > tlo)) return false;
    }
    const float dt = thi - tlo;
    const float tm = 0.5f * (tlo + thi);
    const float hdt = 0.5f * dt;
    // phase at the segment's midpoint x_m = p + tau_m d (relative to mu) and the half
    // segment hdt d: g_k + h_k tau_m = W1'_k.x_m + omega b1_k, h_k hdt = W1'_k.(hdt d)
    const float xmx = fmaf(tm, r.dhx, px), xmy = fmaf(tm, r.dhy, py), xmz = fmaf(tm, r.dhz, pz);
    const float hx = hdt * r.dhx, hy = hdt * r.dhy, hz = hdt * r.dhz;
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
        const float phi = fmaf(u.z, xmz, fmaf(u.y, xmy, fmaf(u.x, xmx, u.w)));
        const float x = fmaf(u.z, hz, fmaf(u.y, hy, u.x * hx));
        acc = fmaf(W2[k], __cosf(phi) * sinc_f(x), acc);
    }
    const float I = dt * (acc + mh.w);
    kap = 1.0f - __expf(-fmaxf(I, 0.0f));
    if (kGraze == kGrazeDefer) {
        // kappa's error from the fp32 chord: |dkappa| <= (1 - kappa) |I| |d dt| / dt with
        // |d dt| <= 2 |d hc| = hc dQ / Q, dQ <= 3.6e-7 (measured maximum of the fp32 Q over
        // grazing C3 rays, R23).  Reported as an exponent e >= ceil(log2(dkappa /
        // kGrazeK0)) (from the float exponents: no division), clamped to 1..7, when dkappa may
        // exceed kGrazeK0 (0: negligible); the pixel's emission then decides, knowing the
        // transmittance in front of the hit (render.cu)
        *graze = false;
        if (q1 < kGrazeQ) {   // (rare)
            const float num = (1.0f - kap) * fabsf(I) * hc * (3.6e-7f / kGrazeK0);
            const float den = q1 * dt;
            const int e = (int)(__float_as_uint(num) >> 23) - (int)(__float_as_uint(den) >> 23) + 1;
            *graze = e > 0 && num > 0.0f;
            *gexp = min(7, max(1, e));
        }
    }
    if (clipped) {
        t_hi = r.t_near;
        t_lo = 0.f;
    } else if (f64) {
        t_hi = (float)t_in64;
        t_lo = (float)(t_in64 - (double)t_hi);
    } else {  // TwoSum(tc, t0): t_in = t_hi + t_lo exactly
        const float s = tc + tlo;
        const float bb = s - tc;
        t_hi = s;
        t_lo = (tc - (s - bb)) + (tlo - bb);
    }
    return true;
}

__device__ __forceinline__ bool before(float ah, float al, uint32_t aid, float bh, float bl, uint32_t bid) {
    return ah < bh || (ah == bh && (al < bl || (al == bl && aid < bid)));
}

}  // namespace
}  // namespace snp
