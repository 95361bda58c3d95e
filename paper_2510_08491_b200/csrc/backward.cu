// backward.cu -- K7: backward of the forward render:
// dL/d{W1, b1, W2, b2, SH} and (optionally) dL/d{mu, q, s} of every primitive for a
// given dL/d(out RGBA).  The per-ray hit order and the T-floor stop are piecewise
// constant in the parameters and carry no gradient.
//
// One warp per pixel.  The warp re-derives its pixel's forward exactly as K6 does --
// every hit of the tile list (conic pre-test + exact_hit), sorted by (t_in, id)
// (R11), front-to-back transmittance with the T < floor stop (Eq. 4) --
// then walks the composited hits back to front:
//   out_rgb = sum_i T_i k_i c_i + T_end bg,  alpha = 1 - T_end,  T_i = prod_{j<i} (1 - k_j)
//   dL/dk_i = G_rgb . (T_i c_i - U_i / (1 - k_i)) + G_a T_end / (1 - k_i),
//             U_i = sum_{j>i} T_j k_j c_j + T_end bg
//   dL/dI_i = dL/dk_i (1 - k_i) for I_i > 0 (Eq. 9), 0 otherwise
//   dL/dc_i = T_i k_i G_rgb (per channel where c_i > 0: c = max(0, SH + 0.5))
// and differentiates Eq. 8 in product form (R3), I = dt (sum_k W2_k cos(phi_k)
// sinc(h_k dt / 2) + b2), phi_k = g_k + h_k tau_m, g_k = W1'_k . p + omega b1_k,
// h_k = W1'_k . d, W1' = omega W1 / ||s||_inf:
//   dI/dW2_k = dt cos(phi_k) S_k,   dI/db2 = dt,
//   dI/db1_k = -omega dt W2_k sin(phi_k) S_k,
//   dI/dW1_k = (omega / ||s||_inf) dt W2_k (-sin(phi_k) S_k (p + tau_m d) + cos(phi_k) S'_k (dt/2) d),
//   S_k = sinc(h_k dt / 2), S' = d sinc / dx.
// Gradients are accumulated with fp32 atomics.  Pixels with more than kBwHits hits are
// redone by one-warp CTAs that hold kBwBigHits in shared memory, and pixels with more
// than that by one-warp CTAs whose arrays live in a global scratch (kBwHugeHits each);
// only beyond that (tile lists of more than 16384 hits per ray) is a pixel skipped,
// counted in counters[kCntBwdSkipped] (reset by every call, reported by snp_get_stats).
#include <algorithm>
#include <type_traits>

#include "hit.cuh"
#include "snp_internal.cuh"

namespace snp {
namespace {

constexpr int kBwWarps = 8;
constexpr int kBwThreads = kBwWarps * 32;
constexpr int kBwHits = 256;
constexpr int kBwQueue = 64;
// pixels with more than kBwHits hits are redone by one-warp CTAs holding kBwBigHits,
// and beyond that by kBwHugeCtas one-warp CTAs with kBwHugeHits in global memory
constexpr int kBwBigHits = 2048;
constexpr int kBwHugeHits = 16384;
constexpr int kBwHugeCtas = 64;

template <int kBwWarps, int kBwHits>
struct BwSmem {
    float th[kBwWarps][kBwHits], tl[kBwWarps][kBwHits], kap[kBwWarps][kBwHits];
    uint32_t id[kBwWarps][kBwHits];
    uint32_t ord[kBwWarps][kBwHits];           // sorted position -> hit slot
    float T[kBwWarps][kBwHits];                // transmittance before each sorted hit
    float gI[kBwWarps][kBwHits];               // dL/dI per sorted hit
    float gc[kBwWarps][kBwHits][3];            // dL/dc per sorted hit (clamped channels: 0)
    int ncomp[kBwWarps];
    // per-warp queue of composited hits awaiting their parameter gradients: the warp
    // drains it 32 hits at a time (all lanes busy) across its successive pixels
    float q_ray[kBwWarps][6][kBwQueue];        // pixel ray, hi + lo
    uint32_t q_vl[kBwWarps][kBwQueue];         // camera index within the batch
    uint32_t q_id[kBwWarps][kBwQueue];
    float q_gI[kBwWarps][kBwQueue];
    float q_gc[kBwWarps][3][kBwQueue];
};

__device__ __forceinline__ void add1(float *p, float a) {
#ifdef SNP_AB_NOATOM
    asm volatile("" ::"f"(a), "l"(p));
#else
    atomicAdd(p, a);
#endif
}

// Four consecutive gradient entries: one 16-byte vector atomic (red.global.add.v4.f32,
// sm_90+) when the arrays are 16-byte aligned (gr.vec), else four scalar atomics.
__device__ __forceinline__ void add4(float *p, float a, float b, float c, float d, bool vec) {
#ifdef SNP_AB_NOATOM   // A/B: the arithmetic without the gradient atomics
    asm volatile("" ::"f"(a), "f"(b), "f"(c), "f"(d), "l"(p));
    return;
#endif
    if (vec) {
        atomicAdd(reinterpret_cast<float4 *>(p), make_float4(a, b, c, d));
    } else {
        atomicAdd(p, a);
        atomicAdd(p + 1, b);
        atomicAdd(p + 2, c);
        atomicAdd(p + 3, d);
    }
}

__device__ __forceinline__ float dsinc_f(float x) {
    // d/dx sin(x)/x = (cos x - sinc x) / x; Taylor -x/3 + x^3/30 below |x| = 0.25
    const float x2 = x * x;
    if (fabsf(x) < 0.25f) return x * fmaf(x2, 1.0f / 30.0f, -1.0f / 3.0f);
    const float ix = rcp_fast(x);
    return (__cosf(x) - __sinf(x) * ix) * ix;
}

// dL/dI (gI) of one (ray, record) hit into the gradients of primitive `prim`: the MLP
// parameters always, the geometry (mu, q, s) when gr.mu is set.  The forward values are
// recomputed exactly as exact_hit (hit.cuh) does; the geometry adjoints follow the
// chain p = t_c d - m (m = mu - C, t_c = d.m), a = Wh d, b = Wh p (Wh = S^-1 R^T),
// A = |a|^2, B = a.b, tau* = -B/A, b_perp = b + tau* a, Q = 1 - |b_perp|^2,
// hc = sqrt(Q/A), [t0, t1] = tau* -/+ hc clipped to [t_near - t_c, t_far - t_c],
// dt = t1 - t0, tau_m = (t0 + t1)/2, W1' = omega W1 / ||s||_inf.
template <int N>
__device__ __forceinline__ void hit_grad(const float4 *__restrict__ rec, const Ray &r, float gI, float omega,
                                         uint32_t prim, const RenderArgs &ra, const BackwardGrads &gr, float xi_t) {
    const float4 mh = rec[kRecMh];
    const float4 ml = rec[kRecMl];
    const float4 w0 = rec[kRecWh0];
    const float4 w1 = rec[kRecWh1];
    const float Wh[9] = {ml.w, w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    const float d[3] = {r.dhx, r.dhy, r.dhz};
    const float tc = fmaf(r.dhz, mh.z, fmaf(r.dhy, mh.y, r.dhx * mh.x));
    const float p[3] = {fmaf(tc, r.dhx, -mh.x) + fmaf(tc, r.dlx, -ml.x),
                        fmaf(tc, r.dhy, -mh.y) + fmaf(tc, r.dly, -ml.y),
                        fmaf(tc, r.dhz, -mh.z) + fmaf(tc, r.dlz, -ml.z)};
    float av[3], bv[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        av[k] = fmaf(Wh[3 * k + 2], d[2], fmaf(Wh[3 * k + 1], d[1], Wh[3 * k] * d[0]));
        bv[k] = fmaf(Wh[3 * k + 2], p[2], fmaf(Wh[3 * k + 1], p[1], Wh[3 * k] * p[0]));
    }
    const float A = fmaf(av[2], av[2], fmaf(av[1], av[1], av[0] * av[0]));
    const float B = fmaf(av[2], bv[2], fmaf(av[1], bv[1], av[0] * bv[0]));
    const float iA = rcp_fast(A);   // (as exact_hit computes it)
    const float ts = -B * iA;
    const float bp[3] = {fmaf(ts, av[0], bv[0]), fmaf(ts, av[1], bv[1]), fmaf(ts, av[2], bv[2])};
    const float Q = 1.0f - fmaf(bp[2], bp[2], fmaf(bp[1], bp[1], bp[0] * bp[0]));
    if (!(Q > 0.0f)) return;
    const float hc = sqrtf(Q * iA);
    const float t0 = ts - hc, t1 = ts + hc;
    const float lo_lim = r.t_near - tc, hi_lim = r.t_far - tc;
    const bool clip_lo = !(t0 > lo_lim), clip_hi = !(t1 < hi_lim);
    const float tlo = clip_lo ? lo_lim : t0;
    const float thi = clip_hi ? hi_lim : t1;
    if (!(thi > tlo)) return;
    const float dt = thi - tlo, tm = 0.5f * (tlo + thi), hdt = 0.5f * dt;
    const float *s3 = ra.scales + 3 * (size_t)prim;
    const float sv[3] = {s3[0], s3[1], s3[2]};
    const int imax = (sv[1] > sv[0]) ? ((sv[2] > sv[1]) ? 2 : 1) : ((sv[2] > sv[0]) ? 2 : 0);
    // (reciprocals once: an IEEE division per use takes its slow path on tiny adjoints)
    const float isv[3] = {rcp_fast(sv[0]), rcp_fast(sv[1]), rcp_fast(sv[2])};
    const float ismax = isv[imax];
    const uint32_t wbase = (uint32_t)N * prim;
    const float s1 = omega * ismax;
    float sumc = mh.w;                    // sum_k W2_k cos(phi_k) S_k + b2
    float gdt = 0.f, gtm = 0.f, gsmax = 0.f;
    float gp[3] = {0.f, 0.f, 0.f};        // dI/dp through the phases
    for (int gq = 0; gq < N / 4; ++gq) {
        const float4 w4 = rec[rec_w2(N) + gq];
        const float w2s[4] = {w4.x, w4.y, w4.z, w4.w};
        float a_w2[4], a_b1[4], a_w1[12];   // this group's four units, added as vectors below
#pragma unroll
        for (int uu = 0; uu < 4; ++uu) {
            const int k = 4 * gq + uu;
            const float4 u = rec[kRecUnits + k];
            const float w2 = w2s[uu];
            const float h = fmaf(u.z, d[2], fmaf(u.y, d[1], u.x * d[0]));
            const float g = fmaf(u.z, p[2], fmaf(u.y, p[1], fmaf(u.x, p[0], u.w)));
            const float phi = fmaf(h, tm, g);
            // (MUFU sin/cos and the forward's sinc: the same approximations as exact_hit)
            float sn, cs;
            __sincosf(phi, &sn, &cs);
            const float x = h * hdt;
            const float S = sinc_f(x);
            const float Sp = dsinc_f(x);
            sumc = fmaf(w2 * cs, S, sumc);
            gdt = fmaf(w2 * cs * Sp, 0.5f * h, gdt);
            gtm = fmaf(-w2 * sn * S, h, gtm);
            const float coef = -dt * w2 * sn * S;            // dI/dphi_k
            const float chs = dt * w2 * cs * Sp * hdt;        // dI/dh_k through the sinc
            gp[0] = fmaf(coef, u.x, gp[0]);
            gp[1] = fmaf(coef, u.y, gp[1]);
            gp[2] = fmaf(coef, u.z, gp[2]);
            // dI/dW1'_k = coef (p + tm d) + chs d
            const float gw[3] = {fmaf(coef, fmaf(tm, d[0], p[0]), chs * d[0]),
                                 fmaf(coef, fmaf(tm, d[1], p[1]), chs * d[1]),
                                 fmaf(coef, fmaf(tm, d[2], p[2]), chs * d[2])};
            gsmax = fmaf(-(gw[0] * u.x + gw[1] * u.y + gw[2] * u.z), ismax, gsmax);
            a_w2[uu] = gI * dt * cs * S;
            a_b1[uu] = gI * omega * coef;
            a_w1[3 * uu + 0] = gI * s1 * gw[0];
            a_w1[3 * uu + 1] = gI * s1 * gw[1];
            a_w1[3 * uu + 2] = gI * s1 * gw[2];
        }
        const uint32_t k0 = wbase + 4 * gq;
        add4(gr.w2 + k0, a_w2[0], a_w2[1], a_w2[2], a_w2[3], gr.vec);
        add4(gr.b1 + k0, a_b1[0], a_b1[1], a_b1[2], a_b1[3], gr.vec);
        // temporal scene: the record's phase offset is omega (b1 + xi_t W_t) (R24)
        if (gr.wt) add4(gr.wt + k0, xi_t * a_b1[0], xi_t * a_b1[1], xi_t * a_b1[2], xi_t * a_b1[3], gr.vec);
#pragma unroll
        for (int v = 0; v < 3; ++v)
            add4(gr.w1 + 3 * k0 + 4 * v, a_w1[4 * v], a_w1[4 * v + 1], a_w1[4 * v + 2], a_w1[4 * v + 3], gr.vec);
    }
    add1(gr.b2 + prim, gI * dt);
    if (!gr.mu) return;
    // ---- geometry
    const float G_dt = gI * fmaf(dt, gdt, sumc), G_tm = gI * dt * gtm;
    const float G_tlo = -G_dt + 0.5f * G_tm, G_thi = G_dt + 0.5f * G_tm;
    const float G_t0 = clip_lo ? 0.f : G_tlo, G_t1 = clip_hi ? 0.f : G_thi;
    float G_tc = (clip_lo ? -G_tlo : 0.f) + (clip_hi ? -G_thi : 0.f);
    float G_ts = G_t0 + G_t1;
    const float G_hc = G_t1 - G_t0;
    const float G_Q = G_hc * hc * 0.5f * rcp_fast(Q);
    float G_A = -G_hc * hc * 0.5f * iA;
    float G_a[3], G_b[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float gbp = -2.0f * bp[k] * G_Q;
        G_b[k] = gbp;
        G_a[k] = ts * gbp;
        G_ts = fmaf(gbp, av[k], G_ts);
    }
    const float G_B = -G_ts * iA;
    G_A = fmaf(G_ts * B, iA * iA, G_A);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        G_a[k] = fmaf(2.0f * av[k], G_A, fmaf(bv[k], G_B, G_a[k]));
        G_b[k] = fmaf(av[k], G_B, G_b[k]);
    }
    float Gp[3] = {gI * gp[0], gI * gp[1], gI * gp[2]};
    float G_Wh[9];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            G_Wh[3 * k + j] = fmaf(G_a[k], d[j], G_b[k] * p[j]);
            Gp[j] = fmaf(Wh[3 * k + j], G_b[k], Gp[j]);
        }
    G_tc = fmaf(Gp[2], d[2], fmaf(Gp[1], d[1], fmaf(Gp[0], d[0], G_tc)));
    // m = mu - C: p = t_c d - m, t_c = d.m
    add1(gr.mu + 3 * (size_t)prim + 0, fmaf(d[0], G_tc, -Gp[0]));
    add1(gr.mu + 3 * (size_t)prim + 1, fmaf(d[1], G_tc, -Gp[1]));
    add1(gr.mu + 3 * (size_t)prim + 2, fmaf(d[2], G_tc, -Gp[2]));
    // Wh[k][j] = R[j][k] / s_k
    float G_s[3], G_R[9];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            acc = fmaf(G_Wh[3 * k + j], Wh[3 * k + j], acc);
            G_R[3 * j + k] = G_Wh[3 * k + j] * isv[k];
        }
        G_s[k] = -acc * isv[k];
    }
    G_s[imax] += gI * gsmax;
#pragma unroll
    for (int k = 0; k < 3; ++k) add1(gr.s + 3 * (size_t)prim + k, G_s[k]);
    // R(q^), q^ = q / |q| (w, x, y, z)
    const float *q4 = ra.rotations + 4 * (size_t)prim;
    const float qn = sqrtf(q4[0] * q4[0] + q4[1] * q4[1] + q4[2] * q4[2] + q4[3] * q4[3]);
    const float iqn = rcp_fast(qn);
    const float w = q4[0] * iqn, x = q4[1] * iqn, y = q4[2] * iqn, z = q4[3] * iqn;
    const float gw_ = 2.0f * (-z * G_R[1] + y * G_R[2] + z * G_R[3] - x * G_R[5] - y * G_R[6] + x * G_R[7]);
    const float gx_ = 2.0f * (y * G_R[1] + z * G_R[2] + y * G_R[3] - 2.0f * x * G_R[4] - w * G_R[5] + z * G_R[6] +
                              w * G_R[7] - 2.0f * x * G_R[8]);
    const float gy_ = 2.0f * (-2.0f * y * G_R[0] + x * G_R[1] + w * G_R[2] + x * G_R[3] + z * G_R[5] - w * G_R[6] +
                              z * G_R[7] - 2.0f * y * G_R[8]);
    const float gz_ = 2.0f * (-2.0f * z * G_R[0] - w * G_R[1] + x * G_R[2] + w * G_R[3] - 2.0f * z * G_R[4] +
                              y * G_R[5] + x * G_R[6] + y * G_R[7]);
    const float dotq = w * gw_ + x * gx_ + y * gy_ + z * gz_;
    add4(gr.q + 4 * (size_t)prim, (gw_ - w * dotq) * iqn, (gx_ - x * dotq) * iqn, (gy_ - y * dotq) * iqn,
         (gz_ - z * dotq) * iqn, gr.vec);
}

// d Y_lm / d dir for the basis of sh_basis_f (rows: coefficient, columns: x, y, z)
__device__ __forceinline__ void sh_basis_grad(float x, float y, float z, float dY[16][3]) {
    const float c1 = 0.4886025119029199f, c2 = 1.0925484305920792f, c3 = 0.31539156525252005f,
                c4 = 0.5462742152960396f, c5 = 0.5900435899266435f, c6 = 2.890611442640554f,
                c7 = 0.4570457994644658f, c8 = 0.3731763325901154f, c9 = 1.445305721320277f;
    const float xx = x * x, yy = y * y, zz = z * z;
    const float t[16][3] = {{0.f, 0.f, 0.f},
                            {0.f, -c1, 0.f},
                            {0.f, 0.f, c1},
                            {-c1, 0.f, 0.f},
                            {c2 * y, c2 * x, 0.f},
                            {0.f, -c2 * z, -c2 * y},
                            {-2.f * c3 * x, -2.f * c3 * y, 4.f * c3 * z},
                            {-c2 * z, 0.f, -c2 * x},
                            {2.f * c4 * x, -2.f * c4 * y, 0.f},
                            {-6.f * c5 * x * y, -3.f * c5 * (xx - yy), 0.f},
                            {c6 * y * z, c6 * x * z, c6 * x * y},
                            {2.f * c7 * x * y, -c7 * (4.f * zz - xx - 3.f * yy), -8.f * c7 * y * z},
                            {-6.f * c8 * x * z, -6.f * c8 * y * z, c8 * (6.f * zz - 3.f * xx - 3.f * yy)},
                            {-c7 * (4.f * zz - 3.f * xx - yy), 2.f * c7 * x * y, -8.f * c7 * x * z},
                            {2.f * c9 * x * z, -2.f * c9 * y * z, c9 * (xx - yy)},
                            {-3.f * c5 * (xx - yy), 6.f * c5 * x * y, 0.f}};
#pragma unroll
    for (int i = 0; i < 16; ++i)
#pragma unroll
        for (int c = 0; c < 3; ++c) dY[i][c] = t[i][c];
}

__device__ __forceinline__ void sh_basis_f(float x, float y, float z, float Y[16]) {
    const float xx = x * x, yy = y * y, zz = z * z;
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
}

// The colour part of the gradients for dL/dc = gc: the SH coefficients (dc/dsh_lm =
// Y_lm(dir) on unclamped channels -- gc is already 0 on clamped ones) and, in primitive
// colour mode, mu through dir = (mu - C) / |mu - C|.  Linear in gc, so in primitive mode
// (dir fixed per view and primitive) the K5 path calls it once per (view, primitive) with
// the summed gc.
template <bool kRay>
__device__ __forceinline__ void colour_grads(const RenderArgs &a, const float4 *rec, const Ray &ray, uint32_t id,
                                             const float gc[3], const BackwardGrads &gr) {
    const int ncoef = (a.sh_degree + 1) * (a.sh_degree + 1);
    // SH colour: dc/dsh_lm = Y_lm(dir) (unclamped channels)
    float dxv, dyv, dzv;
    if (kRay) {
        dxv = ray.dhx; dyv = ray.dhy; dzv = ray.dhz;
    } else {   // dir = normalize(mu - C): the record's compensated camera-relative centre
        const float4 mh = rec[kRecMh], ml = rec[kRecMl];
        const float vx = mh.x + ml.x, vy = mh.y + ml.y, vz = mh.z + ml.z;
        const float nrm = sqrtf(vx * vx + vy * vy + vz * vz);
        const float inv = nrm > 0.f ? 1.0f / nrm : 0.f;
        dxv = nrm > 0.f ? vx * inv : 0.f; dyv = nrm > 0.f ? vy * inv : 0.f; dzv = nrm > 0.f ? vz * inv : 1.f;
    }
    float Y[16];
    sh_basis_f(dxv, dyv, dzv, Y);
    const float g0 = gc[0], g1 = gc[1], g2 = gc[2];
    float *gs = gr.sh + 48 * (size_t)id;
    if (g0 != 0.f || g1 != 0.f || g2 != 0.f) {
        // the 3 ncoef coefficients (RGB innermost), four at a time
        const float gcv[3] = {g0, g1, g2};
#pragma unroll
        for (int f0 = 0; f0 < 48; f0 += 4) {   // (unrolled: Y stays in registers)
            if (f0 < 3 * ncoef) {
                float v4[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int f = f0 + u;
                    v4[u] = f < 3 * ncoef ? Y[f / 3] * gcv[f % 3] : 0.f;
                }
                add4(gs + f0, v4[0], v4[1], v4[2], v4[3], gr.vec);
            }
        }
    }
    if (!kRay && gr.mu && (g0 != 0.f || g1 != 0.f || g2 != 0.f)) {
        // colour direction dir = (mu - C) / |mu - C|: dL/dmu = (I - dir dir^T) dL/ddir / |mu - C|
        const float *shp = a.sh + 48 * (size_t)id;
        float dY[16][3];
        sh_basis_grad(dxv, dyv, dzv, dY);
        float gd[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 16; ++i) {   // (unrolled: dY stays in registers)
            if (i < ncoef) {
                const float e = shp[3 * i] * g0 + shp[3 * i + 1] * g1 + shp[3 * i + 2] * g2;
                gd[0] = fmaf(dY[i][0], e, gd[0]);
                gd[1] = fmaf(dY[i][1], e, gd[1]);
                gd[2] = fmaf(dY[i][2], e, gd[2]);
            }
        }
        const float4 mh = rec[kRecMh], ml = rec[kRecMl];
        const float vx = mh.x + ml.x, vy = mh.y + ml.y, vz = mh.z + ml.z;
        const float nrm = sqrtf(vx * vx + vy * vy + vz * vz);
        if (nrm > 0.f) {
            const float dd = dxv * gd[0] + dyv * gd[1] + dzv * gd[2], inrm = 1.0f / nrm;
            atomicAdd(gr.mu + 3 * (size_t)id + 0, (gd[0] - dxv * dd) * inrm);
            atomicAdd(gr.mu + 3 * (size_t)id + 1, (gd[1] - dyv * dd) * inrm);
            atomicAdd(gr.mu + 3 * (size_t)id + 2, (gd[2] - dzv * dd) * inrm);
        }
    }
}

// Every parameter gradient of one composited hit (dL/dI = gI, dL/dc = gc).
template <int N, bool kRay>
__device__ __forceinline__ void hit_all_grads(const RenderArgs &a, const float4 *rec, const Ray &ray, uint32_t id,
                                              float gI, const float gc[3], float omega, const BackwardGrads &gr,
                                              float xi_t) {
    hit_grad<N>(rec, ray, gI, omega, id, a, gr, xi_t);
    colour_grads<kRay>(a, rec, ray, id, gc, gr);
}

// Processes the first `cnt` (<= 32) entries of the warp's queue, one per lane, and moves
// the rest to the front; returns the new queue length.
template <int N, bool kRay, class Sm>
__device__ __forceinline__ int drain(Sm &sm, int wid, int lane, int qn, int cnt, const RenderArgs &a,
                                     const CamBatch &cb, float omega, const BackwardGrads &gr) {
    if (lane < cnt) {
        Ray r;
        r.dhx = sm.q_ray[wid][0][lane]; r.dhy = sm.q_ray[wid][1][lane]; r.dhz = sm.q_ray[wid][2][lane];
        r.dlx = sm.q_ray[wid][3][lane]; r.dly = sm.q_ray[wid][4][lane]; r.dlz = sm.q_ray[wid][5][lane];
        const uint32_t vl = sm.q_vl[wid][lane], id = sm.q_id[wid][lane];
        r.t_near = cb.cams[vl].t_near;
        r.t_far = cb.cams[vl].t_far;
        const float gc[3] = {sm.q_gc[wid][0][lane], sm.q_gc[wid][1][lane], sm.q_gc[wid][2][lane]};
        const float4 *rec = a.records + ((size_t)(cb.view0 + vl) * (size_t)a.n + id) * rec_f4(N);
        hit_all_grads<N, kRay>(a, rec, r, id, sm.q_gI[wid][lane], gc, omega, gr, cb.cams[vl].xi_t);
    }
    __syncwarp();
    const int rest = qn - cnt;
    // (rest < kBwQueue - 32 + 32: every lane moves at most two entries)
    for (int e = lane; e < rest; e += 32) {
        const int from = cnt + e;
#pragma unroll
        for (int c = 0; c < 6; ++c) sm.q_ray[wid][c][e] = sm.q_ray[wid][c][from];
        sm.q_vl[wid][e] = sm.q_vl[wid][from];
        sm.q_id[wid][e] = sm.q_id[wid][from];
        sm.q_gI[wid][e] = sm.q_gI[wid][from];
#pragma unroll
        for (int c = 0; c < 3; ++c) sm.q_gc[wid][c][e] = sm.q_gc[wid][c][from];
    }
    __syncwarp();
    return rest;
}

// kGlobal: the per-warp arrays live in gscratch (one Sm per CTA) instead of shared memory.
// queue_in: only the listed pixels (count in counters[cnt_in]); else every pixel.  Pixels
// with more hits than kBwHits go to queue_out (count in counters[cnt_out]), or -- without
// one -- are skipped and counted in counters[kCntBwdSkipped].
// skip (K5-based backward): skip[pixel] composited hits of the pixel already have their
// gradients (K5's grad mode emitted them before the pixel overflowed); nullptr = none.
// all_if: if *all_if != 0 the queue is ignored and every pixel is processed (the K5 path's
// entry buffer overflowed: its entries are discarded and this kernel does everything).
template <int N, bool kRay, int kBwWarps, int kBwHits, bool kGlobal>
__global__ void __launch_bounds__(kBwWarps * 32) k_backward(RenderArgs a, CamBatch cb, const float4 *__restrict__ grad,
                                                            BackwardGrads gr, float omega, const uint32_t *queue_in,
                                                            int cnt_in, uint32_t *queue_out, int cnt_out,
                                                            void *gscratch, const uint32_t *skip,
                                                            const unsigned long long *all_if) {
    extern __shared__ __align__(16) unsigned char bw_raw[];
    using Sm = BwSmem<kBwWarps, kBwHits>;
    Sm &sm = kGlobal ? reinterpret_cast<Sm *>(gscratch)[blockIdx.x] : *reinterpret_cast<Sm *>(bw_raw);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const int W = cb.cams[0].W, H = cb.cams[0].H;
    if (all_if && *all_if) {
        queue_in = nullptr;
        skip = nullptr;
    }
    const int64_t npix = queue_in ? (int64_t)a.counters[cnt_in] : (int64_t)cb.nv * W * H;
    int qn = 0;   // entries in this warp's gradient queue
    for (int64_t qi = (int64_t)blockIdx.x * kBwWarps + wid; qi < npix; qi += (int64_t)gridDim.x * kBwWarps) {
        const int64_t pi = queue_in ? (int64_t)queue_in[qi] : qi;
        const int vloc = (int)(pi / ((int64_t)W * H));
        const int rem = (int)(pi - (int64_t)vloc * W * H);
        const int y = rem / W, x = rem - y * W;
        const int64_t view = cb.view0 + vloc;
        const float4 G = grad[(view * H + y) * (int64_t)W + x];
        if (G.x == 0.f && G.y == 0.f && G.z == 0.f && G.w == 0.f) continue;
        const DevCam &cam = cb.cams[vloc];
        const int tile = (y / kTile) * a.tiles_x + (x / kTile);
        const uint32_t beg = a.ranges[2 * (view * a.tiles_per_view + tile)];
        const uint32_t end = a.ranges[2 * (view * a.tiles_per_view + tile) + 1];
        const float4 *recs = a.records + (size_t)view * (size_t)a.n * rec_f4(N);
        const Ray ray = make_ray(cam, x, y);
        const Prec64 g64{a.centers, a.rotations, a.scales, cam.C[0], cam.C[1], cam.C[2]};
        const float pxf = (float)x + 0.5f, pyf = (float)y + 0.5f;
        // ---- every hit of the tile list
        int cnt = 0;
        for (uint32_t e0 = beg; e0 < end; e0 += 32) {
            const uint32_t e = e0 + lane;
            bool hit = false;
            float th = 0.f, tl = 0.f, kap = 0.f;
            uint32_t id = 0;
            if (e < end) {
                id = a.vals[e];
                const float4 *rec = recs + (size_t)id * rec_f4(N);
                const float4 c0 = rec[kRecConic];
                const float cc = rec[kRecConicRgb].x;
                const float dx = pxf - c0.x, dy = pyf - c0.y;
                const float q = fmaf(cc * dy, dy, dx * fmaf(c0.w, dy, c0.z * dx));
                if (q <= 1.0f) hit = exact_hit<N, kGrazeInline>(rec, ray, th, tl, kap, &g64, id);
            }
            const uint32_t m = __ballot_sync(0xffffffffu, hit);
            const int pos = cnt + __popc(m & lt);
            if (hit && pos < kBwHits) {
                sm.th[wid][pos] = th;
                sm.tl[wid][pos] = tl;
                sm.kap[wid][pos] = kap;
                sm.id[wid][pos] = id;
            }
            cnt += __popc(m);
        }
        if (cnt > kBwHits) {   // to the big-capacity pass, or (there) skipped and counted
            if (lane == 0) {
                if (queue_out) queue_out[atomicAdd(a.counters + cnt_out, 1ull)] = (uint32_t)pi;
                else atomicAdd(a.counters + kCntBwdSkipped, 1ull);
            }
            continue;
        }
        __syncwarp();
        // ---- (t_in, id) order by rank
        for (int i = lane; i < cnt; i += 32) {
            const float ti = sm.th[wid][i], li = sm.tl[wid][i];
            const uint32_t ii = sm.id[wid][i];
            int rnk = 0;
            for (int j = 0; j < cnt; ++j)
                rnk += before(sm.th[wid][j], sm.tl[wid][j], sm.id[wid][j], ti, li, ii) ? 1 : 0;
            sm.ord[wid][rnk] = (uint32_t)i;
        }
        __syncwarp();
        // ---- forward transmittance and stop: chunked warp product-scan of (1 - kappa)
        float carryT = 1.f, Tend = 1.f;
        int last = cnt - 1;
        for (int k0 = 0; k0 < cnt; k0 += 32) {
            const int k = k0 + lane;
            const float om = k < cnt ? 1.0f - sm.kap[wid][sm.ord[wid][k]] : 1.0f;
            float incl = om;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const float y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl *= y;
            }
            float excl = __shfl_up_sync(0xffffffffu, incl, 1);
            if (lane == 0) excl = 1.0f;
            const float Tafter = carryT * incl;
            if (k < cnt) sm.T[wid][k] = carryT * excl;
            const uint32_t sb = __ballot_sync(0xffffffffu, k < cnt && Tafter < a.t_floor);
            if (sb) {   // stop after the first hit that takes T below the floor (Eq. 4)
                last = k0 + __ffs(sb) - 1;
                Tend = __shfl_sync(0xffffffffu, Tafter, __ffs(sb) - 1);
                break;
            }
            carryT = __shfl_sync(0xffffffffu, Tafter, 31);
            Tend = carryT;
        }
        // ---- back-to-front adjoints: chunked warp suffix sums of T_k kappa_k c_k
        {
            float U0 = Tend * a.bg[0], U1 = Tend * a.bg[1], U2 = Tend * a.bg[2];
            const float gr_[3] = {G.x, G.y, G.z};
            for (int c0 = (last / 32) * 32; c0 >= 0; c0 -= 32) {
                const int k = c0 + lane;
                const bool valid = k <= last;
                float kp = 0.f, Tk = 0.f, c[3] = {0.f, 0.f, 0.f};
                if (valid) {
                    const int h = (int)sm.ord[wid][k];
                    kp = sm.kap[wid][h];
                    const uint32_t id = sm.id[wid][h];
                    const float4 c4 = hit_rgb<kRay>(recs + (size_t)id * rec_f4(N), a.sh, a.sh_degree, id, ray);
                    c[0] = c4.y; c[1] = c4.z; c[2] = c4.w;
                    Tk = sm.T[wid][k];
                }
                const float w[3] = {Tk * kp * c[0], Tk * kp * c[1], Tk * kp * c[2]};
                // exclusive suffix sums within the chunk (lanes above this one)
                float sfx[3] = {w[0], w[1], w[2]};
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) {
                        const float y = __shfl_down_sync(0xffffffffu, sfx[ch], o);
                        if (lane + o < 32) sfx[ch] += y;
                    }
                }
                const float Uk[3] = {U0 + sfx[0] - w[0], U1 + sfx[1] - w[1], U2 + sfx[2] - w[2]};
                if (valid) {
                    const float iom = rcp_fast(fmaxf(1.0f - kp, 1e-20f));
                    float dk = G.w * Tend * iom;
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) {
                        dk = fmaf(gr_[ch], fmaf(-Uk[ch], iom, Tk * c[ch]), dk);
                        sm.gc[wid][k][ch] = c[ch] > 0.f ? Tk * kp * gr_[ch] : 0.f;
                    }
                    sm.gI[wid][k] = kp > 0.f ? dk * (1.0f - kp) : 0.f;
                }
                U0 += __shfl_sync(0xffffffffu, sfx[0], 0);
                U1 += __shfl_sync(0xffffffffu, sfx[1], 0);
                U2 += __shfl_sync(0xffffffffu, sfx[2], 0);
            }
        }
        if (lane == 0) sm.ncomp[wid] = last + 1;
        __syncwarp();
        // ---- queue the composited hits; drain 32 at a time (all lanes busy)
        const int nc = sm.ncomp[wid];
        for (int k0 = skip ? (int)skip[pi] : 0; k0 < nc;) {
            const int m = min(nc - k0, kBwQueue - qn);
            for (int e = lane; e < m; e += 32) {
                const int k = k0 + e, slot = qn + e;
                sm.q_ray[wid][0][slot] = ray.dhx; sm.q_ray[wid][1][slot] = ray.dhy; sm.q_ray[wid][2][slot] = ray.dhz;
                sm.q_ray[wid][3][slot] = ray.dlx; sm.q_ray[wid][4][slot] = ray.dly; sm.q_ray[wid][5][slot] = ray.dlz;
                sm.q_vl[wid][slot] = (uint32_t)vloc;
                sm.q_id[wid][slot] = sm.id[wid][sm.ord[wid][k]];
                sm.q_gI[wid][slot] = sm.gI[wid][k];
                sm.q_gc[wid][0][slot] = sm.gc[wid][k][0];
                sm.q_gc[wid][1][slot] = sm.gc[wid][k][1];
                sm.q_gc[wid][2][slot] = sm.gc[wid][k][2];
            }
            __syncwarp();
            qn += m;
            k0 += m;
            while (qn >= 32) qn = drain<N, kRay, Sm>(sm, wid, lane, qn, 32, a, cb, omega, gr);
        }
        __syncwarp();
    }
    if (qn > 0) drain<N, kRay, Sm>(sm, wid, lane, qn, qn, a, cb, omega, gr);
}

template <int N, bool kRay, int kW, int kH>
int backward_resident() {
    static int res[64] = {};   // per device (the attribute and the occupancy are per-device)
    int dev = 0;
    cudaGetDevice(&dev);
    int &resident = res[dev < 64 ? dev : 0];
    if (!resident) {
        const int smem = (int)sizeof(BwSmem<kW, kH>);
        cudaFuncSetAttribute(k_backward<N, kRay, kW, kH, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_backward<N, kRay, kW, kH, false>, kW * 32, smem);
        resident = (sms > 0 ? sms : 148) * (per_sm > 0 ? per_sm : 1);
    }
    return resident;
}

// The per-pixel chain.  k5 = false: every pixel (level 1), its overflow through levels 2
// and 3.  k5 = true: only the pixels K5's grad mode queued (bw_queue[0..]), from their
// skip counts, or every pixel if the K5 path's entry buffer overflowed.
template <int N, bool kRay>
cudaError_t launch_backward_n(const RenderArgs &a, const CamBatch &cb, const float *grad, const BackwardGrads &g,
                              float omega, void *scratch, bool k5, cudaStream_t st) {
    const int64_t npix = (int64_t)cb.nv * cb.cams[0].W * cb.cams[0].H;
    if (npix == 0) return cudaSuccess;
    const float4 *g4 = reinterpret_cast<const float4 *>(grad);
    cudaError_t e = cudaMemsetAsync(a.counters + kCntBwdQueue2, 0, sizeof(unsigned long long), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(a.counters + kCntBwdQueue3, 0, sizeof(unsigned long long), st);
    if (e == cudaSuccess && !k5) e = cudaMemsetAsync(a.counters + kCntBwdQueue, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    const int res = backward_resident<N, kRay, kBwWarps, kBwHits>();
    const int64_t want = (npix + kBwWarps - 1) / kBwWarps;
    uint32_t *q1 = a.bw_queue, *q2 = a.bw_queue + npix, *q3 = a.bw_queue + 2 * npix;
    const uint32_t *skip = k5 ? a.bw_skip : nullptr;
    const unsigned long long *all_if = k5 ? a.counters + kCntGradOverflow : nullptr;
    k_backward<N, kRay, kBwWarps, kBwHits, false><<<(unsigned)(want < res ? want : res), kBwThreads,
                                                     sizeof(BwSmem<kBwWarps, kBwHits>), st>>>(
        a, cb, g4, g, omega, k5 ? q1 : nullptr, kCntBwdQueue, q2, kCntBwdQueue2, nullptr, skip, all_if);
    // pixels with more than kBwHits hits: one warp per CTA, kBwBigHits each in shared memory
    k_backward<N, kRay, 1, kBwBigHits, false><<<(unsigned)backward_resident<N, kRay, 1, kBwBigHits>(), 32,
                                                 sizeof(BwSmem<1, kBwBigHits>), st>>>(
        a, cb, g4, g, omega, q2, kCntBwdQueue2, q3, kCntBwdQueue3, nullptr, skip, nullptr);
    // and beyond: kBwHugeHits each in the global scratch
    k_backward<N, kRay, 1, kBwHugeHits, true><<<kBwHugeCtas, 32, 0, st>>>(
        a, cb, g4, g, omega, q3, kCntBwdQueue3, nullptr, 0, scratch, skip, nullptr);
    return cudaGetLastError();
}

// K7f: the parameter gradients of every hit K5's grad mode emitted (one thread per entry;
// skipped wholesale if the entry buffer overflowed -- the per-pixel chain then redoes all)
template <int N, bool kRay>
__global__ void __launch_bounds__(128) k_grad_entries(RenderArgs a, CamBatch cb, const GradEntry *__restrict__ ent,
                                                      BackwardGrads gr, float omega) {
    if (a.counters[kCntGradOverflow]) return;
    // the batch's cameras in shared memory (a dynamic index into the parameter struct
    // would copy it to local memory)
    __shared__ DevCam s_cam[kCamsPerLaunch];
    for (int i = threadIdx.x; i < cb.nv; i += blockDim.x) s_cam[i] = cb.cams[i];
    __syncthreads();
    int64_t nc = (int64_t)a.counters[kCntGradEntries];
    if (nc > a.grad_chunks) nc = a.grad_chunks;
    const int64_t n = nc * kGradChunk;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    auto used = [&](int64_t j) { return j < n && (int)(j & (kGradChunk - 1)) < a.grad_fill[j / kGradChunk]; };
    // software pipeline: the next entry is loaded, and its record prefetched into L1,
    // while this one is differentiated
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool ok = used(i);
    GradEntry e{};
    if (ok) e = ent[i];
    for (; i < n; i += stride) {
        const bool okn = used(i + stride);
        GradEntry en{};
        if (okn) en = ent[i + stride];
        if (ok) {
            const int vloc = (int)(e.pix >> 24);
            SNP_CHECK(vloc < cb.nv && (int64_t)e.id < a.n);
            const DevCam &cam = s_cam[vloc];
            const uint32_t p = e.pix & 0xffffffu;
            const int y = (int)(p / (uint32_t)cam.W), x = (int)(p - (uint32_t)y * (uint32_t)cam.W);
            const Ray ray = make_ray(cam, x, y);
            const float4 *rec = a.records + ((size_t)(cb.view0 + vloc) * (size_t)a.n + e.id) * rec_f4(N);
            if (okn) {
                const char *rn = reinterpret_cast<const char *>(
                    a.records + ((size_t)(cb.view0 + (en.pix >> 24)) * (size_t)a.n + en.id) * rec_f4(N));
#pragma unroll
                for (int b = 0; b < 16 * rec_f4(N); b += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(rn + b));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(a.scales + 3 * (size_t)en.id));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(a.rotations + 4 * (size_t)en.id));
            }
            if (kRay) {
                const float gc[3] = {e.gc0, e.gc1, e.gc2};
                hit_all_grads<N, kRay>(a, rec, ray, e.id, e.gI, gc, omega, gr, cam.xi_t);
            } else {   // colour part per (view, primitive) in k_colour_finalize
                hit_grad<N>(rec, ray, e.gI, omega, e.id, a, gr, cam.xi_t);
                if (e.gc0 != 0.f || e.gc1 != 0.f || e.gc2 != 0.f)
                    atomicAdd(a.gc_acc + (size_t)vloc * a.n + e.id, make_float4(e.gc0, e.gc1, e.gc2, 0.f));
            }
        }
        e = en;
        ok = okn;
    }
}

// ---- K7s: K7f over the entries grouped by (view, primitive).
// The gradient atomics are what bound K7f (an A/B without them: 587 -> 94 us at C3):
// every entry adds ~50 values to its primitive's parameters.  Grouped by key
// vloc * n + primitive (a counting sort: K5 writes each entry's key, k_entry_count
// counts, k_key_* scan, k_entry_count<true> places), the 32 entries of a warp form a few
// runs of one key; each value is summed over its run in shared memory and added once.

constexpr int kRedRows = 64;    // values per flush (two per lane)
constexpr int kRedStride = 33;  // (row of 32 entries + 1: the per-lane column writes and
                                //  per-row reads are both conflict-free)

// A flush row's destination: base + mult * (by_key ? key : primitive).
struct RowDesc {
    float *base;
    uint32_t mult;
    bool by_key;
};

// Row `row` of a flush block: MLP groups g0 .. g0 + ng - 1 (per 4 hidden units: W2 x4,
// b1 x4, W1 x12, [W_t x4]), then, in the last block, b2 [, mu x3, s x3, q x4] [, dL/dc
// x3 -> gc_acc, by key vloc * n + primitive].
template <int N>
__device__ __forceinline__ RowDesc row_desc(const BackwardGrads &gr, const RenderArgs &a, int row, int g0, int ng,
                                            int GR) {
    if (row < ng * GR) {
        const int gi = row / GR, r = row - gi * GR;
        const int k0 = 4 * (g0 + gi);
        if (r < 4) return {gr.w2 + k0 + r, (uint32_t)N, false};
        if (r < 8) return {gr.b1 + k0 + (r - 4), (uint32_t)N, false};
        if (r < 20) return {gr.w1 + 3 * k0 + (r - 8), 3u * N, false};
        return {gr.wt + k0 + (r - 20), (uint32_t)N, false};
    }
    const int t = row - ng * GR;
    if (t == 0) return {gr.b2, 1u, false};
    const int tc = gr.mu ? 11 : 1;
    if (t < tc) {
        if (t < 4) return {gr.mu + (t - 1), 3u, false};
        if (t < 7) return {gr.s + (t - 4), 3u, false};
        return {gr.q + (t - 7), 4u, false};
    }
    return {reinterpret_cast<float *>(a.gc_acc) + (t - tc), 4u, true};
}

// Sums rows [0, nrows) of s (s[row][entry], this warp's 32 entries) over the runs that
// `ends` marks (bit e: entry e ends a run; warp-uniform) and adds each nonzero sum once,
// at desc(row)'s address for the run's primitive pr / key k2.
template <class Desc>
__device__ __forceinline__ void run_flush(float (*s)[kRedStride], int nrows, uint32_t ends, uint32_t pr, uint32_t k2,
                                          Desc desc) {
    __syncwarp();
    const int lane = threadIdx.x & 31;
    const bool h0 = lane < nrows, h1 = lane + 32 < nrows;
    const RowDesc d0 = h0 ? desc(lane) : RowDesc{nullptr, 0u, false};
    const RowDesc d1 = h1 ? desc(lane + 32) : RowDesc{nullptr, 0u, false};
    int start = 0;
    while (ends) {
        const int end = __ffs(ends) - 1;
        ends &= ends - 1;
        const uint32_t rp = __shfl_sync(0xffffffffu, pr, end), rk = __shfl_sync(0xffffffffu, k2, end);
        float a0 = 0.f, a1 = 0.f;
        for (int e = start; e <= end; ++e) {
            a0 += s[lane][e];
            a1 += s[lane + 32][e];
        }
        if (h0 && a0 != 0.f) atomicAdd(d0.base + (size_t)d0.mult * (d0.by_key ? rk : rp), a0);
        if (h1 && a1 != 0.f) atomicAdd(d1.base + (size_t)d1.mult * (d1.by_key ? rk : rp), a1);
        start = end + 1;
    }
    __syncwarp();
}

// hit_grad's values for one entry per lane (ok = false: the lane contributes zeros) into
// the warp's rows, flushed per block of at most kRedRows; dL/dc (primitive colour mode)
// rides in the last block.  Same arithmetic as hit_grad, in the same order.
template <int N, bool kRay>
__device__ __forceinline__ void hit_grad_rows(const float4 *__restrict__ rec, const Ray &r, float gI, float omega,
                                              bool ok, const RenderArgs &ra, const BackwardGrads &gr, float xi_t,
                                              uint32_t prim, uint32_t k2, const float gc[3],
                                              float (*s)[kRedStride], uint32_t ends, const RowDesc *fd) {
    const int lane = threadIdx.x & 31;
    // (the primitive's own parameters first: the shared-memory stores and atomics below
    //  would keep the compiler from hoisting these loads)
    const float *s3 = ra.scales + 3 * (size_t)prim;
    const float sv[3] = {s3[0], s3[1], s3[2]};
    float q4[4] = {0.f, 0.f, 0.f, 0.f};
    if (gr.mu) {
        const float *qp = ra.rotations + 4 * (size_t)prim;
        q4[0] = qp[0]; q4[1] = qp[1]; q4[2] = qp[2]; q4[3] = qp[3];
    }
    const float4 mh = rec[kRecMh];
    const float4 ml = rec[kRecMl];
    const float4 w0 = rec[kRecWh0];
    const float4 w1 = rec[kRecWh1];
    const float Wh[9] = {ml.w, w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    const float d[3] = {r.dhx, r.dhy, r.dhz};
    const float tc = fmaf(r.dhz, mh.z, fmaf(r.dhy, mh.y, r.dhx * mh.x));
    const float p[3] = {fmaf(tc, r.dhx, -mh.x) + fmaf(tc, r.dlx, -ml.x),
                        fmaf(tc, r.dhy, -mh.y) + fmaf(tc, r.dly, -ml.y),
                        fmaf(tc, r.dhz, -mh.z) + fmaf(tc, r.dlz, -ml.z)};
    float av[3], bv[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        av[k] = fmaf(Wh[3 * k + 2], d[2], fmaf(Wh[3 * k + 1], d[1], Wh[3 * k] * d[0]));
        bv[k] = fmaf(Wh[3 * k + 2], p[2], fmaf(Wh[3 * k + 1], p[1], Wh[3 * k] * p[0]));
    }
    const float A = fmaf(av[2], av[2], fmaf(av[1], av[1], av[0] * av[0]));
    const float B = fmaf(av[2], bv[2], fmaf(av[1], bv[1], av[0] * bv[0]));
    const float iA = rcp_fast(A);   // (as exact_hit computes it)
    const float ts = -B * iA;
    const float bp[3] = {fmaf(ts, av[0], bv[0]), fmaf(ts, av[1], bv[1]), fmaf(ts, av[2], bv[2])};
    const float Q = 1.0f - fmaf(bp[2], bp[2], fmaf(bp[1], bp[1], bp[0] * bp[0]));
    ok = ok && Q > 0.0f;
    const float hc = sqrtf(Q * iA);
    const float t0 = ts - hc, t1 = ts + hc;
    const float lo_lim = r.t_near - tc, hi_lim = r.t_far - tc;
    const bool clip_lo = !(t0 > lo_lim), clip_hi = !(t1 < hi_lim);
    const float tlo = clip_lo ? lo_lim : t0;
    const float thi = clip_hi ? hi_lim : t1;
    ok = ok && thi > tlo;
    const float dt = thi - tlo, tm = 0.5f * (tlo + thi), hdt = 0.5f * dt;
    const int imax = (sv[1] > sv[0]) ? ((sv[2] > sv[1]) ? 2 : 1) : ((sv[2] > sv[0]) ? 2 : 0);
    const float isv[3] = {rcp_fast(sv[0]), rcp_fast(sv[1]), rcp_fast(sv[2])};
    const float ismax = isv[imax];
    const float s1 = omega * ismax;
    float sumc = mh.w;
    float gdt = 0.f, gtm = 0.f, gsmax = 0.f;
    float gp[3] = {0.f, 0.f, 0.f};
    const int GR = gr.wt ? 24 : 20;
    const int tail = (gr.mu ? 11 : 1) + (kRay ? 0 : 3);
    int g0 = 0, used = 0;
    auto flush = [&](int ng, int nrows) {
        if (fd && g0 == 0 && ng == N / 4 && nrows == ng * GR + tail)   // (the usual single block: N <= 8)
            run_flush(s, nrows, ends, prim, k2, [&](int row) { return row == (threadIdx.x & 31) ? fd[0] : fd[1]; });
        else
            run_flush(s, nrows, ends, prim, k2, [&](int row) { return row_desc<N>(gr, ra, row, g0, ng, GR); });
    };
#pragma unroll 1
    for (int gq = 0; gq < N / 4; ++gq) {
        if (used + GR > kRedRows) {   // (warp-uniform)
            flush(gq - g0, used);
            g0 = gq;
            used = 0;
        }
        float(*sg)[kRedStride] = s + used;
        const float4 w4 = rec[rec_w2(N) + gq];
        const float w2s[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
        for (int uu = 0; uu < 4; ++uu) {
            const int k = 4 * gq + uu;
            const float4 u = rec[kRecUnits + k];
            const float w2 = w2s[uu];
            const float h = fmaf(u.z, d[2], fmaf(u.y, d[1], u.x * d[0]));
            const float g = fmaf(u.z, p[2], fmaf(u.y, p[1], fmaf(u.x, p[0], u.w)));
            const float phi = fmaf(h, tm, g);
            float sn, cs;
            __sincosf(phi, &sn, &cs);
            const float x = h * hdt;
            const float S = sinc_f(x);
            const float Sp = dsinc_f(x);
            sumc = fmaf(w2 * cs, S, sumc);
            gdt = fmaf(w2 * cs * Sp, 0.5f * h, gdt);
            gtm = fmaf(-w2 * sn * S, h, gtm);
            const float coef = -dt * w2 * sn * S;
            const float chs = dt * w2 * cs * Sp * hdt;
            gp[0] = fmaf(coef, u.x, gp[0]);
            gp[1] = fmaf(coef, u.y, gp[1]);
            gp[2] = fmaf(coef, u.z, gp[2]);
            const float gw[3] = {fmaf(coef, fmaf(tm, d[0], p[0]), chs * d[0]),
                                 fmaf(coef, fmaf(tm, d[1], p[1]), chs * d[1]),
                                 fmaf(coef, fmaf(tm, d[2], p[2]), chs * d[2])};
            gsmax = fmaf(-(gw[0] * u.x + gw[1] * u.y + gw[2] * u.z), ismax, gsmax);
            const float gb1 = gI * omega * coef;
            sg[uu][lane] = ok ? gI * dt * cs * S : 0.f;
            sg[4 + uu][lane] = ok ? gb1 : 0.f;
            sg[8 + 3 * uu + 0][lane] = ok ? gI * s1 * gw[0] : 0.f;
            sg[8 + 3 * uu + 1][lane] = ok ? gI * s1 * gw[1] : 0.f;
            sg[8 + 3 * uu + 2][lane] = ok ? gI * s1 * gw[2] : 0.f;
            if (gr.wt) sg[20 + uu][lane] = ok ? xi_t * gb1 : 0.f;   // phase offset omega (b1 + xi_t W_t) (R24)
        }
        used += GR;
    }
    const int ng = N / 4 - g0;
    if (used + tail > kRedRows) {
        flush(ng, used);
        g0 = N / 4;
        used = 0;
    }
    const int ngl = N / 4 - g0;
    float(*st)[kRedStride] = s + used;
    st[0][lane] = ok ? gI * dt : 0.f;
    int t = 1;
    if (gr.mu) {
        const float G_dt = gI * fmaf(dt, gdt, sumc), G_tm = gI * dt * gtm;
        const float G_tlo = -G_dt + 0.5f * G_tm, G_thi = G_dt + 0.5f * G_tm;
        const float G_t0 = clip_lo ? 0.f : G_tlo, G_t1 = clip_hi ? 0.f : G_thi;
        float G_tc = (clip_lo ? -G_tlo : 0.f) + (clip_hi ? -G_thi : 0.f);
        float G_ts = G_t0 + G_t1;
        const float G_hc = G_t1 - G_t0;
        const float G_Q = G_hc * hc * 0.5f * rcp_fast(Q);
        float G_A = -G_hc * hc * 0.5f * iA;
        float G_a[3], G_b[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float gbp = -2.0f * bp[k] * G_Q;
            G_b[k] = gbp;
            G_a[k] = ts * gbp;
            G_ts = fmaf(gbp, av[k], G_ts);
        }
        const float G_B = -G_ts * iA;
        G_A = fmaf(G_ts * B, iA * iA, G_A);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            G_a[k] = fmaf(2.0f * av[k], G_A, fmaf(bv[k], G_B, G_a[k]));
            G_b[k] = fmaf(av[k], G_B, G_b[k]);
        }
        float Gp[3] = {gI * gp[0], gI * gp[1], gI * gp[2]};
        float G_Wh[9];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                G_Wh[3 * k + j] = fmaf(G_a[k], d[j], G_b[k] * p[j]);
                Gp[j] = fmaf(Wh[3 * k + j], G_b[k], Gp[j]);
            }
        G_tc = fmaf(Gp[2], d[2], fmaf(Gp[1], d[1], fmaf(Gp[0], d[0], G_tc)));
#pragma unroll
        for (int k = 0; k < 3; ++k) st[1 + k][lane] = ok ? fmaf(d[k], G_tc, -Gp[k]) : 0.f;
        float G_s[3], G_R[9];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                acc = fmaf(G_Wh[3 * k + j], Wh[3 * k + j], acc);
                G_R[3 * j + k] = G_Wh[3 * k + j] * isv[k];
            }
            G_s[k] = -acc * isv[k];
        }
        G_s[imax] += gI * gsmax;
#pragma unroll
        for (int k = 0; k < 3; ++k) st[4 + k][lane] = ok ? G_s[k] : 0.f;
        const float qn = sqrtf(q4[0] * q4[0] + q4[1] * q4[1] + q4[2] * q4[2] + q4[3] * q4[3]);
        const float iqn = rcp_fast(qn);
        const float w = q4[0] * iqn, x = q4[1] * iqn, y = q4[2] * iqn, z = q4[3] * iqn;
        const float gw_ = 2.0f * (-z * G_R[1] + y * G_R[2] + z * G_R[3] - x * G_R[5] - y * G_R[6] + x * G_R[7]);
        const float gx_ = 2.0f * (y * G_R[1] + z * G_R[2] + y * G_R[3] - 2.0f * x * G_R[4] - w * G_R[5] +
                                  z * G_R[6] + w * G_R[7] - 2.0f * x * G_R[8]);
        const float gy_ = 2.0f * (-2.0f * y * G_R[0] + x * G_R[1] + w * G_R[2] + x * G_R[3] + z * G_R[5] -
                                  w * G_R[6] + z * G_R[7] - 2.0f * y * G_R[8]);
        const float gz_ = 2.0f * (-2.0f * z * G_R[0] - w * G_R[1] + x * G_R[2] + w * G_R[3] - 2.0f * z * G_R[4] +
                                  y * G_R[5] + x * G_R[6] + y * G_R[7]);
        const float dotq = w * gw_ + x * gx_ + y * gy_ + z * gz_;
        st[7][lane] = ok ? (gw_ - w * dotq) * iqn : 0.f;
        st[8][lane] = ok ? (gx_ - x * dotq) * iqn : 0.f;
        st[9][lane] = ok ? (gy_ - y * dotq) * iqn : 0.f;
        st[10][lane] = ok ? (gz_ - z * dotq) * iqn : 0.f;
        t = 11;
    }
    if (!kRay) {   // (summed per (view, primitive) for k_colour_finalize; the entry's own validity)
#pragma unroll
        for (int c = 0; c < 3; ++c) st[t + c][lane] = gc[c];
    }
    flush(ngl, used + tail);
}

// Counting sort of the entries by key vloc * n + primitive (K5 wrote each slot's key):
// counts per key, exclusive scan in place (block sums, their scan, block scans), then the
// entries' slots go to their key's next position.
constexpr int kScanPer = 4096;   // keys per block (1024 threads x 4)
__device__ __forceinline__ uint32_t block_excl_scan_1024(uint32_t v, uint32_t *s_w, uint32_t *total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const uint32_t w = s_w[lane];
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        s_w[lane] = wi - w;
        if (lane == 31) s_w[32] = wi;
    }
    __syncthreads();
    const uint32_t r = s_w[wid] + incl - v;
    *total = s_w[32];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(1024) k_key_sums(const uint32_t *__restrict__ cnt, int64_t nk, uint32_t *bsum) {
    __shared__ uint32_t s_w[33];
    const int64_t b0 = (int64_t)blockIdx.x * kScanPer;
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t i = b0 + k * 1024 + threadIdx.x;
        if (i < nk) v += cnt[i];
    }
    uint32_t tot;
    block_excl_scan_1024(v, s_w, &tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_key_top(uint32_t *bsum, int64_t nb, unsigned long long *scnt) {
    __shared__ uint32_t s_w[33];
    uint32_t run = 0;
    for (int64_t b = 0; b < nb; b += 1024) {
        const int64_t i = b + threadIdx.x;
        const uint32_t v = i < nb ? bsum[i] : 0u;
        uint32_t tot;
        const uint32_t ex = block_excl_scan_1024(v, s_w, &tot);
        if (i < nb) bsum[i] = run + ex;
        run += tot;
    }
    if (threadIdx.x == 0) scnt[kCntDup] = run;
}

__global__ void __launch_bounds__(1024) k_key_apply(uint32_t *cnt, int64_t nk, const uint32_t *bsum) {
    __shared__ uint32_t s_w[33];
    const int64_t b0 = (int64_t)blockIdx.x * kScanPer + 4 * (int64_t)threadIdx.x;
    uint32_t v[4], sum = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = b0 + k < nk ? cnt[b0 + k] : 0u;
        sum += v[k];
    }
    uint32_t tot;
    uint32_t ex = block_excl_scan_1024(sum, s_w, &tot) + bsum[blockIdx.x];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (b0 + k < nk) cnt[b0 + k] = ex;
        ex += v[k];
    }
}

// (lanes with equal keys -- neighbouring pixels' hits of one primitive -- share one atomic)
template <bool kScatter>
__global__ void __launch_bounds__(256) k_entry_count(RenderArgs a, uint32_t *__restrict__ key_cnt,
                                                     uint32_t *__restrict__ sorted, int64_t nk) {
    int64_t nc = (int64_t)a.counters[kCntGradEntries];
    if (nc > a.grad_chunks) nc = a.grad_chunks;
    if (a.counters[kCntGradOverflow]) nc = 0;
    const int64_t n = nc * kGradChunk;
    const int lane = threadIdx.x & 31;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + threadIdx.x;   // (warp-uniform trip count: i0 steps by whole blocks)
        const bool used = i < n && (int)(i & (kGradChunk - 1)) < a.grad_fill[i / kGradChunk];
        const uint32_t key = used ? a.grad_keys[i] : 0xffffffffu;
        SNP_CHECK(!used || (int64_t)key < nk);
        const uint32_t peers = __match_any_sync(0xffffffffu, key);
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (used && lane == leader) {
            if (kScatter) base = atomicAdd(key_cnt + key, (uint32_t)__popc(peers));
            else atomicAdd(key_cnt + key, (uint32_t)__popc(peers));
        }
        if (kScatter) {
            base = __shfl_sync(0xffffffffu, base, leader);
            SNP_CHECK(!used || (int64_t)(base + __popc(peers)) <= (int64_t)a.grad_chunks * kGradChunk);
            if (used) sorted[base + __popc(peers & ((1u << lane) - 1u))] = (uint32_t)i;
        }
    }
}

template <int N, bool kRay, bool kFromFwd>   // kFromFwd: entries recorded by the forward (FwdEntry)
__global__ void __launch_bounds__(128) k_grad_sorted(RenderArgs a, CamBatch cb, const uint32_t *__restrict__ sorted,
                                                     const unsigned long long *scnt, BackwardGrads gr, float omega) {
    if (a.counters[kCntGradOverflow]) return;
    __shared__ DevCam s_cam[kCamsPerLaunch];
    __shared__ float s_red[4][kRedRows][kRedStride];
    for (int i = threadIdx.x; i < cb.nv; i += blockDim.x) s_cam[i] = cb.cams[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float(*s)[kRedStride] = s_red[wid];
    const int64_t n = (int64_t)scnt[kCntDup];
    // this lane's two flush rows when all values fit one block (N <= 8): fixed per kernel
    const int GR = gr.wt ? 24 : 20;
    const RowDesc fd[2] = {row_desc<N>(gr, a, lane, 0, N / 4, GR), row_desc<N>(gr, a, lane + 32, 0, N / 4, GR)};
    const int64_t step = (int64_t)gridDim.x * 4 * 32;
    int64_t base = ((int64_t)blockIdx.x * 4 + wid) * 32;
    using Entry = typename std::conditional<kFromFwd, FwdEntry, GradEntry>::type;
    const Entry *ent = kFromFwd ? reinterpret_cast<const Entry *>(a.rec_entries)
                                : reinterpret_cast<const Entry *>(a.grad_entries);
    Entry en{};   // (the next iteration's entry, loaded one iteration ahead)
    if (base + lane < n) en = ent[sorted[base + lane]];
    for (; base < n; base += step) {
        const int64_t pos = base + lane;
        const bool valid = pos < n;
        const Entry e = en;   // (zero on lanes past the end)
        en = Entry{};
        if (base + step + lane < n) en = ent[sorted[base + step + lane]];
        const int vloc = valid ? (int)(e.pix >> 24) : 0;
        SNP_CHECK(!valid || (vloc < cb.nv && (int64_t)e.id < a.n));
        const uint32_t k2 = valid ? (uint32_t)vloc * (uint32_t)a.n + e.id : 0xffffffffu;
        const uint32_t nk2 = __shfl_down_sync(0xffffffffu, k2, 1);
        const uint32_t ends = __ballot_sync(0xffffffffu, lane == 31 || nk2 != k2);
        const DevCam &cam = s_cam[vloc];
        const uint32_t p = e.pix & 0xffffffu;
        const int y = (int)(p / (uint32_t)cam.W), x = (int)(p - (uint32_t)y * (uint32_t)cam.W);
        const Ray ray = make_ray(cam, x, y);
        const float4 *rec = a.records + ((size_t)(cb.view0 + vloc) * (size_t)a.n + e.id) * rec_f4(N);
        float gI, gc[3];   // (zero on invalid lanes)
        if constexpr (kFromFwd) {   // dL/dI, dL/dc from dL/d(out), the forward's out and the recorded hit
            gI = 0.f;
            gc[0] = gc[1] = gc[2] = 0.f;
            if (valid) {
                const int64_t gi = ((int64_t)(cb.view0 + vloc) * cam.H + y) * cam.W + x;
                const float4 rgb = hit_rgb<kRay>(rec, a.sh, a.sh_degree, e.id, ray);
                hit_out_grads(a.grad_in[gi], a.fwd[gi], e.T, e.kap, rgb, e.cr, e.cg, e.cb, gI, gc);
            }
        } else {
            gI = e.gI;
            gc[0] = e.gc0;
            gc[1] = e.gc1;
            gc[2] = e.gc2;
        }
        hit_grad_rows<N, kRay>(rec, ray, gI, omega, valid, a, gr, cam.xi_t, e.id, k2, gc, s, ends,
                               (N / 4) * GR + (gr.mu ? 11 : 1) + (kRay ? 0 : 3) <= kRedRows ? fd : nullptr);
        if (kRay) {   // SH at the pixel's ray direction: 3 ncoef (<= 48) values, one flush
            const int ncoef = (a.sh_degree + 1) * (a.sh_degree + 1);
            float Y[16];
            sh_basis_f(ray.dhx, ray.dhy, ray.dhz, Y);
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (i < ncoef) {
                    s[3 * i][lane] = Y[i] * gc[0];
                    s[3 * i + 1][lane] = Y[i] * gc[1];
                    s[3 * i + 2][lane] = Y[i] * gc[2];
                }
            run_flush(s, 3 * ncoef, ends, e.id, k2, [&](int row) { return RowDesc{gr.sh + row, 48u, false}; });
        }
    }
}

// Primitive colour mode: the colour gradients of every (view, primitive) from the summed
// dL/dc of its composited hits (colour_grads is linear in dL/dc).  One thread per
// primitive sums over the batch's views -- dL/dsh = sum_v Y(dir_v) (x) dL/dc_v and the
// mu-through-dir_v terms -- and adds once (a view's direction is the record's
// compensated camera-relative centre, as in colour_grads).
template <int N>
__global__ void __launch_bounds__(128) k_colour_finalize(RenderArgs a, CamBatch cb, BackwardGrads gr) {
    if (a.counters[kCntGradOverflow]) return;
    const int ncoef = (a.sh_degree + 1) * (a.sh_degree + 1);
    for (int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; id < a.n; id += (int64_t)gridDim.x * blockDim.x) {
        float acc[48];
#pragma unroll
        for (int f = 0; f < 48; ++f) acc[f] = 0.f;
        float gmu[3] = {0.f, 0.f, 0.f};
        bool any = false;
        const float *shp = a.sh + 48 * (size_t)id;
        for (int v = 0; v < cb.nv; ++v) {
            const float4 g = a.gc_acc[(size_t)v * a.n + id];
            if (g.x == 0.f && g.y == 0.f && g.z == 0.f) continue;
            any = true;
            // (a composited primitive is visible in the view: its record exists)
            const float4 *rec = a.records + ((size_t)(cb.view0 + v) * (size_t)a.n + id) * rec_f4(N);
            const float4 mh = rec[kRecMh], ml = rec[kRecMl];
            const float vx = mh.x + ml.x, vy = mh.y + ml.y, vz = mh.z + ml.z;
            const float nrm = sqrtf(vx * vx + vy * vy + vz * vz);
            const float inv = nrm > 0.f ? 1.0f / nrm : 0.f;
            const float dxv = nrm > 0.f ? vx * inv : 0.f, dyv = nrm > 0.f ? vy * inv : 0.f,
                        dzv = nrm > 0.f ? vz * inv : 1.f;
            float Y[16];
            sh_basis_f(dxv, dyv, dzv, Y);
            const float gcv[3] = {g.x, g.y, g.z};
#pragma unroll
            for (int f = 0; f < 48; ++f) acc[f] = fmaf(Y[f / 3], gcv[f % 3], acc[f]);
            if (gr.mu && nrm > 0.f) {   // dir = (mu - C) / |mu - C|: dL/dmu = (I - dir dir^T) dL/ddir / |mu - C|
                float dY[16][3];
                sh_basis_grad(dxv, dyv, dzv, dY);
                float gd[3] = {0.f, 0.f, 0.f};
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    if (i < ncoef) {
                        const float e = shp[3 * i] * g.x + shp[3 * i + 1] * g.y + shp[3 * i + 2] * g.z;
                        gd[0] = fmaf(dY[i][0], e, gd[0]);
                        gd[1] = fmaf(dY[i][1], e, gd[1]);
                        gd[2] = fmaf(dY[i][2], e, gd[2]);
                    }
                const float dd = dxv * gd[0] + dyv * gd[1] + dzv * gd[2];
                gmu[0] += (gd[0] - dxv * dd) * inv;
                gmu[1] += (gd[1] - dyv * dd) * inv;
                gmu[2] += (gd[2] - dzv * dd) * inv;
            }
        }
        if (!any) continue;
        float *gs = gr.sh + 48 * (size_t)id;
#pragma unroll
        for (int f0 = 0; f0 < 48; f0 += 4)
            if (f0 < 3 * ncoef)
                add4(gs + f0, acc[f0], f0 + 1 < 3 * ncoef ? acc[f0 + 1] : 0.f, f0 + 2 < 3 * ncoef ? acc[f0 + 2] : 0.f,
                     f0 + 3 < 3 * ncoef ? acc[f0 + 3] : 0.f, gr.vec);
        if (gr.mu) {
            atomicAdd(gr.mu + 3 * (size_t)id + 0, gmu[0]);
            atomicAdd(gr.mu + 3 * (size_t)id + 1, gmu[1]);
            atomicAdd(gr.mu + 3 * (size_t)id + 2, gmu[2]);
        }
    }
}

template <int N, bool kRay>
cudaError_t launch_grad_entries_n(const RenderArgs &a, const CamBatch &cb, const BackwardGrads &g, float omega,
                                  const EntrySort *es, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (es) {   // counting sort by (view, primitive) key, then K7s
        const int64_t nk = (int64_t)cb.nv * a.n;
        const int64_t nb = (nk + kScanPer - 1) / kScanPer;
        if (nb == 0) return cudaSuccess;   // (no primitives: no entries)
        k_entry_count<false><<<(unsigned)(sms * 8), 256, 0, st>>>(a, a.grad_count, nullptr, nk);
        k_key_sums<<<(unsigned)nb, 1024, 0, st>>>(a.grad_count, nk, es->bsum);
        k_key_top<<<1, 1024, 0, st>>>(es->bsum, nb, es->cnt);
        k_key_apply<<<(unsigned)nb, 1024, 0, st>>>(a.grad_count, nk, es->bsum);
        k_entry_count<true><<<(unsigned)(sms * 8), 256, 0, st>>>(a, a.grad_count, es->sorted, nk);
        if (a.from_fwd) k_grad_sorted<N, kRay, true><<<(unsigned)(sms * 8), 128, 0, st>>>(a, cb, es->sorted, es->cnt, g, omega);
        else k_grad_sorted<N, kRay, false><<<(unsigned)(sms * 8), 128, 0, st>>>(a, cb, es->sorted, es->cnt, g, omega);
    } else {
        k_grad_entries<N, kRay><<<(unsigned)(sms * 8), 128, 0, st>>>(a, cb, a.grad_entries, g, omega);
    }
    if (!kRay) k_colour_finalize<N><<<(unsigned)(sms * 8), 128, 0, st>>>(a, cb, g);
    return cudaGetLastError();
}

template <int N>
cudaError_t launch_backward_w(const RenderArgs &a, const CamBatch &cb, const float *grad, const BackwardGrads &g,
                              float omega, void *scratch, bool k5, const EntrySort *es, cudaStream_t st,
                              cudaStream_t st_pix) {
    if (k5) {
        cudaError_t e = a.colour_ray ? launch_grad_entries_n<N, true>(a, cb, g, omega, es, st)
                                     : launch_grad_entries_n<N, false>(a, cb, g, omega, es, st);
        if (e != cudaSuccess) return e;
    }
    return a.colour_ray ? launch_backward_n<N, true>(a, cb, grad, g, omega, scratch, k5, st_pix)
                        : launch_backward_n<N, false>(a, cb, grad, g, omega, scratch, k5, st_pix);
}

}  // namespace

size_t backward_scratch_bytes() { return (size_t)kBwHugeCtas * sizeof(BwSmem<1, kBwHugeHits>); }

cudaError_t launch_backward(const RenderArgs &a, const CamBatch &cb, const float *grad, const BackwardGrads &g,
                            float omega, void *scratch, bool k5, const EntrySort *es, cudaStream_t st,
                            cudaStream_t st_pix) {
    switch (a.n_hidden) {
        case 4: return launch_backward_w<4>(a, cb, grad, g, omega, scratch, k5, es, st, st_pix);
        case 8: return launch_backward_w<8>(a, cb, grad, g, omega, scratch, k5, es, st, st_pix);
        case 16: return launch_backward_w<16>(a, cb, grad, g, omega, scratch, k5, es, st, st_pix);
        case 32: return launch_backward_w<32>(a, cb, grad, g, omega, scratch, k5, es, st, st_pix);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace snp
