// project.cu -- K1: per (view, primitive) projection, cull, binning geometry
// (K1a, k_bin_geom) and render record (K1b, k_records).  Compiled with -fmad=false: the FP64 binning geometry
// below follows the fixed operation order of DESIGN.md "Binning definition"
// so that tile rects and depth keys are bit-exact with
// the CPU oracle's definition.  Every product/sum is written left to right.
//
// Paper anchors: P:235 (ellipsoid mu, s, q), P:249 (||s||_inf normalisation,
// Eq. 5), P:253-283 (MLP, Eq. 6), P:286/P:394 (SH colour), P:298-299 (analytic
// line-ellipsoid intersection), P:368 ("perspectively accurate").
#include <math.h>

#include <algorithm>
#include <cstdlib>

#include "snp_internal.cuh"

namespace snp {
namespace {

__device__ __forceinline__ bool quat_rot(const float *q4, double R[9]) {
    double q0 = q4[0], q1 = q4[1], q2 = q4[2], q3 = q4[3];
    double nq = sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
    if (!(nq > 0.0)) return false;
    double w = q0 / nq, x = q1 / nq, y = q2 / nq, z = q3 / nq;
    R[0] = 1.0 - 2.0 * (y * y + z * z);
    R[1] = 2.0 * (x * y - w * z);
    R[2] = 2.0 * (x * z + w * y);
    R[3] = 2.0 * (x * y + w * z);
    R[4] = 1.0 - 2.0 * (x * x + z * z);
    R[5] = 2.0 * (y * z - w * x);
    R[6] = 2.0 * (x * z - w * y);
    R[7] = 2.0 * (y * z + w * x);
    R[8] = 1.0 - 2.0 * (x * x + y * y);
    return true;
}

// Real SH basis, degrees 0..3 (Condon-Shortley phase, m = -l..l; 3DGS convention).
__device__ __forceinline__ void sh_rgb(int degree, const float4 *sh4, double xd, double yd, double zd,
                                       float rgb[3]) {
    // float4 reads: a 192-byte row stride gives 4-way shared-memory bank conflicts
    // instead of the 16-way of scalar reads
    float sh[48];
#pragma unroll
    for (int k = 0; k < 12; ++k) {
        const float4 t = sh4[k];
        sh[4 * k] = t.x; sh[4 * k + 1] = t.y; sh[4 * k + 2] = t.z; sh[4 * k + 3] = t.w;
    }
    // fp32 is ample here: colour enters the pixel linearly (error ~1e-7)
    const float x = (float)xd, y = (float)yd, z = (float)zd;
    float Y[16];
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
    const int nc = (degree + 1) * (degree + 1);
    float acc[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        if (i < nc) {
            acc[0] += Y[i] * sh[3 * i + 0];
            acc[1] += Y[i] * sh[3 * i + 1];
            acc[2] += Y[i] * sh[3 * i + 2];
        }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float v = acc[c] + 0.5f;
        rgb[c] = v > 0.f ? v : 0.f;
    }
}

// Shared FP64 prelude of K1a and K1b (identical code, so both derive the same
// values): camera-frame centre m = R_wc^T (mu - C), camera-frame rotation
// Rc = R_wc^T R, camera-frame covariance S = Rc diag(s^2) Rc^T, z-range.
struct Geom {
    double R[9], Rc[9], S[9], m[3];
    double zmin, zmax;
};

__device__ __forceinline__ bool geom_prelude(const DevCam &cam, float mu0, float mu1, float mu2, const float q4[4],
                                             float s0f, float s1f, float s2f, Geom &g) {
    if (!quat_rot(q4, g.R)) return false;
    double W[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) W[k] = (double)cam.R[k];
    double dx = (double)mu0 - (double)cam.C[0];
    double dy = (double)mu1 - (double)cam.C[1];
    double dz = (double)mu2 - (double)cam.C[2];
#pragma unroll
    for (int j = 0; j < 3; ++j) g.m[j] = W[0 * 3 + j] * dx + W[1 * 3 + j] * dy + W[2 * 3 + j] * dz;
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            g.Rc[3 * j + k] = W[0 * 3 + j] * g.R[0 * 3 + k] + W[1 * 3 + j] * g.R[1 * 3 + k] + W[2 * 3 + j] * g.R[2 * 3 + k];
    const double s0 = s0f, s1 = s1f, s2 = s2f;
    const double ss0 = s0 * s0, ss1 = s1 * s1, ss2 = s2 * s2;
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int l = 0; l < 3; ++l)
            g.S[3 * j + l] = g.Rc[3 * j + 0] * ss0 * g.Rc[3 * l + 0] + g.Rc[3 * j + 1] * ss1 * g.Rc[3 * l + 1]
                           + g.Rc[3 * j + 2] * ss2 * g.Rc[3 * l + 2];
    const double sz = sqrt(g.S[8]);
    g.zmin = g.m[2] - sz;
    g.zmax = g.m[2] + sz;
    return true;
}

// ============================================================================
// K1a: binning geometry only (critical path of the frame): per (view,
// primitive) cull, tile rect and depth key from 40 B of parameters.
constexpr int kGeomThreads = 256;

__global__ void __launch_bounds__(kGeomThreads) k_bin_geom(ProjectArgs a, CamBatch cb) {
    const int64_t i = (int64_t)blockIdx.x * kGeomThreads + threadIdx.x;
    unsigned long long n_vis = 0;
    if (i < a.n) {
        const float mu0 = __ldg(a.centers + 3 * i), mu1 = __ldg(a.centers + 3 * i + 1),
                    mu2 = __ldg(a.centers + 3 * i + 2);
        const float s0f = __ldg(a.scales + 3 * i), s1f = __ldg(a.scales + 3 * i + 1), s2f = __ldg(a.scales + 3 * i + 2);
        const float4 qv = __ldg(reinterpret_cast<const float4 *>(a.rotations) + i);
        const float q4[4] = {qv.x, qv.y, qv.z, qv.w};
        for (int vloc = 0; vloc < cb.nv; ++vloc) {
            const int64_t view = cb.view0 + vloc;
            const DevCam &cam = cb.cams[vloc];
            const int64_t o = view * a.n + i;
            short4 rect = make_short4(-1, -1, -1, -1);
            uint32_t dep = 0;
            Geom g;
            bool keep = geom_prelude(cam, mu0, mu1, mu2, q4, s0f, s1f, s2f, g);
            if (keep) {
                const double *m = g.m, *S = g.S;
                if (!(g.zmax > 0.0)) keep = false;
                const double fx = cam.fx, fy = cam.fy, cx = cam.cx, cy = cam.cy;
                const double Wd = (double)cam.W, Hd = (double)cam.H;
                const double pn[4][3] = {{fx, 0.0, cx}, {-fx, 0.0, Wd - cx}, {0.0, fy, cy}, {0.0, -fy, Hd - cy}};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double *nn = pn[k];
                    double dot = nn[0] * m[0] + nn[1] * m[1] + nn[2] * m[2];
                    double quad = nn[0] * (nn[0] * S[0] + nn[1] * S[1] + nn[2] * S[2])
                                + nn[1] * (nn[0] * S[3] + nn[1] * S[4] + nn[2] * S[5])
                                + nn[2] * (nn[0] * S[6] + nn[1] * S[7] + nn[2] * S[8]);
                    if (dot + sqrt(quad) < 0.0) keep = false;
                }
                if (keep) {
                    double xlo = -INFINITY, xhi = INFINITY, ylo = -INFINITY, yhi = INFINITY;
                    const double aq = m[2] * m[2] - S[8];
                    if (g.zmin > 0.0 && aq > 0.0) {
                        double bx = m[0] * m[2] - S[2];
                        double cxq = m[0] * m[0] - S[0];
                        double discx = bx * bx - aq * cxq;
                        if (!(discx > 0.0)) discx = 0.0;
                        double rx = sqrt(discx);
                        xlo = fx * ((bx - rx) / aq) + cx;
                        xhi = fx * ((bx + rx) / aq) + cx;
                        double by = m[1] * m[2] - S[5];
                        double cyq = m[1] * m[1] - S[4];
                        double discy = by * by - aq * cyq;
                        if (!(discy > 0.0)) discy = 0.0;
                        double ry = sqrt(discy);
                        ylo = fy * ((by - ry) / aq) + cy;
                        yhi = fy * ((by + ry) / aq) + cy;
                    }
                    const double eps = 1.0 / 256.0;
                    double px0 = ceil(xlo - 0.5 - eps), px1 = floor(xhi - 0.5 + eps);
                    double py0 = ceil(ylo - 0.5 - eps), py1 = floor(yhi - 0.5 + eps);
                    if (px0 < 0.0) px0 = 0.0;
                    if (py0 < 0.0) py0 = 0.0;
                    if (px1 > Wd - 1.0) px1 = Wd - 1.0;
                    if (py1 > Hd - 1.0) py1 = Hd - 1.0;
                    if (!(px0 <= px1) || !(py0 <= py1)) keep = false;
                    if (keep) {
                        rect = make_short4((short)((int)px0 / kTile), (short)((int)py0 / kTile),
                                           (short)((int)px1 / kTile), (short)((int)py1 / kTile));
                        // depth lower bound L <= t_in of every ray (R19)
                        double L = (double)cam.t_near;
                        /* t >= u.x >= u.m - sqrt(u^T S u) for u = m/|m| (support function of E) */
                        double nm = sqrt(m[0] * m[0] + m[1] * m[1] + m[2] * m[2]);
                        double mSm = m[0] * (m[0] * S[0] + m[1] * S[1] + m[2] * S[2])
                                   + m[1] * (m[0] * S[3] + m[1] * S[4] + m[2] * S[5])
                                   + m[2] * (m[0] * S[6] + m[1] * S[7] + m[2] * S[8]);
                        if (nm > 0.0 && mSm >= 0.0) {
                            double l1 = nm - sqrt(mSm) / nm;
                            if (l1 > L) L = l1;
                        }
                        if (g.zmin > L) L = g.zmin;
                        dep = __float_as_uint(__double2float_rd(L));
                    }
                }
            }
            a.rects[o] = rect;
            a.depth[o] = dep;
            n_vis += keep;
        }
    }
    // warp-aggregated visible count
    const uint32_t vb = __reduce_add_sync(0xffffffffu, (uint32_t)n_vis);
    if ((threadIdx.x & 31) == 0 && vb) atomicAdd(a.counters + kCntVisible, (unsigned long long)vb);
}

// ============================================================================
// K1b: render records of the visible (view, primitive) pairs (K1a's rect.x >= 0).
// Off the critical path: it runs on the scene's side stream concurrently with
// K2-K4 and is joined before K5.
constexpr int kProjThreads = 128;

// One slice = the parameters of kProjThreads consecutive primitives, staged with
// cp.async.bulk and reused by every view of the launch.
struct Slice {
    float centers[kProjThreads * 3];
    float rot[kProjThreads * 4];
    float scales[kProjThreads * 3];
    float w1[kProjThreads * 24];
    float b1[kProjThreads * 8];
    float w2[kProjThreads * 8];
    float b2[kProjThreads];
    float sh[kProjThreads * 48];
};
struct ProjSmem {
    Slice buf;
    unsigned long long bar;
};

__device__ __forceinline__ uint32_t psmem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// bit v set: primitive i is visible in view cb.view0 + v (K1a's rect.x >= 0; cb.nv <= 32)
__device__ __forceinline__ uint32_t vis_mask_of(const ProjectArgs &a, const CamBatch &cb, int64_t i) {
    uint32_t m = 0;
    if (i < a.n)
        for (int vloc = 0; vloc < cb.nv; ++vloc)
            if (a.rects[(cb.view0 + vloc) * a.n + i].x >= 0) m |= 1u << vloc;
    return m;
}

__device__ __forceinline__ void issue_slice(const ProjectArgs &a, Slice &dst, unsigned long long *bar, int64_t i0) {
    const int cnt = (int)(a.n - i0 < kProjThreads ? a.n - i0 : kProjThreads);
    const float *src[8] = {a.centers, a.rotations, a.scales, a.w1, a.b1, a.w2, a.b2, a.sh};
    float *d[8] = {dst.centers, dst.rot, dst.scales, dst.w1, dst.b1, dst.w2, dst.b2, dst.sh};
    const int per[8] = {3, 4, 3, 24, 8, 8, 1, 48};
    uint32_t total = 0, bytes[8];
    for (int k = 0; k < 8; ++k) {
        bytes[k] = ((uint32_t)(cnt * per[k] * 4) + 15u) & ~15u;   // arrays are padded in the allocation
        total += bytes[k];
    }
    // the buffer was last read through the generic proxy (previous use, after a barrier)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(psmem_u32(bar)), "r"(total)
                 : "memory");
    for (int k = 0; k < 8; ++k)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                psmem_u32(d[k])),
            "l"(src[k] + i0 * per[k]), "r"(bytes[k]), "r"(psmem_u32(bar))
            : "memory");
}


// One primitive's parameters, wherever they live (shared-memory slice or global).
struct PrimParams {
    const float *center, *scale;
    const float4 *rot, *sh, *w1, *b1, *w2;
    float b2;
};

__device__ __forceinline__ void record_one(const ProjectArgs &a, const CamBatch &cb, const PrimParams &pp,
                                           int64_t i, uint32_t vis_mask) {
    const float mu0 = pp.center[0], mu1 = pp.center[1], mu2 = pp.center[2];
    const float s0f = pp.scale[0], s1f = pp.scale[1], s2f = pp.scale[2];
    const float4 qv = pp.rot[0];
    const float q4[4] = {qv.x, qv.y, qv.z, qv.w};
    for (int vloc = 0; vloc < cb.nv; ++vloc) {
        if (!((vis_mask >> vloc) & 1u)) continue;
        const int64_t view = cb.view0 + vloc;
        const DevCam &cam = cb.cams[vloc];
        const int64_t o = view * a.n + i;
        Geom g;
        geom_prelude(cam, mu0, mu1, mu2, q4, s0f, s1f, s2f, g);   // visible => quaternion is valid
        const double *m = g.m, *Rc = g.Rc, *R = g.R;
        const double zmin = g.zmin;
        const double s0 = s0f, s1 = s1f, s2 = s2f;
        double smax = s0;
        if (s1 > smax) smax = s1;
        if (s2 > smax) smax = s2;
        // silhouette conic in pixel space (tangent cone of the ellipsoid from the camera
        // centre), used by K5 only as a conservative pre-test before the exact intersection
        float cx0 = 0.f, cy0 = 0.f, ca = 0.f, cb2 = 0.f, cc = 0.f;
        {
            double P[9];
            const double is0 = 1.0 / (s0 * s0), is1 = 1.0 / (s1 * s1), is2 = 1.0 / (s2 * s2);
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
                for (int l = 0; l < 3; ++l)
                    P[3 * j + l] = Rc[3 * j] * is0 * Rc[3 * l] + Rc[3 * j + 1] * is1 * Rc[3 * l + 1]
                                 + Rc[3 * j + 2] * is2 * Rc[3 * l + 2];
            double w[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) w[j] = P[3 * j] * m[0] + P[3 * j + 1] * m[1] + P[3 * j + 2] * m[2];
            const double c0 = m[0] * w[0] + m[1] * w[1] + m[2] * w[2] - 1.0;
            if (zmin > 0.0 && c0 > 0.0) {
                double Q[9];
#pragma unroll
                for (int j = 0; j < 3; ++j)
#pragma unroll
                    for (int l = 0; l < 3; ++l) Q[3 * j + l] = c0 * P[3 * j + l] - w[j] * w[l];
                const double A00 = Q[0], A01 = Q[1], A11 = Q[4], l0 = Q[2], l1 = Q[5], kq = Q[8];
                const double det = A00 * A11 - A01 * A01;
                if (det > 0.0 && A00 > 0.0) {
                    const double idet = 1.0 / det;
                    const double u0 = -(A11 * l0 - A01 * l1) * idet;
                    const double v0 = -(A00 * l1 - A01 * l0) * idet;
                    const double qc = kq + l0 * u0 + l1 * v0;
                    if (qc < 0.0) {
                        const double fx = cam.fx, fy = cam.fy;
                        const double iq = -1.0 / qc, ifx = 1.0 / fx, ify = 1.0 / fy;
                        const double an = A00 * iq * (ifx * ifx);
                        const double bn = A01 * iq * (ifx * ify);
                        const double cn = A11 * iq * (ify * ify);
                        const double x0 = fx * u0 + (double)cam.cx, y0 = fy * v0 + (double)cam.cy;
                        const double lmax = 0.5 * (an + cn) + sqrt(0.25 * (an - cn) * (an - cn) + bn * bn);
                        const double delta = ldexp(fabs(x0) + fabs(y0) + 1.0, -21);
                        const double e = 1.0 + delta * sqrt(lmax);
                        const double thr = e * e * (1.0 + 1e-5) + 1e-6;
                        if (isfinite(x0) && isfinite(y0) && isfinite(thr) && fabs(x0) < 1e7 && fabs(y0) < 1e7) {
                            cx0 = (float)x0;
                            cy0 = (float)y0;
                            ca = (float)(an / thr);
                            cb2 = (float)(2.0 * bn / thr);
                            cc = (float)(cn / thr);
                        }
                    }
                }
            }
        }
        // camera-relative centre, compensated (hi + lo)
        const double mw0 = (double)mu0 - (double)cam.C[0];
        const double mw1 = (double)mu1 - (double)cam.C[1];
        const double mw2 = (double)mu2 - (double)cam.C[2];
        const float mh0 = (float)mw0, mh1 = (float)mw1, mh2 = (float)mw2;
        const float ml0 = (float)(mw0 - (double)mh0), ml1 = (float)(mw1 - (double)mh1),
                    ml2 = (float)(mw2 - (double)mh2);
        // colour at dir = normalize(mu - C) (R14)
        float rgb[3];
        {
            double nd = sqrt(mw0 * mw0 + mw1 * mw1 + mw2 * mw2);
            double x = 0.0, y = 0.0, z = 1.0;
            if (nd > 0.0) {
                const double ind = 1.0 / nd;
                x = mw0 * ind; y = mw1 * ind; z = mw2 * ind;
            }
            sh_rgb(a.sh_degree, pp.sh, x, y, z, rgb);
        }
        // whitening Wh = diag(1/s) R^T (world -> unit-sphere frame); fp32 suffices
        float Wh[9];
        {
            const float is[3] = {1.0f / s0f, 1.0f / s1f, 1.0f / s2f};
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int j = 0; j < 3; ++j) Wh[3 * k + j] = (float)R[3 * j + k] * is[k];
        }
        float4 *rec = a.records + o * 16;
        const float b2 = pp.b2;
        rec[kRecConic] = make_float4(cx0, cy0, ca, cb2);
        rec[kRecConicRgb] = make_float4(cc, rgb[0], rgb[1], rgb[2]);
        rec[kRecMh] = make_float4(mh0, mh1, mh2, b2);
        rec[kRecMl] = make_float4(ml0, ml1, ml2, Wh[0]);
        rec[kRecWh0] = make_float4(Wh[1], Wh[2], Wh[3], Wh[4]);
        rec[kRecWh1] = make_float4(Wh[5], Wh[6], Wh[7], Wh[8]);
        // MLP (Eq. 6) with the Eq. 5 normalisation folded in: W1' = omega W1 / ||s||_inf
        const double om = (double)a.omega;
        const float4 *w1v = pp.w1;
        const float4 *b1v = pp.b1;
        const float4 *w2v = pp.w2;
        float w1[24], b1[8];
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            float4 t = w1v[k];
            w1[4 * k] = t.x; w1[4 * k + 1] = t.y; w1[4 * k + 2] = t.z; w1[4 * k + 3] = t.w;
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            float4 t = b1v[k];
            b1[4 * k] = t.x; b1[4 * k + 1] = t.y; b1[4 * k + 2] = t.z; b1[4 * k + 3] = t.w;
        }
        const float scf = (float)(om / smax), omf = a.omega;
#pragma unroll
        for (int k = 0; k < kHidden; ++k)
            rec[kRecUnits + k] = make_float4(scf * w1[3 * k], scf * w1[3 * k + 1], scf * w1[3 * k + 2],
                                             omf * b1[k]);
        rec[kRecW2] = w2v[0];
        rec[kRecW2 + 1] = w2v[1];
    }
}

// One CTA per slice; a slice with no visible primitive is never loaded.
__global__ void __launch_bounds__(kProjThreads, 4) k_records(ProjectArgs a, CamBatch cb) {
    extern __shared__ __align__(128) unsigned char psm_raw[];
    ProjSmem &ps = *reinterpret_cast<ProjSmem *>(psm_raw);
    const int64_t i0 = (int64_t)blockIdx.x * kProjThreads;
    const uint32_t vis = vis_mask_of(a, cb, i0 + threadIdx.x);
    if (!__syncthreads_or(vis != 0)) return;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(psmem_u32(&ps.bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        issue_slice(a, ps.buf, &ps.bar, i0);
    }
    __syncthreads();
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(psmem_u32(&ps.bar))
            : "memory");
    if (vis) {
        const int li = threadIdx.x;
        const Slice &sl = ps.buf;
        PrimParams pp;
        pp.center = sl.centers + 3 * li;
        pp.scale = sl.scales + 3 * li;
        pp.rot = reinterpret_cast<const float4 *>(sl.rot) + li;
        pp.sh = reinterpret_cast<const float4 *>(sl.sh + 48 * li);
        pp.w1 = reinterpret_cast<const float4 *>(sl.w1 + 24 * li);
        pp.b1 = reinterpret_cast<const float4 *>(sl.b1 + 8 * li);
        pp.w2 = reinterpret_cast<const float4 *>(sl.w2 + 8 * li);
        pp.b2 = sl.b2[li];
        record_one(a, cb, pp, i0 + li, vis);
    }
}


// Input validation: q nonzero, s > 0, every value finite.
// bad[0] |= 1 non-finite, 2 zero quaternion, 4 scale <= 0; bad[1] = min bad index.
__global__ void k_validate(ProjectArgs a, int *bad) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    int b = 0;
    double qn = 0.0;
    for (int k = 0; k < 4; ++k) {
        float q = a.rotations[4 * i + k];
        if (!isfinite(q)) b |= 1;
        qn += (double)q * (double)q;
    }
    if (!(qn > 0.0)) b |= 2;
    for (int k = 0; k < 3; ++k) {
        float s = a.scales[3 * i + k], c = a.centers[3 * i + k];
        if (!isfinite(s) || !isfinite(c)) b |= 1;
        if (!(s > 0.f)) b |= 4;
    }
    for (int k = 0; k < 24; ++k) if (!isfinite(a.w1[24 * i + k])) b |= 1;
    for (int k = 0; k < 8; ++k) if (!isfinite(a.b1[8 * i + k]) || !isfinite(a.w2[8 * i + k])) b |= 1;
    if (!isfinite(a.b2[i])) b |= 1;
    for (int k = 0; k < 48; ++k) if (!isfinite(a.sh[48 * i + k])) b |= 1;
    if (b) {
        atomicOr(bad, b);
        atomicMin(bad + 1, (int)i);
    }
}

}  // namespace

cudaError_t launch_bin_geom(const ProjectArgs &a, const CamBatch &cams, cudaStream_t st) {
    if (a.n == 0) return cudaSuccess;
    k_bin_geom<<<(unsigned)((a.n + kGeomThreads - 1) / kGeomThreads), kGeomThreads, 0, st>>>(a, cams);
    return cudaGetLastError();
}

cudaError_t launch_records(const ProjectArgs &a, const CamBatch &cams, cudaStream_t st) {
    if (a.n == 0) return cudaSuccess;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_records, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ProjSmem));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    k_records<<<(unsigned)((a.n + kProjThreads - 1) / kProjThreads), kProjThreads, sizeof(ProjSmem), st>>>(a, cams);
    return cudaGetLastError();
}

cudaError_t launch_validate(const ProjectArgs &a, int *d_bad, cudaStream_t st) {
    if (a.n == 0) return cudaSuccess;
    k_validate<<<(unsigned)((a.n + 255) / 256), 256, 0, st>>>(a, d_bad);
    return cudaGetLastError();
}

}  // namespace snp
