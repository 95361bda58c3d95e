// records.cu -- K1b: the render record (256 B at N = 8) of every visible (view, primitive)
// pair (K1a's rect.x >= 0), see snp_internal.cuh "Render record".  It runs on the
// scene's side stream concurrently with K2-K4 and is joined before K5.
//
// Unlike K1a this file is compiled with FMA contraction and uses a fast FP64
// reciprocal (MUFU seed + 2 Newton steps, full double precision up to the last
// ulp): nothing here is part of the bit-exact binning definition -- the record
// only has to be accurate (fp32 values, a silhouette conic with a safety margin
// of ~1e-5 relative, far above these rounding differences).
//
// Paper anchors: P:235 (ellipsoid mu, s, q), P:249 (||s||_inf normalisation,
// Eq. 5), P:253-283 (MLP, Eq. 6), P:286/P:394 (SH colour), P:298-299 (analytic
// line-ellipsoid intersection), P:368 ("perspectively accurate").
#include <math.h>

#include "snp_internal.cuh"

namespace snp {
namespace {

// 1/x to ~1 ulp: rcp.approx seed (~2^-22) refined by two Newton steps
__device__ __forceinline__ double rcp64(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = __fma_rn(-x, r, 1.0);
    r = __fma_rn(r, e, r);
    e = __fma_rn(-x, r, 1.0);
    return __fma_rn(r, e, r);
}

// Camera frame of one primitive: R(q), Rc = R_wc^T R, m = R_wc^T (mu - C), z_min.
__device__ __forceinline__ void frame_fast(const DevCam &cam, float mu0, float mu1, float mu2, const float q4[4],
                                           float s0f, float s1f, float s2f, double R[9], double Rc[9], double m[3],
                                           double &zmin) {
    const double q0 = q4[0], q1 = q4[1], q2 = q4[2], q3 = q4[3];
    const double inq = rcp64(sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3));   // visible => |q| > 0
    const double w = q0 * inq, x = q1 * inq, y = q2 * inq, z = q3 * inq;
    R[0] = 1.0 - 2.0 * (y * y + z * z);
    R[1] = 2.0 * (x * y - w * z);
    R[2] = 2.0 * (x * z + w * y);
    R[3] = 2.0 * (x * y + w * z);
    R[4] = 1.0 - 2.0 * (x * x + z * z);
    R[5] = 2.0 * (y * z - w * x);
    R[6] = 2.0 * (x * z - w * y);
    R[7] = 2.0 * (y * z + w * x);
    R[8] = 1.0 - 2.0 * (x * x + y * y);
    double W[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) W[k] = (double)cam.R[k];
    const double dx = (double)mu0 - (double)cam.C[0];
    const double dy = (double)mu1 - (double)cam.C[1];
    const double dz = (double)mu2 - (double)cam.C[2];
#pragma unroll
    for (int j = 0; j < 3; ++j) m[j] = W[0 * 3 + j] * dx + W[1 * 3 + j] * dy + W[2 * 3 + j] * dz;
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            Rc[3 * j + k] = W[0 * 3 + j] * R[0 * 3 + k] + W[1 * 3 + j] * R[1 * 3 + k] + W[2 * 3 + j] * R[2 * 3 + k];
    const double s0 = s0f, s1 = s1f, s2 = s2f;
    const double szz = Rc[6] * Rc[6] * (s0 * s0) + Rc[7] * Rc[7] * (s1 * s1) + Rc[8] * Rc[8] * (s2 * s2);
    zmin = m[2] - sqrt(szz);
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

constexpr int kProjThreads = 64;

// One slice = the parameters of kProjThreads consecutive primitives (N hidden units),
// staged with cp.async.bulk and reused by every view of the launch.
template <int N>
struct Slice {
    float centers[kProjThreads * 3];
    float rot[kProjThreads * 4];
    float scales[kProjThreads * 3];
    float w1[kProjThreads * 3 * N];
    float b1[kProjThreads * N];
    float w2[kProjThreads * N];
    float b2[kProjThreads];
    float sh[kProjThreads * 48];
};
template <int N>
struct ProjSmem {
    Slice<N> buf;
    short4 rects[kProjThreads];    // K1a's tile rects of this slice (single-view launches)
    unsigned long long bar_geo;    // centers, rotations, scales, b2 (what the conic needs)
    unsigned long long bar_rest;   // w1, b1, w2, sh: streams in while the conic is computed
};

__device__ __forceinline__ void mbar_wait0(unsigned long long *bar);

__device__ __forceinline__ uint32_t psmem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// bit v set: primitive i is visible in view cb.view0 + v (K1a's rect.x >= 0; cb.nv <= 32)
__device__ __forceinline__ uint32_t vis_mask_of(const ProjectArgs &a, const CamBatch &cb, int64_t i) {
    uint32_t m = 0;
    if (i < a.n)
        for (int vloc = 0; vloc < cb.nv; ++vloc)
            if (a.rects[(cb.view0 + vloc) * a.n + i].x >= 0) m |= 1u << vloc;
    return m;
}

template <int N>
__device__ __forceinline__ void issue_slice(const ProjectArgs &a, Slice<N> &dst, unsigned long long *bar_geo,
                                            unsigned long long *bar_rest, int64_t i0, short4 *rects_dst,
                                            const short4 *rects_src) {
    const int cnt = (int)(a.n - i0 < kProjThreads ? a.n - i0 : kProjThreads);
    const uint32_t rbytes = rects_dst ? (((uint32_t)cnt * 8u + 15u) & ~15u) : 0u;
    const float *src[8] = {a.centers, a.rotations, a.scales, a.b2, a.w1, a.b1, a.w2, a.sh};
    float *d[8] = {dst.centers, dst.rot, dst.scales, dst.b2, dst.w1, dst.b1, dst.w2, dst.sh};
    const int per[8] = {3, 4, 3, 1, 3 * N, N, N, 48};
    uint32_t geo = 0, rest = 0, bytes[8];
    for (int k = 0; k < 8; ++k) {
        bytes[k] = ((uint32_t)(cnt * per[k] * 4) + 15u) & ~15u;   // arrays are padded in the allocation
        (k < 4 ? geo : rest) += bytes[k];
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(psmem_u32(bar_geo)), "r"(geo + rbytes)
                 : "memory");
    if (rects_dst)   // the visibility this CTA needs arrives with its geometry (no separate round trip)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                psmem_u32(rects_dst)),
            "l"(rects_src), "r"(rbytes), "r"(psmem_u32(bar_geo))
            : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(psmem_u32(bar_rest)), "r"(rest)
                 : "memory");
    for (int k = 0; k < 8; ++k)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                psmem_u32(d[k])),
            "l"(src[k] + i0 * per[k]), "r"(bytes[k]), "r"(psmem_u32(k < 4 ? bar_geo : bar_rest))
            : "memory");
}

__device__ __forceinline__ void mbar_wait0(unsigned long long *bar) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(psmem_u32(bar))
            : "memory");
}


// One primitive's parameters, wherever they live (shared-memory slice or global).
struct PrimParams {
    const float *center, *scale;
    const float4 *rot, *sh, *w1, *b1, *w2;
    float b2;
};

template <int N>
__device__ __forceinline__ void record_one(const ProjectArgs &a, const CamBatch &cb, const PrimParams &pp,
                                           int64_t i, uint32_t vis_mask, unsigned long long *bar_rest) {
    const float mu0 = pp.center[0], mu1 = pp.center[1], mu2 = pp.center[2];
    const float s0f = pp.scale[0], s1f = pp.scale[1], s2f = pp.scale[2];
    const float4 qv = pp.rot[0];
    const float q4[4] = {qv.x, qv.y, qv.z, qv.w};
    for (int vloc = 0; vloc < cb.nv; ++vloc) {
        if (!((vis_mask >> vloc) & 1u)) continue;
        const int64_t view = cb.view0 + vloc;
        const DevCam &cam = cb.cams[vloc];
        const int64_t o = view * a.n + i;
        double R[9], Rc[9], m[3], zmin;
        frame_fast(cam, mu0, mu1, mu2, q4, s0f, s1f, s2f, R, Rc, m, zmin);
        const double s0 = s0f, s1 = s1f, s2 = s2f;
        double smax = s0;
        if (s1 > smax) smax = s1;
        if (s2 > smax) smax = s2;
        // silhouette conic in pixel space (tangent cone of the ellipsoid from the camera
        // centre), used by K5 only as a conservative pre-test before the exact intersection
        float cx0 = 0.f, cy0 = 0.f, ca = 0.f, cb2 = 0.f, cc = 0.f;
        {
            double P[9];
            const double is0 = rcp64(s0 * s0), is1 = rcp64(s1 * s1), is2 = rcp64(s2 * s2);
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
            // (zmin is not K1a's bit-exact value: a margin keeps the tangent-cone
            // silhouette to ellipsoids strictly in front of the camera plane)
            if (zmin > 1e-9 * (fabs(m[2]) + 1.0) && c0 > 0.0) {
                double Q[9];
#pragma unroll
                for (int j = 0; j < 3; ++j)
#pragma unroll
                    for (int l = 0; l < 3; ++l) Q[3 * j + l] = c0 * P[3 * j + l] - w[j] * w[l];
                const double A00 = Q[0], A01 = Q[1], A11 = Q[4], l0 = Q[2], l1 = Q[5], kq = Q[8];
                const double det = A00 * A11 - A01 * A01;
                if (det > 0.0 && A00 > 0.0) {
                    const double idet = rcp64(det);
                    const double u0 = -(A11 * l0 - A01 * l1) * idet;
                    const double v0 = -(A00 * l1 - A01 * l0) * idet;
                    const double qc = kq + l0 * u0 + l1 * v0;
                    if (qc < 0.0) {
                        const double fx = cam.fx, fy = cam.fy;
                        const double iq = -rcp64(qc), ifx = cam.ifx, ify = cam.ify;
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
                            const double ithr = rcp64(thr);
                            ca = (float)(an * ithr);
                            cb2 = (float)(2.0 * bn * ithr);
                            cc = (float)(cn * ithr);
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
                const double ind = rcp64(nd);
                x = mw0 * ind; y = mw1 * ind; z = mw2 * ind;
            }
            mbar_wait0(bar_rest);   // (returns at once after the first view)
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
        float4 *rec = a.records + o * rec_f4(N);
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
        const float scf = (float)(om * rcp64(smax)), omf = a.omega;
        // four units at a time: three float4 of W1 rows and one of b1
#pragma unroll
        for (int g = 0; g < N / 4; ++g) {
            float w1[12], b1[4];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const float4 t = w1v[3 * g + k];
                w1[4 * k] = t.x; w1[4 * k + 1] = t.y; w1[4 * k + 2] = t.z; w1[4 * k + 3] = t.w;
            }
            const float4 tb = b1v[g];
            b1[0] = tb.x; b1[1] = tb.y; b1[2] = tb.z; b1[3] = tb.w;
            if (a.w_t) {   // temporal scene: b1 + xi_t W_t at this view's timestamp (R24)
                const float4 wt = __ldg(reinterpret_cast<const float4 *>(a.w_t + (size_t)N * i) + g);
                b1[0] = fmaf(cam.xi_t, wt.x, b1[0]);
                b1[1] = fmaf(cam.xi_t, wt.y, b1[1]);
                b1[2] = fmaf(cam.xi_t, wt.z, b1[2]);
                b1[3] = fmaf(cam.xi_t, wt.w, b1[3]);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                rec[kRecUnits + 4 * g + k] = make_float4(scf * w1[3 * k], scf * w1[3 * k + 1], scf * w1[3 * k + 2],
                                                         omf * b1[k]);
        }
#pragma unroll
        for (int j = 0; j < N / 4; ++j) rec[rec_w2(N) + j] = w2v[j];
    }
}

// One CTA per slice.  The slice load is issued first (its latency overlaps the
// visibility read); a CTA whose slice has no visible primitive only waits for it.
template <int N>
__global__ void __launch_bounds__(kProjThreads, 8) k_records(ProjectArgs a, CamBatch cb) {
    extern __shared__ __align__(128) unsigned char psm_raw[];
    ProjSmem<N> &ps = *reinterpret_cast<ProjSmem<N> *>(psm_raw);
    const int64_t i0 = (int64_t)blockIdx.x * kProjThreads;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(psmem_u32(&ps.bar_geo)) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(psmem_u32(&ps.bar_rest)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // single view with a 16-byte aligned rect row: the rects come with the slice
    const bool rect_smem = cb.nv == 1 && ((cb.view0 * a.n + i0) & 1) == 0;
    if (threadIdx.x == 0)
        issue_slice(a, ps.buf, &ps.bar_geo, &ps.bar_rest, i0, rect_smem ? ps.rects : nullptr,
                    a.rects + cb.view0 * a.n + i0);
    uint32_t vis;
    if (rect_smem) {
        __syncthreads();                 // (publishes the barrier init)
        mbar_wait0(&ps.bar_geo);
        vis = (i0 + threadIdx.x < a.n && ps.rects[threadIdx.x].x >= 0) ? 1u : 0u;
    } else {
        vis = vis_mask_of(a, cb, i0 + threadIdx.x);
    }
    if (!__syncthreads_or(vis != 0)) {   // (also publishes the barrier init)
        mbar_wait0(&ps.bar_geo);         // the copies must land before the CTA's smem is freed
        mbar_wait0(&ps.bar_rest);
        return;
    }
    mbar_wait0(&ps.bar_geo);
    if (vis) {
        const int li = threadIdx.x;
        const Slice<N> &sl = ps.buf;
        PrimParams pp;
        pp.center = sl.centers + 3 * li;
        pp.scale = sl.scales + 3 * li;
        pp.rot = reinterpret_cast<const float4 *>(sl.rot) + li;
        pp.sh = reinterpret_cast<const float4 *>(sl.sh + 48 * li);
        pp.w1 = reinterpret_cast<const float4 *>(sl.w1 + 3 * N * li);
        pp.b1 = reinterpret_cast<const float4 *>(sl.b1 + N * li);
        pp.w2 = reinterpret_cast<const float4 *>(sl.w2 + N * li);
        pp.b2 = sl.b2[li];   // (geometry part of the slice)
        record_one<N>(a, cb, pp, i0 + li, vis, &ps.bar_rest);
    }
}


}  // namespace

namespace {
template <int N>
cudaError_t launch_records_n(const ProjectArgs &a, const CamBatch &cams, cudaStream_t st) {
    static bool attr[64] = {};   // per device (the attribute is a per-device property)
    int dev = 0;
    cudaGetDevice(&dev);
    bool &done = attr[dev < 64 ? dev : 0];
    if (!done) {
        cudaError_t e = cudaFuncSetAttribute(k_records<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(ProjSmem<N>));
        if (e != cudaSuccess) return e;
        done = true;
    }
    k_records<N><<<(unsigned)((a.n + kProjThreads - 1) / kProjThreads), kProjThreads, sizeof(ProjSmem<N>), st>>>(a,
                                                                                                             cams);
    return cudaGetLastError();
}
}  // namespace

cudaError_t launch_records(const ProjectArgs &a, const CamBatch &cams, cudaStream_t st) {
    if (a.n == 0) return cudaSuccess;
    switch (a.n_hidden) {
        case 4: return launch_records_n<4>(a, cams, st);
        case 8: return launch_records_n<8>(a, cams, st);
        case 16: return launch_records_n<16>(a, cams, st);
        case 32: return launch_records_n<32>(a, cams, st);
        default: return cudaErrorInvalidValue;
    }
}
}  // namespace snp
