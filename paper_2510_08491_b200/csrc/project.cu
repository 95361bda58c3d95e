// project.cu -- K1a: per (view, primitive) projection, cull and binning geometry
// (k_bin_geom) and input validation.  Compiled with -fmad=false: the FP64 binning geometry
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
    double inq = 1.0 / nq;   // one division (binning definition)
    double w = q0 * inq, x = q1 * inq, y = q2 * inq, z = q3 * inq;
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

// FP64 prelude of the binning geometry: camera-frame centre m = R_wc^T (mu - C), camera-frame rotation
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

// Tight binning data of a visible (view, primitive): the silhouette as an
// image ellipse (p - c)^T [[A, B], [B, C]] (p - c) <= 1 and the camera-frame centre m and
// covariance S for per-tile depth bounds, as floats (K2 applies margins).  The silhouette
// is the point conic adj(K (m m^T - S) K^T) (the dual conic of the tangent planes through
// the camera centre, whose x / y extents are the rect's above), defined when the
// ellipsoid lies in front of the camera (zmin > 0, m_z^2 > S_zz); otherwise flag 0 and K2
// keeps every rect tile.
__device__ __forceinline__ void tight_geom(const DevCam &cam, const Geom &g, double aq, float4 *t4) {
    const double *m = g.m, *S = g.S;
    const double fx = cam.fx, fy = cam.fy, cx = cam.cx, cy = cam.cy;
    float xc = 0.f, yc = 0.f, A = 0.f, B = 0.f, Cc = 0.f, ok = 0.f;
    if (g.zmin > 0.0 && aq > 0.0) {
        const double M00 = m[0] * m[0] - S[0], M01 = m[0] * m[1] - S[1], M02 = m[0] * m[2] - S[2];
        const double M11 = m[1] * m[1] - S[4], M12 = m[1] * m[2] - S[5], M22 = m[2] * m[2] - S[8];
        // C* = K M K^T
        const double d00 = fx * fx * M00 + 2.0 * fx * cx * M02 + cx * cx * M22;
        const double d01 = fx * fy * M01 + fx * cy * M02 + cx * fy * M12 + cx * cy * M22;
        const double d02 = fx * M02 + cx * M22;
        const double d11 = fy * fy * M11 + 2.0 * fy * cy * M12 + cy * cy * M22;
        const double d12 = fy * M12 + cy * M22;
        const double d22 = M22;
        // point conic = adj(C*)
        const double c00 = d11 * d22 - d12 * d12, c01 = d02 * d12 - d01 * d22, c02 = d01 * d12 - d02 * d11;
        const double c11 = d00 * d22 - d02 * d02, c12 = d01 * d02 - d00 * d12, c22 = d00 * d11 - d01 * d01;
        const double det = c00 * c11 - c01 * c01;
        if (det > 0.0) {
            const double ex = -(c11 * c02 - c01 * c12) / det, ey = -(c00 * c12 - c01 * c02) / det;
            const double qc = c22 + c02 * ex + c12 * ey;   // q at the centre
            if (qc != 0.0 && (c00 > 0.0) == (qc < 0.0)) {  // a real ellipse: interior q / qc > 0
                const double s = -1.0 / qc;
                xc = (float)ex;
                yc = (float)ey;
                A = (float)(c00 * s);
                B = (float)(c01 * s);
                Cc = (float)(c11 * s);
                ok = 1.f;
            }
        }
    }
    t4[0] = make_float4(xc, yc, A, B);
    t4[1] = make_float4(Cc, (float)m[0], (float)m[1], (float)m[2]);
    t4[2] = make_float4((float)S[0], (float)S[1], (float)S[2], (float)S[4]);
    t4[3] = make_float4((float)S[5], (float)S[8], ok, 0.f);
}

// ============================================================================
// K1a: binning geometry only (critical path of the frame): per (view,
// primitive) cull, tile rect and depth key from 40 B of parameters.
constexpr int kGeomThreads = 256;

template <bool kTight>   // tight binning data (a.tight) in its own instantiation
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
                for (int k = 0; k < 4 && keep; ++k) {
                    const double *nn = pn[k];
                    double dot = nn[0] * m[0] + nn[1] * m[1] + nn[2] * m[2];
                    double quad = nn[0] * (nn[0] * S[0] + nn[1] * S[1] + nn[2] * S[2])
                                + nn[1] * (nn[0] * S[3] + nn[1] * S[4] + nn[2] * S[5])
                                + nn[2] * (nn[0] * S[6] + nn[1] * S[7] + nn[2] * S[8]);
                    if (dot < 0.0 && dot * dot > quad) keep = false;   // n.m + sqrt(n^T S n) < 0
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
                        const double iaq = 1.0 / aq;
                        xlo = fx * ((bx - rx) * iaq) + cx;
                        xhi = fx * ((bx + rx) * iaq) + cx;
                        double by = m[1] * m[2] - S[5];
                        double cyq = m[1] * m[1] - S[4];
                        double discy = by * by - aq * cyq;
                        if (!(discy > 0.0)) discy = 0.0;
                        double ry = sqrt(discy);
                        ylo = fy * ((by - ry) * iaq) + cy;
                        yhi = fy * ((by + ry) * iaq) + cy;
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
                        if (kTight) tight_geom(cam, g, aq, a.tight + 4 * o);
                    }
                }
            }
            a.rects[o] = rect;
            a.depth[o] = dep;
            if (kTight && i == 0)
                a.intr[view] = make_float4((float)(1.0 / (double)cam.fx), (float)(1.0 / (double)cam.fy), cam.cx, cam.cy);
            n_vis += keep;
        }
    }
    // warp-aggregated visible count
    const uint32_t vb = __reduce_add_sync(0xffffffffu, (uint32_t)n_vis);
    if ((threadIdx.x & 31) == 0 && vb) atomicAdd(a.counters + kCntVisibleAcc, (unsigned long long)vb);
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
    const int N = a.n_hidden;
    for (int k = 0; k < 3 * N; ++k) if (!isfinite(a.w1[3 * N * i + k])) b |= 1;
    for (int k = 0; k < N; ++k) if (!isfinite(a.b1[N * i + k]) || !isfinite(a.w2[N * i + k])) b |= 1;
    if (!isfinite(a.b2[i])) b |= 1;
    for (int k = 0; k < 48; ++k) if (!isfinite(a.sh[48 * i + k])) b |= 1;
    if (b) {
        atomicOr(bad, b);
        atomicMin(bad + 1, (int)i);
    }
}

}  // namespace

namespace {
__global__ void k_validate_finite(const float *v, int64_t count, int *bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(v[i])) {
            atomicOr(bad, 1);
            atomicMin(bad + 1, (int)(i < 0x7fffffff ? i : 0x7fffffff));
        }
}
}  // namespace

cudaError_t launch_validate_finite(const float *v, int64_t count, int *d_bad, cudaStream_t st) {
    if (count == 0) return cudaSuccess;
    const int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 8);
    k_validate_finite<<<(unsigned)blocks, 256, 0, st>>>(v, count, d_bad);
    return cudaGetLastError();
}

cudaError_t launch_bin_geom(const ProjectArgs &a, const CamBatch &cams, cudaStream_t st) {
    if (a.n == 0) return cudaSuccess;
    const unsigned grid = (unsigned)((a.n + kGeomThreads - 1) / kGeomThreads);
    if (a.tight) k_bin_geom<true><<<grid, kGeomThreads, 0, st>>>(a, cams);
    else k_bin_geom<false><<<grid, kGeomThreads, 0, st>>>(a, cams);
    return cudaGetLastError();
}

cudaError_t launch_validate(const ProjectArgs &a, int *d_bad, cudaStream_t st) {
    if (a.n == 0) return cudaSuccess;
    k_validate<<<(unsigned)((a.n + 255) / 256), 256, 0, st>>>(a, d_bad);
    return cudaGetLastError();
}

}  // namespace snp
