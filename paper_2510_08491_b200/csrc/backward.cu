// backward.cu -- K7: backward of the forward render (first part):
// dL/d{W1, b1, W2, b2, SH} of every primitive for a given dL/d(out RGBA), with the
// ellipsoid geometry (mu, q, s) held fixed.
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
// skipped and counted in counters[kCntBwdSkipped].
#include "hit.cuh"
#include "snp_internal.cuh"

namespace snp {
namespace {

constexpr int kBwWarps = 8;
constexpr int kBwThreads = kBwWarps * 32;
constexpr int kBwHits = 256;

struct BwSmem {
    float th[kBwWarps][kBwHits], tl[kBwWarps][kBwHits], kap[kBwWarps][kBwHits];
    uint32_t id[kBwWarps][kBwHits];
    uint32_t ord[kBwWarps][kBwHits];           // sorted position -> hit slot
    float T[kBwWarps][kBwHits];                // transmittance before each sorted hit
    float gI[kBwWarps][kBwHits];               // dL/dI per sorted hit
    float gc[kBwWarps][kBwHits][3];            // dL/dc per sorted hit (clamped channels: 0)
    int ncomp[kBwWarps];
};

__device__ __forceinline__ float dsinc_f(float x) {
    // d/dx sin(x)/x = (cos x - sinc x) / x; Taylor -x/3 + x^3/30 below |x| = 0.25
    const float x2 = x * x;
    if (fabsf(x) < 0.25f) return x * fmaf(x2, 1.0f / 30.0f, -1.0f / 3.0f);
    return (__cosf(x) - __sinf(x) / x) / x;
}

// dL/dI of one (ray, record) hit into the MLP parameter gradients of primitive `prim`.
template <int N>
__device__ __forceinline__ void hit_grad(const float4 *__restrict__ rec, const Ray &r, float gI, float omega,
                                         float smax, uint32_t prim, float *g_w1, float *g_b1, float *g_w2,
                                         float *g_b2) {
    // the same intermediate values as exact_hit (hit.cuh)
    const float4 mh = rec[kRecMh];
    const float4 ml = rec[kRecMl];
    const float4 w0 = rec[kRecWh0];
    const float4 w1 = rec[kRecWh1];
    const float tc = fmaf(r.dhz, mh.z, fmaf(r.dhy, mh.y, r.dhx * mh.x));
    const float px = fmaf(tc, r.dhx, -mh.x) + fmaf(tc, r.dlx, -ml.x);
    const float py = fmaf(tc, r.dhy, -mh.y) + fmaf(tc, r.dly, -ml.y);
    const float pz = fmaf(tc, r.dhz, -mh.z) + fmaf(tc, r.dlz, -ml.z);
    const float ax = fmaf(w0.y, r.dhz, fmaf(w0.x, r.dhy, ml.w * r.dhx));
    const float ay = fmaf(w1.x, r.dhz, fmaf(w0.w, r.dhy, w0.z * r.dhx));
    const float az = fmaf(w1.w, r.dhz, fmaf(w1.z, r.dhy, w1.y * r.dhx));
    const float bx = fmaf(w0.y, pz, fmaf(w0.x, py, ml.w * px));
    const float by = fmaf(w1.x, pz, fmaf(w0.w, py, w0.z * px));
    const float bz = fmaf(w1.w, pz, fmaf(w1.z, py, w1.y * px));
    const float A = fmaf(az, az, fmaf(ay, ay, ax * ax));
    const float B = fmaf(az, bz, fmaf(ay, by, ax * bx));
    const float iA = 1.0f / A;
    const float ts = -B * iA;
    const float qx = fmaf(ts, ax, bx), qy = fmaf(ts, ay, by), qz = fmaf(ts, az, bz);
    const float q1 = 1.0f - fmaf(qz, qz, fmaf(qy, qy, qx * qx));
    if (!(q1 > 0.0f)) return;
    const float hc = sqrtf(q1 * iA);
    const float t0 = ts - hc, t1 = ts + hc;
    const float lo_lim = r.t_near - tc, hi_lim = r.t_far - tc;
    const float tlo = t0 > lo_lim ? t0 : lo_lim;
    const float thi = t1 < hi_lim ? t1 : hi_lim;
    if (!(thi > tlo)) return;
    const float dt = thi - tlo, tm = 0.5f * (tlo + thi), hdt = 0.5f * dt;
    const uint32_t wbase = (uint32_t)N * prim;
    float gb2 = 0.f;
    gb2 = gI * dt;
    atomicAdd(g_b2 + prim, gb2);
    const float s1 = omega / smax;
    for (int gq = 0; gq < N / 4; ++gq) {
    const float4 w4 = rec[rec_w2(N) + gq];
    const float w2s[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
    for (int uu = 0; uu < 4; ++uu) {
        const int k = 4 * gq + uu;
        const float4 u = rec[kRecUnits + k];
        const float w2 = w2s[uu];
        const float h = fmaf(u.z, r.dhz, fmaf(u.y, r.dhy, u.x * r.dhx));
        const float g = fmaf(u.z, pz, fmaf(u.y, py, fmaf(u.x, px, u.w)));
        const float phi = fmaf(h, tm, g);
        float sn, cs;
        sincosf(phi, &sn, &cs);
        const float x = h * hdt;
        const float S = fabsf(x) < 0.25f ? fmaf(x * x, fmaf(x * x, 8.3333333e-03f, -1.6666667e-01f), 1.0f)
                                         : sinf(x) / x;
        const float Sp = dsinc_f(x);
        atomicAdd(g_w2 + wbase + k, gI * dt * cs * S);
        const float a_sin = -gI * dt * w2 * sn * S;   // dL/dphi_k (through cos)
        atomicAdd(g_b1 + wbase + k, omega * a_sin);
        const float a_h = gI * dt * w2 * cs * Sp * hdt;   // dL/dh_k through the sinc
        // dphi/dW1' = p + tm d, dh/dW1' = d
        const float gx = a_sin * fmaf(tm, r.dhx, px) + a_h * r.dhx;
        const float gy = a_sin * fmaf(tm, r.dhy, py) + a_h * r.dhy;
        const float gz = a_sin * fmaf(tm, r.dhz, pz) + a_h * r.dhz;
        atomicAdd(g_w1 + 3 * (wbase + k) + 0, s1 * gx);
        atomicAdd(g_w1 + 3 * (wbase + k) + 1, s1 * gy);
        atomicAdd(g_w1 + 3 * (wbase + k) + 2, s1 * gz);
    }
    }
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

template <int N, bool kRay>
__global__ void __launch_bounds__(kBwThreads) k_backward(RenderArgs a, CamBatch cb, const float4 *__restrict__ grad,
                                                         BackwardGrads gr, float omega) {
    extern __shared__ __align__(16) unsigned char bw_raw[];
    BwSmem &sm = *reinterpret_cast<BwSmem *>(bw_raw);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const int W = cb.cams[0].W, H = cb.cams[0].H;
    const int64_t npix = (int64_t)cb.nv * W * H;
    for (int64_t pi = (int64_t)blockIdx.x * kBwWarps + wid; pi < npix; pi += (int64_t)gridDim.x * kBwWarps) {
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
                if (q <= 1.0f) hit = exact_hit<N>(rec, ray, th, tl, kap);
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
        if (cnt > kBwHits) {
            if (lane == 0) atomicAdd(a.counters + kCntBwdSkipped, 1ull);
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
        // ---- forward transmittance, stop, and the back-to-front adjoints (one lane)
        if (lane == 0) {
            float T = 1.f;
            int last = cnt - 1;
            for (int k = 0; k < cnt; ++k) {
                sm.T[wid][k] = T;
                T *= 1.0f - sm.kap[wid][sm.ord[wid][k]];
                if (T < a.t_floor) {
                    last = k;
                    break;
                }
            }
            const float Tend = T;
            float U[3] = {Tend * a.bg[0], Tend * a.bg[1], Tend * a.bg[2]};
            for (int k = last; k >= 0; --k) {
                const int h = (int)sm.ord[wid][k];
                const float kp = sm.kap[wid][h];
                const uint32_t id = sm.id[wid][h];
                const float4 c4 = hit_rgb<kRay>(recs + (size_t)id * rec_f4(N), a.sh, a.sh_degree, id, ray);
                const float c[3] = {c4.y, c4.z, c4.w};
                const float Tk = sm.T[wid][k];
                const float om = fmaxf(1.0f - kp, 1e-20f);
                const float gr_[3] = {G.x, G.y, G.z};
                float dk = G.w * Tend / om;
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    dk = fmaf(gr_[ch], Tk * c[ch] - U[ch] / om, dk);
                    sm.gc[wid][k][ch] = c[ch] > 0.f ? Tk * kp * gr_[ch] : 0.f;
                    U[ch] = fmaf(Tk * kp, c[ch], U[ch]);
                }
                sm.gI[wid][k] = kp > 0.f ? dk * (1.0f - kp) : 0.f;
            }
            sm.ncomp[wid] = last + 1;
        }
        __syncwarp();
        // ---- parameter gradients of the composited hits
        const int nc = sm.ncomp[wid];
        const int ncoef = (a.sh_degree + 1) * (a.sh_degree + 1);
        for (int k = lane; k < nc; k += 32) {
            const int h = (int)sm.ord[wid][k];
            const uint32_t id = sm.id[wid][h];
            const float4 *rec = recs + (size_t)id * rec_f4(N);
            const float *s3 = a.scales + 3 * (size_t)id;
            const float smax = fmaxf(s3[0], fmaxf(s3[1], s3[2]));
            hit_grad<N>(rec, ray, sm.gI[wid][k], omega, smax, id, gr.w1, gr.b1, gr.w2, gr.b2);
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
            const float g0 = sm.gc[wid][k][0], g1 = sm.gc[wid][k][1], g2 = sm.gc[wid][k][2];
            float *gs = gr.sh + 48 * (size_t)id;
            for (int i = 0; i < ncoef; ++i) {
                if (g0 != 0.f) atomicAdd(gs + 3 * i + 0, Y[i] * g0);
                if (g1 != 0.f) atomicAdd(gs + 3 * i + 1, Y[i] * g1);
                if (g2 != 0.f) atomicAdd(gs + 3 * i + 2, Y[i] * g2);
            }
        }
        __syncwarp();
    }
}

template <int N, bool kRay>
cudaError_t launch_backward_n(const RenderArgs &a, const CamBatch &cb, const float *grad, const BackwardGrads &g,
                              float omega, cudaStream_t st) {
    static int resident = 0;
    const int smem = (int)sizeof(BwSmem);
    if (!resident) {
        cudaError_t e = cudaFuncSetAttribute(k_backward<N, kRay>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_backward<N, kRay>, kBwThreads, smem);
        resident = (sms > 0 ? sms : 148) * (per_sm > 0 ? per_sm : 1);
    }
    const int64_t npix = (int64_t)cb.nv * cb.cams[0].W * cb.cams[0].H;
    const int64_t want = (npix + kBwWarps - 1) / kBwWarps;
    const unsigned grid = (unsigned)(want < resident ? want : resident);
    if (grid == 0) return cudaSuccess;
    k_backward<N, kRay><<<grid, kBwThreads, smem, st>>>(a, cb, reinterpret_cast<const float4 *>(grad), g, omega);
    return cudaGetLastError();
}

template <int N>
cudaError_t launch_backward_w(const RenderArgs &a, const CamBatch &cb, const float *grad, const BackwardGrads &g,
                              float omega, cudaStream_t st) {
    return a.colour_ray ? launch_backward_n<N, true>(a, cb, grad, g, omega, st)
                        : launch_backward_n<N, false>(a, cb, grad, g, omega, st);
}

}  // namespace

cudaError_t launch_backward(const RenderArgs &a, const CamBatch &cb, const float *grad, const BackwardGrads &g,
                            float omega, cudaStream_t st) {
    switch (a.n_hidden) {
        case 4: return launch_backward_w<4>(a, cb, grad, g, omega, st);
        case 8: return launch_backward_w<8>(a, cb, grad, g, omega, st);
        case 16: return launch_backward_w<16>(a, cb, grad, g, omega, st);
        case 32: return launch_backward_w<32>(a, cb, grad, g, omega, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace snp
