// render.cu -- K5: per-pixel closed-form splatting with exact per-ray order,
// and K6: exact fallback for pixels whose pending buffer overflowed.
//
// Per pixel (ray o = C, unit d), for every primitive listed in its tile
// in (tile | depth-lower-bound) key order:
//   pre-test   silhouette conic (perspective-exact tangent cone) with a margin;
//   exact hit  analytic line-ellipsoid intersection [t_in, t_out]
//              in a compensated camera-relative frame: p = t_c d - m with m and
//              d carried as hi + lo floats, tau = t - t_c;
//   integral   Eq. 8 in product form (R3): I = dt * (sum_k W2_k cos(g_k + h_k tau_m)
//              sinc(h_k dt / 2) + b2), g_k = W1'_k.p + omega b1_k, h_k = W1'_k.d
//              (Eq. 5 normalisation folded into W1' = omega W1 / ||s||_inf, R2);
//   kernel     kappa = 1 - exp(-max(0, I)) (Eq. 9);
//   order      hits wait in a per-pixel pending buffer sorted by exact
//              (t_in, id) and are emitted once t_in < L of the next listed key
//              (L is a lower bound of t_in for every ray, R19), so blending runs in
//              exact per-ray entry order (R11);
//   blend      C += T kappa c, T *= 1 - kappa, stop at T < floor (Eq. 4, R13).
// Records are staged per tile batch into shared memory with cp.async.bulk
// (UBLKCP) + mbarrier transaction counts, 3-stage ring.
#include <math.h>

#include "snp_internal.cuh"

namespace snp {
namespace {

constexpr int kThreads = 256;       // one 16x16 tile, one pixel per thread
constexpr int kWarps = kThreads / 32;
constexpr int kBatch = 64;          // records per stage
constexpr int kStages = 2;
constexpr int kPendMax = 8;         // per-pixel pending buffer (max occupancy 4-10)
constexpr int kFbGrid = 148 * 2;    // K6 blocks
constexpr int kFbCap = 1024;        // K6 stored hits per warp

struct __align__(16) Smem {
    float4 rec[kStages][kBatch][16];          // 32 KB of records (TMA bulk-staged)
    float L[kStages][kBatch + 1];             // depth lower bounds (+ the next batch's first)
    uint32_t id[kStages][kBatch];
    unsigned long long bar[kStages];
    uint32_t submask[kWarps][2];              // records whose conic box touches warp w's 8x4 block
    uint8_t qj[kWarps][64];                   // per-warp compaction queue of candidate pairs:
    uint8_t ql[kWarps][64];                   //   (record slot j, owner lane)
    float r_th[kWarps][32], r_tl[kWarps][32], r_k[kWarps][32], r_L[kWarps][32];
    float r_r[kWarps][32], r_g[kWarps][32], r_b[kWarps][32];
    uint32_t r_id[kWarps][32], r_j[kWarps][32];
    uint32_t own[kWarps][32];                 // per owner lane: mask of result slots it owns
    float p_thi[kPendMax][kThreads];          // pending hits, SoA, column per thread
    float p_tlo[kPendMax][kThreads];
    float p_kap[kPendMax][kThreads];
    float p_r[kPendMax][kThreads];
    float p_g[kPendMax][kThreads];
    float p_b[kPendMax][kThreads];
    uint32_t p_id[kPendMax][kThreads];
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

struct Ray {
    float dhx, dhy, dhz, dlx, dly, dlz;   // unit direction, hi + lo
    float t_near, t_far;
};

__device__ __forceinline__ Ray make_ray(const DevCam &cam, int x, int y) {
    const double u = ((double)x + 0.5 - (double)cam.cx) / (double)cam.fx;
    const double v = ((double)y + 0.5 - (double)cam.cy) / (double)cam.fy;
    double r[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        r[i] = (double)cam.R[3 * i] * u + (double)cam.R[3 * i + 1] * v + (double)cam.R[3 * i + 2];
    const double nd = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    Ray ray;
    const double d0 = r[0] / nd, d1 = r[1] / nd, d2 = r[2] / nd;
    ray.dhx = (float)d0; ray.dlx = (float)(d0 - (double)ray.dhx);
    ray.dhy = (float)d1; ray.dly = (float)(d1 - (double)ray.dhy);
    ray.dhz = (float)d2; ray.dlz = (float)(d2 - (double)ray.dhz);
    ray.t_near = cam.t_near;
    ray.t_far = cam.t_far;
    return ray;
}

// cos / sin after Cody-Waite reduction to [-pi, pi] (the MUFU argument range).
__device__ __forceinline__ float reduce_2pi(float x) {
    const float n = rintf(x * 0.15915494309189535f);
    float r = fmaf(-n, 6.28318548202514648f, x);
    return fmaf(-n, -1.7484556000744487e-07f, r);
}
__device__ __forceinline__ float sinc_f(float x) {
    const float x2 = x * x;
    const float poly = fmaf(x2, fmaf(x2, fmaf(x2, -1.9841270e-04f, 8.3333333e-03f), -1.6666667e-01f), 1.0f);
    const float s = __fdividef(__sinf(reduce_2pi(x)), x);
    return fabsf(x) < 0.25f ? poly : s;
}

// Exact hit + kernel for one (ray, record).  Returns false on a miss.
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
    const float A = fmaf(az, az, fmaf(ay, ay, ax * ax));
    const float B = fmaf(az, bz, fmaf(ay, by, ax * bx));
    const float Cq = fmaf(bz, bz, fmaf(by, by, bx * bx)) - 1.0f;
    const float disc = fmaf(B, B, -A * Cq);
    if (!(disc > 0.0f)) return false;
    const float sq = disc * rsqrtf(disc);
    const float qq = -(B + copysignf(sq, B));
    float t0 = __fdividef(qq, A), t1 = __fdividef(Cq, qq);
    if (t0 > t1) { const float t = t0; t0 = t1; t1 = t; }
    const float lo_lim = r.t_near - tc, hi_lim = r.t_far - tc;
    const bool clipped = !(t0 > lo_lim);
    const float tlo = clipped ? lo_lim : t0;
    const float thi = t1 < hi_lim ? t1 : hi_lim;
    if (!(thi > tlo)) return false;
    const float dt = thi - tlo;
    const float tm = 0.5f * (tlo + thi);
    const float hdt = 0.5f * dt;
    float acc = 0.f;
    const float4 W2a = rec[kRecW2], W2b = rec[kRecW2 + 1];
    const float W2[8] = {W2a.x, W2a.y, W2a.z, W2a.w, W2b.x, W2b.y, W2b.z, W2b.w};
#pragma unroll
    for (int k = 0; k < kHidden; ++k) {
        const float4 u = rec[kRecUnits + k];
        const float h = fmaf(u.z, r.dhz, fmaf(u.y, r.dhy, u.x * r.dhx));
        const float g = fmaf(u.z, pz, fmaf(u.y, py, fmaf(u.x, px, u.w)));
        const float phi = fmaf(h, tm, g);
        acc = fmaf(W2[k], __cosf(reduce_2pi(phi)) * sinc_f(h * hdt), acc);
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

struct PixelState {
    float T, cr, cg, cb;
    int npend;
    bool done;
    bool overflow;
    uint32_t composited;
};

// Emit every pending hit with t_in < L (strictly), smallest first (Eq. 4 front to back).
__device__ __forceinline__ void emit(Smem &sm, PixelState &ps, float L, float t_floor) {
    const int tid = threadIdx.x;
    while (ps.npend > 0) {
        const int k = ps.npend - 1;
        const float th = sm.p_thi[k][tid], tl = sm.p_tlo[k][tid];
        if (!(th < L || (th == L && tl < 0.f))) break;
        const float kap = sm.p_kap[k][tid];
        const float w = ps.T * kap;
        ps.cr = fmaf(w, sm.p_r[k][tid], ps.cr);
        ps.cg = fmaf(w, sm.p_g[k][tid], ps.cg);
        ps.cb = fmaf(w, sm.p_b[k][tid], ps.cb);
        ps.T *= (1.0f - kap);
        ps.npend = k;
        ++ps.composited;
        if (ps.T < t_floor) {
            ps.done = true;
            break;
        }
    }
}

// Insert one hit into the pixel's pending buffer (kept in descending (t_in, id)
// order, smallest at npend-1).  L = key of the hit's own entry: every hit not yet
// seen has t_in >= L, so pending hits below L may be emitted to make room.
__device__ __forceinline__ void insert_hit(Smem &sm, PixelState &ps, float th, float tl, uint32_t id, float kap,
                                           float r, float g, float b, float L, int plimit, float t_floor) {
    const int tid = threadIdx.x;
    if (ps.npend >= plimit) emit(sm, ps, L, t_floor);
    if (ps.done) return;
    if (ps.npend >= plimit) {
        ps.overflow = true;   // K6 re-renders this pixel exactly
        ps.done = true;
        return;
    }
    int k = ps.npend;
    while (k > 0) {
        const float ph = sm.p_thi[k - 1][tid], pl = sm.p_tlo[k - 1][tid];
        const uint32_t pid = sm.p_id[k - 1][tid];
        if (!before(ph, pl, pid, th, tl, id)) break;
        sm.p_thi[k][tid] = ph;
        sm.p_tlo[k][tid] = pl;
        sm.p_id[k][tid] = pid;
        sm.p_kap[k][tid] = sm.p_kap[k - 1][tid];
        sm.p_r[k][tid] = sm.p_r[k - 1][tid];
        sm.p_g[k][tid] = sm.p_g[k - 1][tid];
        sm.p_b[k][tid] = sm.p_b[k - 1][tid];
        --k;
    }
    sm.p_thi[k][tid] = th;
    sm.p_tlo[k][tid] = tl;
    sm.p_id[k][tid] = id;
    sm.p_kap[k][tid] = kap;
    sm.p_r[k][tid] = r;
    sm.p_g[k][tid] = g;
    sm.p_b[k][tid] = b;
    ++ps.npend;
}

__global__ void __launch_bounds__(kThreads, 2) k_render(RenderArgs a, CamBatch cb) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem &sm = *reinterpret_cast<Smem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    const int vloc = blockIdx.y;
    const int64_t view = cb.view0 + vloc;
    const DevCam &cam = cb.cams[vloc];
    const int tx = blockIdx.x % a.tiles_x;
    const int ty = a.row_begin + (blockIdx.x / a.tiles_x) * a.row_stride;
    const int tile = ty * a.tiles_x + tx;
    const int x = tx * kTile + (wid & 1) * 8 + (lane & 7);
    const int y = ty * kTile + (wid >> 1) * 4 + (lane >> 3);
    const bool inside = x < cam.W && y < cam.H;
    const uint32_t beg = a.ranges[2 * (view * a.tiles_per_view + tile)];
    const uint32_t end = a.ranges[2 * (view * a.tiles_per_view + tile) + 1];
    const int nb = (int)((end - beg + kBatch - 1) / kBatch);
    const float4 *recs = a.records + (size_t)view * (size_t)a.n * 16;

    if (tid == 0)
        for (int s = 0; s < kStages; ++s) mbar_init(&sm.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    // producer (warps 0-1): one cp.async.bulk per 256-byte record into slot b % kStages
    auto issue = [&](int b) {
        const int slot = b % kStages;
        const uint32_t e0 = beg + (uint32_t)b * kBatch;
        const uint32_t cnt = min((uint32_t)kBatch, end - e0);
        if (tid == 0) mbar_arrive_expect_tx(&sm.bar[slot], cnt * 256u);
        __syncwarp();
        const int j = tid;  // tid < 64
        if ((uint32_t)j < cnt) {
            const uint32_t id = a.vals[e0 + j];
            sm.id[slot][j] = id;
            sm.L[slot][j] = __uint_as_float((uint32_t)a.keys[e0 + j]);
            bulk_g2s(&sm.rec[slot][j][0], recs + (size_t)id * 16, 256u, &sm.bar[slot]);
        }
        if (j == 0) {
            const uint32_t nx = e0 + cnt;
            sm.L[slot][cnt] = nx < end ? __uint_as_float((uint32_t)a.keys[nx]) : INFINITY;
        }
    };
    int issued = nb < kStages ? nb : kStages;
    if (tid < 64)
        for (int b = 0; b < issued; ++b) issue(b);

    const Ray ray = inside ? make_ray(cam, x, y) : Ray{0, 0, 1, 0, 0, 0, cam.t_near, cam.t_far};
    const float pxf = (float)x + 0.5f, pyf = (float)y + 0.5f;
    // this thread's pre-pass pairs: record pj against the 8x4 blocks of warps ps0 and ps0 + 4
    const int pj = tid & 63, ps0 = tid >> 6;
    const float bx0 = (float)(tx * kTile + (ps0 & 1) * 8) + 0.5f, by0 = (float)(ty * kTile + (ps0 >> 1) * 4) + 0.5f;
    const float by1 = by0 + 8.0f;  // block ps0 + 4 sits two block-rows (8 px) lower
    PixelState ps{1.f, 0.f, 0.f, 0.f, 0, !inside, false, 0u};
    uint32_t tested_end = end;
    uint32_t n_cand = 0, n_hit = 0;
    const int plimit = a.pending_limit;
    __syncthreads();

    int b = 0;
    for (; b < nb; ++b) {
        const int slot = b % kStages;
        mbar_wait(&sm.bar[slot], (uint32_t)((b / kStages) & 1));
        const uint32_t e0 = beg + (uint32_t)b * kBatch;
        const int cnt = (int)min((uint32_t)kBatch, end - e0);
        // ---- pre-pass: which records can touch each warp's 8x4 pixel block
        {
            bool t0 = false, t1 = false;
            if (pj < cnt) {
                const float4 c0 = sm.rec[slot][pj][kRecConic];
                const float cc = sm.rec[slot][pj][kRecConicRgb].x;
                const float hb = 0.5f * c0.w;
                const float det = fmaf(c0.z, cc, -hb * hb);
                if (det > 0.f) {
                    const float rx = sqrtf(cc / det) * 1.001f + 1e-3f;
                    const float ry = sqrtf(c0.z / det) * 1.001f + 1e-3f;
                    const bool ox = c0.x + rx >= bx0 && c0.x - rx <= bx0 + 7.0f;
                    t0 = ox && c0.y + ry >= by0 && c0.y - ry <= by0 + 3.0f;
                    t1 = ox && c0.y + ry >= by1 && c0.y - ry <= by1 + 3.0f;
                } else {
                    t0 = t1 = true;   // no conic (straddles the camera plane / camera inside)
                }
            }
            if (a.debug_flags & 1) t0 = t1 = pj < cnt;
            const uint32_t m0 = __ballot_sync(0xffffffffu, t0);
            const uint32_t m1 = __ballot_sync(0xffffffffu, t1);
            if (lane == 0) {
                sm.submask[ps0][wid & 1] = m0;
                sm.submask[ps0 + 4][wid & 1] = m1;
            }
        }
        __syncthreads();
        // ---- per warp: candidate pairs -> compaction queue -> 32-wide exact rounds
        if (!__all_sync(0xffffffffu, ps.done)) {
            unsigned long long m = (unsigned long long)sm.submask[wid][0] |
                                   ((unsigned long long)sm.submask[wid][1] << 32);
            int qcount = 0;
            auto round = [&](int n) {
                __syncwarp();
                const bool valid = lane < n;
                const int owner = valid ? sm.ql[wid][lane] : lane;
                const int j = valid ? sm.qj[wid][lane] : 0;
                Ray ro;
                ro.dhx = __shfl_sync(0xffffffffu, ray.dhx, owner);
                ro.dhy = __shfl_sync(0xffffffffu, ray.dhy, owner);
                ro.dhz = __shfl_sync(0xffffffffu, ray.dhz, owner);
                ro.dlx = __shfl_sync(0xffffffffu, ray.dlx, owner);
                ro.dly = __shfl_sync(0xffffffffu, ray.dly, owner);
                ro.dlz = __shfl_sync(0xffffffffu, ray.dlz, owner);
                ro.t_near = cam.t_near;   // uniform: lanes outside the image carry a dummy ray
                ro.t_far = cam.t_far;
                sm.own[wid][lane] = 0u;
                bool hit = false;
                if (valid) {
                    float th, tl, kap;
                    const float4 *rec = &sm.rec[slot][j][0];
                    hit = exact_hit(rec, ro, th, tl, kap);
                    if (hit) {
                        const float4 rgb = rec[kRecConicRgb];
                        sm.r_th[wid][lane] = th;
                        sm.r_tl[wid][lane] = tl;
                        sm.r_k[wid][lane] = kap;
                        sm.r_L[wid][lane] = sm.L[slot][j];
                        sm.r_r[wid][lane] = rgb.y;
                        sm.r_g[wid][lane] = rgb.z;
                        sm.r_b[wid][lane] = rgb.w;
                        sm.r_id[wid][lane] = sm.id[slot][j];
                        sm.r_j[wid][lane] = (uint32_t)j;
                    }
                }
                const uint32_t peers = __match_any_sync(0xffffffffu, hit ? owner : 64 + lane);
                __syncwarp();
                if (hit && lane == __ffs(peers) - 1) sm.own[wid][owner] = peers;
                __syncwarp();
                uint32_t mine = sm.own[wid][lane];
                n_hit += __popc(mine);
                while (mine) {   // in queue order == record order for this pixel
                    const int k = __ffs(mine) - 1;
                    mine &= mine - 1u;
                    if (ps.done) continue;
                    insert_hit(sm, ps, sm.r_th[wid][k], sm.r_tl[wid][k], sm.r_id[wid][k], sm.r_k[wid][k],
                               sm.r_r[wid][k], sm.r_g[wid][k], sm.r_b[wid][k], sm.r_L[wid][k], plimit,
                               a.t_floor);
                    if (ps.done && tested_end == end) tested_end = e0 + sm.r_j[wid][k] + 1;
                }
                __syncwarp();
            };
            while (m) {
                const int j = __ffsll(m) - 1;
                m &= m - 1ull;
                const float4 c0 = sm.rec[slot][j][kRecConic];
                const float cc = sm.rec[slot][j][kRecConicRgb].x;
                const float dx = pxf - c0.x, dy = pyf - c0.y;
                const float q = fmaf(cc * dy, dy, dx * fmaf(c0.w, dy, c0.z * dx));
                const bool cand = !ps.done && q <= 1.0f;
                const uint32_t cm = __ballot_sync(0xffffffffu, cand);
                if (cm) {
                    if (cand) {
                        const int pos = qcount + __popc(cm & lt_mask);
                        sm.qj[wid][pos] = (uint8_t)j;
                        sm.ql[wid][pos] = (uint8_t)lane;
                        ++n_cand;
                    }
                    qcount += __popc(cm);
                    if (qcount >= 32) {
                        round(32);
                        const int rem = qcount - 32;
                        uint8_t vj = 0, vl = 0;
                        if (lane < rem) {
                            vj = sm.qj[wid][32 + lane];
                            vl = sm.ql[wid][32 + lane];
                        }
                        __syncwarp();
                        if (lane < rem) {
                            sm.qj[wid][lane] = vj;
                            sm.ql[wid][lane] = vl;
                        }
                        __syncwarp();
                        qcount = rem;
                    }
                }
            }
            if (qcount > 0) round(qcount);
        }
        if (!ps.done) {
            emit(sm, ps, sm.L[slot][cnt], a.t_floor);
            if (ps.done && tested_end == end) tested_end = e0 + cnt;
        }
        const int all_done = __syncthreads_and(ps.done);
        if (all_done) {
            ++b;
            break;
        }
        if (issued < nb) {
            if (tid < 64) issue(issued);
            ++issued;
        }
    }
    // drain: bulk copies still in flight must land before the CTA exits
    for (int bb = b; bb < issued; ++bb) mbar_wait(&sm.bar[bb % kStages], (uint32_t)((bb / kStages) & 1));
    if (!ps.done) emit(sm, ps, INFINITY, a.t_floor);

    if (inside) {
        if (ps.overflow) {
            const unsigned long long slot = atomicAdd(a.counters + kCntFallbackQueue, 1ull);
            if ((int64_t)slot < a.fallback_capacity) {
                a.fallback[2 * slot] = (uint32_t)view;
                a.fallback[2 * slot + 1] = (uint32_t)(y * cam.W + x);
            }
        } else {
            const float4 o = make_float4(fmaf(ps.T, a.bg[0], ps.cr), fmaf(ps.T, a.bg[1], ps.cg),
                                         fmaf(ps.T, a.bg[2], ps.cb), 1.0f - ps.T);
            reinterpret_cast<float4 *>(a.out)[((size_t)view * cam.H + y) * cam.W + x] = o;
        }
    }
    // counters: one atomic per warp per counter
    const unsigned long long tested = inside ? (unsigned long long)(tested_end - beg) : 0ull;
    const unsigned long long v[5] = {tested, n_cand, n_hit, ps.composited, (unsigned long long)ps.overflow};
#pragma unroll
    for (int c = 0; c < 5; ++c) {
        unsigned long long s = v[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (lane == 0 && s) atomicAdd(a.counters + kCntTested + c, s);
    }
}

__device__ __forceinline__ bool fb_hit(const float4 *rec, const Ray &ray, float pxf, float pyf, float &th,
                                       float &tl, float &kap) {
    const float4 c0 = rec[kRecConic];
    const float cc = rec[kRecConicRgb].x;
    const float dx = pxf - c0.x, dy = pyf - c0.y;
    const float q = fmaf(cc * dy, dy, dx * fmaf(c0.w, dy, c0.z * dx));
    if (!(q <= 1.0f)) return false;
    return exact_hit(rec, ray, th, tl, kap);
}

// K6: exact per-pixel fallback (one warp per overflowed pixel).  Phase A stores
// every hit of the tile list once (t_in hi/lo, kappa, id) in a per-warp scratch;
// phase B blends them by repeated selection of the next smallest (t_in, id).
// If a pixel has more than kFbCap hits, phase B recomputes hits instead of
// reading the scratch (same result, slower).
__global__ void __launch_bounds__(256) k_fallback(RenderArgs a, CamBatch cb) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt_mask = (1u << lane) - 1u;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float4 *scratch = a.fb_scratch + gw * kFbCap;
    int64_t nq = (int64_t)a.counters[kCntFallbackQueue];
    if (nq > a.fallback_capacity) nq = a.fallback_capacity;
    for (int64_t qi = gw; qi < nq; qi += nw) {
        const int64_t view = a.fallback[2 * qi];
        if (view < cb.view0 || view >= cb.view0 + cb.nv) continue;
        const DevCam &cam = cb.cams[view - cb.view0];
        const uint32_t pix = a.fallback[2 * qi + 1];
        const int x = (int)(pix % (uint32_t)cam.W), y = (int)(pix / (uint32_t)cam.W);
        const int tile = (y / kTile) * a.tiles_x + (x / kTile);
        const uint32_t beg = a.ranges[2 * (view * a.tiles_per_view + tile)];
        const uint32_t end = a.ranges[2 * (view * a.tiles_per_view + tile) + 1];
        const float4 *recs = a.records + (size_t)view * (size_t)a.n * 16;
        const Ray ray = make_ray(cam, x, y);
        const float pxf = (float)x + 0.5f, pyf = (float)y + 0.5f;
        // phase A
        int count = 0;
        for (uint32_t e0 = beg; e0 < end; e0 += 32) {
            const uint32_t e = e0 + lane;
            float th = 0.f, tl = 0.f, kap = 0.f;
            uint32_t id = 0;
            bool hit = false;
            if (e < end) {
                id = a.vals[e];
                hit = fb_hit(recs + (size_t)id * 16, ray, pxf, pyf, th, tl, kap);
            }
            const uint32_t hm = __ballot_sync(0xffffffffu, hit);
            const int pos = count + __popc(hm & lt_mask);
            if (hit && pos < kFbCap) scratch[pos] = make_float4(th, tl, kap, __uint_as_float(id));
            count += __popc(hm);
        }
        __syncwarp();
        const bool stored = count <= kFbCap;
        // phase B
        float T = 1.f, cr = 0.f, cg = 0.f, cbl = 0.f;
        float lh = -INFINITY, ll = 0.f;
        uint32_t lid = 0;
        bool first = true;
        unsigned long long ncomp = 0;
        while (true) {
            float bh = INFINITY, bl = 0.f, bk = 0.f;
            uint32_t bid = 0xffffffffu;
            bool found = false;
            if (stored) {
                for (int k = lane; k < count; k += 32) {
                    const float4 h = scratch[k];
                    const uint32_t id = __float_as_uint(h.w);
                    if (!first && !before(lh, ll, lid, h.x, h.y, id)) continue;
                    if (!found || before(h.x, h.y, id, bh, bl, bid)) {
                        bh = h.x; bl = h.y; bid = id; bk = h.z; found = true;
                    }
                }
            } else {
                for (uint32_t e = beg + lane; e < end; e += 32) {
                    const uint32_t id = a.vals[e];
                    float th, tl, kap;
                    if (!fb_hit(recs + (size_t)id * 16, ray, pxf, pyf, th, tl, kap)) continue;
                    if (!first && !before(lh, ll, lid, th, tl, id)) continue;
                    if (!found || before(th, tl, id, bh, bl, bid)) {
                        bh = th; bl = tl; bid = id; bk = kap; found = true;
                    }
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float oh = __shfl_xor_sync(0xffffffffu, bh, o);
                const float ol = __shfl_xor_sync(0xffffffffu, bl, o);
                const uint32_t oid = __shfl_xor_sync(0xffffffffu, bid, o);
                const float ok = __shfl_xor_sync(0xffffffffu, bk, o);
                const bool of = __shfl_xor_sync(0xffffffffu, found, o);
                if (of && (!found || before(oh, ol, oid, bh, bl, bid))) {
                    bh = oh; bl = ol; bid = oid; bk = ok; found = true;
                }
            }
            if (!found) break;
            const float4 rgb = recs[(size_t)bid * 16 + kRecConicRgb];
            const float w = T * bk;
            cr = fmaf(w, rgb.y, cr);
            cg = fmaf(w, rgb.z, cg);
            cbl = fmaf(w, rgb.w, cbl);
            T *= (1.f - bk);
            ++ncomp;
            lh = bh; ll = bl; lid = bid; first = false;
            if (T < a.t_floor) break;
        }
        if (lane == 0) {
            reinterpret_cast<float4 *>(a.out)[((size_t)view * cam.H + y) * cam.W + x] =
                make_float4(fmaf(T, a.bg[0], cr), fmaf(T, a.bg[1], cg), fmaf(T, a.bg[2], cbl), 1.f - T);
            atomicAdd(a.counters + kCntComposited, ncomp);
        }
        __syncwarp();
    }
}

}  // namespace

int64_t fallback_scratch_float4() { return (int64_t)kFbGrid * 256 / 32 * kFbCap; }

cudaError_t launch_render(const RenderArgs &a, const CamBatch &cams, cudaStream_t st) {
    static bool attr_set = false;
    const int smem = (int)sizeof(Smem);
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_render, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    dim3 grid((unsigned)(a.tiles_x * a.stripe_rows), (unsigned)cams.nv);
    if (grid.x == 0) return cudaSuccess;
    k_render<<<grid, kThreads, smem, st>>>(a, cams);
    return cudaGetLastError();
}

cudaError_t launch_fallback(const RenderArgs &a, const CamBatch *cams, int n_batches, cudaStream_t st) {
    for (int i = 0; i < n_batches; ++i) k_fallback<<<kFbGrid, 256, 0, st>>>(a, cams[i]);
    return cudaGetLastError();
}

}  // namespace snp
