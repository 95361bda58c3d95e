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
//   order      hits wait in a per-pixel pending list and are blended, smallest
//              (t_in, id) first, once t_in < L of the next unprocessed key (L is a
//              lower bound of t_in for every ray, R19): exact per-ray entry order
//              (R11);
//   blend      C += T kappa c, T *= 1 - kappa, stop at T < floor (Eq. 4, R13).
//
// K5 is persistent and warp-specialised: per CTA one producer warp streams the
// record batches of successive tiles (tile ids from a global atomic queue) into
// a 4-stage shared-memory ring with one cp.async.bulk (UBLKCP) per 256-byte
// record, completing on mbarrier transaction counts; 8 consumer warps (one 8x4
// pixel block each) release slots through per-slot "empty" mbarriers, so there
// is no CTA-wide barrier and the next tile's records arrive while the current
// tile finishes.
#include <math.h>

#include <algorithm>

#include "hit.cuh"
#include "snp_internal.cuh"

namespace snp {
namespace {

constexpr int kConsumers = 8;                      // consumer warps = 8x4 pixel blocks of a tile
constexpr int kThreads = (kConsumers + 1) * 32;    // + 1 producer warp
constexpr int kWarps = kConsumers;
constexpr int kBatch = 32;          // records per stage (one per producer lane)
constexpr int kQueue = 128;         // per-warp candidate ring (power of two, >= 31 + 2 x 32)
// Per hidden width N: the staged record stride (rec_f4(N) float4, made odd so that the
// distinct records one warp reads fall in distinct bank groups: 17 at N = 8) and the
// TMA ring depth (6 at N <= 8: 2 CTAs x ~106 KB per SM; fewer for the longer records).
template <int N>
struct Cfg {
    static constexpr int kRecStride = rec_f4(N) | 1;
#ifdef SNP_AB_STAGES
    static constexpr int kStages = N <= 8 ? SNP_AB_STAGES : (N == 16 ? 4 : 2);
#else
    static constexpr int kStages = N <= 8 ? 6 : (N == 16 ? 4 : 2);
#endif
    static constexpr uint32_t kRecBytes = 16u * rec_f4(N);
};
#ifdef SNP_AB_PEND
constexpr int kPend = SNP_AB_PEND;
#else
constexpr int kPend = 16;           // per-pixel pending hits (sorted ring)
#endif
static_assert((kPend & (kPend - 1)) == 0, "the pending ring needs a power of two");
constexpr int kTileRing = 8;        // tiles in flight tracked for early skipping

template <int N>
struct __align__(16) Smem {
    static constexpr int kStages = Cfg<N>::kStages;
    float4 rec[kStages][kBatch][Cfg<N>::kRecStride];  // records, cp.async.bulk-staged, padded to an odd
                                                      // float4 count so that 8 distinct records read by
                                                      // one warp hit 8 distinct 16-byte bank groups
    float L[kStages][kBatch + 1];             // depth lower bounds (+ the next batch's first)
    uint32_t id[kStages][kBatch];
    // slot metadata written by the producer before its arrive (release)
    int32_t m_tile[kStages];                  // flattened (view, stripe tile) index, -1 = end of work
    int32_t m_cnt[kStages];
    int32_t m_flags[kStages];                 // 1 = first batch of its tile, 2 = last batch
    int32_t m_seq[kStages];                   // tile sequence number within this CTA
    unsigned long long full[kStages];         // TMA transaction barriers (1 arrival + bytes)
    unsigned long long empty[kStages];        // slot released by all consumer warps
    int32_t tdone[kTileRing];                 // consumer warps finished with tile seq % kTileRing
    int32_t next_tile;
    int32_t warps_done;                       // warps of this CTA that have finished (K5 exit signal)
    uint8_t qj[kWarps][kQueue];               // per-warp compaction queue of candidate pairs
    uint8_t ql[kWarps][kQueue];               //   (record slot j, owner lane), a ring from qhead
    float p_thi[kPend][kWarps * 32];          // pending hits, one column per pixel, kept sorted by
                                              // (t_in, id) in a ring starting at the head: t_in's
                                              // high part, kappa, and tin_code(t_in) << 24 | id, so
                                              // that (p_thi, p_id) orders by the compensated t_in
                                              // (hi + lo) then by id
    float p_kap[kPend][kWarps * 32];
    uint32_t p_id[kPend][kWarps * 32];
    uint32_t p_in[kWarps * 32];               // per owner pixel: lanes holding a hit for it this round
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
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// suspend-time hint: the waiting warp sleeps until the phase completes (or the hint
// expires) instead of spinning on issue slots the working warps need
constexpr uint32_t kSuspendNs = 0x989680;
__device__ __forceinline__ bool mbar_try(unsigned long long *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(kSuspendNs)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// t_in = t_hi + t_lo (TwoSum, |t_lo| <= ulp(t_hi)/2) as a 5-bit code of t_lo in units
// of ulp(t_hi)/32, monotone in t_lo: among hits with equal t_hi, (code, id) orders by
// t_in up to 2^-5 ulp (~4e-9 relative), far inside the 1e-7 near-tie window of R23,
// and exact ties (both clipped to t_near: t_lo = 0) fall back to the id (R11).
// Pending entry word: code << 27 | grazing exponent << 24 | primitive id (kMaxPrims).
__device__ __forceinline__ uint32_t tin_code(float th, float tl) {
    const int E = max((int)((__float_as_uint(th) >> 23) & 0xffu), 32);
    const float sc = __uint_as_float((uint32_t)(282 - E) << 23);   // 2^(155 - E) = 32 / ulp(t_hi)
    return (uint32_t)fminf(fmaxf(fmaf(tl, sc, 16.0f), 0.0f), 31.0f);
}
constexpr uint32_t kIdMask = (1u << 24) - 1u;   // kMaxPrims

// The owner lane's view of its pixel's pending ring (the entries live in shared
// memory, column tid; count, head and the largest entry are kept in registers).
struct Pending {
    int n, head;
    float tail_t;
    uint32_t tail_id;
    bool ovf;
};

struct PixelState {
    float T, cr, cg, cb;
    bool done;
    bool overflow;
    uint32_t composited;
};

// Blend, front to back, every pending hit of this thread's pixel with t_in < L
// (strictly): every hit not yet inserted has t_in >= L (R19), so these are
// exactly the next hits of the ray in (t_in, id) order (Eq. 4).  The
// list is sorted, so they are popped from its head.
// K5 grad mode (the backward's forward traversal): the pixel's
// dL/d(out) G and forward result F, and the warp's shared-memory entry staging.
struct GradCtx {
    float4 G, F;
    GradEntry *chunk;     // this warp's current chunk of a.grad_entries (nullptr: none)
    FwdEntry *rchunk;     //   (record mode) of a.rec_entries
    int64_t cbase;        //   its first slot (keys)
    int *cnt;             // its fill count (shared; read and written warp-synchronously)
    uint32_t pix;         // view within the batch << 24 | y * W + x
};

template <int N, bool kRay>
__device__ __forceinline__ void emit(Smem<N> &sm, PixelState &ps, Pending &pd, float L, float t_floor,
                                     const float4 *recs, const RenderArgs &a, const Ray &ray) {
    const int tid = threadIdx.x;
    int n = pd.n;
    int h = pd.head;
    while (n > 0) {
        const float t = sm.p_thi[h][tid];
        if (!(t < L)) break;
        const float kap = sm.p_kap[h][tid];
        const uint32_t word = sm.p_id[h][tid];
        const uint32_t pid = word & kIdMask;
        SNP_CHECK(h >= 0 && h < kPend && n <= kPend && (int64_t)pid < a.n);
        const int gexp = (int)((word >> 24) & 7u);
        // a grazing hit whose fp32 kappa could move this pixel by more than 6e-5 (hit.cuh,
        // kGrazeK0): the pixel goes to K6, which evaluates it with FP64 roots
        if (gexp && (gexp == 7 || ps.T * (float)(1 << gexp) > 2.0f)) {
            atomicAdd(a.counters + kCntGraze, 1ull);   // (rare)
            ps.overflow = true;
            ps.done = true;
            break;
        }
        const float4 rgb = hit_rgb<kRay>(recs + (size_t)pid * rec_f4(N), a.sh, a.sh_degree, pid, ray);
        const float w = ps.T * kap;
        ps.cr = fmaf(w, rgb.y, ps.cr);
        ps.cg = fmaf(w, rgb.z, ps.cg);
        ps.cb = fmaf(w, rgb.w, ps.cb);
        ps.T *= (1.0f - kap);
        ++ps.composited;
        --n;
        h = (h + 1) & (kPend - 1);
        if (ps.T < t_floor) {
            ps.done = true;
            break;
        }
    }
    pd.n = n;
    pd.head = h;
}

// K5 grad / record mode's emission: the same blend (same order and arithmetic) as emit(),
// warp-synchronous (every lane of the warp calls it; `active` = this lane's pixel emits)
// so that the entries' chunk slots come from a ballot instead of shared-memory atomics.
// Grad mode: each composited hit of a pixel with a nonzero dL/d(out) becomes a GradEntry
// (hit_out_grads); record mode: every composited hit becomes a FwdEntry (T in front of
// it, kappa, the colour accumulated up to and including it).
template <int N, bool kRay, bool kRecord>
__device__ __forceinline__ void emit_sync(Smem<N> &sm, PixelState &ps, Pending &pd, bool active, float L,
                                          float t_floor, const float4 *recs, const RenderArgs &a, const Ray &ray,
                                          GradCtx &gx) {
    const int tid = threadIdx.x, lane = tid & 31;
    const uint32_t lt_mask = (1u << lane) - 1u;
    int n = pd.n;
    int h = pd.head;
    bool more = active && n > 0;
    int fill = *gx.cnt;   // (warp-uniform: grad_reserve synchronised the warp)
    const bool has_g = kRecord || gx.G.x != 0.f || gx.G.y != 0.f || gx.G.z != 0.f || gx.G.w != 0.f;
    while (__any_sync(0xffffffffu, more)) {
        bool write = false;
        uint32_t wid_ = 0;
        float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f, v4 = 0.f, v5 = 0.f;   // the entry's payload
        if (more) {
            const float t = sm.p_thi[h][tid];
            if (!(t < L)) {
                more = false;
            } else {
                const float kap = sm.p_kap[h][tid];
                const uint32_t word = sm.p_id[h][tid];
                const uint32_t pid = word & kIdMask;
                SNP_CHECK(h >= 0 && h < kPend && n <= kPend && (int64_t)pid < a.n);
                const int gexp = (int)((word >> 24) & 7u);
                if (gexp && (gexp == 7 || ps.T * (float)(1 << gexp) > 2.0f)) {   // -> K6 / K7 per pixel
                    atomicAdd(a.counters + kCntGraze, 1ull);
                    ps.overflow = true;
                    ps.done = true;
                    more = false;
                } else {
                    const float4 rgb = hit_rgb<kRay>(recs + (size_t)pid * rec_f4(N), a.sh, a.sh_degree, pid, ray);
                    const float Tb = ps.T;
                    const float w = Tb * kap;
                    ps.cr = fmaf(w, rgb.y, ps.cr);
                    ps.cg = fmaf(w, rgb.z, ps.cg);
                    ps.cb = fmaf(w, rgb.w, ps.cb);
                    if (has_g) {
                        wid_ = pid;
                        write = true;
                        if (kRecord) {
                            v0 = Tb; v1 = kap; v2 = ps.cr; v3 = ps.cg; v4 = ps.cb;
                        } else {
                            float gc[3];
                            hit_out_grads(gx.G, gx.F, Tb, kap, rgb, ps.cr, ps.cg, ps.cb, v0, gc);
                            v1 = gc[0]; v2 = gc[1]; v3 = gc[2];
                        }
                    }
                    ps.T *= (1.0f - kap);
                    ++ps.composited;
                    --n;
                    h = (h + 1) & (kPend - 1);
                    if (ps.T < t_floor) {
                        ps.done = true;
                        more = false;
                    }
                    if (n == 0) more = false;
                }
            }
        }
        const uint32_t wm = __ballot_sync(0xffffffffu, write);
        if (write) {
            const int slot = fill + __popc(wm & lt_mask);
            SNP_CHECK(slot >= 0 && slot < kGradChunk);
            if (kRecord ? gx.rchunk != nullptr : gx.chunk != nullptr) {
                if (kRecord) {
                    FwdEntry e;
                    e.pix = gx.pix; e.id = wid_; e.T = v0; e.kap = v1; e.cr = v2; e.cg = v3; e.cb = v4; e.pad = v5;
                    gx.rchunk[slot] = e;
                } else {
                    GradEntry e;
                    e.pix = gx.pix; e.id = wid_; e.gI = v0; e.gc0 = v1; e.gc1 = v2; e.gc2 = v3;
                    gx.chunk[slot] = e;
                }
                if (a.grad_keys)   // K7s's counting sort key
                    a.grad_keys[gx.cbase + slot] = (gx.pix >> 24) * (uint32_t)a.n + wid_;
            }
        }
        fill += __popc(wm);
    }
    if (lane == 0) *gx.cnt = fill;
    pd.n = n;
    pd.head = h;
}

// Owner-local sorted insertion of one hit into this lane's pending ring: appended
// when it is the largest (t_in, id) so far (the usual case: records stream in L
// order), else shifted into place.  A full ring drops the hit and marks the pixel.
template <int N>
__device__ __forceinline__ void insert_local(Smem<N> &sm, Pending &pd, int plimit, float tn, float kn, uint32_t in) {
    const int tid = threadIdx.x;
    if (pd.n >= plimit) {
        pd.ovf = true;
        return;
    }
    int k = pd.n;
    SNP_CHECK(k >= 0 && k < kPend && pd.head >= 0 && pd.head < kPend);
    if (k == 0 || pd.tail_t < tn || (pd.tail_t == tn && pd.tail_id < in)) {
        pd.tail_t = tn;
        pd.tail_id = in;
    } else {
        while (k > 0) {
            const int sp = (pd.head + k - 1) & (kPend - 1);
            const float tp = sm.p_thi[sp][tid];
            const uint32_t ip = sm.p_id[sp][tid];
            if (!(tn < tp || (tn == tp && in < ip))) break;
            const int sd = (pd.head + k) & (kPend - 1);
            sm.p_thi[sd][tid] = tp;
            sm.p_kap[sd][tid] = sm.p_kap[sp][tid];
            sm.p_id[sd][tid] = ip;
            --k;
        }
    }
    const int sd = (pd.head + k) & (kPend - 1);
    sm.p_thi[sd][tid] = tn;
    sm.p_kap[sd][tid] = kn;
    sm.p_id[sd][tid] = in;
    ++pd.n;
}

// kGrad: the backward's forward traversal (no image output): every composited hit of a
// pixel with a nonzero dL/d(out) becomes a GradEntry, written straight to the warp's
// current chunk of a.grad_entries (kGradChunk entries, one global atomic per chunk; fill
// counts in a.grad_fill); an overflowing pixel is queued for K7 with its count of already
// emitted hits.  Two CTAs per SM, as in the forward.
template <int N, bool kRay, bool kEager, int kMode = 0>   // 0 forward, 1 grad mode, 2 record mode
#ifndef SNP_AB_K5_CTAS
#define SNP_AB_K5_CTAS 2
#endif
__global__ void __launch_bounds__(kThreads, SNP_AB_K5_CTAS) k_render(RenderArgs a, CamBatch cb) {
    constexpr bool kGrad = kMode == 1, kRecord = kMode == 2, kEntries = kGrad || kRecord;
    constexpr int kStages = Cfg<N>::kStages;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem<N> &sm = *reinterpret_cast<Smem<N> *>(smem_raw);
    int *gcount = reinterpret_cast<int *>(smem_raw + sizeof(Smem<N>));
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    const int stripe_tiles = a.tiles_x * a.stripe_rows;
    const int total_tiles = stripe_tiles * cb.nv;

    if (kEntries && tid < kConsumers) gcount[tid] = 0;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], kConsumers);
        }
        for (int s = 0; s < kTileRing; ++s) sm.tdone[s] = 0;
        sm.warps_done = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    // K6 may be scheduled as soon as every K5 CTA is resident: it only takes the SM
    // space that finished K5 CTAs free (see k_fallback)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // the last warp of the CTA to finish publishes the CTA's exit (after its queue pushes)
    auto warp_exit = [&]() {
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            if (atomicAdd(&sm.warps_done, 1) == kConsumers) {
                __threadfence();
                atomicAdd(a.counters + kCntK5Done, 1ull);
            }
        }
    };

    if (wid == kConsumers) {
        // =============================== producer warp
#ifdef SNP_INSTRUMENT
        long long p_wait = 0;
        const long long p_start = clock64();
        unsigned long long g_start;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g_start));
#endif
        uint32_t gb = 0;            // global batch counter (ring slot / phase)
        int seq = 0;
        while (true) {
            int t = 0;
            if (lane == 0) {
                t = (int)atomicAdd(a.counters + kCntTileQueue, 1ull);
                if (t < total_tiles) t = (int)a.tile_order[t];   // heaviest tiles first
            }
            t = __shfl_sync(0xffffffffu, t, 0);
            const int slot0 = (int)(gb % kStages);
            if (gb >= kStages) {
                const uint32_t eph = ((gb / kStages) - 1) & 1;
#ifdef SNP_INSTRUMENT
                long long _w0 = clock64();
#endif
                while (!mbar_try(&sm.empty[slot0], eph)) {}
#ifdef SNP_INSTRUMENT
                p_wait += clock64() - _w0;
#endif
            }
            if (t >= total_tiles) {           // end marker
                if (lane == 0) {
                    sm.m_tile[slot0] = -1;
                    sm.m_cnt[slot0] = 0;
                    mbar_arrive_expect_tx(&sm.full[slot0], 0u);
                }
                break;
            }
            const int vloc = t / stripe_tiles;
            const int st = t - vloc * stripe_tiles;
            const int tx = st % a.tiles_x;
            const int ty = a.row_begin + (st / a.tiles_x) * a.row_stride;
            const int64_t view = cb.view0 + vloc;
            const int tile = ty * a.tiles_x + tx;
            const uint32_t beg = a.ranges[2 * (view * a.tiles_per_view + tile)];
            const uint32_t end = a.ranges[2 * (view * a.tiles_per_view + tile) + 1];
            const int nb = max(1, (int)((end - beg + kBatch - 1) / kBatch));
            const float4 *recs = a.records + (size_t)view * (size_t)a.n * rec_f4(N);
            if (lane == 0) *(volatile int32_t *)&sm.tdone[seq % kTileRing] = 0;
            for (int bt = 0; bt < nb; ++bt) {
                const int slot = (int)(gb % kStages);
                if (bt > 0) {
                    if (*(volatile int32_t *)&sm.tdone[seq % kTileRing] >= kConsumers) break;   // all done
                    if (gb >= kStages) {
                        const uint32_t eph = ((gb / kStages) - 1) & 1;
#ifdef SNP_INSTRUMENT
                        long long _w1 = clock64();
#endif
                        while (!mbar_try(&sm.empty[slot], eph)) {}
#ifdef SNP_INSTRUMENT
                        p_wait += clock64() - _w1;
#endif
                    }
                }
                const uint32_t e0 = beg + (uint32_t)bt * kBatch;
                const uint32_t cnt = end > e0 ? min((uint32_t)kBatch, end - e0) : 0u;
                SNP_CHECK(slot < kStages && cnt <= (uint32_t)kBatch && end >= beg);
                if ((uint32_t)lane < cnt) {
                    const uint32_t id = a.vals[e0 + lane];
                    SNP_CHECK((int64_t)id < a.n);
                    sm.id[slot][lane] = id;
                    sm.L[slot][lane] = key_depth(a.keys[e0 + lane]);
                    bulk_g2s(&sm.rec[slot][lane][0], recs + (size_t)id * rec_f4(N), Cfg<N>::kRecBytes,
                             &sm.full[slot]);
                }
                if (lane == 0) {
                    const uint32_t nx = e0 + cnt;
                    sm.L[slot][cnt] = nx < end ? key_depth(a.keys[nx]) : INFINITY;
                    sm.m_tile[slot] = t;
                    sm.m_cnt[slot] = (int)cnt;
                    sm.m_flags[slot] = (bt == 0 ? 1 : 0) | (bt == nb - 1 ? 2 : 0);
                    sm.m_seq[slot] = seq;
                }
                // the arrive (release) publishes id/L/metadata with the phase
                __syncwarp();
                if (lane == 0) mbar_arrive_expect_tx(&sm.full[slot], cnt * Cfg<N>::kRecBytes);
                ++gb;
            }
            ++seq;
        }
#ifdef SNP_INSTRUMENT
        if (lane == 0) {
            atomicAdd(a.counters + 26, (unsigned long long)p_wait);
            atomicAdd(a.counters + 27, (unsigned long long)(clock64() - p_start));
            unsigned long long g_end;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g_end));
            atomicMax(a.counters + 32, ~g_start);
            atomicMax(a.counters + 33, g_end);
            atomicAdd(a.counters + 34, g_end >> 10);
            atomicAdd(a.counters + 35, 1ull);
        }
#endif
        warp_exit();
        return;
    }

    // =============================== consumer warps
#ifdef SNP_INSTRUMENT
    long long ins_wait = 0, ins_round = 0, ins_emit = 0, ins_rounds = 0, ins_lanes = 0, ins_fill = 0, ins_pre = 0,
              ins_setup = 0, ins_finish = 0, ins_touch = 0, ins_empty = 0, ins_ecalls = 0, ins_enone = 0, ins_steps = 0, ins_ins = 0;
    const long long ins_start = clock64();
#endif
    const int plimit = a.pending_limit < kPend ? a.pending_limit : kPend;
    uint32_t n_cand = 0, n_hit = 0, n_comp = 0, n_ovf = 0;
    unsigned long long n_tested = 0;
    // per-tile state
    int cur_seq = -1;
    bool tile_finished = true;    // this warp has written its pixels of the current tile
    int x = 0, y = 0;
    bool inside = false;
    int64_t view = 0;
    const DevCam *cam = &cb.cams[0];
    const float4 *recs = a.records;
    Ray ray{0, 0, 1, 0, 0, 0, 0, 0};
    float pxf = 0.f, pyf = 0.f, bx0 = 0.f, by0 = 0.f;
    PixelState ps{1.f, 0.f, 0.f, 0.f, true, false, 0u};
    Pending pd{0, 0, 0.f, 0u, false};
    GradCtx gx{make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f), nullptr, nullptr, 0, gcount + wid, 0u};
    int64_t gchunk = -1;   // (kGrad) index of gx.chunk; -2: the chunk table is exhausted
    // (kGrad) switch to a fresh chunk when this emission call (need entries at most)
    // might not fit: the old one's fill goes to a.grad_fill (warp-uniform)
    auto grad_reserve = [&](int need) {
        __syncwarp();
        const int c = *gx.cnt;
        SNP_CHECK(c >= 0 && c <= kGradChunk);
        if (need == 0 || (gchunk >= 0 && c + need <= kGradChunk)) return;
        long long k = -2;
        if (lane == 0) {
            if (gchunk >= 0) a.grad_fill[gchunk] = c;
            if (gchunk != -2) {
                k = (long long)atomicAdd(a.counters + kCntGradEntries, 1ull);
                if (k >= a.grad_chunks) {
                    atomicExch(a.counters + kCntGradOverflow, 1ull);
                    k = -2;
                }
            }
            *gx.cnt = 0;
        }
        gchunk = __shfl_sync(0xffffffffu, k, 0);
        gx.cbase = gchunk >= 0 ? gchunk * kGradChunk : 0;
        if (kRecord) gx.rchunk = gchunk >= 0 ? a.rec_entries + gx.cbase : nullptr;
        else gx.chunk = gchunk >= 0 ? a.grad_entries + gx.cbase : nullptr;
        __syncwarp();
    };
    int64_t gpi = 0;   // (kGrad) pixel index within the camera batch

    auto finish_tile = [&]() {   // write this warp's pixels; count the warp as done with the tile
        if (kGrad) {
            if (inside && ps.overflow) {   // K7 redoes the pixel, from its emitted hits on
                const unsigned long long q = atomicAdd(a.counters + kCntBwdQueue, 1ull);
                a.bw_queue[q] = (uint32_t)gpi;
                a.bw_skip[gpi] = ps.composited;
            }
        } else if (inside) {
            if (ps.overflow) {
                if (kRecord) {   // the backward's per-pixel K7 takes it from its recorded hits on
                    const unsigned long long qb = atomicAdd(a.counters + kCntBwdQueue, 1ull);
                    a.bw_queue[qb] = (uint32_t)gpi;
                    a.bw_skip[gpi] = ps.composited;
                }
                const unsigned long long q = atomicAdd(a.counters + kCntFallbackQueue, 1ull);
                if ((int64_t)q < a.fallback_capacity)
                    atomicExch(a.fallback + q, (1ull << 63) | ((unsigned long long)view << 32) |
                                                   (unsigned long long)(uint32_t)(y * cam->W + x));
                ++n_ovf;
            } else {
                const float4 o = make_float4(fmaf(ps.T, a.bg[0], ps.cr), fmaf(ps.T, a.bg[1], ps.cg),
                                             fmaf(ps.T, a.bg[2], ps.cb), 1.0f - ps.T);
                SNP_CHECK(x >= 0 && x < cam->W && y >= 0 && y < cam->H);
                reinterpret_cast<float4 *>(a.out)[((size_t)view * cam->H + y) * cam->W + x] = o;
            }
        }
        n_comp += ps.composited;
        tile_finished = true;
        __syncwarp();
        if (lane == 0) atomicAdd(&sm.tdone[cur_seq % kTileRing], 1);
    };

    for (uint32_t gb = 0;; ++gb) {
        const int slot = (int)(gb % kStages);
#ifdef SNP_INSTRUMENT
        long long _t0 = clock64();
#endif
        while (!mbar_try(&sm.full[slot], (gb / kStages) & 1)) {}
#ifdef SNP_INSTRUMENT
        ins_wait += clock64() - _t0;
#endif
        const int t = sm.m_tile[slot];
        if (t < 0) break;                      // end of work (no release needed)
        const int cnt = sm.m_cnt[slot];
        const int flags = sm.m_flags[slot];
#ifdef SNP_INSTRUMENT
        long long _s0 = clock64();
#endif
        if (flags & 1) {                       // first batch of a new tile: set up the pixels
            cur_seq = sm.m_seq[slot];
            const int vloc = t / stripe_tiles;
            const int st = t - vloc * stripe_tiles;
            const int tx = st % a.tiles_x;
            const int ty = a.row_begin + (st / a.tiles_x) * a.row_stride;
            view = cb.view0 + vloc;
            cam = &cb.cams[vloc];
            recs = a.records + (size_t)view * (size_t)a.n * rec_f4(N);
            const int bx = tx * kTile + (wid & 1) * 8, by = ty * kTile + (wid >> 1) * 4;
            x = bx + (lane & 7);
            y = by + (lane >> 3);
            inside = x < cam->W && y < cam->H;
            ray = inside ? make_ray(*cam, x, y) : Ray{0, 0, 1, 0, 0, 0, cam->t_near, cam->t_far};
            pxf = (float)x + 0.5f;
            pyf = (float)y + 0.5f;
            bx0 = (float)bx + 0.5f;
            by0 = (float)by + 0.5f;
            ps = PixelState{1.f, 0.f, 0.f, 0.f, !inside, false, 0u};
            pd = Pending{0, 0, 0.f, 0u, false};
            if (kEntries) {
                gpi = ((int64_t)vloc * cam->H + y) * cam->W + x;
                if (kGrad) {
                    const int64_t gi = ((int64_t)view * cam->H + y) * cam->W + x;
                    gx.G = inside ? a.grad_in[gi] : make_float4(0.f, 0.f, 0.f, 0.f);
                    gx.F = inside ? a.fwd[gi] : make_float4(0.f, 0.f, 0.f, 0.f);
                }
                gx.pix = ((uint32_t)vloc << 24) | (uint32_t)(inside ? y * cam->W + x : 0);
            }
            sm.p_in[tid] = 0u;
            tile_finished = false;
        }
#ifdef SNP_INSTRUMENT
        ins_setup += clock64() - _s0;
#endif
        if (!tile_finished) {
#ifdef SNP_INSTRUMENT
            long long _p0 = clock64();
#endif
            if (!ps.done) n_tested += (unsigned long long)cnt;
            // records whose conic box touches this warp's 8x4 block
            bool touch = false;
            if (lane < cnt) {
                const float4 c0 = sm.rec[slot][lane][kRecConic];
                const float cc = sm.rec[slot][lane][kRecConicRgb].x;
                const float hb = 0.5f * c0.w;
                const float det = fmaf(c0.z, cc, -hb * hb);
                if (det > 0.f) {
                    // half extents of the conic's bounding box, with a 0.1% + 1e-3 px margin
                    // (which also covers the approximate reciprocal and square roots)
                    const float rdet = rcp_fast(det);
                    const float vx = cc * rdet, vy = c0.z * rdet;
                    const float rx = vx * rsqrtf(vx) * 1.001f + 1e-3f;
                    const float ry = vy * rsqrtf(vy) * 1.001f + 1e-3f;
                    touch = c0.x + rx >= bx0 && c0.x - rx <= bx0 + 7.0f && c0.y + ry >= by0 &&
                            c0.y - ry <= by0 + 3.0f;
                } else {
                    touch = true;   // no conic (straddles the camera plane / camera inside)
                }
                if (a.debug_flags & 1) touch = true;
            }
            uint32_t m = __ballot_sync(0xffffffffu, touch);
#ifdef SNP_INSTRUMENT
            ins_pre += clock64() - _p0;
#endif
            int qcount = 0, qhead = 0;
            auto round = [&](int n) {
#ifdef SNP_INSTRUMENT
                long long _r0 = clock64();
                ++ins_rounds;
                ins_lanes += n;
#endif
                __syncwarp();
                const bool valid = lane < n;
                const int qi = (qhead + lane) & (kQueue - 1);
                const int owner = valid ? sm.ql[wid][qi] : lane;
                const int j = valid ? sm.qj[wid][qi] : 0;
                Ray ro;
                ro.dhx = __shfl_sync(0xffffffffu, ray.dhx, owner);
                ro.dhy = __shfl_sync(0xffffffffu, ray.dhy, owner);
                ro.dhz = __shfl_sync(0xffffffffu, ray.dhz, owner);
                ro.dlx = __shfl_sync(0xffffffffu, ray.dlx, owner);
                ro.dly = __shfl_sync(0xffffffffu, ray.dly, owner);
                ro.dlz = __shfl_sync(0xffffffffu, ray.dlz, owner);
                ro.t_near = cam->t_near;
                ro.t_far = cam->t_far;
                bool hit = false, graze = false;
                int gexp = 0;
                float th = 0.f, tl = 0.f, kap = 0.f;
                SNP_CHECK(!valid || (j < cnt && owner < 32));
                const uint32_t idj = sm.id[slot][j];

                if (valid)
                    hit = exact_hit<N, kGrazeDefer>(&sm.rec[slot][j][0], ro, th, tl, kap, nullptr, idj, &graze, &gexp);

                n_hit += hit;
#ifdef SNP_INSTRUMENT
                long long _i0 = clock64();
#endif
                // route every hit to its owner pixel's lane, which inserts it into its
                // own sorted ring: each hitting lane adds its bit to the owner's mask; the
                // owner then fetches its hits one per step by shuffle (no cross-lane
                // writes to a ring, no dependent shared-memory round trips per step)
                const uint32_t idn = hit ? (tin_code(th, tl) << 27) | ((uint32_t)gexp << 24) | idj : 0u;
                if (hit) atomicOr(&sm.p_in[wid * 32 + owner], 1u << lane);
                __syncwarp();
                uint32_t inc = sm.p_in[tid];
                sm.p_in[tid] = 0u;
                const int steps = __reduce_max_sync(0xffffffffu, (uint32_t)__popc(inc));
#ifdef SNP_INSTRUMENT
                ins_steps += steps;
#endif
                for (int r = 0; r < steps; ++r) {
                    const int src = inc ? __ffs(inc) - 1 : lane;
                    const float tn = __shfl_sync(0xffffffffu, th, src);
                    const float kn = __shfl_sync(0xffffffffu, kap, src);
                    const uint32_t in = __shfl_sync(0xffffffffu, idn, src);
                    if (inc) {
                        inc &= inc - 1u;
                        insert_local<N>(sm, pd, plimit, tn, kn, in);
                    }
                }
#ifdef SNP_INSTRUMENT
                ins_ins += clock64() - _i0;
                ins_round += clock64() - _r0;
#endif
            };
            // Single call site for the exact round and for emission (keeps the hot code
            // inside the instruction cache).
            int jlast = -1;
            while (true) {
                // fill the queue from the records that touch this warp's block
#ifdef SNP_INSTRUMENT
                long long _f0 = clock64();
#endif
                // two records per step (independent loads and tests); the queue holds
                // up to 31 + 2 x 32 pairs
                while (m && qcount < 32) {
                    const int j1 = __ffs(m) - 1;
                    m &= m - 1u;
                    const int j2 = m ? __ffs(m) - 1 : j1;
                    const bool two = m != 0u;
                    m &= m - 1u;
                    jlast = two ? j2 : j1;
                    const float4 c1 = sm.rec[slot][j1][kRecConic];
                    const float cc1 = sm.rec[slot][j1][kRecConicRgb].x;
                    const float4 c2 = sm.rec[slot][j2][kRecConic];
                    const float cc2 = sm.rec[slot][j2][kRecConicRgb].x;
                    const float dx1 = pxf - c1.x, dy1 = pyf - c1.y;
                    const float dx2 = pxf - c2.x, dy2 = pyf - c2.y;
                    const float q1 = fmaf(cc1 * dy1, dy1, dx1 * fmaf(c1.w, dy1, c1.z * dx1));
                    const float q2 = fmaf(cc2 * dy2, dy2, dx2 * fmaf(c2.w, dy2, c2.z * dx2));
                    const bool cand1 = !ps.done && q1 <= 1.0f;
                    const bool cand2 = two && !ps.done && q2 <= 1.0f;
                    const uint32_t cm1 = __ballot_sync(0xffffffffu, cand1);
                    const uint32_t cm2 = __ballot_sync(0xffffffffu, cand2);
                    const int n1 = __popc(cm1);
                    SNP_CHECK(qcount + __popc(cm1) + __popc(cm2) <= kQueue);
                    if (cand1) {
                        const int pos = (qhead + qcount + __popc(cm1 & lt_mask)) & (kQueue - 1);
                        sm.qj[wid][pos] = (uint8_t)j1;
                        sm.ql[wid][pos] = (uint8_t)lane;
                    }
                    if (cand2) {
                        const int pos = (qhead + qcount + n1 + __popc(cm2 & lt_mask)) & (kQueue - 1);
                        sm.qj[wid][pos] = (uint8_t)j2;
                        sm.ql[wid][pos] = (uint8_t)lane;
                    }
                    n_cand += cand1 + cand2;
                    qcount += n1 + __popc(cm2);
#ifdef SNP_INSTRUMENT
                    ins_touch += 1 + two;
                    ins_empty += (cm1 == 0u) + (two && cm2 == 0u);
#endif
                }
#ifdef SNP_INSTRUMENT
                ins_fill += clock64() - _f0;
#endif
                int rem = 0, jn = jlast + 1;
                if (qcount > 0) {
                    round(qcount < 32 ? qcount : 32);
                    rem = qcount > 32 ? qcount - 32 : 0;
                    qhead = (qhead + 32) & (kQueue - 1);
                    // every hit this warp has not inserted yet comes from a record >= the
                    // oldest queued one (or > jlast), so that record's L bounds its t_in
                    if (rem > 0) jn = sm.qj[wid][qhead];
                    qcount = rem;
                }
                // records after jlast that do not touch this warp's block cannot hit its
                // pixels: the next touching one (or the next batch) bounds what is left
                if (rem == 0) jn = m ? __ffs(m) - 1 : cnt;
                const bool batch_end = (m == 0u) && rem == 0;
                if (!ps.done && pd.ovf) {   // a hit was dropped: nothing may be blended
                    ps.overflow = true;
                    ps.done = true;
                }
                // batch end: everything in later batches has t_in >= L of the next key;
                // mid-batch: every hit not inserted yet comes from record jn or later, so
                // L[jn] bounds it.  Default: only when the pending list runs nearly full;
                // kEager: after every exact round -- shorter pending lists (fewer K6
                // pixels), earlier termination; chosen per scene from the overflow rate
                const bool do_emit = !ps.done && (batch_end || pd.n > (kEager ? 0 : plimit - 4));
                if (kEntries) {
                    const uint32_t need = __reduce_add_sync(0xffffffffu, do_emit ? (uint32_t)pd.n : 0u);
                    if (need) {   // (warp-uniform: rounds without an emitting lane skip both)
                        grad_reserve((int)need);
                        emit_sync<N, kRay, kRecord>(sm, ps, pd, do_emit,
                                           batch_end ? ((flags & 2) ? INFINITY : sm.L[slot][cnt]) : sm.L[slot][jn],
                                           a.t_floor, recs, a, ray, gx);
                    }
                } else if (do_emit) {
#ifdef SNP_INSTRUMENT
                    long long _e0 = clock64();
                    ++ins_ecalls;
                    ins_enone += (pd.n == 0);
#endif
                    emit<N, kRay>(sm, ps, pd,
                                  batch_end ? ((flags & 2) ? INFINITY : sm.L[slot][cnt]) : sm.L[slot][jn],
                                  a.t_floor, recs, a, ray);
#ifdef SNP_INSTRUMENT
                    ins_emit += clock64() - _e0;
#endif
                }
                if (batch_end) break;
            }
#ifdef SNP_INSTRUMENT
            long long _z0 = clock64();
#endif
            if ((flags & 2) || __all_sync(0xffffffffu, ps.done)) finish_tile();
#ifdef SNP_INSTRUMENT
            ins_finish += clock64() - _z0;
#endif
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[slot]);
    }
#ifdef SNP_INSTRUMENT
    if (lane == 0) {
        atomicAdd(a.counters + 16, (unsigned long long)ins_wait);
        atomicAdd(a.counters + 17, (unsigned long long)ins_round);
        atomicAdd(a.counters + 18, (unsigned long long)ins_emit);
        atomicAdd(a.counters + 19, (unsigned long long)ins_rounds);
        atomicAdd(a.counters + 20, (unsigned long long)ins_lanes);
        atomicAdd(a.counters + 21, (unsigned long long)(clock64() - ins_start));
        atomicAdd(a.counters + 22, (unsigned long long)ins_fill);
        atomicAdd(a.counters + 23, (unsigned long long)ins_pre);
        atomicAdd(a.counters + 24, (unsigned long long)ins_setup);
        atomicAdd(a.counters + 25, (unsigned long long)ins_finish);
        atomicAdd(a.counters + 37, (unsigned long long)ins_touch);
        atomicAdd(a.counters + 38, (unsigned long long)ins_empty);
        atomicAdd(a.counters + 36, (unsigned long long)ins_steps);
        atomicAdd(a.counters + 41, (unsigned long long)ins_ins);
    }
    {
        const unsigned long long ec = __reduce_add_sync(0xffffffffu, (uint32_t)ins_ecalls);
        const unsigned long long en = __reduce_add_sync(0xffffffffu, (uint32_t)ins_enone);
        if (lane == 0) {
            atomicAdd(a.counters + 39, ec);
            atomicAdd(a.counters + 40, en);
        }
    }
#endif
    __syncwarp();
    if (kEntries) {
        __syncwarp();
        if (lane == 0 && gchunk >= 0) a.grad_fill[gchunk] = *gx.cnt;
    }
    if (kGrad) {   // (the backward's traversal leaves the forward's statistics alone)
        warp_exit();
        return;
    }
    const uint32_t v[5] = {(uint32_t)n_tested, n_cand, n_hit, n_comp, n_ovf};
#pragma unroll
    for (int c = 0; c < 5; ++c) {
        const uint32_t s = __reduce_add_sync(0xffffffffu, v[c]);   // per-warp totals fit 32 bits
        if (lane == 0 && s) atomicAdd(a.counters + kCntTested + c, (unsigned long long)s);
    }
    warp_exit();
}

template <int N>
__device__ __forceinline__ bool fb_hit(const float4 *rec, const Ray &ray, float pxf, float pyf, float &th,
                                       float &tl, float &kap, const Prec64 &g64, uint32_t id) {
    const float4 c0 = rec[kRecConic];
    const float cc = rec[kRecConicRgb].x;
    const float dx = pxf - c0.x, dy = pyf - c0.y;
    const float q = fmaf(cc * dy, dy, dx * fmaf(c0.w, dy, c0.z * dx));
    if (!(q <= 1.0f)) return false;
    return exact_hit<N, kGrazeInline>(rec, ray, th, tl, kap, &g64, id);
}

// K6: exact per-pixel fallback, one CTA per overflowed pixel.  Phase A: the
// 256 threads split the tile list and store every hit (t_in hi/lo, kappa, id) in
// shared memory.  Phase B: bitonic sort by (t_in, id) (R11).  Phase C:
// T before each hit = prefix product of (1 - kappa) (block scan); a hit blends
// iff T before it is >= floor (Eq. 4 with the stop rule, R13); colours are
// fetched in parallel and reduced.  Pixels with more than kFbHits hits use a
// block-wide repeated selection instead (same result, slower).
constexpr int kFbThreads = 256;
constexpr int kFbHits = 2048;
constexpr int kFbIlp = 4;
constexpr int kFbRank = 512;
constexpr int kFbPer = kFbHits / kFbThreads;   // 8 sorted entries per thread in phase C

struct FbSmem {
    float t[kFbHits], l[kFbHits], k[kFbHits];
    uint32_t id[kFbHits];
    uint16_t idx[kFbHits];
    float wsum[kFbThreads / 32][4];
    float wprod[kFbThreads / 32];
    int count;
    int last;
};

__device__ __forceinline__ bool fb_less(const FbSmem &s, int a, int b, int n) {
    if (b >= n) return a < n;          // padding sorts last
    if (a >= n) return false;
    return before(s.t[a], s.l[a], s.id[a], s.t[b], s.l[b], s.id[b]);
}

__device__ __forceinline__ unsigned long long ld_vol64(const unsigned long long *p) {
    return *reinterpret_cast<const volatile unsigned long long *>(p);
}

// overlap = true (one camera batch): launched as K5's programmatic dependent; entries
// are claimed one at a time as K5 queues them, and the CTA leaves once every K5 CTA has
// exited and no entry is left.  overlap = false: K5 has completed; CTAs stride over the
// queue and take the entries of this batch's views.
template <int N, bool kRay>
__global__ void __launch_bounds__(kFbThreads) k_fallback(RenderArgs a, CamBatch cb) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ FbSmem sm;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // the pixels K6w could not hold (second half of the queue buffer)
    const unsigned long long *big = a.fallback + a.fallback_capacity;
    int64_t nq = (int64_t)a.counters[kCntBigQueue];
    if (nq > a.fallback_capacity) nq = a.fallback_capacity;
    for (int64_t qi = blockIdx.x; qi < nq; qi += gridDim.x) {
        const unsigned long long ent = big[qi];
        const int64_t view = (int64_t)((ent >> 32) & 0x7fffffffull);
        if (view < cb.view0 || view >= cb.view0 + cb.nv) continue;
        const DevCam &cam = cb.cams[view - cb.view0];
        const uint32_t pix = (uint32_t)ent;
        const int x = (int)(pix % (uint32_t)cam.W), y = (int)(pix / (uint32_t)cam.W);
        const int tile = (y / kTile) * a.tiles_x + (x / kTile);
        const uint32_t beg = a.ranges[2 * (view * a.tiles_per_view + tile)];
        const uint32_t end = a.ranges[2 * (view * a.tiles_per_view + tile) + 1];
        const float4 *recs = a.records + (size_t)view * (size_t)a.n * rec_f4(N);
        const Ray ray = make_ray(cam, x, y);
        const Prec64 g64{a.centers, a.rotations, a.scales, cam.C[0], cam.C[1], cam.C[2]};
        const float pxf = (float)x + 0.5f, pyf = (float)y + 0.5f;
        if (tid == 0) sm.count = 0;
        __syncthreads();
#ifdef SNP_INSTRUMENT
        const long long _fa = clock64();
#endif
        // ---- phase A: every hit of the tile list, once
        // kFbIlp independent records per thread per step: the id and conic loads of a
        // step are all in flight together (the loop is latency-bound otherwise)
        for (uint32_t e0 = beg + tid; e0 < end; e0 += kFbThreads * kFbIlp) {
            uint32_t ids[kFbIlp];
            bool cand[kFbIlp];
#pragma unroll
            for (int u = 0; u < kFbIlp; ++u) {
                const uint32_t e = e0 + (uint32_t)(u * kFbThreads);
                ids[u] = e < end ? a.vals[e] : 0xffffffffu;
            }
#pragma unroll
            for (int u = 0; u < kFbIlp; ++u) {
                cand[u] = false;
                if (ids[u] != 0xffffffffu) {
                    const float4 *rec = recs + (size_t)ids[u] * rec_f4(N);
                    const float4 c0 = rec[kRecConic];
                    const float cc = rec[kRecConicRgb].x;
                    const float dx = pxf - c0.x, dy = pyf - c0.y;
                    cand[u] = fmaf(cc * dy, dy, dx * fmaf(c0.w, dy, c0.z * dx)) <= 1.0f;
                }
            }
#pragma unroll
            for (int u = 0; u < kFbIlp; ++u) {
                float th, tl, kap;
                if (cand[u] && exact_hit<N, kGrazeInline>(recs + (size_t)ids[u] * rec_f4(N), ray, th, tl, kap, &g64, ids[u])) {
                    const int pos = atomicAdd(&sm.count, 1);
                    if (pos < kFbHits) {
                        sm.t[pos] = th; sm.l[pos] = tl; sm.k[pos] = kap; sm.id[pos] = ids[u];
                    }
                }
            }
        }
        __syncthreads();
        const int n = sm.count;
#ifdef SNP_INSTRUMENT
        const long long _fb = clock64();
        if (tid == 0) {
            atomicAdd(a.counters + 28, (unsigned long long)(_fb - _fa));
            atomicAdd(a.counters + 31, (unsigned long long)n + ((unsigned long long)(end - beg) << 32));
        }
#endif
        float T = 1.f, cr = 0.f, cg = 0.f, cbl = 0.f;
        unsigned long long ncomp = 0;
        if (n <= kFbHits) {
            // ---- phase B: sort of indices.  Up to kFbRank hits: rank sort (the rank of
            // hit i is the number of hits before it in the strict total order (t_in, id);
            // one pass, no block barriers).  Above: bitonic network.
            if (n <= kFbRank) {
                // g = 256 / n rounded down to a power of two (<= 32) lanes share one hit's count
                int g = 1;
                while (g < 32 && g * 2 * n <= kFbThreads) g <<= 1;
                const int part = tid & (g - 1);
                for (int i0 = tid / g; i0 < (n + kFbThreads / g - 1) / (kFbThreads / g) * (kFbThreads / g);
                     i0 += kFbThreads / g) {
                    const int i = i0 < n ? i0 : n - 1;
                    const float ti = sm.t[i], li = sm.l[i];
                    const uint32_t di = sm.id[i];
                    int r = 0;
                    for (int j = part; j < n; j += g) r += before(sm.t[j], sm.l[j], sm.id[j], ti, li, di);
                    for (int o = 1; o < g; o <<= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
                    if (part == 0 && i0 < n) sm.idx[r] = (uint16_t)i;
                }
                __syncthreads();
            } else {
            int n2 = 1;
            while (n2 < n) n2 <<= 1;
            for (int i = tid; i < n2; i += kFbThreads) sm.idx[i] = (uint16_t)i;
            __syncthreads();
            for (int kk = 2; kk <= n2; kk <<= 1) {
                for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                    for (int i = tid; i < n2; i += kFbThreads) {
                        const int ixj = i ^ jj;
                        if (ixj > i) {
                            const int p = sm.idx[i], q = sm.idx[ixj];
                            const bool asc = (i & kk) == 0;
                            if (asc ? fb_less(sm, q, p, n) : fb_less(sm, p, q, n)) {
                                sm.idx[i] = (uint16_t)q;
                                sm.idx[ixj] = (uint16_t)p;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            }
#ifdef SNP_INSTRUMENT
            if (tid == 0) atomicAdd(a.counters + 29, (unsigned long long)(clock64() - _fb));
#endif
            // ---- phase C: transmittance before each sorted hit by a block product scan
            float om[kFbPer];
            float prod = 1.f;
#pragma unroll
            for (int r = 0; r < kFbPer; ++r) {
                const int i = tid * kFbPer + r;
                om[r] = i < n ? 1.f - sm.k[sm.idx[i]] : 1.f;
                prod *= om[r];
            }
            float inc = prod;   // inclusive product over threads 0..tid
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const float v = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc *= v;
            }
            if (lane == 31) sm.wprod[wid] = inc;
            if (tid == 0) sm.last = -1;
            __syncthreads();
            float Tb = __shfl_up_sync(0xffffffffu, inc, 1);   // exclusive product within the warp
            if (lane == 0) Tb = 1.f;
            for (int w = 0; w < wid; ++w) Tb *= sm.wprod[w];
            float wr = 0.f, wg = 0.f, wb = 0.f;
            int last = -1;
            float t_end = 1.f;
#pragma unroll
            for (int r = 0; r < kFbPer; ++r) {
                const int i = tid * kFbPer + r;
                if (i < n && Tb >= a.t_floor) {
                    const int h = sm.idx[i];
                    const float kap = sm.k[h];
                    const float4 rgb = hit_rgb<kRay>(recs + (size_t)sm.id[h] * rec_f4(N), a.sh, a.sh_degree,
                                                     sm.id[h], ray);
                    const float w = Tb * kap;
                    wr = fmaf(w, rgb.y, wr);
                    wg = fmaf(w, rgb.z, wg);
                    wb = fmaf(w, rgb.w, wb);
                    last = i;
                    t_end = Tb * om[r];
                }
                Tb *= om[r];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                wr += __shfl_xor_sync(0xffffffffu, wr, o);
                wg += __shfl_xor_sync(0xffffffffu, wg, o);
                wb += __shfl_xor_sync(0xffffffffu, wb, o);
            }
            if (lane == 0) {
                sm.wsum[wid][0] = wr; sm.wsum[wid][1] = wg; sm.wsum[wid][2] = wb;
            }
            if (last >= 0) atomicMax(&sm.last, last);
            __syncthreads();
            const int lst = sm.last;
            if (last >= 0 && last == lst) sm.wsum[0][3] = t_end;   // unique owner of the last blended hit
            __syncthreads();
            for (int w = 0; w < kFbThreads / 32; ++w) {
                cr += sm.wsum[w][0]; cg += sm.wsum[w][1]; cbl += sm.wsum[w][2];
            }
            T = lst >= 0 ? sm.wsum[0][3] : 1.f;
            ncomp = (unsigned long long)(lst + 1);
        } else {
#ifdef SNP_INSTRUMENT
            if (tid == 0) atomicAdd(a.counters + 30, 1ull);
#endif
            // ---- too many hits for shared memory: block-wide repeated selection
            float lh = -INFINITY, ll = 0.f;
            uint32_t lid = 0;
            bool first = true;
            while (true) {
                float bh = INFINITY, bl = 0.f, bk = 0.f;
                uint32_t bid = 0xffffffffu;
                for (uint32_t e = beg + tid; e < end; e += kFbThreads) {
                    const uint32_t id = a.vals[e];
                    float th, tl, kap;
                    if (!fb_hit<N>(recs + (size_t)id * rec_f4(N), ray, pxf, pyf, th, tl, kap, g64, id)) continue;
                    if (!first && !before(lh, ll, lid, th, tl, id)) continue;
                    if (before(th, tl, id, bh, bl, bid)) { bh = th; bl = tl; bid = id; bk = kap; }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const float oh = __shfl_xor_sync(0xffffffffu, bh, o);
                    const float ol = __shfl_xor_sync(0xffffffffu, bl, o);
                    const uint32_t oid = __shfl_xor_sync(0xffffffffu, bid, o);
                    const float ok = __shfl_xor_sync(0xffffffffu, bk, o);
                    if (before(oh, ol, oid, bh, bl, bid)) { bh = oh; bl = ol; bid = oid; bk = ok; }
                }
                __syncthreads();
                if (lane == 0) { sm.t[wid] = bh; sm.l[wid] = bl; sm.id[wid] = bid; sm.k[wid] = bk; }
                __syncthreads();
                for (int w = 0; w < kFbThreads / 32; ++w)
                    if (before(sm.t[w], sm.l[w], sm.id[w], bh, bl, bid)) {
                        bh = sm.t[w]; bl = sm.l[w]; bid = sm.id[w]; bk = sm.k[w];
                    }
                if (bid == 0xffffffffu) break;
                const float4 rgb = hit_rgb<kRay>(recs + (size_t)bid * rec_f4(N), a.sh, a.sh_degree, bid, ray);
                const float w = T * bk;
                cr = fmaf(w, rgb.y, cr);
                cg = fmaf(w, rgb.z, cg);
                cbl = fmaf(w, rgb.w, cbl);
                T *= (1.f - bk);
                ++ncomp;
                lh = bh; ll = bl; lid = bid; first = false;
                if (T < a.t_floor) break;
            }
        }
        if (tid == 0) {
            reinterpret_cast<float4 *>(a.out)[((size_t)view * cam.H + y) * cam.W + x] =
                make_float4(fmaf(T, a.bg[0], cr), fmaf(T, a.bg[1], cg), fmaf(T, a.bg[2], cbl), 1.f - T);
            atomicAdd(a.counters + kCntComposited, ncomp);
        }
        __syncthreads();
    }
}

// K6w: exact per-pixel fallback, one warp per overflowed pixel (the pixels K5 queues:
// pending overflow or a grazing hit, R23).  Small enough (one warp, 7 KB of
// shared memory) to run on the SMs beside K5's two CTAs: launched as K5's programmatic
// dependent, its CTAs are resident while K5 runs and take pixels as K5 queues them, so
// the fallback work overlaps K5 instead of following it.  Per pixel: every hit of the
// tile list (conic pre-test, exact hit with the FP64 grazing branch), (t_in, id) order
// by rank (R11), transmittance by a chunked warp product-scan with the stop rule
// (Eq. 4, R13), colours summed over the warp.  A pixel with more than kFwHits
// hits goes to the block-wide K6 (k_fallback) that runs after.
constexpr int kFwHits = 384;
struct FwSmem {
    float th[kFwHits], tl[kFwHits], kap[kFwHits];
    uint32_t id[kFwHits];
    uint16_t ord[kFwHits];
};

template <int N, bool kRay>
__global__ void __launch_bounds__(32) k_fallback_warp(RenderArgs a, CamBatch cb, int overlap) {
    if (!overlap) asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ FwSmem sm;
    const int lane = threadIdx.x;
    const uint32_t lt = (1u << lane) - 1u;
    int64_t nq = overlap ? 0 : (int64_t)a.counters[kCntFallbackQueue];
    if (nq > a.fallback_capacity) nq = a.fallback_capacity;
    for (int64_t it = blockIdx.x;; it += gridDim.x) {
        unsigned long long ent = 0;
        int64_t qi = it;
        if (lane == 0) {
            if (overlap) {
                qi = (int64_t)atomicAdd(a.counters + kCntFallbackClaim, 1ull);
                while (qi < a.fallback_capacity) {
                    ent = ld_vol64(a.fallback + qi);
                    if (ent) break;
                    if (ld_vol64(a.counters + kCntK5Done) == (unsigned long long)a.k5_grid) {
                        ent = ld_vol64(a.fallback + qi);   // (pushed before K5's exit signal)
                        break;
                    }
                    __nanosleep(500);
                }
            } else {
                ent = qi < nq ? a.fallback[qi] : ~0ull;
            }
        }
        ent = __shfl_sync(0xffffffffu, ent, 0);
        qi = __shfl_sync(0xffffffffu, qi, 0);
        if (overlap ? ent == 0 : ent == ~0ull) break;
        if (!(ent >> 63)) continue;
        const int64_t view = (int64_t)((ent >> 32) & 0x7fffffffull);
        if (view < cb.view0 || view >= cb.view0 + cb.nv) continue;
        if (lane == 0) a.fallback[qi] = 0ull;   // consumed: the queue is all zero between renders
        const DevCam &cam = cb.cams[view - cb.view0];
        const uint32_t pix = (uint32_t)ent;
        const int x = (int)(pix % (uint32_t)cam.W), y = (int)(pix / (uint32_t)cam.W);
        SNP_CHECK(y < cam.H);
        const int tile = (y / kTile) * a.tiles_x + (x / kTile);
        const uint32_t beg = a.ranges[2 * (view * a.tiles_per_view + tile)];
        const uint32_t end = a.ranges[2 * (view * a.tiles_per_view + tile) + 1];
        SNP_CHECK(beg <= end);
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
                hit = fb_hit<N>(recs + (size_t)id * rec_f4(N), ray, pxf, pyf, th, tl, kap, g64, id);
            }
            const uint32_t m = __ballot_sync(0xffffffffu, hit);
            const int pos = cnt + __popc(m & lt);
            if (hit && pos < kFwHits) {
                sm.th[pos] = th;
                sm.tl[pos] = tl;
                sm.kap[pos] = kap;
                sm.id[pos] = id;
            }
            cnt += __popc(m);
        }
        if (cnt > kFwHits) {   // to the block-wide K6
            if (lane == 0) {
                const unsigned long long b = atomicAdd(a.counters + kCntBigQueue, 1ull);
                if ((int64_t)b < a.fallback_capacity) a.fallback[a.fallback_capacity + b] = ent;
            }
            continue;
        }
        __syncwarp();
        // ---- (t_in, id) order by rank
        for (int i = lane; i < cnt; i += 32) {
            const float ti = sm.th[i], li = sm.tl[i];
            const uint32_t ii = sm.id[i];
            int rnk = 0;
            for (int j = 0; j < cnt; ++j) rnk += before(sm.th[j], sm.tl[j], sm.id[j], ti, li, ii) ? 1 : 0;
            SNP_CHECK(rnk >= 0 && rnk < cnt);
            sm.ord[rnk] = (uint16_t)i;
        }
        __syncwarp();
        // ---- composite: chunked warp product-scan of (1 - kappa), stop after the first hit
        // that takes T below the floor
        float carryT = 1.f, cr = 0.f, cg = 0.f, cbl = 0.f;
        int ncomp = cnt;
        for (int k0 = 0; k0 < cnt; k0 += 32) {
            const int k = k0 + lane;
            const bool valid = k < cnt;
            const int h = valid ? (int)sm.ord[k] : 0;
            const float kap = valid ? sm.kap[h] : 0.f;
            float incl = 1.0f - kap;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const float yv = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl *= yv;
            }
            float excl = __shfl_up_sync(0xffffffffu, incl, 1);
            if (lane == 0) excl = 1.0f;
            const float Tb = carryT * excl, Ta = carryT * incl;
            const uint32_t sb = __ballot_sync(0xffffffffu, valid && Ta < a.t_floor);
            const int stop = sb ? __ffs(sb) - 1 : 32;   // last composited lane of this chunk
            if (valid && lane <= stop) {
                const uint32_t id = sm.id[h];
                const float4 c = hit_rgb<kRay>(recs + (size_t)id * rec_f4(N), a.sh, a.sh_degree, id, ray);
                const float w = Tb * kap;
                cr = fmaf(w, c.y, cr);
                cg = fmaf(w, c.z, cg);
                cbl = fmaf(w, c.w, cbl);
            }
            if (sb) {
                carryT = __shfl_sync(0xffffffffu, Ta, stop);
                ncomp = k0 + stop + 1;
                break;
            }
            carryT = __shfl_sync(0xffffffffu, Ta, 31);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            cr += __shfl_xor_sync(0xffffffffu, cr, o);
            cg += __shfl_xor_sync(0xffffffffu, cg, o);
            cbl += __shfl_xor_sync(0xffffffffu, cbl, o);
        }
        if (lane == 0) {
            reinterpret_cast<float4 *>(a.out)[((size_t)view * cam.H + y) * cam.W + x] =
                make_float4(fmaf(carryT, a.bg[0], cr), fmaf(carryT, a.bg[1], cg), fmaf(carryT, a.bg[2], cbl),
                            1.f - carryT);
            atomicAdd(a.counters + kCntComposited, (unsigned long long)ncomp);
        }
        __syncwarp();
    }
    // (the grid completes only after K5: later work in the stream sees both)
    if (overlap) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// One CTA per camera batch: histogram of the slots over 256 length buckets
// (bucket 0 = longest list), exclusive scan, scatter.  The order inside a bucket is
// arbitrary: tiles are independent, so the rendered frame does not depend on it.
__global__ void __launch_bounds__(1024) k_tile_order(RenderArgs a, CamBatch cb, uint32_t *order) {
    pdl_prologue();
    __shared__ uint32_t hist[256];
    __shared__ uint32_t wsum[32];
    const int stripe_tiles = a.tiles_x * a.stripe_rows;
    const int total = stripe_tiles * cb.nv;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid < 256) hist[tid] = 0;
    __syncthreads();
    auto bucket = [&](int t) -> int {
        const int vloc = t / stripe_tiles;
        const int st = t - vloc * stripe_tiles;
        const int tx = st % a.tiles_x;
        const int ty = a.row_begin + (st / a.tiles_x) * a.row_stride;
        const int64_t slot = (int64_t)(cb.view0 + vloc) * a.tiles_per_view + ty * a.tiles_x + tx;
        const uint32_t len = a.ranges[2 * slot + 1] - a.ranges[2 * slot];
        if (len == 0) return 255;
        const int lz = __clz(len);                                  // len in [2^(31-lz), 2^(32-lz))
        const int frac = (int)((len << lz << 1) >> 29);             // 3 bits below the leading one
        const int lg8 = (31 - lz) * 8 + frac;                       // ~ 8 log2(len)
        return 254 - (lg8 < 254 ? lg8 : 254);
    };
    for (int t = tid; t < total; t += 1024) atomicAdd(&hist[bucket(t)], 1u);
    __syncthreads();
    if (tid < 256) {   // exclusive scan over the 256 buckets (8 warps)
        const uint32_t v = hist[tid];
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[wid] = x;
        hist[tid] = x - v;   // exclusive within the warp
    }
    __syncthreads();
    if (tid < 256) {
        uint32_t before = 0;
        for (int w = 0; w < wid; ++w) before += wsum[w];
        hist[tid] += before;
    }
    __syncthreads();
    for (int t = tid; t < total; t += 1024) order[atomicAdd(&hist[bucket(t)], 1u)] = (uint32_t)t;
}

}  // namespace

namespace {
constexpr int kMaxDevices = 64;
template <int N, bool kRay, bool kEager>
int render_grid_n(int tiles) {
    // persistent grid: every CTA that fits, all SMs.  Cached per device (the shared-memory
    // attribute and the occupancy are per-device properties; a process may drive several)
    static int resident[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    int &res = resident[dev < kMaxDevices ? dev : 0];
    if (!res) {
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(k_render<N, kRay, kEager>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(Smem<N>));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render<N, kRay, kEager>, kThreads, sizeof(Smem<N>));
        res = std::max(1, sms) * std::max(1, per_sm);
    }
    return std::min(tiles, res);
}

template <int N, bool kRay, bool kEager>
cudaError_t launch_render_n(const RenderArgs &a, const CamBatch &cams, int tiles, cudaStream_t st) {
    const int smem = (int)sizeof(Smem<N>);
    const int grid = render_grid_n<N, kRay, kEager>(tiles);   // (sets the attribute on this device)
    if (a.record) {   // (same grid: K6w counts K5's CTAs; + the warps' chunk fill counts)
        static bool attr[kMaxDevices] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        bool &done = attr[dev < kMaxDevices ? dev : 0];
        if (!done) {
            cudaError_t e = cudaFuncSetAttribute(k_render<N, kRay, kEager, 2>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem + 64);
            if (e != cudaSuccess) return e;
            done = true;
        }
        k_render<N, kRay, kEager, 2><<<grid, kThreads, smem + 64, st>>>(a, cams);
    } else {
        k_render<N, kRay, kEager><<<grid, kThreads, smem, st>>>(a, cams);
    }
    return cudaGetLastError();
}

template <int N, bool kRay>
cudaError_t launch_fallback_n(const RenderArgs &a, const CamBatch *cams, int n_batches, cudaStream_t st) {
    // K6w: 2 one-warp CTAs per SM (they fit beside K5's two CTAs); K6: every CTA that fits
    static int fw[kMaxDevices] = {}, fb[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const int d = dev < kMaxDevices ? dev : 0;
    if (!fw[d]) {
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fallback<N, kRay>, kFbThreads, 0);
        fb[d] = std::max(1, sms) * std::max(1, per_sm);
        fw[d] = 2 * std::max(1, sms);
    }
    const int overlap = n_batches == 1 ? 1 : 0;
    for (int i = 0; i < n_batches; ++i) {
        cudaError_t e = launch_hi(k_fallback_warp<N, kRay>, dim3(fw[d]), dim3(32), 0, st, a, cams[i], overlap);
        if (e != cudaSuccess) return e;
    }
    for (int i = 0; i < n_batches; ++i) {
        cudaError_t e = launch_hi(k_fallback<N, kRay>, dim3(fb[d]), dim3(kFbThreads), 0, st, a, cams[i]);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

template <int N>
cudaError_t launch_render_w(const RenderArgs &a, const CamBatch &cams, int tiles, cudaStream_t st) {
    if (a.eager_emit)
        return a.colour_ray ? launch_render_n<N, true, true>(a, cams, tiles, st)
                            : launch_render_n<N, false, true>(a, cams, tiles, st);
    return a.colour_ray ? launch_render_n<N, true, false>(a, cams, tiles, st)
                        : launch_render_n<N, false, false>(a, cams, tiles, st);
}
template <int N>
int render_grid_w(bool ray, bool eager, int tiles) {
    if (eager) return ray ? render_grid_n<N, true, true>(tiles) : render_grid_n<N, false, true>(tiles);
    return ray ? render_grid_n<N, true, false>(tiles) : render_grid_n<N, false, false>(tiles);
}
template <int N>
cudaError_t launch_fallback_w(const RenderArgs &a, const CamBatch *cams, int n_batches, cudaStream_t st) {
    return a.colour_ray ? launch_fallback_n<N, true>(a, cams, n_batches, st)
                        : launch_fallback_n<N, false>(a, cams, n_batches, st);
}
}  // namespace

namespace {
template <int N, bool kRay>
cudaError_t launch_render_grad_n(const RenderArgs &a, const CamBatch &cams, cudaStream_t st) {
    const int smem = (int)(sizeof(Smem<N>) + 64);
    static int res[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    int &resident = res[dev < kMaxDevices ? dev : 0];
    if (!resident) {
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaError_t e = cudaFuncSetAttribute(k_render<N, kRay, false, 1>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render<N, kRay, false, 1>, kThreads, smem);
        resident = std::max(1, sms) * std::max(1, per_sm);
    }
    const int tiles = a.tiles_x * a.stripe_rows * cams.nv;
    k_render<N, kRay, false, 1><<<std::min(tiles, resident), kThreads, smem, st>>>(a, cams);
    return cudaGetLastError();
}
template <int N>
cudaError_t launch_render_grad_w(const RenderArgs &a, const CamBatch &cams, cudaStream_t st) {
    return a.colour_ray ? launch_render_grad_n<N, true>(a, cams, st) : launch_render_grad_n<N, false>(a, cams, st);
}
}  // namespace

cudaError_t launch_render_grad(const RenderArgs &a, const CamBatch &cams, cudaStream_t st) {
    if (a.tiles_x * a.stripe_rows * cams.nv == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(a.counters + kCntTileQueue, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    switch (a.n_hidden) {
        case 4: return launch_render_grad_w<4>(a, cams, st);
        case 8: return launch_render_grad_w<8>(a, cams, st);
        case 16: return launch_render_grad_w<16>(a, cams, st);
        case 32: return launch_render_grad_w<32>(a, cams, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_render(const RenderArgs &a, const CamBatch &cams, bool reset_queue, cudaStream_t st) {
    const int tiles = a.tiles_x * a.stripe_rows * cams.nv;
    if (tiles == 0) return cudaSuccess;
    if (reset_queue) {
        cudaError_t e = cudaMemsetAsync(a.counters + kCntTileQueue, 0, sizeof(unsigned long long), st);
        if (e != cudaSuccess) return e;
    }
    switch (a.n_hidden) {
        case 4: return launch_render_w<4>(a, cams, tiles, st);
        case 8: return launch_render_w<8>(a, cams, tiles, st);
        case 16: return launch_render_w<16>(a, cams, tiles, st);
        case 32: return launch_render_w<32>(a, cams, tiles, st);
        default: return cudaErrorInvalidValue;
    }
}

int render_grid(int n_hidden, bool colour_ray, bool eager, int tiles) {
    switch (n_hidden) {
        case 4: return render_grid_w<4>(colour_ray, eager, tiles);
        case 16: return render_grid_w<16>(colour_ray, eager, tiles);
        case 32: return render_grid_w<32>(colour_ray, eager, tiles);
        default: return render_grid_w<8>(colour_ray, eager, tiles);
    }
}

cudaError_t launch_tile_order(const RenderArgs &a, const CamBatch &cams, uint32_t *order, cudaStream_t st) {
    if (a.tiles_x * a.stripe_rows * cams.nv == 0) return cudaSuccess;
    return launch_hi(k_tile_order, dim3(1), dim3(1024), 0, st, a, cams, order);
}

cudaError_t launch_fallback(const RenderArgs &a, const CamBatch *cams, int n_batches, cudaStream_t st) {
    switch (a.n_hidden) {
        case 4: return launch_fallback_w<4>(a, cams, n_batches, st);
        case 8: return launch_fallback_w<8>(a, cams, n_batches, st);
        case 16: return launch_fallback_w<16>(a, cams, n_batches, st);
        case 32: return launch_fallback_w<32>(a, cams, n_batches, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace snp
