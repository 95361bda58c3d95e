// binning.cu -- K2 (count, scan, warp-aggregated key duplication) and K4
// (tile ranges).  Key layout (R19): view << (tile_bits + 19) |
// tile << 19 | bits(L) >> 12, L the fp32 depth lower bound from K1; value = primitive
// index.  Emission order: view, primitive, stripe rows, columns -- the order the
// stable sort (K3) then preserves among equal keys.  The paper itself names no
// tiles; "depth-sorted" is realised per ray in K5 on top of this order.
#include "snp_internal.cuh"

namespace snp {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 2;                       // items per thread (blocked)
constexpr int kScanTile = kScanThreads * kScanItems;  // 512 items per block

struct ItemInfo {
    uint32_t count;
    int32_t x0, w, r_first;
};

__device__ __forceinline__ ItemInfo item_info(const BinArgs &a, int64_t o) {
    ItemInfo it{0, 0, 0, 0};
    short4 r = a.rects[o];
    if (r.x < 0) return it;
    int32_t y0 = r.y, y1 = r.w;
    int32_t first = y0 > a.row_begin ? y0 : a.row_begin;
    int32_t k = (first - a.row_begin + a.row_stride - 1) / a.row_stride;
    int32_t rf = a.row_begin + k * a.row_stride;
    if (rf > y1) return it;
    int32_t rows = (y1 - rf) / a.row_stride + 1;
    it.x0 = r.x;
    it.w = r.z - r.x + 1;
    it.r_first = rf;
    it.count = (uint32_t)(rows * it.w);
    return it;
}

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t *smem_warp, uint32_t &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) smem_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = lane < (kScanThreads / 32) ? smem_warp[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
            if (lane >= d) w += y;
        }
        if (lane < (kScanThreads / 32)) smem_warp[lane] = w;
    }
    __syncthreads();
    total = smem_warp[kScanThreads / 32 - 1];
    uint32_t before = wid ? smem_warp[wid - 1] : 0;
    return before + x - v;
}

constexpr unsigned long long kStAgg = 1ull << 62;   // block status: aggregate published
constexpr unsigned long long kStInc = 2ull << 62;   //               inclusive prefix published
constexpr unsigned long long kStVal = (1ull << 62) - 1ull;

// Decoupled look-back over the duplication blocks (one warp): returns the number of
// keys of all blocks before `blk`.  Lane l polls block blk-1-l; the nearest block
// with an inclusive prefix ends the walk.
__device__ __forceinline__ unsigned long long dup_lookback(const unsigned long long *status, int64_t blk) {
    const int lane = threadIdx.x & 31;
    unsigned long long sum = 0;
    int64_t q = blk - 1;
    while (q >= 0) {
        const int64_t me = q - lane;
        unsigned long long v = kStInc;   // (before block 0: an inclusive prefix of 0)
        if (me >= 0) {
            do {
                v = *reinterpret_cast<const volatile unsigned long long *>(status + me);
            } while ((v & ~kStVal) == 0);
        }
        const uint32_t inc = __ballot_sync(0xffffffffu, (v & kStInc) != 0);
        const int stop = inc ? __ffs(inc) - 1 : 31;   // nearest inclusive within the window
        unsigned long long x = lane <= stop ? (v & kStVal) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        sum += x;
        if (inc) break;
        q -= 32;
    }
    return sum;
}

// Single pass: counts the keys of a block of 512 items, gets the block's output
// offset by a decoupled look-back over the earlier blocks (block order from an
// atomic ticket, so every earlier block is resident or done), forms per-item
// offsets and emits keys warp-aggregated: the 256 items of a warp own a contiguous
// output range; lanes walk it 32 keys at a time (coalesced 8-byte key + 4-byte
// value stores), each lane finding its key's item by binary search over the warp's
// item offsets in shared memory.  The last block writes the key count.
// Tight binning (scene flag SNP_BIN_CONIC_TILES): does the silhouette
// ellipse (d^T [[A, B], [B, C]] d <= 1, d = p - centre) reach the rectangle [dx0, dx1] x
// [dy0, dy1] of a tile's pixel centres (offsets from the centre)?  The minimum of the
// quadratic over the rectangle is at the centre when the centre is inside, else on an
// edge (the clamped vertex of the edge's 1D quadratic).  Margins: the rectangle is grown
// by 1/256 px, the threshold by 1e-3 (the float data and the fp32 hit test, hit.cuh).
__device__ __forceinline__ bool ellipse_meets_rect(float A, float B, float C, float dx0, float dx1, float dy0,
                                                   float dy1) {
    if (dx0 <= 0.f && 0.f <= dx1 && dy0 <= 0.f && 0.f <= dy1) return true;
    float qmin = INFINITY;
    const float xs[2] = {dx0, dx1}, ys[2] = {dy0, dy1};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const float X = xs[k];
        const float dy = fminf(fmaxf(-B * X / C, dy0), dy1);
        qmin = fminf(qmin, A * X * X + 2.0f * B * X * dy + C * dy * dy);
        const float Y = ys[k];
        const float dx = fminf(fmaxf(-B * Y / A, dx0), dx1);
        qmin = fminf(qmin, A * dx * dx + 2.0f * B * dx * Y + C * Y * Y);
    }
    return qmin <= 1.0f + 1e-3f;
}

// Tight binning (SNP_BIN_TILE_DEPTH): a per-tile depth lower bound.  For any unit u,
// every point x of the ellipsoid has |x| >= u.x >= u.m - sqrt(u^T S u) (its support
// function), so with u the tile's central ray this bounds t_in of every ray (the unit
// ray's t = |x|), and is tight for rays near u.  Rounded down with a 4e-6 relative margin
// (float data); the key keeps the larger of it and K1a's bound.
__device__ __forceinline__ float tile_depth_bound(const float4 &f1, const float4 &f2, const float4 &f3,
                                                  const float4 &intr, int col, int row) {
    const float px = (float)(col * kTile) + 0.5f * kTile, py = (float)(row * kTile) + 0.5f * kTile;
    float u0 = (px - intr.z) * intr.x, u1 = (py - intr.w) * intr.y, u2 = 1.0f;
    const float inv = rsqrtf(u0 * u0 + u1 * u1 + 1.0f);
    u0 *= inv; u1 *= inv; u2 *= inv;
    const float um = u0 * f1.y + u1 * f1.z + u2 * f1.w;
    const float S00 = f2.x, S01 = f2.y, S02 = f2.z, S11 = f2.w, S12 = f3.x, S22 = f3.y;
    const float uSu = S00 * u0 * u0 + S11 * u1 * u1 + S22 * u2 * u2 + 2.0f * (S01 * u0 * u1 + S02 * u0 * u2 + S12 * u1 * u2);
    if (!(uSu >= 0.f)) return 0.f;
    const float r = sqrtf(uSu);
    return (um - r) - 4e-6f * (fabsf(um) + r) - 1e-30f;
}

template <bool kTight>   // tight binning (a.tight) in its own instantiation: the default one is unchanged
__global__ void __launch_bounds__(kScanThreads) k_scan_dup(BinArgs a) {
    pdl_prologue();
    __shared__ uint32_t sw[32];
    __shared__ int64_t s_blk;
    __shared__ unsigned long long s_gbase;
    __shared__ uint32_t s_off[kScanTile + 8];   // per item exclusive offset (block-relative)
    __shared__ uint32_t s_hist[8][256];         // digit histograms of the keys this block emits
    __shared__ int32_t s_x0[kScanTile], s_w[kScanTile], s_rf[kScanTile];   // item geometry, read once
    __shared__ uint32_t s_dep[kScanTile];
    for (int i = threadIdx.x; i < a.passes * 256; i += kScanThreads) (&s_hist[0][0])[i] = 0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        const int64_t t = (int64_t)atomicAdd(a.dup_status + gridDim.x, 1ull);
        s_blk = t;
        if (t == (int64_t)gridDim.x - 1) a.dup_status[gridDim.x] = 0ull;   // last ticket: reset
    }
    // K4 writes only the non-empty tiles' ranges: clear all of them here
    for (int64_t j = (int64_t)blockIdx.x * kScanThreads + threadIdx.x; j < 2 * a.n_slots;
         j += (int64_t)gridDim.x * kScanThreads)
        a.ranges[j] = 0u;
    __syncthreads();
    const int64_t blk = s_blk;
    const int64_t total_items = a.n * a.n_views;
    const int64_t blk0 = blk * kScanTile;
    const int64_t base = blk0 + (int64_t)threadIdx.x * kScanItems;
    uint32_t cnt[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        ItemInfo it{0, 0, 1, 0};
        if (base + k < total_items) it = item_info(a, base + k);
        cnt[k] = it.count;
        const int li = threadIdx.x * kScanItems + k;
        s_x0[li] = it.x0;
        s_w[li] = it.w > 0 ? it.w : 1;
        s_rf[li] = it.r_first;
        s_dep[li] = (it.count && base + k < total_items) ? (a.depth[base + k] >> kDepthDrop) : 0u;
        s += cnt[k];
    }
    uint32_t tot;
    uint32_t ex = block_exclusive_scan(s, sw, tot);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        s_off[threadIdx.x * kScanItems + k] = ex;
        ex += cnt[k];
    }
    if (threadIdx.x == kScanThreads - 1) s_off[kScanTile] = ex;   // block total
    if (wid == 0) {
        if (lane == 0) {
            if (blk == 0) atomicExch(a.dup_status, kStInc | (unsigned long long)tot);
            else atomicExch(a.dup_status + blk, kStAgg | (unsigned long long)tot);
        }
        const unsigned long long excl = blk == 0 ? 0ull : dup_lookback(a.dup_status, blk);
        if (lane == 0) {
            if (blk > 0) atomicExch(a.dup_status + blk, kStInc | (excl + tot));
            s_gbase = excl;
            if (blk == (int64_t)gridDim.x - 1) {
                // (every block has published its aggregate, so K1a is long complete)
                a.counters[kCntVisible] = atomicAdd(a.counters + kCntVisibleAcc, 0ull);   // (K4 clears it)
                a.counters[kCntDup] = excl + tot;
                a.counters[kCntCapOverflow] = excl + tot > (unsigned long long)a.capacity ? 1ull : 0ull;
            }
        }
    }
    __syncthreads();
    const uint64_t gbase = s_gbase;
    // warp wid owns items [wid*256, wid*256+256) of this block
    const int i0 = wid * 32 * kScanItems;
    const uint32_t wbeg = s_off[i0];
    const uint32_t wend = (wid == kScanThreads / 32 - 1) ? s_off[kScanTile] : s_off[i0 + 32 * kScanItems];
    const uint64_t view_shift = (uint64_t)a.tile_bits + kDepthBits;
    uint32_t n_dead = 0;
    for (uint32_t e = wbeg + lane; e < wend; e += 32) {
        // largest item j in [i0, i0+256) with s_off[j] <= e (and count > 0)
        int lo = i0, hi = i0 + 32 * kScanItems - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (s_off[mid] <= e) lo = mid; else hi = mid - 1;
        }
        const int64_t o = blk0 + lo;
        const uint32_t w = (uint32_t)s_w[lo];
        const uint32_t k = e - s_off[lo];
        const int32_t ri = (int32_t)(k / w);
        const int32_t c = (int32_t)(k - (uint32_t)ri * w);
        const int32_t row = s_rf[lo] + ri * a.row_stride;
        const uint64_t view = (uint64_t)(o / a.n);
        const uint32_t prim = (uint32_t)(o - (int64_t)view * a.n);
        const uint64_t tile = (uint64_t)row * (uint64_t)a.tiles_x + (uint64_t)(s_x0[lo] + c);
        SNP_CHECK(lo >= i0 && lo < i0 + 32 * kScanItems && row < a.tiles_y && s_x0[lo] + c < a.tiles_x);
        uint64_t key = (view << view_shift) | (tile << kDepthBits) | (uint64_t)s_dep[lo];
        if (kTight) {   // tight binning: drop tiles the silhouette misses, per-tile depth bounds
            const float4 *t4 = a.tight + 4 * o;
            const float4 f3 = __ldg(t4 + 3);
            if (f3.z != 0.f) {
                const int col = s_x0[lo] + c;
                if (a.bin_flags & 1) {
                    const float4 f0 = __ldg(t4), f1c = __ldg(t4 + 1);
                    const float x0 = (float)(col * kTile) + 0.5f - 1.0f / 256.0f, y0 = (float)(row * kTile) + 0.5f - 1.0f / 256.0f;
                    const float w = (float)(kTile - 1) + 2.0f / 256.0f;
                    if (!ellipse_meets_rect(f0.z, f0.w, f1c.x, x0 - f0.x, x0 + w - f0.x, y0 - f0.y, y0 + w - f0.y)) {
                        key = kDeadKey;
                        ++n_dead;
                    }
                }
                if (key != kDeadKey && (a.bin_flags & 2)) {
                    const float Lt = tile_depth_bound(__ldg(t4 + 1), __ldg(t4 + 2), f3, __ldg(a.intr + view), col, row);
                    const float Lp = __uint_as_float(a.depth[o]);
                    if (Lt > Lp) {
                        const uint64_t dep = (uint64_t)(__float_as_uint(Lt) >> kDepthDrop);
                        key = (key & ~((1ull << kDepthBits) - 1ull)) | dep;
                    }
                }
            }
        }
        const uint64_t g = gbase + e;
        if (g < (uint64_t)a.capacity) {
            a.keys[g] = key;
            a.vals[g] = prim;
            for (int p = 0; p < a.passes; ++p) atomicAdd(&s_hist[p][(key >> (8 * p)) & 255u], 1u);
        }
    }
    if (kTight) {
        const uint32_t d = __reduce_add_sync(0xffffffffu, n_dead);
        if (lane == 0 && d) atomicAdd(a.counters + kCntDeadKeysAcc, (unsigned long long)d);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < a.passes * 256; i += kScanThreads) {
        const uint32_t v = (&s_hist[0][0])[i];
        if (v) atomicAdd(a.hist + i, v);
    }
}

__global__ void k_tile_ranges(const uint64_t *keys, const unsigned long long *counters, int64_t capacity,
                              int32_t tile_bits, int32_t tiles, uint32_t *ranges, unsigned long long *dup_status,
                              int64_t dup_blocks, uint32_t *hist, int32_t hist_words) {
    pdl_prologue();
    // the first render of this binning needs clean render counters, the next frame's K2
    // clean block states and digit histograms (no memset node)
    if (blockIdx.x == 0 && threadIdx.x <= kCntRenderLast - kCntTested)
        const_cast<unsigned long long *>(counters)[kCntTested + threadIdx.x] = 0ull;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long *c = const_cast<unsigned long long *>(counters);
        c[kCntVisibleAcc] = 0ull;
        c[kCntDeadKeys] = c[kCntDeadKeysAcc];   // (K2 is complete)
        c[kCntDeadKeysAcc] = 0ull;
    }
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < dup_blocks; j += (int64_t)gridDim.x * blockDim.x)
        dup_status[j] = 0ull;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < hist_words; j += (int64_t)gridDim.x * blockDim.x)
        hist[j] = 0u;
    int64_t n = (int64_t)counters[kCntDup];
    if (n > capacity) n = capacity;
    const uint64_t tmask = (1ull << tile_bits) - 1ull;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (keys[i] == kDeadKey) continue;   // (tight binning: sorted after every live key)
        const uint64_t vt = keys[i] >> kDepthBits;
        const uint64_t slot = (vt >> tile_bits) * (uint64_t)tiles + (vt & tmask);
        SNP_CHECK((vt & tmask) < (uint64_t)tiles);
        if (i == 0 || (keys[i - 1] >> kDepthBits) != vt) ranges[2 * slot] = (uint32_t)i;
        if (i == n - 1 || (keys[i + 1] >> kDepthBits) != vt) ranges[2 * slot + 1] = (uint32_t)(i + 1);
    }
}

}  // namespace

int64_t bin_scan_blocks(int64_t items) { return (items + kScanTile - 1) / kScanTile; }

cudaError_t launch_dup(const BinArgs &a, cudaStream_t st) {
    const int64_t nb = bin_scan_blocks(a.n * a.n_views);
    if (nb == 0) {
        cudaError_t e = cudaMemsetAsync(a.counters + kCntDup, 0, sizeof(unsigned long long), st);
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(a.counters + kCntCapOverflow, 0, sizeof(unsigned long long), st);
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(a.counters + kCntVisible, 0, sizeof(unsigned long long), st);
        if (e != cudaSuccess) return e;
        if (a.n_slots > 0) e = cudaMemsetAsync(a.ranges, 0, sizeof(uint32_t) * 2 * (size_t)a.n_slots, st);
        return e;
    }
    cudaError_t e0 = a.tight ? launch_hi(k_scan_dup<true>, dim3((unsigned)nb), dim3(kScanThreads), 0, st, a)
                             : launch_hi(k_scan_dup<false>, dim3((unsigned)nb), dim3(kScanThreads), 0, st, a);
    if (e0 != cudaSuccess) return e0;
    return cudaGetLastError();
}

cudaError_t launch_tile_ranges(const uint64_t *keys, const unsigned long long *counters, int64_t capacity,
                               int32_t tile_bits, int32_t tiles, uint32_t *ranges, const BinArgs &b,
                               cudaStream_t st) {
    cudaError_t e = cudaSuccess;
    if (capacity == 0) return cudaSuccess;
    int64_t blocks = (capacity + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    e = launch_hi(k_tile_ranges, dim3((unsigned)blocks), dim3(256), 0, st, keys, counters, capacity, tile_bits, tiles,
                  ranges, b.dup_status, bin_scan_blocks(b.n * b.n_views), b.hist, (int32_t)(b.passes * 256));
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace snp
