// Stage (d): (depth, index) order of the passed splats and tile binning.
//
// Reference: argsort(depth, kind="stable") over passed splats
// (sc/raster.py:319) followed by the counting sort bin_tiles
// (sc/_kernels.py:137-165).  B200 version, all on device, no host sync:
//   1. stable LSD radix sort (4 x 8 bits) of the f32 depth keys of all
//      survivors (non-passed keys are 0xFFFFFFFF and sink to the end); the
//      input is in survivor order, so equal keys stay index-ordered;
//   2. tie-fix: runs of equal f32 keys are re-ordered by (f64 depth, index),
//      which makes the order identical to the reference's f64 argsort;
//   3. per-splat tile counts -> exclusive scan -> entry emission
//      (tile id, survivor index) in depth order;
//   4. stable LSD radix sort of the entries by tile id (2 x 8 bits), i.e.
//      the reference's stable counting sort by tile;
//   5. tile offsets (the reference's `counts` array).
// Every kernel reads its element count from device memory, so the whole
// frame stays asynchronous (and CUDA-graph capturable).
#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace sc {

// ---------------------------------------------------------------------------
// generic exclusive scan of uint32 (3 phases), n read from device or host
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t dev_count(const unsigned long long *n_dev, int64_t n_host)
{
    return n_dev ? std::min<int64_t>((int64_t)*n_dev, n_host) : n_host;
}

template <int THREADS>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t *s_warp, uint32_t &total)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NW = THREADS / 32;
    uint32_t v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) s_warp[wid] = v;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = lane < NW ? s_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NW) s_warp[lane] = w;
    }
    __syncthreads();
    total = s_warp[NW - 1];
    const uint32_t r = (wid ? s_warp[wid - 1] : 0u) + v - x;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t *in, const unsigned long long *n_dev,
                                                              int64_t n_host, uint32_t *part)
{
    __shared__ uint32_t s_warp[32];
    const int64_t n = dev_count(n_dev, n_host);
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    uint32_t sum = 0;
    if (base < n) {
        for (int j = 0; j < kScanItems; j++) {
            const int64_t i = base + (int64_t)j * kScanThreads + threadIdx.x;
            if (i < n) sum += in[i];
        }
    }
    uint32_t total;
    block_excl_scan<kScanThreads>(sum, s_warp, total);
    if (threadIdx.x == 0) part[blockIdx.x] = total;
}

// Each block adds up the raw sums of the blocks before it (a few thousand L2-resident
// words at most), so no single-CTA pass over the partials sits between the two kernels;
// the last active block writes the total.
__global__ void __launch_bounds__(kScanThreads) k_scan_down(const uint32_t *in, uint32_t *out,
                                                            const unsigned long long *n_dev, int64_t n_host,
                                                            const uint32_t *part, unsigned long long *total_out,
                                                            int64_t *stat_out)
{
    __shared__ uint32_t s_warp[32];
    const int64_t n = dev_count(n_dev, n_host);
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    if (base >= n) {
        if (n <= 0 && blockIdx.x == 0 && threadIdx.x == 0) {
            if (total_out) *total_out = 0;
            if (stat_out) *stat_out = 0;
        }
        return;
    }
    uint32_t pre = 0;
    {
        uint32_t acc = 0;
        for (int64_t i = threadIdx.x; i < (int64_t)blockIdx.x; i += kScanThreads) acc += __ldcg(part + i);
        block_excl_scan<kScanThreads>(acc, s_warp, pre);   // pre = total over the block
    }
    // blocked arrangement: thread t owns items [base + t*16, base + t*16 + 16), moved as 4 x uint4
    static_assert(kScanItems == 16, "vector path assumes 16 items per thread");
    uint32_t v[kScanItems];
    uint32_t sum = 0;
    const int64_t my = base + (int64_t)threadIdx.x * kScanItems;
    const bool full = my + kScanItems <= n;
    if (full) {
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const uint4 x = __ldcs(reinterpret_cast<const uint4 *>(in + my) + q);
            v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < kScanItems; j++) v[j] = my + j < n ? in[my + j] : 0u;
    }
#pragma unroll
    for (int j = 0; j < kScanItems; j++) sum += v[j];
    uint32_t total;
    uint32_t run = block_excl_scan<kScanThreads>(sum, s_warp, total) + pre;
    if (threadIdx.x == 0 && base + kScanTile >= n) {   // the last active block
        if (total_out) *total_out = (unsigned long long)pre + total;
        if (stat_out) *stat_out = (int64_t)pre + total;
    }
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        const uint32_t x = v[j];
        v[j] = run;
        run += x;
    }
    if (full) {
#pragma unroll
        for (int q = 0; q < 4; q++)
            reinterpret_cast<uint4 *>(out + my)[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < kScanItems; j++)
            if (my + j < n) out[my + j] = v[j];
    }
}

cudaError_t scan_excl(const uint32_t *in, uint32_t *out, const unsigned long long *n_dev, int64_t n_max,
                      uint32_t *part, unsigned long long *total_out, int64_t *stat_out, cudaStream_t st)
{
    const int64_t nblk = std::max<int64_t>(1, (n_max + kScanTile - 1) / kScanTile);
    SC_LAUNCH(k_scan_reduce, (int)nblk, kScanThreads, 0, st, in, n_dev, n_max, part);
    SC_LAUNCH(k_scan_down, (int)nblk, kScanThreads, 0, st, in, out, n_dev, n_max, part, total_out, stat_out);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// LSD radix sort (8-bit digits), stable, reduce-then-scan per pass:
//   upsweep:   per 4096-key tile, digit counts -> counts[digit][tile]
//   scan:      one exclusive scan over the digit-major matrix = every
//              (digit, tile) global scatter base (no inter-tile chains)
//   downsweep: persistent CTAs taking tiles from an atomic ticket; a tile's
//              keys/values arrive by TMA bulk copy into one of two shared
//              buffers while the previous tile is ranked and scattered; stable
//              warp-private ranking (8-ballot match, or match.any for the
//              block sort's last pass), staging in shared memory, digit-run
//              coalesced write-out.
// ---------------------------------------------------------------------------
// 4096-key tiles, 256 threads x 16 keys, 2 CTAs per SM (~120 registers): 8 warps share each
// tile barrier (512 x 8 keys: 16 warps, 64 registers, 3 % slower sort; 128 threads cannot
// hold the one-thread-per-digit scan phase)
#ifndef SC_RADIX_THREADS
#define SC_RADIX_THREADS 256
#endif
constexpr int kOsThreads = SC_RADIX_THREADS;
constexpr int kOsItems = 4096 / SC_RADIX_THREADS;
static_assert(kOsThreads >= 256, "the scan phase has one thread per digit");
constexpr int kOsTile = kOsThreads * kOsItems;
constexpr int kOsWarps = kOsThreads / 32;
static_assert(kOsTile == kRadixTile, "matrix sizing in api.cu assumes kRadixTile keys per tile");

// lanes of the warp holding the same 8-bit digit: 8 ballots, constant cost
// (match.any's cost grows with the number of distinct values in the warp)
// per bit: predicate straight from the digit, ballot, sign mask, one 3-input
// logic op (m &= ~(ballot ^ mask)): 4 instructions
__device__ __forceinline__ uint32_t match_digit8(uint32_t d)
{
    uint32_t m = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; b++) {
        uint32_t bal, sm;
        asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
            "and.b32 t, %2, %3;\n\t"
            "setp.ne.u32 p, t, 0;\n\t"
            "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t"
            "selp.b32 %1, -1, 0, p;\n\t}"
            : "=r"(bal), "=r"(sm)
            : "r"(d), "r"(1u << b));
        m &= ~(bal ^ sm);
    }
    return m;
}

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void os_mbar_init(uint64_t *bar)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void os_mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "OS_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra OS_DONE;\n\t"
        "bra OS_WAIT;\n\t"
        "OS_DONE:\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// one thread: expect the bytes on bar, then bulk-copy the two pieces
__device__ __forceinline__ void os_bulk_load(uint64_t *bar, void *dk, const void *sk, uint32_t bk, void *dv,
                                             const void *sv, uint32_t bv)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bk + bv)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dk)),
                 "l"(sk), "r"(bk), "r"(smem_addr(bar))
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dv)),
                 "l"(sv), "r"(bv), "r"(smem_addr(bar))
                 : "memory");
}

// Tile tickets: tiles are handed out in order by an atomic counter; each CTA
// ends by taking one ticket past the end; the last CTA to finish resets the
// pair for the next sweep (kernels on a stream run one after the other).
__device__ __forceinline__ void ticket_release(unsigned long long *next, unsigned long long *done)
{
    __threadfence();
    if (atomicAdd(done, 1ull) == (unsigned long long)gridDim.x - 1) {
        *next = 0;
        *done = 0;
        __threadfence();
    }
}

// Upsweep, warp per tile: a warp takes a whole 4096-key tile from the ticket,
// histograms it into its private shared counters and writes the tile's 256
// counts itself -- no CTA barrier per tile (a CTA-cooperative upsweep spent its
// time in two barriers per tile: 90 vs ~60 us per depth pass, far view).
#ifndef SC_UPW_BATCH
#define SC_UPW_BATCH 4
#endif
constexpr int kUpwBatch = SC_UPW_BATCH;   // uint4 loads per lane per batch (double-buffered)
#ifndef SC_UP_THREADS
#define SC_UP_THREADS 256
#endif
constexpr int kUpThreads = SC_UP_THREADS, kUpWarps = kUpThreads / 32;   // upsweep: warp per tile
__global__ void __launch_bounds__(kUpThreads, 2) k_radix_up(const uint32_t *__restrict__ keys,
                                                             const unsigned long long *n_dev, int64_t n_host,
                                                             int shift, uint32_t *counts,
                                                             unsigned long long *scan_n,
                                                             unsigned long long *tk_next, unsigned long long *tk_done)
{
    __shared__ uint32_t h[kUpWarps][256];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t n = dev_count(n_dev, n_host);
    // the count matrix is [256][tiles of this frame] (not of the capacity): the scan and the
    // downsweep use the same device-side tile count
    const int64_t ntiles = (n + kOsTile - 1) / kOsTile;
    if (blockIdx.x == 0 && tid == 0) *scan_n = 256ull * (unsigned long long)ntiles;
    uint32_t *hw = h[wid];
#pragma unroll
    for (int q = 0; q < 8; q++) hw[lane + 32 * q] = 0;
    __syncwarp();
    constexpr int kBatches = kOsTile / (32 * 4 * kUpwBatch);
    for (;;) {
        unsigned long long tt = 0;
        if (lane == 0) tt = atomicAdd(tk_next, 1ull);
        const int64_t t = (int64_t)__shfl_sync(0xffffffffu, tt, 0);
        if (t >= ntiles) break;
        const int64_t base = t * kOsTile;
        if (base + kOsTile <= n) {
            uint4 ka[kUpwBatch], kb[kUpwBatch];
            auto load = [&](int bi, uint4 *dst) {
#pragma unroll
                for (int q = 0; q < kUpwBatch; q++)
                    dst[q] = __ldcs(reinterpret_cast<const uint4 *>(keys + base) + (bi * kUpwBatch + q) * 32 + lane);
            };
            auto count = [&](const uint4 *src) {
#pragma unroll
                for (int q = 0; q < kUpwBatch; q++) {
                    atomicAdd(&hw[(src[q].x >> shift) & 0xFFu], 1u);
                    atomicAdd(&hw[(src[q].y >> shift) & 0xFFu], 1u);
                    atomicAdd(&hw[(src[q].z >> shift) & 0xFFu], 1u);
                    atomicAdd(&hw[(src[q].w >> shift) & 0xFFu], 1u);
                }
            };
            load(0, ka);
#pragma unroll 1
            for (int bi = 0; bi < kBatches; bi += 2) {
                load(bi + 1, kb);
                count(ka);
                if (bi + 2 < kBatches) load(bi + 2, ka);
                count(kb);
            }
        } else {
            for (int64_t e = base + lane; e < n && e < base + kOsTile; e += 32) atomicAdd(&hw[(keys[e] >> shift) & 0xFFu], 1u);
        }
        __syncwarp();
        // digit-major: the matrix's exclusive scan is every (digit, tile) base; empty tiles write zeros
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int d = lane + 32 * q;
            counts[(int64_t)d * ntiles + t] = hw[d];
            hw[d] = 0;
        }
        __syncwarp();
    }
    __syncthreads();
    if (tid == 0) ticket_release(tk_next, tk_done);
}

// (the ranked tile is staged back into its own input buffer for the write-out)
template <typename V>
struct OsSmem {
    uint32_t in_k[2][kOsTile];
    V in_v[2][kOsTile];
    uint16_t wcnt[kOsWarps][256];
};

// MATCH_ANY: rank with match.any (fast when a warp holds few distinct digits,
// e.g. the block sort's high byte: screen rows follow depth order) instead of
// the constant-cost 8-ballot match.
// IDX_IN (first depth pass of the frame path, V = uint2): the input values are the
// packed pixel windows alone (u32, the projection writes no index) and the output
// value is (input position = survivor index, window).
#ifndef SC_RADIX_WUNROLL
#define SC_RADIX_WUNROLL 2
#endif
constexpr int kRadixWUnroll = SC_RADIX_WUNROLL;
template <typename V, bool MATCH_ANY, bool IDX_IN = false>
__global__ void __launch_bounds__(kOsThreads, 2) k_radix_down(const uint32_t *__restrict__ keys_in,
                                                              const V *__restrict__ vals_in,
                                                              uint32_t *__restrict__ keys_out,
                                                              V *__restrict__ vals_out,
                                                              const unsigned long long *n_dev, int64_t n_host,
                                                              int shift, const uint32_t *__restrict__ bases,
                                                              int64_t /* capacity tiles (unused) */,
                                                              unsigned long long *tk_next,
                                                              unsigned long long *tk_done)
{
    constexpr int kPerWarp = kOsTile / kOsWarps;
    extern __shared__ __align__(128) uint4 s_dyn4[];
    OsSmem<V> &sm = *reinterpret_cast<OsSmem<V> *>(s_dyn4);
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ uint32_t s_gofs[256];     // global scatter base - tile-local start of each digit

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t n = dev_count(n_dev, n_host);
    const int64_t ntiles = (n + kOsTile - 1) / kOsTile;
    auto issue = [&](int64_t t, int b) {
        const int64_t base = t * kOsTile;
        const uint32_t c = (uint32_t)std::min<int64_t>(kOsTile, n - base);
        // sizes rounded up to 16 B (the key / value buffers carry 16 bytes of slack)
        if constexpr (IDX_IN)
            os_bulk_load(&s_bar[b], sm.in_k[b], keys_in + base, (c * 4u + 15u) & ~15u, sm.in_v[b],
                         reinterpret_cast<const uint32_t *>(vals_in) + base, (c * 4u + 15u) & ~15u);
        else
            os_bulk_load(&s_bar[b], sm.in_k[b], keys_in + base, (c * 4u + 15u) & ~15u, sm.in_v[b], vals_in + base,
                         (c * (uint32_t)sizeof(V) + 15u) & ~15u);
    };
    __shared__ int64_t s_tile;
    __shared__ uint32_t s_dsum[256 / 32];   // per-warp digit totals of the scan phase
    for (int i = tid; i < kOsWarps * 256; i += kOsThreads) (&sm.wcnt[0][0])[i] = 0;
    if (tid == 0) {
        os_mbar_init(&s_bar[0]);
        os_mbar_init(&s_bar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_tile = (int64_t)atomicAdd(tk_next, 1ull);
        if (s_tile < ntiles) issue(s_tile, 0);
    }
    __syncthreads();
    int64_t tile = s_tile;
    uint32_t phase0 = 0, phase1 = 0;
    int b = 0;
    const uint32_t lt = lanemask_lt();
    while (tile < ntiles) {
        __syncthreads();   // buffer b^1 (previous tile) fully written out; s_tile read by all
        if (tid == 0) {   // the next tile's ticket and its TMA load, one tile ahead
            s_tile = (int64_t)atomicAdd(tk_next, 1ull);
            if (s_tile < ntiles) issue(s_tile, b ^ 1);
        }
        uint32_t gb = 0;
        if (tid < 256) gb = bases[(int64_t)tid * ntiles + tile];   // (matrix stride: this frame's tiles)
        const int64_t base = tile * kOsTile;
        const int cnt = (int)std::min<int64_t>(kOsTile, n - base);
        if (b == 0) {
            os_mbar_wait(&s_bar[0], phase0);
            phase0 ^= 1u;
        } else {
            os_mbar_wait(&s_bar[1], phase1);
            phase1 ^= 1u;
        }
        // (no barrier: every thread observed the TMA's mbarrier itself, and the warp counters
        // were zeroed before the loop-top barrier)

        // stable warp-private ranking: warp w owns the contiguous slice
        // [w * 256, (w + 1) * 256) and keeps running per-digit counts
        uint32_t k[kOsItems], rk[kOsItems];
        V v[kOsItems];
        auto rank = [&](auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;   // no bounds checks on full tiles
            uint32_t peers[kOsItems];
#pragma unroll
            for (int j = 0; j < kOsItems; j++) {
                const int i = wid * kPerWarp + j * 32 + lane;
                k[j] = sm.in_k[b][i];
                if constexpr (IDX_IN)
                    v[j] = make_uint2((uint32_t)(base + i), reinterpret_cast<const uint32_t *>(sm.in_v[b])[i]);
                else
                    v[j] = sm.in_v[b][i];
                const bool ok = FULL || i < cnt;
                if constexpr (MATCH_ANY)
                    peers[j] = __match_any_sync(0xffffffffu, ok ? ((k[j] >> shift) & 0xFFu) : 256u + (uint32_t)lane);
                else if constexpr (FULL)
                    peers[j] = match_digit8((k[j] >> shift) & 0xFFu);
                else
                    peers[j] = match_digit8((k[j] >> shift) & 0xFFu) & __ballot_sync(0xffffffffu, ok);
            }
#pragma unroll
            for (int j = 0; j < kOsItems; j++) {
                const bool ok = FULL || wid * kPerWarp + j * 32 + lane < cnt;
                const uint32_t d = (k[j] >> shift) & 0xFFu;
                const uint32_t r = __popc(peers[j] & lt);
                const uint32_t prev = ok ? sm.wcnt[wid][d] : 0u;
                __syncwarp();
                if (ok && r == 0) sm.wcnt[wid][d] = (uint16_t)(prev + __popc(peers[j]));
                __syncwarp();
                rk[j] = prev + r;
            }
        };
        if (cnt == kOsTile)
            rank(std::true_type{});
        else
            rank(std::false_type{});
        __syncthreads();
        // thread = digit: its per-warp counts, the tile-local digit start (block scan), then
        // wcnt[w][d] = digit start + exclusive prefix over warps (the scatter base of warp w)
        uint32_t wc[kOsWarps];
        uint32_t tot = 0;
        if (tid < 256) {
#pragma unroll
            for (int w = 0; w < kOsWarps; w++) {
                wc[w] = sm.wcnt[w][tid];
                tot += wc[w];
            }
        }
        {
            // exclusive scan over the 256 digits: warp scans, one barrier, each thread adds the
            // totals of the warps before its own (<= 7 broadcast reads)
            uint32_t ds = 0;
            if (tid < 256) {
                uint32_t x = tot;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (lane == 31) s_dsum[wid] = x;
                ds = x - tot;
            }
            __syncthreads();
            if (tid < 256)
                for (int w = 0; w < wid; w++) ds += s_dsum[w];
            if (tid < 256) {
                uint32_t run = ds;
#pragma unroll
                for (int w = 0; w < kOsWarps; w++) {
                    sm.wcnt[w][tid] = (uint16_t)run;
                    run += wc[w];
                }
                s_gofs[tid] = gb - ds;   // output index = s_gofs[d] + tile position (mod 2^32)
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kOsItems; j++) {
            if (wid * kPerWarp + j * 32 + lane < cnt) {
                const uint32_t d = (k[j] >> shift) & 0xFFu;
                const uint32_t pos = sm.wcnt[wid][d] + rk[j];
                sm.in_k[b][pos] = k[j];
                sm.in_v[b][pos] = v[j];
            }
        }
        __syncthreads();
        // coalesced write-out: consecutive positions of one digit are contiguous in the output
        // (unrolled 2x with 256-thread CTAs; 4x bursts of loads then stores ran 2-3 % slower per pass)
#pragma unroll kRadixWUnroll
        for (int i = tid; i < cnt; i += kOsThreads) {
            const uint32_t key = sm.in_k[b][i];
            const uint32_t dst = s_gofs[(key >> shift) & 0xFFu] + (uint32_t)i;
            keys_out[dst] = key;
            vals_out[dst] = sm.in_v[b][i];
        }
        // the next tile's warp counters (the write-out does not read them; the loop-top
        // barrier orders this before the next ranking)
        for (int i = tid; i < kOsWarps * 256 / 8; i += kOsThreads) reinterpret_cast<uint4 *>(&sm.wcnt[0][0])[i] = make_uint4(0, 0, 0, 0);
        // generic-proxy writes to buffer b above; its next refill is a TMA (async-proxy) write
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        b ^= 1;
        tile = s_tile;   // written by thread 0 before the tile's barriers
    }
    if (tid == 0) ticket_release(tk_next, tk_done);
}

template <typename V>
static cudaError_t radix_down_attr()
{
    const int bytes = (int)sizeof(OsSmem<V>);
    cudaError_t e = smem_attr_once(reinterpret_cast<const void *>(k_radix_down<V, false>), bytes);
    if (e == cudaSuccess) e = smem_attr_once(reinterpret_cast<const void *>(k_radix_down<V, true>), bytes);
    if constexpr (std::is_same<V, uint2>::value)
        if (e == cudaSuccess) e = smem_attr_once(reinterpret_cast<const void *>(k_radix_down<V, false, true>), bytes);
    return e;
}

static int sm_count_sort() { return sm_count(); }

// Sorts (keys, vals) on key bits [bit_lo, bit_hi) (bits below bit_lo ride
// along); the result ends in the buffers returned through keys_res / vals_res
// (ping-pong between a and b).
template <typename V>
static cudaError_t radix_sort(uint32_t *ka, V *va, uint32_t *kb, V *vb, const unsigned long long *n_dev, int64_t n_max,
                              int bit_lo, int bit_hi, const Ws &ws, uint32_t **keys_res, V **vals_res, cudaStream_t st,
                              bool last_match_any = false, bool first_idx_in = false)
{
    cudaError_t e = radix_down_attr<V>();
    if (e != cudaSuccess) return e;
    const int npass = std::max(1, (bit_hi - bit_lo + 7) / 8);
    const int64_t ntiles = std::max<int64_t>(1, (n_max + kOsTile - 1) / kOsTile);
    const int nsm = sm_count_sort();
    uint32_t *ki = ka, *ko = kb;
    V *vi = va, *vo = vb;
    for (int p = 0; p < npass; p++) {
        const int shift = bit_lo + 8 * p;
        SC_LAUNCH(k_radix_up, (int)std::min<int64_t>((ntiles + kUpWarps - 1) / kUpWarps, (int64_t)nsm * 2),
                  kUpThreads, 0, st, ki, n_dev, n_max, shift, ws.rs_counts, &ws.ctr->rs_scan_n, &ws.ctr->rs_next,
                  &ws.ctr->rs_done);
        e = scan_excl(ws.rs_counts, ws.rs_counts, &ws.ctr->rs_scan_n, 256 * ntiles, ws.scan_part, nullptr, nullptr, st);
        if (e != cudaSuccess) return e;
#ifndef SC_RADIX_CPS
#define SC_RADIX_CPS 2
#endif
        const int grid = (int)std::min<int64_t>(ntiles, (int64_t)nsm * SC_RADIX_CPS);
        if (last_match_any && p == npass - 1)
            SC_LAUNCH((k_radix_down<V, true>), grid, kOsThreads, sizeof(OsSmem<V>), st, ki, vi, ko, vo, n_dev, n_max,
                      shift, ws.rs_counts, ntiles, &ws.ctr->rs_next, &ws.ctr->rs_done);
        else if (first_idx_in && p == 0)   // input values: u32 windows at va (index = position)
            SC_LAUNCH((k_radix_down<V, false, std::is_same<V, uint2>::value>), grid, kOsThreads, sizeof(OsSmem<V>), st,
                      ki, vi, ko, vo, n_dev, n_max, shift, ws.rs_counts, ntiles, &ws.ctr->rs_next, &ws.ctr->rs_done);
        else
            SC_LAUNCH((k_radix_down<V, false>), grid, kOsThreads, sizeof(OsSmem<V>), st, ki, vi, ko, vo, n_dev, n_max,
                      shift, ws.rs_counts, ntiles, &ws.ctr->rs_next, &ws.ctr->rs_done);
        std::swap(ki, ko);
        std::swap(vi, vo);
    }
    *keys_res = ki;
    *vals_res = vi;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// stage-level API depth keys: frame-adaptive 32-bit quantisation of the f64
// depth over the passed splats' exact [dmin, dmax] (monotone non-decreasing,
// so key order agrees with f64 order wherever keys differ; equal keys go to
// the tie-fix).  The frame path quantises over the instance spheres' depth
// range inside the projection kernel instead (no depth64 round trip).
// ---------------------------------------------------------------------------
__global__ void k_depth_keys(const double *depth64, const unsigned long long *n_dev, int64_t n_host,
                             const Counters *ctr, uint32_t *keys, uint2 *pv)
{
    const int64_t n = dev_count(n_dev, n_host);
    const double dmin = __longlong_as_double((long long)~ctr->dmin_inv);
    const double dmax = __longlong_as_double((long long)ctr->dmax);
    constexpr double kTop = 4294967040.0;   // < 0xFFFFFFFF, which marks non-passed splats
    const double scale = (ctr->passed > 0 && dmax > dmin) ? kTop / (dmax - dmin) : 0.0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const double d = depth64[k];
        uint32_t key = 0xFFFFFFFFu;
        if (d >= 0.0) key = (uint32_t)fmin(floor((d - dmin) * scale), kTop);
        keys[k] = key;
        pv[k] = make_uint2((uint32_t)k, 0u);
    }
}

__global__ void k_extract_order(const uint2 *pv, const unsigned long long *n_dev, int64_t n_host, uint32_t *order)
{
    const int64_t n = dev_count(n_dev, n_host);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        order[k] = pv[k].x;
}

// ---------------------------------------------------------------------------
// entries: per passed splat (depth order) count, scan, emit (tile, survivor)
// ---------------------------------------------------------------------------
// The rect of each splat is gathered once here (depth order) and kept
// contiguous in (rlo, rhi) so the emission pass reads it coalesced.
__global__ void k_entry_count(const uint32_t *order, const ushort4 *rect, const unsigned long long *n_dev,
                              int64_t n_host, uint32_t *cnt, uint32_t *rlo, uint32_t *rhi)
{
    const int64_t n = dev_count(n_dev, n_host);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const ushort4 r = rect[order[k]];
        cnt[k] = (uint32_t)(r.y - r.x) * (uint32_t)(r.w - r.z);
        rlo[k] = (uint32_t)r.x | ((uint32_t)r.y << 16);
        rhi[k] = (uint32_t)r.z | ((uint32_t)r.w << 16);
    }
}

__global__ void k_entry_emit(const uint32_t *order, const uint32_t *rlo, const uint32_t *rhi, const uint32_t *off,
                             const unsigned long long *n_dev, int64_t n_host, int n_tx, uint32_t *ekey,
                             uint32_t *eval, const unsigned long long *e_total, unsigned long long *e_eff, int64_t cap_e,
                             sc_frame_stats *stats)
{
    const int64_t n = dev_count(n_dev, n_host);
    const bool over = (int64_t)*e_total > cap_e;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *e_eff = over ? 0ull : *e_total;
        if (over) atomicOr((unsigned long long *)&stats->overflow, 2ull);
    }
    if (over) return;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t sv = order[k];
        const uint32_t a = rlo[k], b = rhi[k];
        const ushort4 r = make_ushort4(a & 0xFFFF, a >> 16, b & 0xFFFF, b >> 16);
        uint32_t o = off[k];
        for (int y = r.z; y < r.w; y++)
            for (int x = r.x; x < r.y; x++) {
                ekey[o] = (uint32_t)(y * n_tx + x);
                eval[o] = sv;
                o++;
            }
    }
}

// tile_off[t] = first entry index with tile >= t, for t in [0, n_tiles] (the
// reference's `counts`; stage-level API only)
__global__ void k_tile_offsets(const uint32_t *ekey, const unsigned long long *e_dev, int64_t cap_e, int64_t n_tiles,
                               uint32_t *tile_off)
{
    const int64_t E = std::min<int64_t>((int64_t)*e_dev, cap_e);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= E; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t prev = i > 0 ? (int64_t)ekey[i - 1] : -1;
        const int64_t cur = i < E ? (int64_t)ekey[i] : n_tiles;
        for (int64_t t = prev + 1; t <= cur; t++) tile_off[t] = (uint32_t)i;
    }
}

// ---------------------------------------------------------------------------
// Frame-path binning: 8x4 pixel blocks instead of 16x16 tiles.
//
// Each passed splat (in depth order) emits one entry per 8x4 block its pixel
// window touches; block b of tile t has id 8 t + b (b = 2 row + col: x in
// [8 col, 8 col + 7], y in [4 row, 4 row + 3]), so a tile's blocks are
// contiguous.  The sort key is id << 10 | the window clipped to the block
// (x0 | x1 << 3 | y0 << 6 | y1 << 8, block-relative); the radix sort only
// sorts the id bits, so the clipped window rides along.  Being a stable sort
// of the depth-ordered emission, block list (t, b) is exactly the depth-order
// subsequence of the reference's tile-t entry list whose window touches
// block b (the only entries the reference composites onto those pixels):
// one blend warp walks one list.
// ---------------------------------------------------------------------------
constexpr int kCodeBits = 10;

// block entries of one passed splat (depth order), window from the sort payload
__device__ __forceinline__ uint32_t block_count(int x0, int x1, int y0, int y1)
{
    return (uint32_t)((x1 / 8 - x0 / 8 + 1) * (y1 / 4 - y0 / 4 + 1));
}

__device__ __forceinline__ uint32_t bentry_count(uint2 v, const sc_window *wins, int width, int height)
{
    int x0, x1, y0, y1;
    return unpack_window(v.y, v.x, wins, width, height, x0, x1, y0, y1) ? block_count(x0, x1, y0, y1) : 0u;
}

// Emission tiles: kEmitTile consecutive passed splats (depth order) per CTA
// iteration, warp w owning the contiguous kEmitPerWarp splats [w * 512, w * 512
// + 512) of the tile.  Pass 1 writes per-(tile, warp) entry totals, one
// exclusive scan turns them into output bases, pass 2 emits (every warp on its
// own, no CTA barrier): no per-splat count array round trip through HBM.
constexpr int kEmitThreads = 256;
constexpr int kEmitTile = 4096;
constexpr int kEmitPerWarp = kEmitTile / (kEmitThreads / 32);

// pass 1: the entry total of every (tile, warp) range of kEmitPerWarp splats

__global__ void __launch_bounds__(kEmitThreads) k_bentry_tiles(const uint2 *__restrict__ pv, const sc_window *wins,
                                                               const unsigned long long *n_dev, int64_t n_host,
                                                               int64_t ntiles_max, int width, int height,
                                                               uint32_t *warp_tot)
{
    const int64_t n = dev_count(n_dev, n_host);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t t = blockIdx.x; t < ntiles_max; t += gridDim.x) {
        const int64_t wbase = t * kEmitTile + (int64_t)wid * kEmitPerWarp;
        uint32_t c = 0;
        if (wbase < n) {
#pragma unroll 4
            for (int r = 0; r < kEmitPerWarp / 32; r++) {
                const int64_t k = wbase + r * 32 + lane;
                if (k < n) c += bentry_count(__ldg(pv + k), wins, width, height);
            }
        }
        c = __reduce_add_sync(0xffffffffu, c);
        if (lane == 0) warp_tot[t * (kEmitThreads / 32) + wid] = c;
    }
}

#ifndef SC_EMIT_LANE_MAX
#define SC_EMIT_LANE_MAX 5   // per-lane walk while no splat of the group has more blocks, else lane = entry (A/B: 2-3 +1.7 %, 16 +0.4 %)
#endif
// one warp: the (contiguous) entries of 32 consecutive passed splats, starting
// at output obase; returns their total
__device__ __forceinline__ uint32_t emit_group(uint2 cv, bool valid, uint32_t obase, const sc_window *wins, int width,
                                               int height, int n_tx, uint32_t *ekey, uint32_t *eval, int lane)
{
    // Warp-cooperative, load-balanced: lane l produces output o = step + l; the
    // owning splat is found by an upper-bound search over the warp's exclusive
    // counts (5 shuffles).  Splats covering thousands of blocks (close to the
    // camera) do not serialise one thread, and the stores are coalesced.
    int x0 = 1, x1 = 0, y0 = 1, y1 = 0;
    uint32_t sv = 0, cnt = 0;
    if (valid) {
        sv = cv.x;
        if (unpack_window(cv.y, cv.x, wins, width, height, x0, x1, y0, y1)) cnt = block_count(x0, x1, y0, y1);
    }
    uint32_t incl = cnt;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, s);
        if (lane >= s) incl += y;
    }
    const uint32_t excl = incl - cnt;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (__reduce_max_sync(0xffffffffu, cnt) <= (uint32_t)SC_EMIT_LANE_MAX) {
        // small splats (the common case): each lane writes its own entries, row by row;
        // the warp's outputs are one contiguous range, so the stores stay within a few lines
        uint32_t o = obase + excl;
        if (cnt) {
            for (int by = y0 / 4; by <= y1 / 4; by++) {
                const int ry0 = max(y0 - 4 * by, 0), ry1 = min(y1 - 4 * by, 3);
                const uint32_t row = (uint32_t)(((by >> 2) * n_tx) * 8 + (by & 3) * 2);
                for (int bx = x0 / 8; bx <= x1 / 8; bx++) {
                    const int rx0 = max(x0 - 8 * bx, 0), rx1 = min(x1 - 8 * bx, 7);
                    const uint32_t id = row + (uint32_t)((bx >> 1) * 8 + (bx & 1));
                    ekey[o] = (id << kCodeBits) | (uint32_t)(rx0 | (rx1 << 3) | (ry0 << 6) | (ry1 << 8));
                    eval[o] = sv;
                    o++;
                }
            }
        }
        return total;
    }
    for (uint32_t o0 = 0; o0 < total; o0 += 32) {
        const uint32_t o = o0 + lane;
        int s = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const uint32_t e = __shfl_sync(0xffffffffu, excl, s + step);
            if (e <= o) s += step;
        }
        const uint32_t li = o - __shfl_sync(0xffffffffu, excl, s);
        const int X0 = __shfl_sync(0xffffffffu, x0, s), X1 = __shfl_sync(0xffffffffu, x1, s);
        const int Y0 = __shfl_sync(0xffffffffu, y0, s), Y1 = __shfl_sync(0xffffffffu, y1, s);
        const uint32_t v = __shfl_sync(0xffffffffu, sv, s);
        if (o < total) {
            const int w = X1 / 8 - X0 / 8 + 1;
            // li / w without an integer division (li < 2^24: one correction step is exact)
            int qy = (int)((float)li * __frcp_rn((float)w));
            int rx = (int)li - qy * w;
            if (rx < 0) { qy--; rx += w; } else if (rx >= w) { qy++; rx -= w; }
            const int bx = X0 / 8 + rx, by = Y0 / 4 + qy;
            const int rx0 = max(X0 - 8 * bx, 0), rx1 = min(X1 - 8 * bx, 7);
            const int ry0 = max(Y0 - 4 * by, 0), ry1 = min(Y1 - 4 * by, 3);
            const uint32_t id = (uint32_t)(((by >> 2) * n_tx + (bx >> 1)) * 8 + (by & 3) * 2 + (bx & 1));
            ekey[obase + o] = (id << kCodeBits) | (uint32_t)(rx0 | (rx1 << 3) | (ry0 << 6) | (ry1 << 8));
            eval[obase + o] = v;
        }
    }
    return total;
}

__global__ void __launch_bounds__(kEmitThreads) k_bentry_emit(const uint2 *__restrict__ pv, const sc_window *wins,
                                                              const uint32_t *warp_off, const unsigned long long *n_dev,
                                                              int64_t n_host, int width, int height, int n_tx,
                                                              uint32_t *ekey, uint32_t *eval,
                                                              const unsigned long long *e_total,
                                                              unsigned long long *e_eff, int64_t cap_e,
                                                              sc_frame_stats *stats)
{
    const int64_t n = dev_count(n_dev, n_host);
    const bool over = (int64_t)*e_total > cap_e;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *e_eff = over ? 0ull : *e_total;
        stats->block_entries = (int64_t)*e_total;
        if (over) atomicOr((unsigned long long *)&stats->overflow, 2ull);
    }
    if (over) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t ntiles = (n + kEmitTile - 1) / kEmitTile;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        // this warp's range of the tile and its output base (scan of the (tile, warp) totals)
        const int64_t wbase = t * kEmitTile + (int64_t)wid * kEmitPerWarp;
        uint32_t o = warp_off[t * (kEmitThreads / 32) + wid];
        // the next group's pairs are loaded while this group is emitted
        uint2 cv_next = wbase + lane < n ? __ldg(pv + wbase + lane) : make_uint2(0u, kWinEmpty);
        for (int r = 0; r < kEmitPerWarp / 32; r++) {
            const int64_t g0 = wbase + r * 32;
            if (g0 >= n) break;
            const int64_t k = g0 + lane;
            const uint2 cv = cv_next;
            if (r + 1 < kEmitPerWarp / 32 && k + 32 < n) cv_next = __ldg(pv + k + 32);
            o += emit_group(cv, k < n, o, wins, width, height, n_tx, ekey, eval, lane);
        }
    }
}

// boff[b] = first entry with block id >= b, for b in [0, n_blocks]: one thread
// per block, binary search over the sorted keys (~log2 E dependent loads whose
// upper levels are shared through L1/L2): ~32 B per probe instead of a full read
// of the E keys.
__global__ void k_block_offsets(const uint32_t *__restrict__ ekey, const unsigned long long *e_dev, int64_t cap_e,
                                int64_t n_blocks, uint32_t *boff)
{
    const int64_t E = std::min<int64_t>((int64_t)*e_dev, cap_e);
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= n_blocks;
         b += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = E;   // first i in [0, E] with block(i) >= b
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)(__ldg(ekey + mid) >> kCodeBits) < b) lo = mid + 1; else hi = mid;
        }
        boff[b] = (uint32_t)lo;
    }
}

static int grid_for(int64_t n, int threads)
{
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, (int64_t)sm_count_sort() * 16));
}

static int bits_for(int64_t n)
{
    int b = 0;
    while ((1ll << b) < n) b++;
    return b;
}

// n_dev: survivor count (device).  Input: ws.key_a (depth keys) + ws.pv_a
// ((survivor index, packed window) or (index, 0)) in survivor order.
// Always: depth sort + tie-fix (order = passed survivors by (depth, index)).
// blocks = true (frame path): block lists (entries_out = survivor per entry,
// keys_out = id << 10 | window, ws.boff).  blocks = false (stage-level API,
// parity with the reference): *order_out, tile entries and ws.tile_off,
// exactly bin_tiles' output.
cudaError_t launch_bin(const Ws &ws, const sc_scene &scene, const sc_survivor *surv, const unsigned long long *n_dev,
                       int64_t n_max, const sc_camera &cam, const sc_window *wins, sc_frame_stats *stats, bool blocks,
                       uint32_t **order_out, uint32_t **entries_out, uint32_t **keys_out, uint32_t *dbg_order,
                       cudaStream_t st)
{
    cudaError_t e;
    uint32_t *keys_s = nullptr;
    uint2 *pv_s = nullptr;
    if (!blocks)   // stage-level API: keys from the exact depth range (the frame path's come from the projection)
        SC_LAUNCH(k_depth_keys, grid_for(n_max, 256), 256, 0, st, ws.depth64, n_dev, n_max, ws.ctr, ws.key_a, ws.pv_a);
    // frame path: the projection wrote u32 windows at pv_a (the survivor index is the position)
    e = radix_sort<uint2>(ws.key_a, ws.pv_a, ws.key_b, ws.pv_b, n_dev, n_max, 0, 32, ws, &keys_s, &pv_s, st, false,
                          blocks);
    if (e != cudaSuccess) return e;
    const unsigned long long *p_dev = &ws.ctr->passed;   // passed splats lead the sorted order
    // the depth sort's other key / payload buffers are free now: the tie-run list and the
    // f64 depths of long tie runs go there
    uint32_t *key_free = keys_s == ws.key_a ? ws.key_b : ws.key_a;
    uint2 *pv_free = pv_s == ws.pv_a ? ws.pv_b : ws.pv_a;
    e = launch_tiefix(scene, surv, cam, keys_s, pv_s, blocks ? nullptr : ws.depth64, p_dev, n_max, key_free,
                      reinterpret_cast<double *>(pv_free), ws.ctr, stats, st);
    if (e != cudaSuccess) return e;
    if (dbg_order)   // debug copy-out of the (depth, index) order of the passed survivors
        SC_LAUNCH(k_extract_order, grid_for(n_max, 256), 256, 0, st, pv_s, p_dev, n_max, dbg_order);
    uint32_t *ek = nullptr, *ev = nullptr;
    if (blocks) {
        // per-(tile, warp) entry totals (free key buffer) -> output bases -> emission
        const int64_t etiles = std::max<int64_t>(1, (n_max + kEmitTile - 1) / kEmitTile);
        const int egrid = (int)std::min<int64_t>(etiles, (int64_t)sm_count_sort() * 8);
        uint32_t *wtot = key_free;   // etiles x 8 words <= max(capS, 4096)
        SC_LAUNCH(k_bentry_tiles, egrid, kEmitThreads, 0, st, pv_s, wins, p_dev, n_max, etiles, cam.width, cam.height,
                  wtot);
        e = scan_excl(wtot, wtot, nullptr, etiles * (kEmitThreads / 32), ws.scan_part, &ws.ctr->entries, nullptr, st);
        if (e != cudaSuccess) return e;
        SC_LAUNCH(k_bentry_emit, egrid, kEmitThreads, 0, st, pv_s, wins, wtot, p_dev, n_max, cam.width,
                  cam.height, ws.n_tx, ws.ekey_a, ws.eval_a, &ws.ctr->entries, &ws.ctr->entries_eff, ws.capE, stats);
        const int64_t n_blocks = 8 * ws.n_tiles;
        // last pass (block-id high byte ~ screen rows, which follow depth order): few distinct
        // digits per warp, match.any ranks them faster than the ballot match
        e = radix_sort<uint32_t>(ws.ekey_a, ws.eval_a, ws.ekey_b, ws.eval_b, &ws.ctr->entries_eff, ws.capE, kCodeBits,
                                 kCodeBits + bits_for(n_blocks), ws, &ek, &ev, st, true);
        if (e != cudaSuccess) return e;
        SC_LAUNCH(k_block_offsets, (int)((n_blocks + 1 + 255) / 256), 256, 0, st, ek, &ws.ctr->entries_eff, ws.capE,
                  n_blocks, ws.boff);
        if (order_out) *order_out = nullptr;
    } else {
        // free after the tie-fix: both key buffers and the other payload buffer; after the
        // order is extracted the sorted payload buffer holds the per-splat entry counts
        uint32_t *order = reinterpret_cast<uint32_t *>(pv_free);
        uint32_t *cnt = reinterpret_cast<uint32_t *>(pv_s);
        uint32_t *rlo = ws.key_a, *rhi = ws.key_b;
        SC_LAUNCH(k_extract_order, grid_for(n_max, 256), 256, 0, st, pv_s, p_dev, n_max, order);
        SC_LAUNCH(k_entry_count, grid_for(n_max, 256), 256, 0, st, order, ws.rect, p_dev, n_max, cnt, rlo, rhi);
        e = scan_excl(cnt, cnt, p_dev, n_max, ws.scan_part, &ws.ctr->entries, &stats->entries, st);
        if (e != cudaSuccess) return e;
        SC_LAUNCH(k_entry_emit, grid_for(n_max, 256), 256, 0, st, order, rlo, rhi, cnt, p_dev, n_max,
                  ws.n_tx_ref, ws.ekey_a, ws.eval_a, &ws.ctr->entries, &ws.ctr->entries_eff, ws.capE, stats);
        e = radix_sort<uint32_t>(ws.ekey_a, ws.eval_a, ws.ekey_b, ws.eval_b, &ws.ctr->entries_eff, ws.capE, 0,
                                 std::max(1, bits_for(ws.n_tiles_ref)), ws, &ek, &ev, st);
        if (e != cudaSuccess) return e;
        SC_LAUNCH(k_tile_offsets, grid_for(ws.capE + 1, 256), 256, 0, st, ek, &ws.ctr->entries_eff, ws.capE,
                  ws.n_tiles_ref, ws.tile_off);
        if (order_out) *order_out = order;
    }
    *entries_out = ev;
    if (keys_out) *keys_out = ek;
    return cudaGetLastError();
}

}  // namespace sc
