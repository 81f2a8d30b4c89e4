// tcgen05 / TMEM / mbarrier PTX wrappers (sm_100a) and the fused 16->32->32->1
// visibility-MLP tile used by the cull kernel and the batched forward.
#pragma once
#include "common.cuh"

namespace sc {

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_LOOP:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra WAIT_DONE;\n\t"
        "bra WAIT_LOOP;\n\t"
        "WAIT_DONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// whole warp: allocate ncols TMEM columns, base address written to *dst (smem)
__device__ __forceinline__ void tmem_alloc(uint32_t *dst, uint32_t ncols)
{
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols)
{
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// Shared-memory matrix descriptor, K-major, no swizzle ("interleaved" core
// matrices of 8 rows x 16 bytes).  lbo = byte stride between core matrices
// along K, sbo = byte stride between 8-row groups along M/N.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;   // descriptor version 1 (sm_100)
    return d;                 // base offset 0, layout type 0 = SWIZZLE_NONE
}

// Instruction descriptor, kind::f16: A = B = fp16, D = f32, both K-major.
template <int M, int N>
__host__ __device__ constexpr uint32_t idesc_f16()
{
    return (1u << 4)                       // D format f32
           | (0u << 7) | (0u << 10)        // A, B = f16
           | ((uint32_t)(N >> 3) << 17)    // N / 8
           | ((uint32_t)(M >> 4) << 24);   // M / 16
}

__device__ __forceinline__ void mma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t *bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// Warp-collective: lane i reads TMEM lane (taddr.lane + i), 32 consecutive
// 32-bit columns starting at taddr.col.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float *v)
{
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}

// 16 consecutive columns (fewer live registers than x32: the cull kernel runs
// 12 CTAs per SM)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *v)
{
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}

// ---------------------------------------------------------------------------
// Fused MLP tile: 128 rows x 16 fp16 inputs -> logit per row.
//   layer 1: D1[128x32] = A1[128x16] . W1^T        (1 MMA, K = 16)   TMEM cols [0, 32)
//   epilogue: +b1, ReLU, fp16 -> A2 (smem)
//   layer 2: D2[128x32] = A2[128x32] . W2^T        (2 MMAs, K = 16 each) TMEM cols [32, 64)
//   epilogue: +b2, ReLU, dot w3 + b3 on CUDA cores (N = 1 is below the MMA minimum)
// smem operands in the no-swizzle K-major canonical layout:
//   byte(r, k) = (r / 8) * (KC * 128) + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2
// ---------------------------------------------------------------------------
struct __align__(128) MlpSmem {
    // a1 (layer-1 input) and a2 (layer-2 input) share storage: MMA 1 has completed
    // before a2 is written, MMA 2 before the next tile's a1 is
    union {
        __align__(128) __half a1[128 * 16];
        __align__(128) __half a2[128 * 32];
    };
    __align__(128) __half w1[32 * 16];
    __align__(128) __half w2[32 * 32];
    // biases ride the MMAs: D += ONES . BIAS^T with ONES rows (1, 1, 0, ..) (one 8-row core
    // matrix pair read by every row group: SBO = 0) and BIAS rows (b_hi, b_lo, 0, ..), b_hi
    // = fp16(b), b_lo = fp16(b - b_hi): the f32 bias to ~2^-22 relative
    __align__(128) __half ones[8 * 16];
    __align__(128) __half bias1[32 * 16];
    __align__(128) __half bias2[32 * 16];
    __align__(16) float w3[32];
    float b3;
    uint32_t tmem_base;
    __align__(8) uint64_t bar;
};

constexpr uint32_t kTmemCols = 32;   // D1, then D2 in the same columns (D1 is read out before MMA 2)

__device__ __forceinline__ int core_off(int r, int k, int kc_total)
{
    return (r >> 3) * (kc_total * 64) + (k >> 3) * 64 + (r & 7) * 8 + (k & 7);   // in halves
}

// All threads of the CTA: copy one model's weights into the smem layout.
__device__ __forceinline__ void mlp_load_weights(MlpSmem &sm, const sc_vis_weights *w, int tid, int nthreads)
{
    const __half *w1 = reinterpret_cast<const __half *>(w->w1);
    const __half *w2 = reinterpret_cast<const __half *>(w->w2);
    for (int i = tid; i < 32 * 16; i += nthreads) sm.w1[core_off(i >> 4, i & 15, 2)] = w1[i];
    for (int i = tid; i < 32 * 32; i += nthreads) sm.w2[core_off(i >> 5, i & 31, 4)] = w2[i];
    for (int i = tid; i < 32 * 16; i += nthreads) {
        const int n = i >> 4, k = i & 15;
        __half v1 = __float2half_rn(0.0f), v2 = v1;
        if (k < 2) {
            const float b1 = w->b1[n], b2 = w->b2[n];
            const __half h1 = __float2half_rn(b1), h2 = __float2half_rn(b2);
            v1 = k == 0 ? h1 : __float2half_rn(b1 - __half2float(h1));
            v2 = k == 0 ? h2 : __float2half_rn(b2 - __half2float(h2));
        }
        sm.bias1[core_off(n, k, 2)] = v1;
        sm.bias2[core_off(n, k, 2)] = v2;
    }
    for (int i = tid; i < 32; i += nthreads) sm.w3[i] = w->w3[i];
    if (tid == 0) sm.b3 = w->b3;
}

// Thread `row` stores its 16 fp16 inputs (two 16-byte core-matrix rows).
__device__ __forceinline__ void mlp_store_row(MlpSmem &sm, int row, uint4 lo, uint4 hi)
{
    uint4 *base = reinterpret_cast<uint4 *>(sm.a1 + (row >> 3) * 128 + (row & 7) * 8);
    base[0] = lo;        // k 0..7
    base[8] = hi;        // k 8..15  (+128 bytes)
}

// (a, b) -> fp16x2 {lo = relu(a), hi = relu(b)}, round to nearest (cvt.rn.relu.f16x2.f32)
__device__ __forceinline__ uint32_t pack_h2_relu(float a, float b)
{
    uint32_t r;
    asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
    return r;
}

__device__ __forceinline__ uint32_t pack_h2(float a, float b)
{
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}

#ifndef SC_MLP_FFMA2
#define SC_MLP_FFMA2 1
#endif
// packed f32 pair in one 64-bit register (f32x2 arithmetic, sm_100)
__device__ __forceinline__ uint64_t pack_f2(float a, float b)
{
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void unpack_f2(uint64_t r, float &a, float &b)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c)
{
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

// Runs the three layers for the tile whose inputs are in sm.a1 if any thread
// passes `pred` (the first barrier doubles as that vote); returns whether it
// ran, the logit of this thread's row in *logit.  Must be called by all 128
// threads.
__device__ __forceinline__ bool mlp_tile(MlpSmem &sm, int tid, uint32_t &phase, bool pred, float *logit_out)
{
    constexpr uint32_t kIdesc = idesc_f16<128, 32>();
    fence_async_smem();
    tc_fence_before();
    if (!__syncthreads_or(pred)) return false;
    if (tid == 0) {
        tc_fence_after();
        mma_f16_ss(sm.tmem_base, smem_desc(smem_u32(sm.a1), 128, 256), smem_desc(smem_u32(sm.w1), 128, 256),
                   kIdesc, 0);
        mma_f16_ss(sm.tmem_base, smem_desc(smem_u32(sm.ones), 128, 0), smem_desc(smem_u32(sm.bias1), 128, 256),
                   kIdesc, 1);
        mma_commit(&sm.bar);
    }
    mbar_wait(&sm.bar, phase);
    phase ^= 1u;
    tc_fence_after();
    const uint32_t lane_sel = (uint32_t)(tid & ~31) << 16;
    float v[16];
    {
        uint4 *dst = reinterpret_cast<uint4 *>(sm.a2 + (tid >> 3) * 256 + (tid & 7) * 8);
#pragma unroll
        for (int half = 0; half < 2; half++) {
            tmem_ld16(sm.tmem_base + lane_sel + 16 * half, v);
#pragma unroll
            for (int kc = 0; kc < 2; kc++) {
                // relu(acc) rounded to fp16 (the bias is in acc): the relu rides the f32 -> f16x2 conversion
                const float *u = v + kc * 8;
                dst[(2 * half + kc) * 8] = make_uint4(pack_h2_relu(u[0], u[1]), pack_h2_relu(u[2], u[3]),
                                                      pack_h2_relu(u[4], u[5]), pack_h2_relu(u[6], u[7]));
            }
        }
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
        tc_fence_after();
        const uint32_t a2 = smem_u32(sm.a2), w2 = smem_u32(sm.w2);
        mma_f16_ss(sm.tmem_base, smem_desc(a2, 128, 512), smem_desc(w2, 128, 512), kIdesc, 0);
        mma_f16_ss(sm.tmem_base, smem_desc(a2 + 256, 128, 512), smem_desc(w2 + 256, 128, 512), kIdesc, 1);
        mma_f16_ss(sm.tmem_base, smem_desc(smem_u32(sm.ones), 128, 0), smem_desc(smem_u32(sm.bias2), 128, 256),
                   kIdesc, 1);
        mma_commit(&sm.bar);
    }
    mbar_wait(&sm.bar, phase);
    phase ^= 1u;
    tc_fence_after();
#if SC_MLP_FFMA2
    // layer 3 as two interleaved partial sums on packed f32x2 FMAs (FFMA2: half the FMA issue)
    uint64_t acc = pack_f2(sm.b3, 0.0f);
#pragma unroll
    for (int half = 0; half < 2; half++) {
        tmem_ld16(sm.tmem_base + lane_sel + 16 * half, v);
#pragma unroll
        for (int n4 = 0; n4 < 4; n4++) {
            const float4 w = reinterpret_cast<const float4 *>(sm.w3)[4 * half + n4];
            acc = ffma2(pack_f2(fmaxf(v[4 * n4], 0.0f), fmaxf(v[4 * n4 + 1], 0.0f)), pack_f2(w.x, w.y), acc);
            acc = ffma2(pack_f2(fmaxf(v[4 * n4 + 2], 0.0f), fmaxf(v[4 * n4 + 3], 0.0f)), pack_f2(w.z, w.w), acc);
        }
    }
    float l0, l1;
    unpack_f2(acc, l0, l1);
    const float logit = l0 + l1;
#else
    float logit = sm.b3;
#pragma unroll
    for (int half = 0; half < 2; half++) {
        tmem_ld16(sm.tmem_base + lane_sel + 16 * half, v);
#pragma unroll
        for (int n4 = 0; n4 < 4; n4++) {
            const float4 w = reinterpret_cast<const float4 *>(sm.w3)[4 * half + n4];
            logit += fmaxf(v[4 * n4], 0.0f) * w.x;
            logit += fmaxf(v[4 * n4 + 1], 0.0f) * w.y;
            logit += fmaxf(v[4 * n4 + 2], 0.0f) * w.z;
            logit += fmaxf(v[4 * n4 + 3], 0.0f) * w.w;
        }
    }
#endif
    tc_fence_before();
    *logit_out = logit;
    return true;
}

// CTA prologue / epilogue for kernels that use mlp_tile (blockDim = 128).
__device__ __forceinline__ void mlp_setup(MlpSmem &sm, int tid)
{
    if (tid < 32) tmem_alloc(&sm.tmem_base, kTmemCols);
    for (int i = tid; i < 8 * 16; i += blockDim.x) sm.ones[i] = __float2half_rn((i & 7) < 2 && i < 64 ? 1.0f : 0.0f);
    if (tid == 0) {
        mbar_init(&sm.bar, 1);
        mbar_fence_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
}

__device__ __forceinline__ void mlp_teardown(MlpSmem &sm, int tid)
{
    tc_fence_before();
    __syncthreads();
    if (tid < 32) {
        tc_fence_after();
        tmem_dealloc(sm.tmem_base, kTmemCols);
    }
}

}  // namespace sc
