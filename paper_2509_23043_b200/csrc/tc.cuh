// tc.cuh -- the tcgen05 building blocks of the IsingFormer's dense products (sm_100a).
//
// One CTA computes D[128][N] = A[128][K] . B[N][K]^T on the 5th-generation tensor cores:
//   * operands are bf16 in shared memory in the K-major, no-swizzle canonical layout: 8x8-element
//     "core matrices" of 128 contiguous bytes (row r at +16 r); core matrices adjacent along K are
//     LBO = 128 B apart, those adjacent along M / N are SBO = K/8 * 128 B apart;
//   * one elected thread issues tcgen05.mma.cta_group::1.kind::f16 (M = 128, N <= 256, K = 16
//     per instruction) with the fp32 accumulator in TMEM (lane = row, column = output), and
//     tcgen05.commit arrives on an mbarrier when the MMAs retire;
//   * the epilogue warps read their rows back with tcgen05.ld.32x32b (warp w: lanes 32 (w % 4) ..).
// Near-fp32 accuracy from bf16 tensor cores ("bf16x3"): every fp32 operand x is split into
// x_hi = bf16(x) and x_lo = bf16(x - x_hi), and D = A_hi B_hi + A_hi B_lo + A_lo B_hi.  The split
// residuals and the dropped A_lo B_lo term leave ~2^-16 (1.5e-5) relative error per product: logits
// agree with the fp32 CUDA-core engine to ~1e-5 and with the fp64 oracle within the same 2e-4 the
// fp32 engine is held to (plain bf16 would be ~4e-3 per product).
#pragma once
#include <cuda_bf16.h>

#include <cstdint>

namespace tapt_tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Byte offset of element (row, k) in the canonical K-major no-swizzle layout with K columns.
__host__ __device__ constexpr uint32_t kmajor_off(int row, int k, int K) {
    return (uint32_t)((row >> 3) * (K / 8) * 128 + (k >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2);
}

// Shared-memory matrix descriptor (sm100 version 1, SWIZZLE_NONE, base offset 0).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// Instruction descriptor, kind::f16: bf16 A and B (K-major), fp32 D, M x N.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// generic-proxy shared-memory writes (operand tiles) become visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void bar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Wait for phase `parity`; traps after ~2^31 polls (an MMA that never retires must not hang the GPU).
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
    for (uint32_t k = 0;; ++k) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if (k > (1u << 31)) __trap();
    }
}

// TMEM allocation by one full warp; the base address lands in *slot (shared memory).
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free(uint32_t base, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(ncols) : "memory");
}

// 16 consecutive fp32 accumulator columns of this thread's row (lane = row within the warp's 32).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    __syncwarp();  // .sync.aligned: the whole warp executes it together
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// x = hi + lo with hi = bf16(x), lo = bf16(x - hi)
__device__ __forceinline__ void split_bf16(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
    hi = __float2bfloat16_rn(x);
    lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

// Store 8 consecutive k of one row (a 16-byte core-matrix row) of the hi and lo operand tiles.
__device__ __forceinline__ void store_row8(uint8_t* hi_tile, uint8_t* lo_tile, int row, int k0, int K,
                                           const float (&x)[8]) {
    __nv_bfloat16 h[8], l[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) split_bf16(x[i], h[i], l[i]);
    const uint32_t off = kmajor_off(row, k0, K);
    *reinterpret_cast<uint4*>(hi_tile + off) = *reinterpret_cast<const uint4*>(h);
    *reinterpret_cast<uint4*>(lo_tile + off) = *reinterpret_cast<const uint4*>(l);
}

// Issue D[128][N] (+)= A . B^T as bf16x3 from one thread: A tiles [128][K], B tiles [N][K].
template <int N, int K>
__device__ __forceinline__ void mma_x3(uint32_t tmem_d, const uint8_t* a_hi, const uint8_t* a_lo, const uint8_t* b_hi,
                                       const uint8_t* b_lo) {
    constexpr uint32_t LBO = 128, SBO = (K / 8) * 128;
    constexpr uint32_t idesc = idesc_bf16(128, N);
    const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
#pragma unroll
    for (int kk = 0; kk < K / 16; ++kk) {
        const uint32_t o = kk * 256;  // two core matrices along K per instruction
        mma_bf16(tmem_d, sdesc(ah + o, LBO, SBO), sdesc(bh + o, LBO, SBO), idesc, kk > 0 ? 1u : 0u);
        mma_bf16(tmem_d, sdesc(ah + o, LBO, SBO), sdesc(bl + o, LBO, SBO), idesc, 1u);
        mma_bf16(tmem_d, sdesc(al + o, LBO, SBO), sdesc(bh + o, LBO, SBO), idesc, 1u);
    }
}

}  // namespace tapt_tc
