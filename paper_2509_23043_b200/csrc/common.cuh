// common.cuh -- device-side building blocks shared by every TAPT kernel.
//
// RNG: the reference's counter-based splitmix64 (proj/include/tapt/rng.hpp:21-32,58-65).
// Draw k (1-based) of a stream whose state is s0 is  mix_final(s0 + k*phi), so any
// draw can be computed from (stream state, counter) with no sequential state.
//
// Heat-bath decision (proj/src/mcmc.cpp:13-15,38):  uniform() < p  with
// uniform = (x>>11)*2^-53.  The host turns p into the integer threshold
// T = ceil(p*2^53), so the device decides with integers only:  (x>>11) < T.
// Fast path: only the high 32 bits of x are produced; they decide unless they
// equal the high word of T*2^11-1 (probability 2^-32), in which case the exact
// 64-bit test is redone.
#pragma once
#include <cstdint>

namespace tapt_dev {

constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kM1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kM2 = 0x94D049BB133111EBull;

__host__ __device__ __forceinline__ uint64_t mix_final(uint64_t z) {
    z = (z ^ (z >> 30)) * kM1;
    z = (z ^ (z >> 27)) * kM2;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t draw(uint64_t s0, uint64_t k) { return mix_final(s0 + k * kPhi); }

// High word of mix_final(z): the last xor-shift only needs z_hi for the top word.
__device__ __forceinline__ uint32_t mix_final_hi(uint64_t z) {
    z = (z ^ (z >> 30)) * kM1;
    z = (z ^ (z >> 27)) * kM2;
    const uint32_t h = static_cast<uint32_t>(z >> 32);
    return h ^ (h >> 31);
}

// High word of T*2^11 - 1 (T in [0, 2^53]); T = 0 maps to 0 and is resolved by the tie path.
__host__ __device__ __forceinline__ uint32_t thr_hi(uint64_t T) {
    return T == 0 ? 0u : static_cast<uint32_t>(((T << 11) - 1ull) >> 32);
}

// Runtime copies of 4 and 32: multiplying by an opaque register keeps a right shift of the
// high word on the FMA pipe (IMAD.HI) instead of the ALU pipe (SHF).
struct MixConsts {
    uint32_t k4, k32;
    uint32_t nib[8];  // nib[k] = 2^(34-4k) (k >= 1): hi(N * nib[k]) = N >> (4k-2)
    uint32_t sh[8];   // sh[m] = 2^(32-m) (m >= 1): hi(v * sh[m]) = v >> m
};

inline MixConsts make_mix_consts() {
    MixConsts c{4u, 32u, {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u}, {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u}};
    for (int k = 1; k < 8; ++k) c.nib[k] = 1u << (34 - 4 * k);
    for (int m = 1; m < 8; ++m) c.sh[m] = 1u << (32 - m);
    return c;
}

// High word of (z ^ z>>30) * M1 ^ ... * M2, i.e. mix_final(z) BEFORE its last xor-shift.
// Variant bits (instruction-mix choices, identical results; measured on B200 with
// tools/probe_variants.sh and tools/k1_variants.sh; default 6 = bits 2|4 since the index scratch
// (TAPT_K1_IDXS) took the threshold-index shift off the ALU pipe; before that 12 = bits 4|8):
//   V & 1: high-word right shifts as IMAD.HI by 4 / 32 (FMA pipe) instead of SHF (ALU pipe)  [slower]
//   V & 2: first 64-bit multiply as an explicit IMAD.WIDE + IMAD + IMAD chain (PTX)           [+3% with IDXS: 3 ops, not 4]
//   V & 4: tie band tracked as a running min (k1_lattice.cu)                                   [+4%]
//   V & 8: threshold-index shift as IMAD.HI on the FMA pipe (k1_lattice.cu)                    [+3%; unused with IDXS]
//   V & 64 / V & 128: the first / second high-word right shift as an immediate-form IMAD.HI (inline PTX)
//   V & 32: first 64-bit multiply as two IMAD + one IMAD.WIDE with a 64-bit addend (3 ops, not 4)
// The last multiply only needs its high word: IMAD.HI + IMAD + IMAD.
template <int V>
__device__ __forceinline__ uint32_t mix_pre_hi(uint32_t zl, uint32_t zh, const MixConsts& c) {
    constexpr uint32_t A_LO = (uint32_t)kM1, A_HI = (uint32_t)(kM1 >> 32);
    constexpr uint32_t B_LO = (uint32_t)kM2, B_HI = (uint32_t)(kM2 >> 32);
    uint32_t t;
    asm("shf.r.clamp.b32 %0, %1, %2, 30;" : "=r"(t) : "r"(zl), "r"(zh));
    zl ^= t;
    if constexpr ((V & 64) != 0) {  // immediate-form IMAD.HI (ptxas keeps an inline mul.hi by 4)
        uint32_t s;
        asm("mul.hi.u32 %0, %1, 4;" : "=r"(s) : "r"(zh));
        zh ^= s;
    } else {
        zh ^= (V & 1) ? __umulhi(zh, c.k4) : (zh >> 30);
    }
    if constexpr ((V & 32) != 0) {
        asm("{\n\t.reg .u32 x;\n\t.reg .u64 c, w;\n\t"
            "mul.lo.u32 x, %2, %5;\n\t"
            "mad.lo.u32 x, %3, %4, x;\n\t"
            "mov.b64 c, {0, x};\n\t"
            "mad.wide.u32 w, %2, %4, c;\n\t"
            "mov.b64 {%0, %1}, w;\n\t}"
            : "=r"(t), "=r"(zh)
            : "r"(zl), "r"(zh), "n"(A_LO), "n"(A_HI));
        zl = t;
    } else if constexpr ((V & 2) != 0) {
        asm("{\n\t.reg .u64 w;\n\t"
            "mul.wide.u32 w, %2, %4;\n\t"
            "mov.b64 {%0, %1}, w;\n\t"
            "mad.lo.u32 %1, %2, %5, %1;\n\t"
            "mad.lo.u32 %1, %3, %4, %1;\n\t}"
            : "=r"(t), "=r"(zh)
            : "r"(zl), "r"(zh), "n"(A_LO), "n"(A_HI));
        zl = t;
    } else {
        const uint64_t w = (uint64_t)zl * A_LO;
        zh = zh * A_LO + zl * A_HI + (uint32_t)(w >> 32);
        zl = (uint32_t)w;
    }
    asm("shf.r.clamp.b32 %0, %1, %2, 27;" : "=r"(t) : "r"(zl), "r"(zh));
    zl ^= t;
    if constexpr ((V & 128) != 0) {
        uint32_t s;
        asm("mul.hi.u32 %0, %1, 32;" : "=r"(s) : "r"(zh));
        zh ^= s;
    } else {
        zh ^= (V & 1) ? __umulhi(zh, c.k32) : (zh >> 27);
    }
    return __umulhi(zl, B_LO) + zh * B_LO + zl * B_HI;
}

// K independent chains of mix_pre_hi, written stage by stage so the instruction stream
// interleaves the chains (ptxas otherwise tends to emit one dependent chain at a time).
template <int K>
__device__ __forceinline__ void mix_pre_hi_k(const uint32_t (&zl0)[K], const uint32_t (&zh0)[K], uint32_t (&out)[K]) {
    constexpr uint32_t A_LO = (uint32_t)kM1, A_HI = (uint32_t)(kM1 >> 32);
    constexpr uint32_t B_LO = (uint32_t)kM2, B_HI = (uint32_t)(kM2 >> 32);
    uint32_t zl[K], zh[K], t[K];
#pragma unroll
    for (int c = 0; c < K; ++c) asm("shf.r.clamp.b32 %0, %1, %2, 30;" : "=r"(t[c]) : "r"(zl0[c]), "r"(zh0[c]));
#pragma unroll
    for (int c = 0; c < K; ++c) {
        zl[c] = zl0[c] ^ t[c];
        zh[c] = zh0[c] ^ (zh0[c] >> 30);
    }
#pragma unroll
    for (int c = 0; c < K; ++c) {
        const uint64_t w = (uint64_t)zl[c] * A_LO;
        zh[c] = zh[c] * A_LO + zl[c] * A_HI + (uint32_t)(w >> 32);
        zl[c] = (uint32_t)w;
    }
#pragma unroll
    for (int c = 0; c < K; ++c) asm("shf.r.clamp.b32 %0, %1, %2, 27;" : "=r"(t[c]) : "r"(zl[c]), "r"(zh[c]));
#pragma unroll
    for (int c = 0; c < K; ++c) {
        zl[c] ^= t[c];
        zh[c] ^= zh[c] >> 27;
    }
#pragma unroll
    for (int c = 0; c < K; ++c) out[c] = __umulhi(zl[c], B_LO) + zh[c] * B_LO + zl[c] * B_HI;
}

// Heat-bath decision on h = mix_pre_hi(z) against U = thr_hi(T):  the final xor-shift
// of mix_final only flips bit 0 of the high word, so whenever |h - U| >= 2 the decision
// equals (h < U).  Shifts NOT(up) into w (w = 2w + [h >= U]) via the carry of h - U and
// returns h - U, whose value in {-1, 0, 1} flags the rare case that needs the exact test.
__device__ __forceinline__ uint32_t decide_acc(uint32_t h, uint32_t U, uint32_t& w) {
    uint32_t d;
    asm("sub.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %1, %1;" : "=r"(d), "+r"(w) : "r"(h), "r"(U));
    return d;
}

// Exact decision on a full draw.
__host__ __device__ __forceinline__ bool below(uint64_t x, uint64_t T) { return (x >> 11) < T; }

// Metropolis decision with a tabulated threshold over integer energy differences
// (swap Eq. 1 / proposal Eq. 2):  accept iff uniform < exp(c * dE).
//   dE >= 0          -> always (exp >= 1 > uniform)
//   0 < -dE < K      -> tab[-dE]
//   K <= -dE <= kz   -> threshold 1 (exp(c*dE)*2^53 in (0,1])
//   -dE > kz         -> threshold 0 (exp underflows to 0)
struct MetroTable {
    const uint64_t* tab;  // per row: K entries, tab[0] = 2^53
    const uint32_t* off;  // row offset into tab
    const uint32_t* K;    // row length
    const int64_t* kz;    // largest -dE with nonzero probability (-1: none beyond table)
    const uint8_t* always;  // row accepts everything (c == 0)
    const double* c;        // row coefficient: accept iff uniform < exp(-c k), k = -dE
};

__device__ __forceinline__ bool metro_accept(const MetroTable& t, int row, int64_t dE, uint64_t x) {
    if (dE >= 0 || t.always[row]) return true;
    const int64_t k = -dE;
    uint64_t T;
    if (k < static_cast<int64_t>(t.K[row]))
        T = t.tab[t.off[row] + k];
    else
        T = (k <= t.kz[row]) ? 1ull : 0ull;
    return below(x, T);
}

// ------------------------------------------------------- bulk copies (TMA) --
// 1D bulk copy global -> shared through the copy engine, completed on an mbarrier: one thread
// arms the barrier with the byte count and issues the copies; every thread waits on the phase.

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// bytes: a multiple of 16; both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Wait for the barrier phase `parity`; traps after ~2^31 polls (a copy that never lands must not
// hang the GPU: the launch fails and the host raises CudaError).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
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

// Order this thread's earlier generic-proxy shared-memory accesses before later async-proxy ones.
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------ bit slicing --

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (c & (a | b)); }

// Add a 3-plane sliced value (u0 + 2u1 + 4u2) into a K-plane sliced counter.
template <int K>
__device__ __forceinline__ void sliced_add3(uint32_t (&C)[K], uint32_t u0, uint32_t u1, uint32_t u2) {
    uint32_t carry = C[0] & u0;
    C[0] ^= u0;
    uint32_t s = C[1] ^ u1 ^ carry;
    carry = maj3(C[1], u1, carry);
    C[1] = s;
    s = C[2] ^ u2 ^ carry;
    carry = maj3(C[2], u2, carry);
    C[2] = s;
#pragma unroll
    for (int k = 3; k < K; ++k) {
        const uint32_t c = C[k] & carry;
        C[k] ^= carry;
        carry = c;
    }
}

// Add a 1-plane value into a K-plane sliced counter.
template <int K>
__device__ __forceinline__ void sliced_add1(uint32_t (&C)[K], uint32_t u) {
    uint32_t carry = u;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint32_t c = C[k] & carry;
        C[k] ^= carry;
        carry = c;
    }
}

// 32x32 bit transpose across a warp: afterwards lane b holds, in bit l, bit b of
// lane l's input word.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t w) {
    const int lane = threadIdx.x & 31;
    const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        const int j = 16 >> s;
        const uint32_t m = masks[s];
        const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, w, j);
        w = (lane & j) ? ((w & ~m) | ((o & ~m) >> j)) : ((w & m) | ((o & m) << j));
    }
    return w;
}

// Per-replica totals of a K-plane sliced counter summed over the warp: lane b
// returns sum over lanes of the value held for replica (bit) b.
// Planes that are zero in every lane (high planes of small per-thread counts) are skipped after
// one warp vote.
template <int K>
__device__ __forceinline__ uint32_t warp_sliced_total(const uint32_t (&C)[K]) {
    uint32_t tot = 0;
#pragma unroll
    for (int k = 0; k < K; ++k)
        if (__any_sync(0xFFFFFFFFu, C[k] != 0u)) tot += static_cast<uint32_t>(__popc(warp_transpose32(C[k]))) << k;
    return tot;
}

// Lane b receives sum over lanes of v[b] (butterfly reduce-scatter, 31 shuffles).
__device__ __forceinline__ int32_t warp_reduce_scatter32(int32_t (&v)[32]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        const int j = 16 >> s;  // partner distance; keep half of the entries each stage
#pragma unroll
        for (int e = 0; e < j; ++e) {
            // entries e and e+j: lanes with bit j clear keep e, others keep e+j
            const bool hi = (lane & j) != 0;
            const int32_t send = hi ? v[e] : v[e + j];
            const int32_t recv = __shfl_xor_sync(0xFFFFFFFFu, send, j);
            if (hi)
                v[e + j] += recv;
            else
                v[e] += recv;
            // compact: the kept entry goes to position e
            v[e] = hi ? v[e + j] : v[e];
        }
    }
    return v[0];
}

}  // namespace tapt_dev
