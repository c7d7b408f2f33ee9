// k1_lattice.cu -- K1: fused parallel-tempering kernel for periodic 2D/3D lattices
// with +-J0 nearest-neighbour bonds (BASELINE configs 1, 2, 3, 5).
//
// One CTA owns one group of W <= 32 replicas of one instance; its spins live in
// shared memory for the whole launch in multi-replica coding (word = site, bit =
// replica).  An instance with R > 32 slots is a thread-block cluster of R/32 CTAs
// that exchange per-replica energies through DSMEM once per sweep, so the
// replica-exchange pass runs in-kernel with no host round trip.
//
// Per sweep: colour 0 then colour 1 of the checkerboard.  For a site word, the
// 2*dim neighbour words give, bit-sliced over the 32 replicas, the count q of
// neighbours with J*s_j = +1 (so l = J0*(2q - z)); q is spread into 4-bit
// nibbles so each replica's threshold-table index is one shift+mask.  Every
// replica then needs one counter-addressed splitmix64 draw:
//     draw index  k = draw_base + t*n + i + 1     (site rank i: no clamps)
// which is the reference's per-site stream position (mcmc.cpp:30-45 advances the
// stream once per free site in ascending order), so the result is bit-exact with
// the colour-order restatement in oracle/tapt_oracle.c.
// Energies are recomputed exactly during the colour-1 half: in a bipartite
// lattice every bond has exactly one colour-1 end, so summing unsatisfied bonds
// of colour-1 sites counts each bond once:  E = J0 * (2*U - n*dim).
#include <cuda_runtime.h>

#include "pt_common.cuh"

namespace tapt_dev {

template <int DIM>
__device__ __forceinline__ int colour_site(int j, int c, const LatDims& d, int& x, int& y, int& z) {
    // j's low bit picks one of two consecutive rows (opposite colour parity), so a
    // warp's loads alternate between even and odd words: no shared-memory bank
    // conflicts for rows of >= 32 sites.
    const int rb = j & 1, q = j >> 1;
    const int m = q & ((1 << d.log2hx) - 1);
    const int row = ((q >> d.log2hx) << 1) | rb;
    y = row & ((1 << d.log2Ly) - 1);
    z = (DIM == 3) ? (row >> d.log2Ly) : 0;
    x = (m << 1) | ((y + z + c) & 1);
    return x + (row << d.log2Lx);
}

// Bit-sliced count of neighbours with J*s_j = +1: returns planes q0 (1), q1 (2), q2 (4).
template <int DIM, bool DIS, int PACK = 1>
__device__ __forceinline__ void k1_stencil(const uint32_t* __restrict__ w, const uint8_t* __restrict__ bonds, int i,
                                           int x, int y, int z, const LatDims& d, uint32_t& q0, uint32_t& q1,
                                           uint32_t& q2, const uint32_t* bm = nullptr, int nfold = 0) {
    const int Lx = 1 << d.log2Lx, Ly = 1 << d.log2Ly;
#if TAPT_K1_IDX2
    // periodic neighbours by masked add on the packed index (power-of-two extents)
    // (PACK > 1: the slowest dimension is folded to nfold = n/PACK sites, so its mask shrinks)
    const int mx = Lx - 1;
    const int my = (PACK > 1 && DIM == 2) ? ((nfold - 1) & ~(Lx - 1)) : ((Ly - 1) << d.log2Lx);
#if TAPT_K1_XSEL
    // bit-field select (mask ? stepped : i) as one LOP3 each (the compiler's form shares i & ~mx and
    // spends an AND and an OR per neighbour)
    uint32_t ixp, ixm;
    asm("lop3.b32 %0, %1, %2, %3, 0xB8;" : "=r"(ixp) : "r"(i), "r"(mx), "r"(i + 1));
    asm("lop3.b32 %0, %1, %2, %3, 0xB8;" : "=r"(ixm) : "r"(i), "r"(mx), "r"(i - 1));
    uint32_t p0 = w[ixp];
    uint32_t p1 = w[ixm];
#else
    uint32_t p0 = w[(i & ~mx) | ((i + 1) & mx)];
    uint32_t p1 = w[(i & ~mx) | ((i - 1) & mx)];
#endif
    uint32_t p2 = w[(i & ~my) | ((i + Lx) & my)];
    uint32_t p3 = w[(i & ~my) | ((i - Lx) & my)];
    uint32_t p4 = 0, p5 = 0;
    if constexpr (DIM == 3) {
        const int P = Lx * Ly;
        const int mz = PACK > 1 ? ((nfold - 1) & ~(P - 1)) : ((Ly - 1) << (d.log2Lx + d.log2Ly));
        p4 = w[(i & ~mz) | ((i + P) & mz)];
        p5 = w[(i & ~mz) | ((i - P) & mz)];
    }
    (void)x;
    (void)y;
    (void)z;
#else
    static_assert(PACK == 1, "packed narrow groups use the masked-add neighbour indices");
    const int rowb = i - x;
    uint32_t p0 = w[rowb + ((x + 1) & (Lx - 1))];
    uint32_t p1 = w[rowb + ((x - 1) & (Lx - 1))];
    const int ip = i + ((y == Ly - 1) ? -(Ly - 1) * Lx : Lx);
    const int im = i + ((y == 0) ? (Ly - 1) * Lx : -Lx);
    uint32_t p2 = w[ip], p3 = w[im];
    uint32_t p4 = 0, p5 = 0;
    if constexpr (DIM == 3) {
        const int P = Lx * Ly;
        const int Lz = Ly;
        const int kp = i + ((z == Lz - 1) ? -(Lz - 1) * P : P);
        const int km = i + ((z == 0) ? (Lz - 1) * P : -P);
        p4 = w[kp];
        p5 = w[km];
    }
#endif
    if constexpr (PACK > 1) {
        // Packed narrow groups: the word holds PACK sites i + k*n/PACK (k-th field of 32/PACK replica
        // bits), i.e. the lattice is folded PACK times along its slowest dimension.  The masked adds
        // above wrapped inside the folded lattice; a neighbour across the fold seam is the next /
        // previous field of the wrapped word, i.e. the word rotated by one field.
        constexpr int FW = 32 / PACK;
        const int S = DIM == 3 ? (Lx * Ly) : Lx;  // stride of the folded dimension
        const bool seam_p = (i + S) >= nfold, seam_m = i < S;
        uint32_t& pp = DIM == 3 ? p4 : p2;
        uint32_t& pm = DIM == 3 ? p5 : p3;
        if (seam_p) pp = __funnelshift_r(pp, pp, FW);  // field k takes field k+1 of the wrapped word
        if (seam_m) pm = __funnelshift_l(pm, pm, FW);  // field k takes field k-1
    }
    if constexpr (DIS && PACK > 1) {
        // one bond byte per folded site: direction d's sign mask is field k all-ones iff byte k has bit d
        constexpr int FW = 32 / PACK;
        constexpr uint32_t F1 = FW == 16 ? 0xFFFFu : 0xFFu;
        uint32_t m[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < PACK; ++k) {
            const uint32_t bb = bonds[i + k * nfold];
#pragma unroll
            for (int dd = 0; dd < 2 * DIM; ++dd) m[dd] |= ((bb >> dd) & 1u) * (F1 << (k * FW));
        }
        p0 ^= m[0];
        p1 ^= m[1];
        p2 ^= m[2];
        p3 ^= m[3];
        if constexpr (DIM == 3) {
            p4 ^= m[4];
            p5 ^= m[5];
        }
    } else if constexpr (DIS) {
        const uint32_t bb = bonds[i];  // bit d set: bond in direction d has J = -J0
#if TAPT_K1_BLUT
        if (bm) {  // the six sign masks of this byte from a 64-row shared-memory table (2 loads, no shifts)
            const uint4 m0 = *reinterpret_cast<const uint4*>(bm + 8 * bb);
            const uint2 m1 = *reinterpret_cast<const uint2*>(bm + 8 * bb + 4);
            p0 ^= m0.x;
            p1 ^= m0.y;
            p2 ^= m0.z;
            p3 ^= m0.w;
            if constexpr (DIM == 3) {
                p4 ^= m1.x;
                p5 ^= m1.y;
            }
        } else
#endif
        {
        p0 ^= 0u - (bb & 1u);
        p1 ^= 0u - ((bb >> 1) & 1u);
        p2 ^= 0u - ((bb >> 2) & 1u);
        p3 ^= 0u - ((bb >> 3) & 1u);
        if constexpr (DIM == 3) {
            p4 ^= 0u - ((bb >> 4) & 1u);
            p5 ^= 0u - ((bb >> 5) & 1u);
        }
        }
    }
    if constexpr (DIM == 3) {
        const uint32_t sa = p0 ^ p1 ^ p2, ca = maj3(p0, p1, p2);
        const uint32_t sb = p3 ^ p4 ^ p5, cb = maj3(p3, p4, p5);
        q0 = sa ^ sb;
        const uint32_t c0 = sa & sb;
        q1 = ca ^ cb ^ c0;
        q2 = maj3(ca, cb, c0);
    } else {
        const uint32_t sa = p0 ^ p1 ^ p2, ca = maj3(p0, p1, p2);
        q0 = sa ^ p3;
        const uint32_t c0 = sa & p3;
        q1 = ca ^ c0;
        q2 = ca & c0;
    }
}

// Planes of the number of unsatisfied bonds at a site whose new word is s:
// bond d is satisfied iff s == p_d, so #unsat = s ? z - q : q.
template <int DIM>
__device__ __forceinline__ void unsat_planes(uint32_t s, uint32_t q0, uint32_t q1, uint32_t q2, uint32_t& u0,
                                             uint32_t& u1, uint32_t& u2) {
    uint32_t r0, r1, r2;  // z - q
    if constexpr (DIM == 3) {
        r0 = q0;
        r1 = ~q1 ^ q0;
        r2 = ~q2 ^ (q1 & q0);
    } else {
        r0 = q0;
        r1 = q1 ^ q0;
        r2 = ~(q0 | q1 | q2);
    }
    u0 = (s & r0) | (~s & q0);
    u1 = (s & r1) | (~s & q1);
    u2 = (s & r2) | (~s & q2);
}

// Nibble spread: bits 0..2 of nibble k of N[m] = q of replica 4k+m (bit 3 is don't-care:
// every reader masks with 7).  Pairs (q0,q1) of even / odd replicas are formed first.
__device__ __forceinline__ void nibbles(uint32_t q0, uint32_t q1, uint32_t q2, uint32_t (&N)[4]) {
#if TAPT_K1_NIB2
    const uint32_t e01 = (q0 & 0x55555555u) | ((q1 << 1) & 0xAAAAAAAAu);
    const uint32_t o01 = ((q0 >> 1) & 0x55555555u) | (q1 & 0xAAAAAAAAu);
    constexpr uint32_t M = 0x33333333u;
    N[0] = (e01 & M) | ((q2 << 2) & ~M);
    N[1] = (o01 & M) | ((q2 << 1) & ~M);
    N[2] = ((e01 >> 2) & M) | (q2 & ~M);
    N[3] = ((o01 >> 2) & M) | ((q2 >> 1) & ~M);
#else
    constexpr uint32_t K1 = 0x11111111u;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const uint32_t a = (q0 >> m) & K1;
        const uint32_t b = (m >= 1 ? (q1 >> (m - 1)) : (q1 << 1)) & (K1 << 1);
        const uint32_t c = (m >= 2 ? (q2 >> (m - 2)) : (q2 << (2 - m))) & (K1 << 2);
        N[m] = a | b | c;
    }
#endif
}

struct K1Smem {
    PTShared S;
    uint32_t Uhi[kW][8];   // per own buffer: high words of T*2^11-1 for its current slot
    uint64_t T64[kW][8];   // per own buffer: exact thresholds (tie path)
};

// Dynamic shared memory: [threshold-offset scratch of the launch shape |] spin words | bond bytes |
// staged slot thresholds and stream states; the control block is static.
__host__ __device__ constexpr size_t k1_words_offset() { return 0; }
// Stride (threads) of the per-thread threshold-offset scratch of a launch shape; 0: no scratch.
__host__ __device__ constexpr int k1_scratch_stride(int sp, int maxt) {
    return (TAPT_K1_IDXS && sp * maxt <= 1536) ? maxt : 0;
}
__host__ __device__ constexpr size_t k1_stage_offset(int n, bool dis) {
    return (k1_words_offset() + (size_t)n * 4 + (dis ? (size_t)n : 0) + 15) & ~size_t(15);
}

// TAPT_K1_IDXS: threshold offsets as bytes in shared memory.  Word j of a site's 8 scratch words
// (thread-interleaved: word (u, j) of thread tid sits at [(u*8 + j)*STRIDE + tid]) takes the even
// (j < 4) or odd (j >= 4) nibbles of N[j & 3] as bytes 4*q, so replica b = 8y + 4*odd + m reads byte y
// of word m + 4*odd.
template <int STRIDE>
__host__ __device__ constexpr int k1_index_byte(int u, int b) {
    return ((u * 8 + (b & 3) + 4 * ((b >> 2) & 1)) * STRIDE) * 4 + (b >> 3);
}
template <int STRIDE>
__device__ __forceinline__ void k1_index_bytes(uint32_t* scr_w, int u, const uint32_t (&N)[4]) {
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        scr_w[(u * 8 + m) * STRIDE] = (N[m] << 2) & 0x1C1C1C1Cu;
        scr_w[(u * 8 + 4 + m) * STRIDE] = (N[m] >> 2) & 0x1C1C1C1Cu;
    }
}

// PACK > 1: lane b is replica b % (32/PACK) of the word's field b / (32/PACK), whose site counter is dph
// per field further on.
template <int STRIDE, int PACK = 1>
__device__ __forceinline__ uint32_t k1_decide_exact_scr(const K1Smem& sm, int W, uint64_t phi_i, const uint8_t* scr,
                                                        int u, uint64_t dph = 0) {
    constexpr int FW = kW / PACK;
    uint32_t nw = 0;
    for (int b = 0; b < W; ++b) {
        const uint32_t idx = scr[k1_index_byte<STRIDE>(u, b)] >> 2;
        if constexpr (PACK > 1) {
            const int rb = b & (FW - 1);
            const uint64_t x = mix_final(sm.S.sb[rb] + phi_i + (uint64_t)(b / FW) * dph);
            if (below(x, sm.T64[rb][idx])) nw |= 1u << b;
        } else {
            const uint64_t x = mix_final(sm.S.sb[b] + phi_i);
            if (below(x, sm.T64[b][idx])) nw |= 1u << b;
        }
    }
    return nw;
}

// Heat-bath decisions for one site word over the W replicas of this CTA.
__device__ __forceinline__ uint32_t k1_decide_exact(const K1Smem& sm, int W, uint64_t phi_i, const uint32_t (&N)[4]) {
    uint32_t nw = 0;
    for (int b = 0; b < W; ++b) {
        const uint32_t idx = (N[b & 3] >> (4 * (b >> 2))) & 7u;
        const uint64_t x = mix_final(sm.S.sb[b] + phi_i);
        if (below(x, sm.T64[b][idx])) nw |= 1u << b;
    }
    return nw;
}

// Fast-path decisions for SP site words (independent chains interleaved): replica b of
// site u draws mix(sb[b] + i_u*phi) and compares with the threshold of its own q.  The
// loop runs b descending so the carry chain leaves NOT(up_b) at bit b.  NV = 32: full
// group, fully unrolled; NV = 0: partial group (runtime count nv), rolled loop.
// V & 4: track the tie band as a running min of (h - U + 1) instead of OR-ing compares.
// STRIDE > 0 (TAPT_K1_IDXS): the threshold offsets 4*q of the site's 32 replicas were stored as bytes in
// the thread's shared-memory scratch (k1_index_bytes), so a replica's offset is one LDS.U8 with an
// immediate address instead of a shift and a mask on the ALU pipe.
template <int NV, int V, int SP, int STRIDE = 0, int PACK = 1>
__device__ __forceinline__ void k1_decide(const K1Smem& sm, int nv, const uint64_t (&ph)[SP],
                                          const uint32_t (&N)[SP][4], const MixConsts& mc, uint32_t (&w)[SP],
                                          bool& tie, const uint8_t* scr = nullptr, uint64_t dph = 0) {
    static_assert(PACK == 1 || (NV == kW && STRIDE > 0 && (V & 16) == 0), "packed groups: all 32 lanes, index scratch");
    constexpr int FW = kW / PACK;  // lanes per field (= replicas of the group)
    [[maybe_unused]] uint64_t phf[SP][PACK];  // PACK > 1: site counter of each field of each word
    if constexpr (PACK > 1) {
#pragma unroll
        for (int u = 0; u < SP; ++u)
#pragma unroll
            for (int k = 0; k < PACK; ++k) phf[u][k] = ph[u] + (uint64_t)k * dph;
    }
    constexpr int U = NV ? NV : 1;
    const int cnt = NV ? NV : nv;
    uint32_t tmin = 0xFFFFFFFFu;
    if constexpr (NV == kW && (V & 16) != 0) {
        // two replicas (b, b-1) x SP sites per step: 2*SP chains interleaved stage by stage
#pragma unroll
        for (int b = kW - 1; b >= 1; b -= 2) {
            constexpr int K = 2 * SP;
            uint32_t zl[K], zh[K], h[K], thr[K];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int bb = b - e;
                const uint64_t base = sm.S.sb[bb];
                const int m = bb & 3, sh = 4 * (bb >> 2);
#pragma unroll
                for (int u = 0; u < SP; ++u) {
                    const uint64_t z = base + ph[u];
                    zl[e * SP + u] = (uint32_t)z;
                    zh[e * SP + u] = (uint32_t)(z >> 32);
                    if constexpr ((V & 8) != 0) {
                        const uint32_t ix = (sh >= 4 ? __umulhi(N[u][m], mc.nib[sh >> 2]) : (N[u][m] << 2)) & 0x1Cu;
                        thr[e * SP + u] =
                            *reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(&sm.Uhi[bb][0]) + ix);
                    } else {
                        thr[e * SP + u] = sm.Uhi[bb][(N[u][m] >> sh) & 7u];
                    }
                }
            }
            mix_pre_hi_k<K>(zl, zh, h);
#pragma unroll
            for (int e = 0; e < 2; ++e)
#pragma unroll
                for (int u = 0; u < SP; ++u) {
                    const uint32_t dd = decide_acc(h[e * SP + u], thr[e * SP + u], w[u]);
                    tmin = min(tmin, dd + (TAPT_K1_UM1 ? 0u : 1u));
                }
        }
        tie |= tmin <= 2u;
    } else {
#pragma unroll U
    for (int b = cnt - 1; b >= 0; --b) {
        int rb = b, fk = 0;  // replica of the group, field of the word
        if constexpr (PACK > 1) {
            rb = b & (FW - 1);
            fk = b / FW;
        }
        const uint64_t base = sm.S.sb[rb];
        const int m = b & 3, sh = 4 * (b >> 2);
        uint32_t dmin[SP];
#pragma unroll
        for (int u = 0; u < SP; ++u) {
            uint32_t thr;
            if constexpr (STRIDE > 0) {
                // IDXS = 1: ptxas merges the byte reads into word loads + PRMT; 2: one LDS.U8 per decision
                const uint32_t ix = TAPT_K1_IDXS == 2 ? *(reinterpret_cast<const volatile uint8_t*>(scr) + k1_index_byte<STRIDE>(u, b))
                                                      : scr[k1_index_byte<STRIDE>(u, b)];
                thr = *reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(&sm.Uhi[rb][0]) + ix);
            } else if constexpr ((V & 8) != 0) {  // shift on the FMA pipe: (N >> sh) << 2 == hi(N * 2^(34-sh)) & 0x1C
                const uint32_t ix = (sh >= 4 ? __umulhi(N[u][m], mc.nib[sh >> 2]) : (N[u][m] << 2)) & 0x1Cu;
                thr = *reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(&sm.Uhi[b][0]) + ix);
            } else {
                thr = sm.Uhi[b][(N[u][m] >> sh) & 7u];
            }
            uint64_t phv = ph[u];
            if constexpr (PACK > 1) phv = phf[u][fk];
#if TAPT_K1_PHOPQ
            uint32_t zl_, zh_;  // explicit carry-chain add: IADD3 + IADD3.X / IMAD.X instead of IMAD.WIDE + IMAD.IADD
            asm("add.cc.u32 %0, %2, %4;\n\taddc.u32 %1, %3, %5;"
                : "=r"(zl_), "=r"(zh_)
                : "r"((uint32_t)base), "r"((uint32_t)(base >> 32)), "r"((uint32_t)phv), "r"((uint32_t)(phv >> 32)));
            const uint32_t h = mix_pre_hi<V>(zl_, zh_, mc);
#else
            const uint64_t z = base + phv;
            const uint32_t h = mix_pre_hi<V>((uint32_t)z, (uint32_t)(z >> 32), mc);
#endif
            const uint32_t dd = decide_acc(h, thr, w[u]);
            dmin[u] = dd;
            if constexpr (TAPT_K1_UM1 && TAPT_K1_MIN3 && (V & 4) != 0 && SP == 2) {
            } else if constexpr ((V & 4) != 0)
                tmin = min(tmin, dd + (TAPT_K1_UM1 ? 0u : 1u));
            else
                tie |= (dd + (TAPT_K1_UM1 ? 0u : 1u) <= 2u);
        }
        // tables hold U - 1: the band is d in {0, 1, 2} itself, and one 3-input min covers two sites
        if constexpr (TAPT_K1_UM1 && TAPT_K1_MIN3 && (V & 4) != 0 && SP == 2) tmin = min(tmin, min(dmin[0], dmin[1]));
    }
    if constexpr ((V & 4) != 0) tie |= tmin <= 2u;
    }
}

// MINB: CTAs per SM the register allocation must allow (2 for the 256-thread small-lattice shape)
// BULK: per-item state loads as copy-engine bulk copies (large tiles; see the load below).
// NAR: unrolled decisions for 16- and 8-replica groups (narrow groups).  Both
// are separate instantiations because the extra code shifts the hot loop's code generation: with the
// narrow paths compiled in, 2D shapes measured up to 4 % faster and 3D shapes up to 1.2 % slower, so
// 3D shapes carry them only when the launch uses narrow groups (tools/cfg_ab.sh, tools/k1_ab.sh).
// PACK: sites per word of a narrow group (2: 16 replicas, 4: 8 replicas): the lattice is folded PACK times
// along its slowest dimension and a word holds the PACK folded sites, so the per-site work (stencil, nibble
// spread, offset bytes, energy planes) is amortised over 32 decisions again.  Needs full groups and an even
// number of planes per fold (both colours stay aligned); launch_k1_t checks.
template <int DIM, bool DIS, bool CLU, int SP, int MAXT, int MINB = 1, bool BULK = false, bool NAR = true, int PACK = 1>
__global__ void __launch_bounds__(MAXT, MINB) k1_lattice_pt(const PTArgs a, const LatDims d) {
    static_assert(PACK == 1 || (!BULK && TAPT_K1_IDXS), "packed groups: small lattices with the index scratch");
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __shared__ K1Smem sm;  // static: table addresses fold into LDS immediates
    constexpr size_t kScr0 = (size_t)k1_scratch_stride(SP, MAXT) * SP * 8 * 4;
    uint32_t* words = reinterpret_cast<uint32_t*>(smem_raw + kScr0);
    uint8_t* bonds = reinterpret_cast<uint8_t*>(words + a.n);
    // staged once per launch / item: heat-bath thresholds of every slot and the instance's stream
    // states, so that the per-sweep table and stream-base refresh reads no global memory
    uint64_t* thrS = reinterpret_cast<uint64_t*>(smem_raw + kScr0 + k1_stage_offset(a.n, a.bonds != nullptr));
    uint64_t* strS = thrS + (size_t)a.R * 8;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    constexpr int KV = DIM == 3 ? TAPT_K1_VARIANT3 : TAPT_K1_VARIANT;  // decision instruction mix
    // threshold offsets of the thread's SP site words as bytes, at the front of the dynamic block so that
    // their addresses are the thread's offset + an immediate
    constexpr int XS = k1_scratch_stride(SP, MAXT);
    static_assert(!(TAPT_K1_IDXS && TAPT_K1_PIPE), "the index scratch holds one site pair at a time");
    uint32_t* const scr_w = reinterpret_cast<uint32_t*>(smem_raw) + tid;
    const uint8_t* const scr_b = reinterpret_cast<const uint8_t*>(scr_w);
    const int cl = blockIdx.x / a.G, grp = blockIdx.x % a.G;
    const int n = a.n, W = a.W, nv = own_count(a, grp);
    const int nfold = PACK > 1 ? n / PACK : n;  // words of the (folded) lattice
    const int half = (PACK > 1 ? nfold : n) >> 1, nsub = half / SP;
    // site-counter step from one field of a word to the next
    [[maybe_unused]] const uint64_t dph = PACK > 1 ? (uint64_t)nfold * kPhi : 0ull;
    const int tl = a.sched ? pt_timeline(cl, a.sched_clusters) : 0;
    const int it0 = a.sched ? a.sched_ptr[tl] : 0, it1 = a.sched ? a.sched_ptr[tl + 1] : 1;
    for (int e = tid; e < a.R * 8; e += nt) {
        const int r = e >> 3, k = e & 7;
        thrS[e] = k < a.nidx ? a.thr[(size_t)r * a.nidx + k] : 0ull;
    }
    // BULK (tiles of >= 16384 sites, config 5: +0.5 %): spin words and bond bytes of each item come
    // in as bulk copies (copy engine, mbarrier).  Smaller tiles use uint4 loads, in an instantiation
    // without this code (with it, config 2 measured 4.5 % slower even when the path was unused).
    // sign masks of the 64 bond bytes: row bb = {-(bb & 1), -(bb >> 1 & 1), ...} (TAPT_K1_BLUT; the
    // config-5 shape only: +0.4 % there on top of XSEL, -1.6 % on config 3)
    __shared__ __align__(16) uint32_t bmask[(DIS && BULK && TAPT_K1_BLUT) ? 64 : 1][8];
    if constexpr (DIS && BULK && TAPT_K1_BLUT) {
        for (int e = tid; e < 64 * 8; e += nt) bmask[e >> 3][e & 7] = 0u - (((uint32_t)(e >> 3) >> (e & 7)) & 1u);
    }
    __shared__ uint64_t tile_bar;
    constexpr bool bulk = BULK;
    uint32_t tile_phase = 0;
    if constexpr (BULK) {
        if (tid == 0) mbar_init(&tile_bar);
        __syncthreads();
    }
    for (int it = it0; it < it1; ++it) {
    const SchedItem item = a.sched ? a.sched[it] : SchedItem{cl, 0, a.energy_only ? 1 : a.n_sweeps, -1, -1};
    const int inst = item.inst;
    if (item.wait >= 0) pt_wait_flag(a, item.wait);

    // ---- load this CTA's spins (and the instance's bond signs) into shared memory
    if constexpr (bulk) {
        fence_proxy_async_smem();  // the previous item's generic accesses before the copy engine writes
        __syncthreads();
        if (tid == 0) {
            // a split job's words were written by another SM's generic stores (flag-ordered)
            asm volatile("fence.proxy.async.global;" ::: "memory");
            const uint32_t wb = (uint32_t)n * 4u, bb = DIS ? (uint32_t)n : 0u;
            mbar_expect_tx(&tile_bar, wb + bb);
            bulk_g2s(words, a.words + ((size_t)inst * a.G + grp) * n, wb, &tile_bar);
            if constexpr (DIS) bulk_g2s(bonds, a.bonds + (size_t)inst * n, bb, &tile_bar);
        }
    } else {
        if constexpr (PACK > 1) {
            const uint32_t* src = a.words + ((size_t)inst * a.G + grp) * n;
            for (int k = tid; k < nfold; k += nt) {
                uint32_t v = 0;
#pragma unroll
                for (int f = 0; f < PACK; ++f) v |= (src[k + f * nfold] & ((1u << (kW / PACK)) - 1u)) << (f * (kW / PACK));
                words[k] = v;
            }
        } else {
        const uint4* src = reinterpret_cast<const uint4*>(a.words + ((size_t)inst * a.G + grp) * n);
        uint4* dst = reinterpret_cast<uint4*>(words);
        for (int k = tid; k < (n >> 2); k += nt) dst[k] = src[k];
        }
        if constexpr (DIS) {
            const uint4* bs = reinterpret_cast<const uint4*>(a.bonds + (size_t)inst * n);
            uint4* bd = reinterpret_cast<uint4*>(bonds);
            for (int k = tid; k < (n >> 4); k += nt) bd[k] = bs[k];
        }
    }
    pt_load_perm(a, sm.S, inst);
    for (int r = tid; r < a.R; r += nt) strS[r] = a.streams[(size_t)inst * a.R + r];
    if constexpr (bulk) {
        mbar_wait(&tile_bar, tile_phase);
        tile_phase ^= 1u;
    }
    __syncthreads();

    // swap passes before this item: sweeps T = t+1 in (t0, t0+s0] with swap_every | T
    uint64_t pass = a.p0;
    if (a.swap_every > 0 && item.s0 > 0)
        pass += (a.t0 + item.s0) / (uint64_t)a.swap_every - a.t0 / (uint64_t)a.swap_every;
    int par = 0;
    for (int s = item.s0; s < item.s1; ++s) {
        const uint64_t t = a.t0 + (uint64_t)s;
        par = (int)(t & 1);
        // per-buffer tables and stream bases for the slots the buffers occupy now
        for (int e = tid; e < nv * 8; e += nt) {
            const int b = e >> 3, k = e & 7;
            const int slot = sm.S.slot_of[grp * W + b];
            const uint64_t T = thrS[slot * 8 + k];
            // UM1: store U - 1 (clamped at 0) so that h - (U - 1) is both the carry of the decision
            // and the tie band {0, 1, 2} (h = U - 1 falls in the band and is redone exactly)
            sm.Uhi[b][k] = TAPT_K1_UM1 ? max(thr_hi(T), 1u) - 1u : thr_hi(T);
            sm.T64[b][k] = T;
        }
        {  // pt_stream_bases with the staged stream states
            const uint64_t k0 = a.draw_base + t * (uint64_t)a.n_free + 1ull;
            for (int b = tid; b < nv; b += nt) sm.S.sb[b] = strS[sm.S.slot_of[grp * W + b]] + k0 * kPhi;
        }
        __syncthreads();

        uint32_t C[kCnt];
#pragma unroll
        for (int k = 0; k < kCnt; ++k) C[k] = 0;

        const int c_end = TAPT_K1_EPOST ? 3 : 2;
        for (int cc = (a.energy_only ? (TAPT_K1_EPOST ? 2 : 1) : 0); cc < c_end; ++cc) {
            // cc = 0, 1: colour halves; with TAPT_K1_EPOST the energy is a third pass (cc = 2)
            // over colour 1, so no energy state stays live across the decision loop
            const int c = cc > 1 ? 1 : cc;
            const bool decide = !a.energy_only && cc < 2;
            const bool count = TAPT_K1_EPOST ? (cc == 2) : (c == 1);
            // Software-pipelined over this thread's site pairs: the neighbour sums of the next
            // pair (other-colour words, not written during this half) are formed before the
            // decisions of the current pair, hiding the shared-memory latency of the stencil.
            int is[SP];
            uint32_t q[SP][3], N[SP][4];
            auto stencil = [&](int jj, int (&is_)[SP], uint32_t (&q_)[SP][3], uint32_t (&N_)[SP][4]) {
#pragma unroll
                for (int u = 0; u < SP; ++u) {
                    int x, y, z;
                    is_[u] = colour_site<DIM>(jj + u * nsub, c, d, x, y, z);
                    k1_stencil<DIM, DIS, PACK>(words, bonds, is_[u], x, y, z, d, q_[u][0], q_[u][1], q_[u][2],
                                               (DIS && BULK && TAPT_K1_BLUT) ? &bmask[0][0] : nullptr, nfold);
                    nibbles(q_[u][0], q_[u][1], q_[u][2], N_[u]);
                    if constexpr (XS > 0) k1_index_bytes<XS>(scr_w, u, N_[u]);
                }
            };
            if (tid < nsub) stencil(tid, is, q, N);
            for (int j = tid; j < nsub; j += nt) {
                int isn[SP];
                uint32_t qn[SP][3], Nn[SP][4];
                if (TAPT_K1_PIPE && j + nt < nsub) stencil(j + nt, isn, qn, Nn);
                uint32_t nw[SP];
                if (!decide) {
#pragma unroll
                    for (int u = 0; u < SP; ++u) nw[u] = words[is[u]];
                } else {
                    uint64_t ph[SP];
#pragma unroll
                    for (int u = 0; u < SP; ++u) {
                        ph[u] = (uint64_t)(uint32_t)is[u] * kPhi;
#if TAPT_K1_PHOPQ
                        asm volatile("" : "+l"(ph[u]));  // keep base + ph a 64-bit add (no IMAD.WIDE re-multiply)
#endif
                        nw[u] = 0;  // NOT(up) bits, replica b at bit b
                    }
                    bool tie = false;
                    // full 32-, 16- and 8-replica groups unrolled (narrow groups spread an instance over
                    // more CTAs when instances are few); partial groups take the rolled loop
                    if constexpr (PACK > 1)
                        k1_decide<kW, KV, SP, XS, PACK>(sm, kW, ph, N, a.mc, nw, tie, scr_b, dph);
                    else if (nv == kW)
                        k1_decide<kW, KV, SP, XS>(sm, nv, ph, N, a.mc, nw, tie, scr_b);
                    else if (NAR && nv == 16)
                        k1_decide<16, KV, SP, XS>(sm, nv, ph, N, a.mc, nw, tie, scr_b);
                    else if (NAR && nv == 8)
                        k1_decide<8, KV, SP, XS>(sm, nv, ph, N, a.mc, nw, tie, scr_b);
                    else
                        k1_decide<0, KV, SP, XS>(sm, nv, ph, N, a.mc, nw, tie, scr_b);
                    const uint32_t vmask = (PACK > 1 || nv >= 32) ? 0xFFFFFFFFu : ((1u << nv) - 1u);
#pragma unroll
                    for (int u = 0; u < SP; ++u) nw[u] = ~nw[u] & vmask;
                    if (tie) {  // probability ~ 2^-31 per decision: redo the words exactly
#pragma unroll
                        for (int u = 0; u < SP; ++u)
                            nw[u] = XS > 0 ? k1_decide_exact_scr<(XS > 0 ? XS : 1), PACK>(sm, PACK > 1 ? kW : nv, ph[u],
                                                                                          scr_b, u, dph)
                                           : k1_decide_exact(sm, nv, ph[u], N[u]);
                    }
#pragma unroll
                    for (int u = 0; u < SP; ++u) words[is[u]] = nw[u];
                }
                if (count) {
#pragma unroll
                    for (int u = 0; u < SP; ++u) {
                        uint32_t v0, v1, v2;
                        unsat_planes<DIM>(nw[u], q[u][0], q[u][1], q[u][2], v0, v1, v2);
                        sliced_add3<kCnt>(C, v0, v1, v2);
                    }
                }
                if (j + nt < nsub) {
                    if (!TAPT_K1_PIPE) stencil(j + nt, isn, qn, Nn);
#pragma unroll
                    for (int u = 0; u < SP; ++u) {
                        is[u] = isn[u];
#pragma unroll
                        for (int k = 0; k < 3; ++k) q[u][k] = qn[u][k];
#pragma unroll
                        for (int k = 0; k < 4; ++k) N[u][k] = Nn[u][k];
                    }
                }
            }
            __syncthreads();
        }
        // exact energies: E = J0 * (2*U - n*dim)
        {
            const uint32_t tot = warp_sliced_total<kCnt>(C);
            if constexpr (PACK > 1)
                atomicAdd(&sm.S.Ucnt[lane & (kW / PACK - 1)], tot);  // the fields of a word are the same replicas
            else if (lane < nv)
                atomicAdd(&sm.S.Ucnt[lane], tot);
            __syncthreads();
            if (tid < nv) {
                sm.S.Eown[par][tid] = d.J0 * (2 * (int)sm.S.Ucnt[tid] - n * DIM);
                sm.S.Ucnt[tid] = 0;
            }
        }
        if (a.energy_only) break;
        pt_epilogue<CLU, CtaTeam, PACK>(a, sm.S, words, inst, grp, t, pass);
    }
    if (a.energy_only) {
        __syncthreads();
        for (int b = tid; b < nv; b += nt) a.E[(size_t)inst * a.B + grp * W + b] = sm.S.Eown[par][b];
        continue;
    }
    // ---- write back
    {
        if constexpr (PACK > 1) {
            uint32_t* dst = a.words + ((size_t)inst * a.G + grp) * n;
            constexpr uint32_t F1 = (1u << (kW / PACK)) - 1u;
            for (int k = tid; k < nfold; k += nt) {
                const uint32_t v = words[k];
#pragma unroll
                for (int f = 0; f < PACK; ++f) dst[k + f * nfold] = (v >> (f * (kW / PACK))) & F1;
            }
        } else {
        uint4* dst = reinterpret_cast<uint4*>(a.words + ((size_t)inst * a.G + grp) * n);
        const uint4* src = reinterpret_cast<const uint4*>(words);
        for (int k = tid; k < (n >> 2); k += nt) dst[k] = src[k];
        }
    }
    pt_finish<CLU>(a, sm.S, inst, grp, par);
    if (item.signal >= 0) pt_signal_flag<CLU>(a, item.signal, grp);
    __syncthreads();  // shared memory is reused by the next item
    }
}

size_t k1_smem_bytes(int n, bool dis, int R) {
    // dynamic part without the launch shape's threshold-offset scratch, which launch_k1_t adds (the static
    // K1Smem block is accounted by the compiler): words, bond bytes, then the staged slot thresholds
    // [R][8] and stream states [R]
    return k1_stage_offset(n, dis) + (size_t)R * 9 * 8;
}

// resident != null: report how many clusters (or CTAs, without a cluster) of this launch shape
// are co-resident on the device instead of launching.
template <int DIM, bool DIS, bool CLU>
static cudaError_t launch_k1_t(const PTArgs& a, const LatDims& d, int threads, cudaStream_t st, int* resident,
                               char* name) {
    // launch shapes: 2 interleaved site words per thread-iteration at 257..768 threads (640 is the
    // config-5 default: <= 102 registers, 5 warps per scheduler), 1 at > 768, 4 at < 256
    const bool bulk = (a.n & 15) == 0 && a.n >= 16384;
    constexpr bool NAR3 = DIM == 2;  // 3D: narrow decision paths only in the narrow-group instantiations
    const bool narrow = a.W < kW;
    // (SP, MAXT, MINB, BULK, NAR) of the instantiation this launch shape selects
    const int pick = threads > 768                ? 0
                     : threads > 640              ? 1
                     : threads > 512 && bulk && !narrow ? 9
                     : threads > 512              ? 8
                     : threads > 256 && narrow    ? 2
                     : threads > 256 && bulk      ? 3
                     : threads > 256              ? 4
                     : threads == 256 && narrow   ? 5
                     : threads == 256             ? 6
                                                  : 7;
    // packed narrow groups (PACK template parameter): full 16- or 8-replica groups on a lattice whose
    // slowest dimension folds into 32/W parts of an even number of planes
    int pack = 1;
    if (narrow && TAPT_K1_IDXS && TAPT_K1_PACK && (a.W == 16 || a.W == 8) && a.B % a.W == 0 && threads > 128 &&
        threads <= 512) {
        const int pk = kW / a.W, Ls = 1 << d.log2Ly;  // extent of the slowest dimension (3D lattices are cubic)
        if (Ls >= 2 * pk && (a.n / pk / 2) % 2 == 0) pack = pk;
    }
    // one word per thread-iteration (SP = 1) when two would leave threads of a 512-thread CTA without work
    const bool sp1 = pack > 1 && threads > 256 && TAPT_K1_PACK_SP1 && a.n / pack / 4 < threads;
    const int ppick = pack == 1 ? -1 : (sp1 ? 4 : threads > 256 ? 0 : 2) + (pack == 4 ? 1 : 0);
    static void (*const ptable[6])(const PTArgs, const LatDims) = {
        k1_lattice_pt<DIM, DIS, CLU, 2, 512, 1, false, true, 2>, k1_lattice_pt<DIM, DIS, CLU, 2, 512, 1, false, true, 4>,
        k1_lattice_pt<DIM, DIS, CLU, 2, 256, TAPT_K1_MINB256, false, true, 2>,
        k1_lattice_pt<DIM, DIS, CLU, 2, 256, TAPT_K1_MINB256, false, true, 4>,
        k1_lattice_pt<DIM, DIS, CLU, 1, 512, 1, false, true, 2>, k1_lattice_pt<DIM, DIS, CLU, 1, 512, 1, false, true, 4>};
    static const int pshape[6][5] = {{2, 512, 1, 0, 1}, {2, 512, 1, 0, 1}, {2, 256, TAPT_K1_MINB256, 0, 1},
                                     {2, 256, TAPT_K1_MINB256, 0, 1}, {1, 512, 1, 0, 1}, {1, 512, 1, 0, 1}};
    static const int shape[10][5] = {{1, 1024, 1, 0, 1}, {2, 768, 1, 0, 1},   {2, 512, 1, 0, 1}, {2, 512, 1, 1, NAR3},
                                    {2, 512, 1, 0, NAR3}, {2, 256, TAPT_K1_MINB256, 0, 1}, {2, 256, TAPT_K1_MINB256, 0, NAR3}, {4, 256, 1, 0, 1},
                                    {2, 640, 1, 0, 1}, {2, 640, 1, 1, NAR3}};
    static void (*const table[10])(const PTArgs, const LatDims) = {
        k1_lattice_pt<DIM, DIS, CLU, 1, 1024>,          k1_lattice_pt<DIM, DIS, CLU, 2, 768>,
        k1_lattice_pt<DIM, DIS, CLU, 2, 512, 1, false, true>, k1_lattice_pt<DIM, DIS, CLU, 2, 512, 1, true, NAR3>,
        k1_lattice_pt<DIM, DIS, CLU, 2, 512, 1, false, NAR3>, k1_lattice_pt<DIM, DIS, CLU, 2, 256, TAPT_K1_MINB256, false, true>,
        k1_lattice_pt<DIM, DIS, CLU, 2, 256, TAPT_K1_MINB256, false, NAR3>, k1_lattice_pt<DIM, DIS, CLU, 4, 256>,
        k1_lattice_pt<DIM, DIS, CLU, 2, 640>, k1_lattice_pt<DIM, DIS, CLU, 2, 640, 1, true, NAR3>};
    auto fn = ppick >= 0 ? ptable[ppick] : table[pick];
    const int* v = ppick >= 0 ? pshape[ppick] : shape[pick];
    const size_t smem = k1_smem_bytes(a.n, DIS, a.R) + (size_t)k1_scratch_stride(v[0], v[1]) * v[0] * 32;
    if (name) {
        if (pack > 1)
            snprintf(name, 96, "k1_lattice_pt<%d,%d,%d,%d,%d,%d,%d,%d,%d>", DIM, (int)DIS, (int)CLU, v[0], v[1], v[2],
                     v[3], v[4], pack);
        else
        snprintf(name, 96, "k1_lattice_pt<%d,%d,%d,%d,%d,%d,%d,%d>", DIM, (int)DIS, (int)CLU, v[0], v[1], v[2], v[3],
                 v[4]);
        return cudaSuccess;
    }
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((a.sched ? a.sched_clusters : a.I) * a.G));
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    if (CLU) {
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)a.G;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    if (resident) {
        if (CLU) return cudaOccupancyMaxActiveClusters(resident, (const void*)fn, &cfg);
        int per_sm = 0, dev = 0, nsm = 0;
        cudaError_t q = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
        if (q == cudaSuccess) q = cudaGetDevice(&dev);
        if (q == cudaSuccess) q = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        *resident = per_sm * nsm;
        return q;
    }
    return pt_launch(fn, cfg.gridDim.x, (unsigned)threads, smem, st, CLU ? (unsigned)a.G : 1u, a, d);
}

static cudaError_t k1_dispatch(const PTArgs& a, const LatDims& d, int threads, bool cluster, cudaStream_t st,
                               int* resident, char* name = nullptr) {
    const bool dis = a.bonds != nullptr;
    if (d.dim == 2) {
        if (dis)
            return cluster ? launch_k1_t<2, true, true>(a, d, threads, st, resident, name)
                           : launch_k1_t<2, true, false>(a, d, threads, st, resident, name);
        return cluster ? launch_k1_t<2, false, true>(a, d, threads, st, resident, name)
                       : launch_k1_t<2, false, false>(a, d, threads, st, resident, name);
    }
    if (dis)
        return cluster ? launch_k1_t<3, true, true>(a, d, threads, st, resident, name)
                       : launch_k1_t<3, true, false>(a, d, threads, st, resident, name);
    return cluster ? launch_k1_t<3, false, true>(a, d, threads, st, resident, name)
                   : launch_k1_t<3, false, false>(a, d, threads, st, resident, name);
}

cudaError_t launch_k1(const PTArgs& a, const LatDims& d, int threads, bool cluster, cudaStream_t st) {
    return k1_dispatch(a, d, threads, cluster, st, nullptr);
}

// Name of the instantiation (template arguments) a launch with these arguments selects.
void k1_variant_name(const PTArgs& a, const LatDims& d, int threads, bool cluster, char* out) {
    out[0] = 0;
    k1_dispatch(a, d, threads, cluster, nullptr, nullptr, out);
}

// Co-resident clusters (cluster launches) or CTAs of the K1 launch shape (balanced schedule).
int k1_resident_units(const PTArgs& a, const LatDims& d, int threads, bool cluster) {
    int r = 0;
    return k1_dispatch(a, d, threads, cluster, nullptr, &r) == cudaSuccess ? r : 0;
}

}  // namespace tapt_dev

// ---------------------------------------------------------------------------
// Decision-rate probe: the irreducible per-update work of K1 with no stencil and no
// memory traffic -- one counter-addressed splitmix64 draw (high word), one threshold
// lookup in shared memory, one compare, one bit insert -- in the same unrolled 2x32
// form as the sweep loop.  Its rate is the measured ALU ceiling used as the roofline
// denominator by bench.py.
namespace tapt_dev {

template <int V>
__global__ void __launch_bounds__(512) k_decision_probe(uint32_t iters, uint32_t* sink, MixConsts mc) {
    __shared__ K1Smem sm;
    constexpr int XS = TAPT_K1_IDXS ? 512 : 0;  // the sweep kernel's scratch-indexed thresholds
    __shared__ uint32_t idx_scr[XS ? 2 * 8 * XS : 1];
    const int tid = threadIdx.x;
    for (int e = tid; e < kW * 8; e += blockDim.x) sm.Uhi[e >> 3][e & 7] = 0x80000000u + (uint32_t)e * 977u;
    for (int e = tid; e < kW; e += blockDim.x) sm.S.sb[e] = 0x1234567ull * (e + 1);
    __syncthreads();
    const uint32_t gid = blockIdx.x * blockDim.x + tid;
    uint32_t N[2][4];
    for (int m = 0; m < 4; ++m) {
        N[0][m] = gid * 0x9E3779B9u + m;
        N[1][m] = gid * 0x85EBCA6Bu + m;
    }
    uint32_t* const scr_w = idx_scr + (XS ? tid : 0);
    if constexpr (XS > 0) {
        k1_index_bytes<(XS > 0 ? XS : 1)>(scr_w, 0, N[0]);
        k1_index_bytes<(XS > 0 ? XS : 1)>(scr_w, 1, N[1]);
    }
    uint32_t acc = 0;
    bool tie = false;
    for (uint32_t it = 0; it < iters; ++it) {
        const uint64_t ph[2] = {(uint64_t)(2 * gid + it * 7919u) * kPhi, (uint64_t)(2 * gid + it * 7919u) * kPhi + kPhi};
        uint32_t w[2] = {0, 0};
        k1_decide<kW, V, 2, XS>(sm, kW, ph, N, mc, w, tie, reinterpret_cast<const uint8_t*>(scr_w));
        if constexpr (XS > 0) {  // keep the offsets changing (one word of the scratch per iteration)
            scr_w[(it & 15) * XS] = (scr_w[(it & 15) * XS] ^ (w[0] >> 3) ^ (w[1] << 1)) & 0x1C1C1C1Cu;
        } else {
            N[0][it & 3] ^= w[0] >> 3;
            N[1][it & 3] ^= w[1] << 1;
        }
        acc += w[0] ^ w[1];
    }
    sink[gid] = acc + (tie ? 1u : 0u);
}

cudaError_t launch_decision_probe(int blocks, int threads, uint32_t iters, uint32_t* sink, cudaStream_t st,
                                  int variant) {
    const MixConsts mc = make_mix_consts();
    switch (variant < 0 ? TAPT_K1_VARIANT3 : variant) {  // default: the config-5 (3D) kernel's variant
#define TAPT_PROBE_CASE(v) \
    case v: k_decision_probe<v><<<blocks, threads, 0, st>>>(iters, sink, mc); break;
        TAPT_PROBE_CASE(0) TAPT_PROBE_CASE(1) TAPT_PROBE_CASE(2) TAPT_PROBE_CASE(3)
        TAPT_PROBE_CASE(4) TAPT_PROBE_CASE(5) TAPT_PROBE_CASE(6) TAPT_PROBE_CASE(7)
        TAPT_PROBE_CASE(8) TAPT_PROBE_CASE(9) TAPT_PROBE_CASE(10) TAPT_PROBE_CASE(11)
        TAPT_PROBE_CASE(12) TAPT_PROBE_CASE(13) TAPT_PROBE_CASE(14) TAPT_PROBE_CASE(15)
        TAPT_PROBE_CASE(22) TAPT_PROBE_CASE(70) TAPT_PROBE_CASE(134) TAPT_PROBE_CASE(198) TAPT_PROBE_CASE(28) TAPT_PROBE_CASE(36) TAPT_PROBE_CASE(38) TAPT_PROBE_CASE(44)
#undef TAPT_PROBE_CASE
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace tapt_dev
