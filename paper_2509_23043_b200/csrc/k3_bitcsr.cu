// k3_bitcsr.cu -- K3: bit-sliced parallel-tempering kernel for integer CSR graphs with small
// couplings and fields (BASELINE config 4: |J| in {1, 2}, h in {-2, 0, 16}), colour-class order.
//
// One thread owns a site word (32 replicas, bit b = replica b), as in K1:
//   * Unit-weight adjacency.  A coupling J_ij becomes |J| entries that point at w_j (J > 0) or at
//     its complement ~w_j (J < 0); a field h_i becomes |h| entries that point at a constant
//     all-ones (h > 0) or all-zeros word; rows are padded with the zeros word to 16 * nch
//     entries.  An entry is a byte offset into the instance's word image [w | ~w | ONES | ZEROS],
//     so entry e contributes bit x_e = [J s_j > 0] (or [h > 0]) and
//         acc = sum_e x_e,   S' = sum|J| + |h|,   l = h + sum_j J s_j = 2 acc - S'.
//   * acc is a bit-sliced popcount: a carry-save tree over each 16-entry chunk (11 full and 4 half
//     adders, no masks, no weights), 4 planes for S' <= 15 and 7 for the "heavy" rows (S' <= 127).
//   * Decisions: K1's carry-chain test on the pre-xorshift high word against per-buffer threshold
//     rows with a compile-time stride; a replica's threshold is LDS [base_i + 8 acc + imm(b)].
//   * Energies by flip bookkeeping, bit-sliced: the unsatisfied weight of site i in state s is
//     U(s) = s ? S' - acc : acc (bonds and field), and E changes by 2 (U(new) - U(old)).  Each
//     thread adds U(new) + (2^P - 1 - U(old)) to sliced counters and counts the constants.
//   * Teams: 4 warps (128 threads) per instance with their own named barrier; up to 4 instances
//     per CTA share one staged copy of the graph and of the slot threshold table, and progress
//     independently (no CTA-wide barrier inside the sweep loop).
//   * Split sites (Q = 2, 4; few instances per GPU): a team of 128 Q threads, Q adjacent lanes per
//     site.  Every lane of the group forms the site's bit-sliced count (broadcast loads) and decides
//     the replicas B = Q j + q of its lane q; the group ORs its bits into the word with shuffles.
//     With 4Q warps per instance instead of 4, the per-site dependency chain (the latency that
//     bounds an instance when its SM runs nothing else) is ~1/Q as long.  Energies are kept as
//     integers per owned replica (8 dU per flip, from the same acc the threshold index uses).
// The draw of replica b at site i in sweep t is the reference's per-site stream position
// (mcmc.cpp:30-45), so the chain is bit-identical to K2's colour order and to the oracle
// (oracle/tapt_oracle.c): tests/test_gpu_parity.py.
#include <cuda_runtime.h>

#include "pt_common.cuh"

namespace tapt_dev {

constexpr int kT3 = 128;     // threads per instance team
constexpr int kIPB3 = 4;     // max instance teams per CTA
constexpr int kRow3 = 132;   // threshold row stride (entries) of the per-buffer table
constexpr int kC3 = 12;      // sliced energy-counter planes (per-thread weight per sweep < 4096)
#ifndef TAPT_K3_IDXS
#define TAPT_K3_IDXS 0   // (measured -1 % on config 4: the gathers already load the LSU) light rows: threshold offsets 8*acc as bytes in a per-thread shared-memory scratch
#endif
#ifndef TAPT_K3_UM1
#define TAPT_K3_UM1 1    // threshold rows hold U - 1: the tie band is d in {0, 1, 2}; two decisions share a 3-input min
#endif
#ifndef TAPT_K3_CADD
#define TAPT_K3_CADD 1   // stream base + counter as an explicit carry-chain add
#endif
#ifndef TAPT_K3_VARIANT
#define TAPT_K3_VARIANT TAPT_K1_VARIANT  // mix_pre_hi instruction mix (common.cuh; V & 32 measured: no gain)
#endif

__device__ __forceinline__ void fa(uint32_t a, uint32_t b, uint32_t c, uint32_t& s, uint32_t& co) {
    s = a ^ b ^ c;
    co = maj3(a, b, c);
}
__device__ __forceinline__ void ha(uint32_t a, uint32_t b, uint32_t& s, uint32_t& co) {
    s = a ^ b;
    co = a & b;
}

// Bit-sliced popcount of the 16 entries of one chunk: P[0..4] (sum <= 16).
__device__ __forceinline__ void chunk_count(const uint8_t* W2, const uint32_t* ap, uint32_t (&P)[5]) {
    uint32_t x[16];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint4 e = *reinterpret_cast<const uint4*>(ap + 4 * k);
        x[4 * k + 0] = *reinterpret_cast<const uint32_t*>(W2 + e.x);
        x[4 * k + 1] = *reinterpret_cast<const uint32_t*>(W2 + e.y);
        x[4 * k + 2] = *reinterpret_cast<const uint32_t*>(W2 + e.z);
        x[4 * k + 3] = *reinterpret_cast<const uint32_t*>(W2 + e.w);
    }
    uint32_t s1, s2, s3, s4, s5, c1, c2, c3, c4, c5;
    fa(x[0], x[1], x[2], s1, c1);
    fa(x[3], x[4], x[5], s2, c2);
    fa(x[6], x[7], x[8], s3, c3);
    fa(x[9], x[10], x[11], s4, c4);
    fa(x[12], x[13], x[14], s5, c5);
    uint32_t t1, t2, d1, d2, d3;  // ones: s1..s5, x15
    fa(s1, s2, s3, t1, d1);
    fa(s4, s5, x[15], t2, d2);
    ha(t1, t2, P[0], d3);
    uint32_t u1, u2, u3, e1, e2, e3, e4;  // twos: c1..c5, d1..d3
    fa(c1, c2, c3, u1, e1);
    fa(c4, c5, d1, u2, e2);
    fa(d2, d3, u1, u3, e3);
    ha(u2, u3, P[1], e4);
    uint32_t v1, f1, f2;  // fours: e1..e4
    fa(e1, e2, e3, v1, f1);
    ha(v1, e4, P[2], f2);
    P[3] = f1 ^ f2;  // eights
    P[4] = f1 & f2;
}

// 4 planes -> nibbles: nibble k of N[m] = (P0..P3) of replica 4k+m.
__device__ __forceinline__ void nibbles4(uint32_t P0, uint32_t P1, uint32_t P2, uint32_t P3, uint32_t (&N)[4]) {
    const uint32_t e01 = (P0 & 0x55555555u) | ((P1 << 1) & 0xAAAAAAAAu);
    const uint32_t o01 = ((P0 >> 1) & 0x55555555u) | (P1 & 0xAAAAAAAAu);
    const uint32_t e23 = (P2 & 0x55555555u) | ((P3 << 1) & 0xAAAAAAAAu);
    const uint32_t o23 = ((P2 >> 1) & 0x55555555u) | (P3 & 0xAAAAAAAAu);
    constexpr uint32_t M = 0x33333333u;
    N[0] = (e01 & M) | ((e23 << 2) & ~M);
    N[1] = (o01 & M) | ((o23 << 2) & ~M);
    N[2] = ((e01 >> 2) & M) | (e23 & ~M);
    N[3] = ((o01 >> 2) & M) | (o23 & ~M);
}

// 8 * (nibble of replica b) as a byte offset (bits 3..6), and 128 * (high nibble) for heavy rows.
template <int SH>
__device__ __forceinline__ uint32_t nib8(uint32_t N) {
    if constexpr (SH >= 3)
        return (N >> (SH - 3)) & 0x78u;
    else
        return (N << (3 - SH)) & 0x78u;
}
template <int SH>
__device__ __forceinline__ uint32_t nib128(uint32_t N) {
    if constexpr (SH >= 7)
        return (N >> (SH - 7)) & 0x380u;
    else
        return (N << (7 - SH)) & 0x380u;
}

// Decisions of the 32 replicas of one site word, descending b so that the carry chain leaves
// NOT(up_b) in bit b.  Ub: byte address of this site's threshold base (per-buffer rows).
// z = stream base + counter, high word of the mix before its last xor-shift
__device__ __forceinline__ uint32_t k3_mix(uint64_t base, uint64_t ph, const MixConsts& mc) {
#if TAPT_K3_CADD
    uint32_t zl, zh;
    asm("add.cc.u32 %0, %2, %4;\n\taddc.u32 %1, %3, %5;"
        : "=r"(zl), "=r"(zh)
        : "r"((uint32_t)base), "r"((uint32_t)(base >> 32)), "r"((uint32_t)ph), "r"((uint32_t)(ph >> 32)));
    return mix_pre_hi<TAPT_K3_VARIANT>(zl, zh, mc);
#else
    const uint64_t z = base + ph;
    return mix_pre_hi<TAPT_K3_VARIANT>((uint32_t)z, (uint32_t)(z >> 32), mc);
#endif
}

// Light rows with TAPT_K3_IDXS: byte y of scratch word m + 4*odd of the thread (words STRIDE apart) holds
// 8*acc of replica 8y + 4*odd + m (even / odd nibbles of N[m]).
template <int STRIDE>
__host__ __device__ constexpr int k3_index_byte(int b) {
    return (((b & 3) + 4 * ((b >> 2) & 1)) * STRIDE) * 4 + (b >> 3);
}
template <int STRIDE>
__device__ __forceinline__ void k3_index_bytes(uint32_t* scr_w, const uint32_t (&N)[4]) {
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        scr_w[m * STRIDE] = (N[m] << 3) & 0x78787878u;
        scr_w[(4 + m) * STRIDE] = (N[m] >> 1) & 0x78787878u;
    }
}

template <bool HEAVY, int B, int STRIDE>
__device__ __forceinline__ uint32_t k3_decide_one(const uint8_t* Ub, const uint32_t (&N)[4], const uint32_t (&Nh)[4],
                                                  const PTShared& S, uint64_t ph, const MixConsts& mc, uint32_t& w,
                                                  const uint8_t* scr) {
    constexpr int m = B & 3, sh = 4 * (B >> 2);
    uint32_t ix;
    if constexpr (!HEAVY && STRIDE > 0) {
        ix = *(reinterpret_cast<const volatile uint8_t*>(scr) + k3_index_byte<(STRIDE > 0 ? STRIDE : 1)>(B));
    } else {
        ix = nib8<sh>(N[m]);
        if constexpr (HEAVY) ix += nib128<sh>(Nh[m]);
    }
    const uint32_t thr = *reinterpret_cast<const uint32_t*>(Ub + ix + B * kRow3 * 4);
    return decide_acc(k3_mix(S.sb[B], ph, mc), thr, w);
}

template <bool HEAVY, int B, int STRIDE>
__device__ __forceinline__ void k3_decide_rec(const uint8_t* Ub, const uint32_t (&N)[4], const uint32_t (&Nh)[4],
                                              const PTShared& S, uint64_t ph, const MixConsts& mc, uint32_t& w,
                                              uint32_t& tmin, const uint8_t* scr) {
    static_assert(B & 1, "pairs (B, B - 1)");
    const uint32_t d1 = k3_decide_one<HEAVY, B, STRIDE>(Ub, N, Nh, S, ph, mc, w, scr);
    const uint32_t d0 = k3_decide_one<HEAVY, B - 1, STRIDE>(Ub, N, Nh, S, ph, mc, w, scr);
    if constexpr (TAPT_K3_UM1)
        tmin = min(tmin, min(d1, d0));
    else
        tmin = min(min(tmin, d1 + 1u), d0 + 1u);
    if constexpr (B > 1) k3_decide_rec<HEAVY, B - 2, STRIDE>(Ub, N, Nh, S, ph, mc, w, tmin, scr);
}

// Exact 64-bit decisions (tie band, p ~ 2^-31 per site word).
__device__ __noinline__ uint32_t k3_decide_exact(const PTArgs& a, const PTShared& S, int off, uint32_t A0, uint32_t A1,
                                                 uint32_t A2, uint32_t A3, uint32_t A4, uint32_t A5, uint32_t A6,
                                                 uint64_t ph, int nv) {
    const uint32_t A[7] = {A0, A1, A2, A3, A4, A5, A6};
    uint32_t up = 0;
    for (int b = 0; b < nv; ++b) {
        int acc = 0;
        for (int p = 0; p < 7; ++p) acc |= (int)((A[p] >> b) & 1u) << p;
        const uint64_t T = a.thr[(size_t)S.slot_of[b] * a.nidx + off + 2 * acc];
        if (below(mix_final(S.sb[b] + ph), T)) up |= 1u << b;
    }
    return up;
}

// Sliced U(s) = s ? S' - acc : acc over P planes, for s = new and s = old, and
// C += U(new) + (2^P - 1 - U(old)) (P + 1 planes, one ripple through the counters).
template <int P>
__device__ __forceinline__ void k3_energy(uint32_t (&C)[kC3], const uint32_t (&A)[7], uint32_t sp, uint32_t nw,
                                          uint32_t old) {
    uint32_t T[P + 1];
    uint32_t c = 0xFFFFFFFFu, ct = 0;  // D = S' + ~acc + 1 (carry c); T = U(new) + ~U(old) (carry ct)
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const uint32_t sb = (uint32_t)((int32_t)(sp << (31 - p)) >> 31);
        const uint32_t na = ~A[p];
        const uint32_t D = sb ^ na ^ c;
        c = maj3(sb, na, c);
        const uint32_t un = (nw & D) | (~nw & A[p]);
        const uint32_t uo = ~((old & D) | (~old & A[p]));
        if (p == 0)
            ha(un, uo, T[0], ct);
        else
            fa(un, uo, ct, T[p], ct);
    }
    T[P] = ct;
    uint32_t cc;
    ha(C[0], T[0], C[0], cc);
#pragma unroll
    for (int k = 1; k <= P; ++k) fa(C[k], T[k], cc, C[k], cc);
#pragma unroll
    for (int k = P + 1; k < kC3; ++k) ha(C[k], cc, C[k], cc);
}

struct Csr3 {
    const uint4* meta;         // [n_free] by class position: site, rank, adj start, off+32768 | nch<<16 | S'<<20
    const uint32_t* adj;       // [nadj] byte offsets into the instance word image
    const uint32_t* class_ptr; // [n_classes+1]
    int n_classes;
    int nadj;
    int n2;                    // words of the instance image (2n + 2, rounded up to 4)
    int nidx4;                 // staged slot-table row stride (nidx rounded up to 4)
};

// Split sites: spread bit j of x to bit Q j.
template <int Q>
__device__ __forceinline__ uint32_t spread_q(uint32_t x) {
    if constexpr (Q == 4) {
        x &= 0xFFu;
        x = (x | (x << 12)) & 0x000F000Fu;
        x = (x | (x << 6)) & 0x03030303u;
        return (x | (x << 3)) & 0x11111111u;
    } else {
        x &= 0xFFFFu;
        x = (x | (x << 8)) & 0x00FF00FFu;
        x = (x | (x << 4)) & 0x0F0F0F0Fu;
        x = (x | (x << 2)) & 0x33333333u;
        return (x | (x << 1)) & 0x55555555u;
    }
}

// Split sites: decision of replica B = Q J + q (N nibble k of N[m] is replica 4k + m, so B sits in
// Ns[J % (4/Q)] = N[Q (J % (4/Q)) + q] at nibble J / (4/Q)).  Ubq / sbq: this lane's first row / base.
template <bool HEAVY, int Q, int J>
__device__ __forceinline__ void k3q_decide_rec(const uint8_t* Ubq, const uint32_t (&Ns)[4 / Q],
                                               const uint32_t (&Nhs)[4 / Q], const uint64_t* sbq, uint64_t ph,
                                               const MixConsts& mc, uint32_t& w, uint32_t& tmin,
                                               uint32_t (&ix8)[32 / Q]) {
    constexpr int r = J % (4 / Q), sh = 4 * (J / (4 / Q));
    uint32_t ix = nib8<sh>(Ns[r]);
    if constexpr (HEAVY) ix += nib128<sh>(Nhs[r]);
    ix8[J] = ix;
    const uint32_t thr = *reinterpret_cast<const uint32_t*>(Ubq + ix + Q * J * kRow3 * 4);
    tmin = min(tmin, decide_acc(k3_mix(sbq[Q * J], ph, mc), thr, w) + (TAPT_K3_UM1 ? 0u : 1u));
    if constexpr (J > 0) k3q_decide_rec<HEAVY, Q, J - 1>(Ubq, Ns, Nhs, sbq, ph, mc, w, tmin, ix8);
}

// Process one class position (site) of this team's instance.
template <bool HW, int STRIDE>
__device__ __forceinline__ void k3_site(const PTArgs& a, const PTShared& S, const uint4 md, uint8_t* W2,
                                        const uint32_t* adj, const uint8_t* ub0, int n, uint32_t vmask, int nv,
                                        uint32_t (&C)[kC3], int& corr, uint32_t* scr_w) {
    const uint32_t i = md.x;
    const uint64_t ph = (uint64_t)(md.y & 0xFFFFFFu) * kPhi;
    const int off = (int)(md.w & 0xFFFFu) - 32768;
    const int nch = (int)((md.w >> 16) & 15u);
    const uint32_t sp = (md.w >> 20) & 127u;
    const bool heavy = HW && ((md.w >> 27) & 1u);
    const uint32_t* ap = adj + md.z;
    uint32_t A[7];
    if (heavy) {  // A = hc + sum over chunks of (count << weight), 7 planes
        const uint32_t hc = md.y >> 24;
#pragma unroll
        for (int p = 0; p < 7; ++p) A[p] = ((hc >> p) & 1u) ? 0xFFFFFFFFu : 0u;
        for (int ch = 0; ch < nch; ++ch) {
            uint32_t P[5];
            chunk_count(W2, ap + 16 * ch, P);
            uint32_t c;
            if ((md.w >> (28 + ch)) & 1u) {  // weight 2: planes 1..5
                ha(A[1], P[0], A[1], c);
#pragma unroll
                for (int p = 2; p < 6; ++p) fa(A[p], P[p - 1], c, A[p], c);
                A[6] ^= c;
            } else {
                ha(A[0], P[0], A[0], c);
#pragma unroll
                for (int p = 1; p < 5; ++p) fa(A[p], P[p], c, A[p], c);
                ha(A[5], c, A[5], c);
                A[6] ^= c;
            }
        }
    } else {
        uint32_t P[5];
        chunk_count(W2, ap, P);
#pragma unroll
        for (int p = 0; p < 5; ++p) A[p] = P[p];
        A[5] = A[6] = 0;
    }
    uint32_t N[4], Nh[4];
    nibbles4(A[0], A[1], A[2], A[3], N);
    if constexpr (HW) nibbles4(A[4], A[5], A[6], 0u, Nh);
    const uint32_t old = *reinterpret_cast<const uint32_t*>(W2 + 4 * i);
    // the site's threshold base as one register (otherwise 4*off is re-added in every decision)
    uint32_t ubr = (uint32_t)__cvta_generic_to_shared(ub0) + (uint32_t)(4 * off);
    asm("mov.b32 %0, %0;" : "+r"(ubr));
    const uint8_t* Ub = reinterpret_cast<const uint8_t*>(__cvta_shared_to_generic(ubr));
    uint32_t w = 0, tmin = 0xFFFFFFFFu;
    if constexpr (!HW && STRIDE > 0) k3_index_bytes<(STRIDE > 0 ? STRIDE : 1)>(scr_w, N);
    k3_decide_rec<HW, kW - 1, STRIDE>(Ub, N, Nh, S, ph, a.mc, w, tmin, reinterpret_cast<const uint8_t*>(scr_w));
    uint32_t nw = ~w & vmask;
    if (tmin <= 2u) nw = k3_decide_exact(a, S, off, A[0], A[1], A[2], A[3], A[4], A[5], A[6], ph, nv);
    nw |= old & ~vmask;
    *reinterpret_cast<uint32_t*>(W2 + 4 * i) = nw;
    *reinterpret_cast<uint32_t*>(W2 + 4 * (n + i)) = ~nw;
    if (heavy) {
        k3_energy<7>(C, A, sp, nw, old);
        corr += 127;
    } else {
        k3_energy<4>(C, A, sp, nw, old);
        corr += 15;
    }
}

// Split sites: lane q of the site's group of Q lanes decides replicas Q j + q and adds
// 8 (U(new) - U(old)) of each to dU[j].  Called by the whole warp (full-mask shuffles); lanes past
// the end of the class (on = false) repeat a valid site and store nothing.
template <bool HW, int Q>
__device__ __forceinline__ void k3q_site(const PTArgs& a, const PTShared& S, const uint4 md, uint8_t* W2,
                                         const uint32_t* adj, const uint8_t* ubq, int n, uint32_t vmask, int nv, int q,
                                         bool on, int (&dU)[32 / Q]) {
    const uint32_t i = md.x;
    const uint64_t ph = (uint64_t)(md.y & 0xFFFFFFu) * kPhi;
    const int off = (int)(md.w & 0xFFFFu) - 32768;
    const int nch = (int)((md.w >> 16) & 15u);
    const int sp = (int)((md.w >> 20) & 127u);
    const bool heavy = HW && ((md.w >> 27) & 1u);
    const uint32_t* ap = adj + md.z;
    uint32_t A[7];
    if (heavy) {
        const uint32_t hc = md.y >> 24;
#pragma unroll
        for (int p = 0; p < 7; ++p) A[p] = ((hc >> p) & 1u) ? 0xFFFFFFFFu : 0u;
        for (int ch = 0; ch < nch; ++ch) {
            uint32_t P[5];
            chunk_count(W2, ap + 16 * ch, P);
            uint32_t c;
            if ((md.w >> (28 + ch)) & 1u) {
                ha(A[1], P[0], A[1], c);
#pragma unroll
                for (int p = 2; p < 6; ++p) fa(A[p], P[p - 1], c, A[p], c);
                A[6] ^= c;
            } else {
                ha(A[0], P[0], A[0], c);
#pragma unroll
                for (int p = 1; p < 5; ++p) fa(A[p], P[p], c, A[p], c);
                ha(A[5], c, A[5], c);
                A[6] ^= c;
            }
        }
    } else {
        uint32_t P[5];
        chunk_count(W2, ap, P);
#pragma unroll
        for (int p = 0; p < 5; ++p) A[p] = P[p];
        A[5] = A[6] = 0;
    }
    uint32_t N[4], Nh[4] = {0u, 0u, 0u, 0u};
    nibbles4(A[0], A[1], A[2], A[3], N);
    if constexpr (HW) nibbles4(A[4], A[5], A[6], 0u, Nh);
    uint32_t Ns[4 / Q], Nhs[4 / Q];
#pragma unroll
    for (int r = 0; r < 4 / Q; ++r) {
        const int m = Q * r + q;
        Ns[r] = m == 0 ? N[0] : m == 1 ? N[1] : m == 2 ? N[2] : N[3];
        Nhs[r] = m == 0 ? Nh[0] : m == 1 ? Nh[1] : m == 2 ? Nh[2] : Nh[3];
    }
    const uint32_t old = *reinterpret_cast<const uint32_t*>(W2 + 4 * i);
    uint32_t ubr = (uint32_t)__cvta_generic_to_shared(ubq) + (uint32_t)(4 * off);
    asm("mov.b32 %0, %0;" : "+r"(ubr));
    const uint8_t* Ub = reinterpret_cast<const uint8_t*>(__cvta_shared_to_generic(ubr));
    uint32_t w = 0, tmin = 0xFFFFFFFFu, ix8[32 / Q];
    k3q_decide_rec<HW, Q, 32 / Q - 1>(Ub, Ns, Nhs, &S.sb[q], ph, a.mc, w, tmin, ix8);
    uint32_t nw = spread_q<Q>(~w) << q;
#pragma unroll
    for (int d = 1; d < Q; d <<= 1) nw |= __shfl_xor_sync(0xFFFFFFFFu, nw, d);
    nw &= vmask;
    if (__any_sync(0xFFFFFFFFu, tmin <= 2u))
        nw = k3_decide_exact(a, S, off, A[0], A[1], A[2], A[3], A[4], A[5], A[6], ph, nv);
    nw |= old & ~vmask;
    if (on && q == 0) {
        *reinterpret_cast<uint32_t*>(W2 + 4 * i) = nw;
        *reinterpret_cast<uint32_t*>(W2 + 4 * (n + i)) = ~nw;
    }
    const uint32_t fl = on ? (nw ^ old) >> q : 0u, up = nw >> q;
    const int s8 = 8 * sp;
#pragma unroll
    for (int j = 0; j < 32 / Q; ++j) {
        const int d = 2 * (int)ix8[j] - s8;  // 8 (U(0) - U(1)) = 8 (2 acc - S')
        const int sg = -(int)((up >> (Q * j)) & 1u), f = -(int)((fl >> (Q * j)) & 1u);
        dU[j] += ((d ^ sg) - sg) & f;  // flipped: -d to up, +d to down
    }
}

// IPB: instance teams per CTA.  One instantiation per IPB so that each launch shape gets the whole
// register file for its threads (3 teams: 167 registers, +2 % on config 4 over a 512-thread bound).
// Q: lanes per site (1: one thread per site word; 2, 4: split sites, IPB = 1).
template <bool BAL, int IPB, int Q>
__global__ void __launch_bounds__(kT3 * Q * IPB, 1) k3_bitcsr_pt(const PTArgs a, const Csr3 g) {
    constexpr int TT = kT3 * Q;  // threads per instance team
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __shared__ PTShared SS[kIPB3];
    __shared__ int corr_sh[kIPB3];
    __shared__ uint64_t str_sh[kIPB3][kW];  // the instance's dynamics stream states by slot
    const int n = a.n, nidx = a.nidx, n_free = (int)a.n_free;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    const int ipb = nt / TT, kin = tid / TT, ti = tid - kin * TT;
    const SubTeam tm{ti, TT, 1 + kin};
    const int nv = own_count(a, 0);
    const uint32_t vmask = nv >= 32 ? 0xFFFFFFFFu : ((1u << nv) - 1u);
    // shared memory: Uslot [R][nidx4] | adj [nadj] | meta [n_free] (uint4) | class_ptr [n_classes+1] |
    // per team: Ub [32][kRow3] | W2 [n2]
    constexpr int XS = (TAPT_K3_IDXS && Q == 1) ? kT3 * IPB : 0;  // scratch stride (threads); 8 words per thread
    uint32_t* const scr_w = reinterpret_cast<uint32_t*>(smem_raw) + tid;
    uint32_t* Uslot = reinterpret_cast<uint32_t*>(smem_raw) + 8 * XS;
    uint32_t* adj = Uslot + (size_t)a.R * g.nidx4;
    uint4* meta = reinterpret_cast<uint4*>(adj + ((g.nadj + 3) & ~3));
    uint32_t* cptr = reinterpret_cast<uint32_t*>(meta + n_free);
    uint32_t* team0 = cptr + ((g.n_classes + 1 + 3) & ~3);
    const size_t team_words = (size_t)kW * kRow3 + g.n2;
    uint32_t* Ubuf = team0 + (size_t)kin * team_words;
    uint32_t* W2w = Ubuf + (size_t)kW * kRow3;
    uint8_t* W2 = reinterpret_cast<uint8_t*>(W2w);
    PTShared& S = SS[kin];
    for (int k = tid; k < a.R * g.nidx4; k += nt) {
        const int r = k / g.nidx4, x = k - r * g.nidx4;
        const uint32_t U = x < nidx ? thr_hi(a.thr[(size_t)r * nidx + x]) : 0u;
        Uslot[k] = TAPT_K3_UM1 ? max(U, 1u) - 1u : U;  // U - 1: h - (U - 1) in {0, 1, 2} is the tie band
    }
    for (int k = tid; k < g.nadj; k += nt) adj[k] = g.adj[k];
    for (int k = tid; k < n_free; k += nt) meta[k] = g.meta[k];
    for (int k = tid; k <= g.n_classes; k += nt) cptr[k] = g.class_ptr[k];
    pt_stage_swap(a);
    __syncthreads();  // the last CTA-wide barrier: teams are independent from here on

    const int unit = (int)blockIdx.x * ipb + kin;
    int it0, it1;
    if (BAL) {
        if (unit >= a.sched_clusters) return;
        it0 = a.sched_ptr[pt_timeline(unit, a.sched_clusters)];
        it1 = a.sched_ptr[pt_timeline(unit, a.sched_clusters) + 1];
    } else {
        if (unit >= a.I) return;
        it0 = 0;
        it1 = 1;
    }
    const uint8_t* ub0 = reinterpret_cast<const uint8_t*>(Ubuf);
    for (int it = it0; it < it1; ++it) {
        const SchedItem item = BAL ? a.sched[it] : SchedItem{unit, 0, a.n_sweeps, -1, -1};
        const int inst = item.inst;
        if (BAL && item.wait >= 0) pt_wait_flag(a, item.wait, tm);
        const uint64_t t0 = a.t0 + (uint64_t)item.s0;
        {
            const uint32_t* src = a.words + (size_t)inst * n;
            for (int k = ti; k < n; k += TT) {
                const uint32_t v = src[k];
                W2w[k] = v;
                W2w[n + k] = ~v;
            }
            if (ti == 0) {
                W2w[2 * n] = 0xFFFFFFFFu;
                W2w[2 * n + 1] = 0u;
            }
        }
        pt_load_perm(a, S, inst, tm);
        for (int r = ti; r < a.R; r += TT) str_sh[kin][r] = a.streams[(size_t)inst * a.R + r];
        for (int b = ti; b < nv; b += TT) S.Eown[(t0 + 1) & 1][b] = a.E[(size_t)inst * a.B + b];
        tm.sync();

        uint64_t pass = a.p0;
        if (a.swap_every > 0 && item.s0 > 0) pass += t0 / (uint64_t)a.swap_every - a.t0 / (uint64_t)a.swap_every;
        int par = (int)((t0 + 1) & 1);
        for (int s = item.s0; s < item.s1; ++s) {
            const uint64_t t = a.t0 + (uint64_t)s;
            const int prev = par;
            par = (int)(t & 1);
            {  // per-buffer stream bases for sweep t (pt_stream_bases with the staged stream states)
                const uint64_t k0 = a.draw_base + t * (uint64_t)a.n_free + 1ull;
                for (int b = ti; b < nv; b += TT) S.sb[b] = str_sh[kin][S.slot_of[b]] + k0 * kPhi;
            }
            // per-buffer threshold rows for the slots the buffers occupy this sweep
            for (int e = ti; e < kW * (kRow3 / 4); e += TT) {
                const int b = e / (kRow3 / 4), x4 = e - b * (kRow3 / 4);
                if (b < nv && 4 * x4 < g.nidx4)
                    reinterpret_cast<uint4*>(Ubuf)[e] =
                        reinterpret_cast<const uint4*>(Uslot + (size_t)S.slot_of[b] * g.nidx4)[x4];
            }
            tm.sync();
            if constexpr (Q > 1) {
                const int q = ti & (Q - 1);
                const uint8_t* ubq = ub0 + q * kRow3 * 4;
                int dU[32 / Q];
#pragma unroll
                for (int j = 0; j < 32 / Q; ++j) dU[j] = 0;
                for (int c = 0; c < g.n_classes; ++c) {
                    const int c0 = (int)cptr[c], c1 = (int)cptr[c + 1];
                    for (int base = c0; base < c1; base += TT / Q) {
                        const int qq = base + ti / Q;
                        const bool on = qq < c1;
                        const uint4 md = meta[on ? qq : c1 - 1];
                        const bool hw = __any_sync(0xFFFFFFFFu, on && ((md.w >> 27) & 1u));
                        if (hw)
                            k3q_site<true, Q>(a, S, md, W2, adj, ubq, n, vmask, nv, q, on, dU);
                        else
                            k3q_site<false, Q>(a, S, md, W2, adj, ubq, n, vmask, nv, q, on, dU);
                    }
                    tm.sync();
                }
                // E_b += 2 dU_b: dU (in eighths) summed over the lanes of the same q, then over warps
#pragma unroll
                for (int j = 0; j < 32 / Q; ++j) {
                    int v = dU[j];
#pragma unroll
                    for (int d = Q; d < 32; d <<= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
                    if (lane < Q && v != 0) atomicAdd(&S.Ucnt[Q * j + lane], (uint32_t)v);
                }
                tm.sync();
                for (int b = ti; b < nv; b += TT) {
                    S.Eown[par][b] = S.Eown[prev][b] + ((int32_t)S.Ucnt[b] >> 2);
                    S.Ucnt[b] = 0;
                }
                pt_epilogue<false>(a, S, W2w, inst, 0, t, pass, tm);
                continue;
            }
            uint32_t C[kC3];
#pragma unroll
            for (int k = 0; k < kC3; ++k) C[k] = 0;
            int corr = 0;
            for (int c = 0; c < g.n_classes; ++c) {
                const int c0 = (int)cptr[c], c1 = (int)cptr[c + 1];
                for (int base = c0; base < c1; base += kT3) {  // warp-uniform trip count
                    const int q = base + ti;
                    const bool on = q < c1;
                    const uint4 md = on ? meta[q] : make_uint4(0, 0, 0, 0);
                    const bool hw = __any_sync(0xFFFFFFFFu, on && ((md.w >> 27) & 1u));
                    if (on) {
                        if (hw)
                            k3_site<true, XS>(a, S, md, W2, adj, ub0, n, vmask, nv, C, corr, scr_w);
                        else
                            k3_site<false, XS>(a, S, md, W2, adj, ub0, n, vmask, nv, C, corr, scr_w);
                    }
                }
                tm.sync();
            }
            // E_b += 2 (sum over threads of C_b - sum of the per-site constants).  The 4 warps' sliced
            // counters are summed bit-sliced through shared memory (the threshold rows, rebuilt at the
            // start of every sweep, serve as scratch), then each warp transposes a quarter of the planes.
            {
                constexpr int kP = kC3 + 2;  // planes of the 4-warp sum
                const int wq = ti >> 5;      // warp in the team
                uint32_t* scr = Ubuf;        // [3][kC3][32] counters of warps 1..3 | [kP][32] sum | [4] corr
                uint32_t* sum = scr + 3 * kC3 * 32;
                int* csc = reinterpret_cast<int*>(sum + kP * 32);
                int cw = corr;
#pragma unroll
                for (int d = 16; d >= 1; d >>= 1) cw += __shfl_xor_sync(0xFFFFFFFFu, cw, d);
                if (wq > 0) {
#pragma unroll
                    for (int k = 0; k < kC3; ++k) scr[((wq - 1) * kC3 + k) * 32 + lane] = C[k];
                }
                if (lane == 0) csc[wq] = cw;
                tm.sync();
                if (wq == 0) {
                    uint32_t A[kP];
#pragma unroll
                    for (int k = 0; k < kC3; ++k) A[k] = C[k];
                    A[kC3] = A[kC3 + 1] = 0;
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        uint32_t c;
                        ha(A[0], scr[(q * kC3) * 32 + lane], A[0], c);
#pragma unroll
                        for (int k = 1; k < kC3; ++k) fa(A[k], scr[(q * kC3 + k) * 32 + lane], c, A[k], c);
                        ha(A[kC3], c, A[kC3], c);
                        A[kC3 + 1] ^= c;
                    }
#pragma unroll
                    for (int k = 0; k < kP; ++k) sum[k * 32 + lane] = A[k];
                    if (lane == 0) corr_sh[kin] = csc[0] + csc[1] + csc[2] + csc[3];
                }
                tm.sync();
                uint32_t tot = 0;
#pragma unroll
                for (int k = 0; k < kP; k += 4)
                    if (k + wq < kP) tot += (uint32_t)__popc(warp_transpose32(sum[(k + wq) * 32 + lane])) << (k + wq);
                if (lane < nv) atomicAdd(&S.Ucnt[lane], tot);
                tm.sync();
                for (int b = ti; b < nv; b += kT3) {
                    S.Eown[par][b] = S.Eown[prev][b] + 2 * ((int32_t)S.Ucnt[b] - corr_sh[kin]);
                    S.Ucnt[b] = 0;
                }
            }
            pt_epilogue<false>(a, S, W2w, inst, 0, t, pass, tm);
        }
        {
            uint32_t* dst = a.words + (size_t)inst * n;
            for (int k = ti; k < n; k += TT) dst[k] = W2w[k];
        }
        pt_finish<false>(a, S, inst, 0, par, tm);
        if (BAL && item.signal >= 0) pt_signal_flag<false>(a, item.signal, 0, tm);
        tm.sync();  // the team's shared memory is reused by the next item
    }
}

size_t k3_smem_bytes(int R, int nidx, int nadj, int nfree, int n, int ncls, int ipb) {
    const size_t nidx4 = ((size_t)nidx + 3) & ~size_t(3), n2 = ((size_t)2 * n + 2 + 3) & ~size_t(3);
    // (the index scratch of the one-lane-per-site shapes is counted for every shape: 8 words per thread)
    return ((TAPT_K3_IDXS ? (size_t)8 * kT3 * ipb : 0) + (size_t)R * nidx4 + (((size_t)nadj + 3) & ~size_t(3)) + 4 * (size_t)nfree +
            (((size_t)ncls + 1 + 3) & ~size_t(3)) +
            (size_t)ipb * ((size_t)kW * kRow3 + n2)) * 4;
}

int k3_row_stride() { return kRow3; }

template <int IPB, int Q>
static cudaError_t k3_shape_t(const PTArgs& a, const Csr3& g, size_t smem) {
    cudaError_t e =
        cudaFuncSetAttribute(k3_bitcsr_pt<false, IPB, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k3_bitcsr_pt<true, IPB, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return e;
}

template <int IPB, int Q>
static cudaError_t k3_run_t(const PTArgs& a, const Csr3& g, cudaStream_t st, int* resident) {
    const size_t smem = k3_smem_bytes(a.R, a.nidx, g.nadj, (int)a.n_free, a.n, g.n_classes, IPB);
    cudaError_t e = k3_shape_t<IPB, Q>(a, g, smem);
    if (e != cudaSuccess) return e;
    if (resident) {  // co-resident instance teams: CTAs per SM x SMs x IPB
        int per_sm = 0, dev = 0, nsm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k3_bitcsr_pt<true, IPB, Q>, kT3 * Q * IPB, smem);
        if (e == cudaSuccess) e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        *resident = per_sm * nsm * IPB;
        return e;
    }
    const unsigned grid = a.sched ? (unsigned)((a.sched_clusters + IPB - 1) / IPB) : (unsigned)((a.I + IPB - 1) / IPB);
    if (a.sched)
        k3_bitcsr_pt<true, IPB, Q><<<grid, kT3 * Q * IPB, smem, st>>>(a, g);
    else
        k3_bitcsr_pt<false, IPB, Q><<<grid, kT3 * Q * IPB, smem, st>>>(a, g);
    return cudaGetLastError();
}

// shape = IPB for one lane per site (IPB 1..4); -2 / -4: split sites with Q = 2 / 4 lanes (IPB 1)
static cudaError_t k3_run(const PTArgs& a, const Csr3& g, int shape, cudaStream_t st, int* resident) {
    switch (shape) {
        case -4: return k3_run_t<1, 4>(a, g, st, resident);
        case -2: return k3_run_t<1, 2>(a, g, st, resident);
        case 1: return k3_run_t<1, 1>(a, g, st, resident);
        case 2: return k3_run_t<2, 1>(a, g, st, resident);
        case 3: return k3_run_t<3, 1>(a, g, st, resident);
        default: return k3_run_t<4, 1>(a, g, st, resident);
    }
}

// Co-resident instance teams of the K3 launch shape (balanced schedule).
int k3_resident_units(const PTArgs& a, const Csr3& g, int shape) {
    int r = 0;
    return k3_run(a, g, shape, nullptr, &r) == cudaSuccess ? r : 0;
}

cudaError_t launch_k3(const PTArgs& a, const Csr3& g, int shape, cudaStream_t st) {
    return k3_run(a, g, shape, st, nullptr);
}

}  // namespace tapt_dev
