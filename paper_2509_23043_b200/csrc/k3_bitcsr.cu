// k3_bitcsr.cu -- K3: bit-sliced parallel-tempering kernel for integer CSR graphs with small
// couplings (BASELINE config 4: |J| in {1, 2}, sum |J| per site <= 63), colour-class order.
//
// K2 gives each site word to four lanes and sums the neighbour contributions of its 32
// replicas in byte lanes (~72 instructions per update on config 4).  K3 follows K1 instead:
// one thread owns a site word (32 replicas, bit b = replica b) and
//   * accumulates acc_b = sum over neighbours of |J| [J s_j > 0] in bit planes (weighted
//     ripple adds, 4 planes; 6 for "heavy" sites with sum |J| > 15),
//   * spreads the planes into nibbles (N[m] nibble k = acc of replica 4k+m),
//   * decides the 32 replicas with K1's carry-chain test against per-buffer threshold rows
//     laid out with a compile-time stride, so a replica's threshold is LDS [4*idx + imm]:
//     l = h - sum|J| + 2 acc, idx = l - lmin = off_i + 2 acc,
//   * counts energies exactly: every edge is scored once, at its later-updated endpoint (its
//     "early" neighbours -- earlier colour classes and clamped sites -- come first in the
//     site's adjacency), as weighted unsatisfied-bond planes into sliced counters; plus the
//     field terms.  E_b = 2 U_b + Ek[inst] (Ek: the clamped-only terms and -sum of weights).
// Same streams, tables, permutation, swap epilogue and observables as K1/K2 (pt_common.cuh);
// results are identical to K2's colour order (tests/test_gpu_parity.py).
#include <cuda_runtime.h>

#include "pt_common.cuh"

namespace tapt_dev {

constexpr int kUS = 128;     // threshold row stride (entries) of the per-buffer table
constexpr int kC3 = 10;      // sliced energy-counter planes (per-thread unsat weight per sweep < 1024)
constexpr int kTPI = 128;    // threads per instance
constexpr int kIPB3 = 2;     // instances per CTA

// Adjacency entry: bits 0..23 neighbour index, bit 24 sign of J (1: J < 0), bits 25..30 |J|.
__device__ __forceinline__ uint32_t adj_col(uint32_t e) { return e & 0xFFFFFFu; }
__device__ __forceinline__ uint32_t adj_sign(uint32_t e) { return (uint32_t)((int32_t)(e << 7) >> 31); }
__device__ __forceinline__ uint32_t adj_bit(uint32_t e, int k) { return (uint32_t)((int32_t)(e << (6 - k)) >> 31); }

// P += a0 + 2 a1 (a 2-bit addend per replica): one half adder, one full adder, then the carry.
template <int K>
__device__ __forceinline__ void plane_add2(uint32_t (&P)[K], uint32_t a0, uint32_t a1) {
    const uint32_t c0 = P[0] & a0;
    P[0] ^= a0;
    uint32_t c = maj3(P[1], a1, c0);
    P[1] ^= a1 ^ c0;
#pragma unroll
    for (int p = 2; p < K; ++p) {
        const uint32_t t = P[p] & c;
        P[p] ^= c;
        c = t;
    }
}

// P += v * w for an edge entry: the |J| bits 0, 1 through plane_add2, bits 2..5 (rare) one by one.
template <int K>
__device__ __forceinline__ void plane_add_edge(uint32_t (&P)[K], uint32_t v, uint32_t e);

// Bit-sliced add of plane v with weight 2^k into planes P[0..K).
template <int K>
__device__ __forceinline__ void plane_add(uint32_t (&P)[K], uint32_t v, int k) {
    uint32_t c = v;
#pragma unroll
    for (int p = 0; p < K; ++p) {
        if (p >= k) {
            const uint32_t t = P[p] & c;
            P[p] ^= c;
            c = t;
        }
    }
}

template <int K>
__device__ __forceinline__ void plane_addw(uint32_t (&P)[K], uint32_t v, uint32_t w) {
#pragma unroll
    for (int k = 0; k < K; ++k)
        if ((w >> k) & 1u) plane_add<K>(P, v, k);
}

template <int K>
__device__ __forceinline__ void plane_add_edge(uint32_t (&P)[K], uint32_t v, uint32_t e) {
    plane_add2<K>(P, v & adj_bit(e, 0), v & adj_bit(e, 1));
    if (e & 0x78000000u) {  // |J| >= 4
#pragma unroll
        for (int k = 2; k < 6 && k < K; ++k)
            if ((e >> (25 + k)) & 1u) plane_add<K>(P, v, k);
    }
}

// C += T for a 6-plane site sum T into the K-plane counters (ripple of full adders).
template <int K>
__device__ __forceinline__ void planes_accumulate(uint32_t (&C)[K], const uint32_t (&T)[6]) {
    uint32_t c = 0;
#pragma unroll
    for (int p = 0; p < 6; ++p) {
        const uint32_t s = C[p] ^ T[p] ^ c;
        c = maj3(C[p], T[p], c);
        C[p] = s;
    }
#pragma unroll
    for (int p = 6; p < K; ++p) {
        const uint32_t t = C[p] & c;
        C[p] ^= c;
        c = t;
    }
}

// 4 planes -> nibbles: nibble k of N[m] = (P0..P3) of replica 4k+m.
__device__ __forceinline__ void nibbles4(const uint32_t (&P)[4], uint32_t (&N)[4]) {
    const uint32_t e01 = (P[0] & 0x55555555u) | ((P[1] << 1) & 0xAAAAAAAAu);
    const uint32_t o01 = ((P[0] >> 1) & 0x55555555u) | (P[1] & 0xAAAAAAAAu);
    const uint32_t e23 = (P[2] & 0x55555555u) | ((P[3] << 1) & 0xAAAAAAAAu);
    const uint32_t o23 = ((P[2] >> 1) & 0x55555555u) | (P[3] & 0xAAAAAAAAu);
    constexpr uint32_t M = 0x33333333u;
    N[0] = (e01 & M) | ((e23 << 2) & ~M);
    N[1] = (o01 & M) | ((o23 << 2) & ~M);
    N[2] = ((e01 >> 2) & M) | (e23 & ~M);
    N[3] = ((o01 >> 2) & M) | (o23 & ~M);
}

struct Csr3 {
    const uint32_t* rowptr;  // [n+1] into adj
    const uint32_t* adj;     // [nnz] col | sign << 24 | |J| << 25, early neighbours first
    const uint32_t* meta;    // [n] (off_i + 32768) | n_early << 16 | heavy << 31 (free sites)
    const int32_t* h;        // [n]
    const uint32_t* rank;    // [n]
};

template <bool HEAVY>
__device__ __forceinline__ uint32_t k3_decide(const uint32_t* Ub, int off, const uint32_t (&N)[4], const uint32_t (&Nh)[4],
                                              const PTShared& S, uint64_t ph, const MixConsts& mc, bool& tie) {
    uint32_t w = 0, tmin = 0xFFFFFFFFu;
#pragma unroll
    for (int b = kW - 1; b >= 0; --b) {
        const int m = b & 3, sh = 4 * (b >> 2);
        uint32_t acc = (N[m] >> sh) & 15u;
        if constexpr (HEAVY) acc += ((Nh[m] >> sh) & 3u) << 4;
        const uint32_t thr = Ub[b * kUS + off + 2 * (int)acc];
        const uint64_t z = S.sb[b] + ph;
        const uint32_t h = mix_pre_hi<TAPT_K1_VARIANT>((uint32_t)z, (uint32_t)(z >> 32), mc);
        tmin = min(tmin, decide_acc(h, thr, w) + 1u);
    }
    tie |= tmin <= 2u;
    return w;  // NOT(up) bits
}

template <bool HEAVY>
__device__ __forceinline__ uint32_t k3_decide_exact(const PTArgs& a, const PTShared& S, int off,
                                                    const uint32_t (&N)[4], const uint32_t (&Nh)[4], uint64_t ph, int nv) {
    uint32_t up = 0;
    for (int b = 0; b < nv; ++b) {
        const int m = b & 3, sh = 4 * (b >> 2);
        uint32_t acc = (N[m] >> sh) & 15u;
        if (HEAVY) acc += ((Nh[m] >> sh) & 3u) << 4;
        const uint64_t T = a.thr[(size_t)S.slot_of[b] * a.nidx + off + 2 * acc];
        if (below(mix_final(S.sb[b] + ph), T)) up |= 1u << b;
    }
    return up;
}

__global__ void __launch_bounds__(kTPI * kIPB3, 2) k3_bitcsr_pt(const PTArgs a, const Csr3 g3, const CsrArgs g,
                                                                  const int32_t* Ek) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __shared__ PTShared SS[kIPB3];
    const int n = a.n, nidx = a.nidx;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    const int kin = tid / kTPI, ti = tid - kin * kTPI;  // instance slot, thread within it
    const int inst0 = blockIdx.x * kIPB3;
    const int nin = min(kIPB3, a.I - inst0);
    const bool active = kin < nin;
    const int nv = own_count(a, 0);
    const uint32_t vmask = nv >= 32 ? 0xFFFFFFFFu : ((1u << nv) - 1u);
    // shared memory: Uslot [R][nidx] | Ubuf [ipb][32][kUS] | words [ipb][n] | staged graph
    uint32_t* Uslot = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* Ubuf = Uslot + (size_t)a.R * nidx;
    uint32_t* wbase = Ubuf + (size_t)kIPB3 * kW * kUS;
    uint32_t* rp = wbase + (size_t)kIPB3 * n;
    uint32_t* adj = rp + (n + 1);
    uint32_t* meta = adj + g.nnz;
    uint32_t* rk = meta + n;
    uint32_t* cs = rk + n;
    for (int k = tid; k <= n; k += nt) rp[k] = g3.rowptr[k];
    for (int k = tid; k < g.nnz; k += nt) adj[k] = g3.adj[k];
    for (int k = tid; k < n; k += nt) {
        meta[k] = g3.meta[k];
        rk[k] = g3.rank[k];
    }
    for (int k = tid; k < (int)g.n_free; k += nt) cs[k] = g.class_sites[k];
    for (int k = tid; k < a.R * nidx; k += nt) Uslot[k] = thr_hi(a.thr[k]);
    for (int q = 0; q < nin; ++q) {
        const int ik = inst0 + q;
        for (int k = tid; k < n; k += nt) wbase[(size_t)q * n + k] = a.words[(size_t)ik * n + k];
        pt_load_perm(a, SS[q], ik);
    }
    __syncthreads();

    PTShared& S = SS[active ? kin : 0];
    uint32_t* words = wbase + (size_t)(active ? kin : 0) * n;
    const uint32_t* Ub = Ubuf + (size_t)(active ? kin : 0) * kW * kUS;
    uint64_t pass = a.p0;
    int par = 0;
    for (int s = 0; s < a.n_sweeps; ++s) {
        const uint64_t t = a.t0 + (uint64_t)s;
        par = (int)(t & 1);
        for (int q = 0; q < nin; ++q) pt_stream_bases(a, SS[q], inst0 + q, 0, t);
        // per-buffer threshold rows for the slots the buffers occupy this sweep
        for (int e = tid; e < nin * kW * kUS; e += nt) {
            const int q = e / (kW * kUS), r = e - q * kW * kUS, b = r / kUS, x = r - b * kUS;
            Ubuf[e] = (b < nv && x < nidx) ? Uslot[SS[q].slot_of[b] * nidx + x] : 0u;
        }
        __syncthreads();
        uint32_t C[kC3];
#pragma unroll
        for (int k = 0; k < kC3; ++k) C[k] = 0;
        for (int c = 0; c < g.n_classes; ++c) {
            const uint32_t c0 = g.class_ptr[c], c1 = g.class_ptr[c + 1];
            for (uint32_t q = c0 + (uint32_t)ti; active && q < c1; q += (uint32_t)kTPI) {
                const uint32_t i = cs[q];
                const uint32_t mt = meta[i];
                const int off = (int)(mt & 0xFFFFu) - 32768;
                const uint32_t r0 = rp[i], r1 = rp[i + 1], nearly = (mt >> 16) & 0x7FFFu;
                const bool heavy = (mt >> 31) != 0;
                uint32_t P[6] = {0, 0, 0, 0, 0, 0};
                for (uint32_t k = r0; k < r1; ++k) {
                    const uint32_t e = adj[k];
                    plane_add_edge<6>(P, words[adj_col(e)] ^ adj_sign(e), e);
                }
                uint32_t N[4], Nh[4];
                {
                    const uint32_t P4[4] = {P[0], P[1], P[2], P[3]};
                    nibbles4(P4, N);
                    const uint32_t H4[4] = {P[4], P[5], 0u, 0u};
                    nibbles4(H4, Nh);
                }
                const uint64_t ph = (uint64_t)rk[i] * kPhi;
                bool tie = false;
                uint32_t nw = heavy ? k3_decide<true>(Ub, off, N, Nh, S, ph, a.mc, tie)
                                    : k3_decide<false>(Ub, off, N, Nh, S, ph, a.mc, tie);
                nw = ~nw & vmask;
                if (tie) nw = heavy ? k3_decide_exact<true>(a, S, off, N, Nh, ph, nv)
                                    : k3_decide_exact<false>(a, S, off, N, Nh, ph, nv);
                words[i] = nw;
                // energy: early edges (final on both ends now) and the field as weighted
                // unsatisfied planes of this site (< 64), then folded into the counters
                uint32_t U[6] = {0, 0, 0, 0, 0, 0};
                for (uint32_t k = r0; k < r0 + nearly; ++k) {
                    const uint32_t e = adj[k];
                    plane_add_edge<6>(U, nw ^ words[adj_col(e)] ^ adj_sign(e), e);
                }
                const int hi = g3.h[i];
                if (hi != 0) plane_addw<6>(U, hi > 0 ? ~nw : nw, (uint32_t)(hi > 0 ? hi : -hi));
                planes_accumulate<kC3>(C, U);
            }
            __syncthreads();
        }
        // E_b = 2 U_b + Ek: reduce the per-thread planes of each instance's warps
        {
            const uint32_t tot = warp_sliced_total<kC3>(C);
            if (active && lane < nv) atomicAdd(&S.Ucnt[lane], tot);
            __syncthreads();
            for (int e = tid; e < nin * nv; e += nt) {
                const int q = e / nv, b = e - q * nv;
                SS[q].Eown[par][b] = 2 * (int32_t)SS[q].Ucnt[b] + Ek[inst0 + q];
                SS[q].Ucnt[b] = 0;
            }
        }
        uint64_t pass_k = pass;
        for (int q = 0; q < nin; ++q) {
            pass_k = pass;
            pt_epilogue<false>(a, SS[q], wbase + (size_t)q * n, inst0 + q, 0, t, pass_k);
        }
        pass = pass_k;
    }
    for (int q = 0; q < nin; ++q)
        for (int k = tid; k < n; k += nt) a.words[(size_t)(inst0 + q) * n + k] = wbase[(size_t)q * n + k];
    for (int q = 0; q < nin; ++q) pt_finish<false>(a, SS[q], inst0 + q, 0, par);
}

size_t k3_smem_bytes(int n, int R, int nidx, int nnz, int nfree) {
    return ((size_t)R * nidx + (size_t)kIPB3 * kW * kUS + (size_t)kIPB3 * n + (n + 1) + nnz + 2 * (size_t)n + nfree) * 4;
}

cudaError_t launch_k3(const PTArgs& a, const CsrArgs& g, const uint32_t* rowptr3, const uint32_t* adj3,
                      const uint32_t* meta3, const int32_t* h, const int32_t* Ek, cudaStream_t st) {
    const size_t smem = k3_smem_bytes(a.n, a.R, a.nidx, g.nnz, (int)g.n_free);
    cudaError_t e = cudaFuncSetAttribute(k3_bitcsr_pt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const Csr3 g3{rowptr3, adj3, meta3, h, g.rank};
    k3_bitcsr_pt<<<(a.I + kIPB3 - 1) / kIPB3, kTPI * kIPB3, smem, st>>>(a, g3, g, Ek);
    return cudaGetLastError();
}

}  // namespace tapt_dev
