// k2_csr.cu -- K2: fused parallel-tempering kernel for arbitrary integer Ising graphs
// (fields, clamps, any degree): factorization circuits (BASELINE config 4), open or
// clamped lattices, and the reference-order schedule used for bit-exact parity with
// the unmodified gibbs_sweep (proj/src/mcmc.cpp:30-45).
//
// Sites are visited class by class (class_ptr/class_sites): greedy colour classes for
// the parallel chain, or dependency levels for index order (level(i) = 1 + max level of
// lower-index neighbours: sites of one level are independent, and every lower-index
// neighbour of i sits on an earlier level while every higher-index one sits on a later
// level, so the level schedule reproduces the sequential index-ascending sweep).
//
// Local fields, byte-SWAR over 32 replicas: with the neighbour word v = w_j, negated for
// J < 0, acc = sum |J| * bit  counts into 8 words x 4 byte lanes (replica 8k+m in byte k
// of A[m]); then l = h_i - sum|J| + 2*acc exactly, and the threshold table is indexed by
// l - lmin.  Decisions use the carry-chain test of K1 (decide_acc).  Energies are tracked per
// replica by exact integer dE = 2*s_old*l on flips.
//
// Work split: four lanes share one site word (lane `sub` owns replicas 8k + 2*sub + {0,1});
// the neighbour walk is split over the four lanes and reduced with shuffles.  When an
// instance fits one CTA (R <= 32) a CTA carries up to kIPB instances that share the staged
// CSR and the threshold table; lane group q works on instance q % ipb, so every colour class
// gives each group several sites and the class barriers are amortised.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "pt_common.cuh"

namespace tapt_dev {

constexpr int kTPS = 4;  // lanes per site word
constexpr int kIPB = 4;  // max instances per CTA

__device__ __forceinline__ uint32_t prmt(uint32_t x, uint32_t y, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(y), "r"(sel));
    return r;
}

// Shared-memory image of the graph (the whole CSR is staged once per launch when it fits):
//   rowptr [n+1] u32 | col [nnz] u32 | hs [n] i32 | rank [n] u32 | class_sites [n_free] u32 | J [nnz] i8
__host__ __device__ inline size_t k2_graph_bytes(int n, int nnz, int nfree) {
    return ((size_t)(n + 1) + nnz + 2 * (size_t)n + nfree) * 4 + (((size_t)nnz + 15) & ~size_t(15));
}

// Graph arrays as seen by the sweep: shared-memory copies (SMEMG) or the global CSR.
struct K2Graph {
    const uint32_t* rowptr;
    const uint32_t* col;
    const int8_t* J;
    const int32_t* hs;  // h_i - sum |J_ik|
    const uint32_t* rank;
    const uint32_t* class_sites;
};

// BAL: run a balanced schedule's items (one instance per CTA); otherwise one pass over this CTA's
// instances (the loop below folds away and the register allocation is the single-pass one).
template <bool CLU, bool SMEMG, bool BAL>
__global__ void __launch_bounds__(TAPT_K2_MAXT, 1) k2_csr_pt(const PTArgs a, const CsrArgs g, const int ipb) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __shared__ PTShared SS[kIPB];
    const int nidx = a.nidx, n = a.n, W = a.W;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    // instances [inst0, inst0 + nin) of this CTA (ipb > 1 only without clusters: G == 1); with a
    // balanced schedule (ipb = 1) the cluster runs its items one after another
    const int grp = ipb > 1 ? 0 : (int)(blockIdx.x % a.G);
    const int cl = ipb > 1 ? (int)blockIdx.x : (int)(blockIdx.x / a.G);
    const int nv = own_count(a, grp);
    uint32_t* Uslot = reinterpret_cast<uint32_t*>(smem_raw);  // [R][nidx] high threshold words by slot
    uint32_t* wbase = Uslot + (size_t)a.R * nidx;               // [ipb][n]
    const int nfree = (int)g.n_free;
    // this thread's lane group, instance and position among that instance's groups
    const int grp_id = tid / kTPS, ngroups = nt / kTPS;
    const int mykin = grp_id % ipb;  // instance slot inside the CTA
    const int gi = grp_id / ipb, ngi = ngroups / ipb;
    K2Graph G;
    if constexpr (SMEMG) {  // stage the CSR next to the spins: every neighbour walk stays on-chip
        uint32_t* rp = wbase + (size_t)ipb * n;
        uint32_t* co = rp + (n + 1);
        int32_t* hh = reinterpret_cast<int32_t*>(co + g.nnz);
        uint32_t* rk = reinterpret_cast<uint32_t*>(hh + n);
        uint32_t* cs = rk + n;
        int8_t* jj = reinterpret_cast<int8_t*>(cs + nfree);
        for (int k = tid; k <= n; k += nt) rp[k] = g.rowptr[k];
        for (int k = tid; k < g.nnz; k += nt) {
            co[k] = g.col[k];
            jj[k] = g.J[k];  // shared couplings; per-instance couplings stay in global memory
        }
        for (int k = tid; k < n; k += nt) {
            hh[k] = TAPT_K2_HS ? g.hs[k] : g.h[k];
            rk[k] = g.rank[k];
        }
        for (int k = tid; k < nfree; k += nt) cs[k] = g.class_sites[k];
        G = K2Graph{rp, co, jj, hh, rk, cs};  // per-instance couplings: G.J set per item
    } else {
        G = K2Graph{g.rowptr, g.col, g.J, TAPT_K2_HS ? g.hs : g.h, g.rank, g.class_sites};
    }
    const int sub = tid & (kTPS - 1), m0 = 2 * sub;
    const uint32_t vmask = nv >= 32 ? 0xFFFFFFFFu : ((1u << nv) - 1u);
    const uint32_t mine = (0x03030303u << m0) & vmask;  // replicas of this lane
    // U - 1 (clamped at 0): the carry of h - (U - 1) and the tie band h - (U - 1) in {0, 1, 2}
    // come out of one subtraction (decisions with h = U - 1 fall in the band and are redone)
    for (int k = tid; k < a.R * nidx; k += nt) Uslot[k] = max(thr_hi(a.thr[k]), 1u) - 1u;

    const int tl = BAL ? pt_timeline(cl, a.sched_clusters) : 0;
    const int it0 = BAL ? a.sched_ptr[tl] : 0, it1 = BAL ? a.sched_ptr[tl + 1] : 1;
    for (int it = it0; it < it1; ++it) {
    const SchedItem item = BAL ? a.sched[it] : SchedItem{ipb > 1 ? cl * ipb : cl, 0, a.n_sweeps, -1, -1};
    const int inst0 = item.inst;
    const int nin = min(ipb, a.I - inst0);
    const bool active = mykin < nin;
    const int inst = inst0 + (active ? mykin : 0);
    PTShared& S = SS[active ? mykin : 0];
    uint32_t* words = wbase + (size_t)(active ? mykin : 0) * n;
    if (g.nJ > 1) G.J = g.J + (size_t)inst * g.nnz;  // per-instance couplings stay in global memory
    if (BAL && item.wait >= 0) pt_wait_flag(a, item.wait);
    const uint64_t t0 = a.t0 + (uint64_t)item.s0;  // first sweep of this item
    for (int kin = 0; kin < nin; ++kin) {
        const int ik = inst0 + kin;
        uint32_t* wk = wbase + (size_t)kin * n;
        for (int k = tid; k < n; k += nt) wk[k] = a.words[((size_t)ik * a.G + grp) * n + k];
        pt_load_perm(a, SS[kin], ik);
        for (int b = tid; b < nv; b += nt) SS[kin].Eown[(t0 + 1) & 1][b] = a.E[(size_t)ik * a.B + grp * W + b];
    }
    __syncthreads();

    // swap passes before this item: sweeps T = t+1 in (a.t0, t0] with swap_every | T
    uint64_t pass = a.p0;
    if (a.swap_every > 0 && item.s0 > 0) pass += t0 / (uint64_t)a.swap_every - a.t0 / (uint64_t)a.swap_every;
    int par = (int)((t0 + 1) & 1);
    for (int s = item.s0; s < item.s1; ++s) {
        const uint64_t t = a.t0 + (uint64_t)s;
        const int prev = par;
        par = (int)(t & 1);
        for (int kin = 0; kin < nin; ++kin) pt_stream_bases(a, SS[kin], inst0 + kin, grp, t);
        __syncthreads();
        // this lane's 8 replicas: threshold rows of their current slots, offset by -lmin so that
        // Uslot[trl + l] is the entry of local field l.  (A per-sweep copy of the rows indexed by
        // buffer with a compile-time stride, making the address 4l + an immediate, measured 4-9 %
        // slower on config 4: 32 KB more shared memory per CTA and bank conflicts.)
        int trl[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int b = 8 * (j >> 1) + m0 + (j & 1);
            trl[j] = (b < nv ? S.slot_of[grp * W + b] * nidx : 0) - g.lmin;
        }
        int32_t dE[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) dE[j] = 0;

        for (int c = 0; c < g.n_classes; ++c) {
            const uint32_t c0 = g.class_ptr[c], c1 = g.class_ptr[c + 1];
            // warp-uniform trip count (full-mask shuffles stay legal); lane groups past the end
            // of the class or without an instance run predicated off
            for (uint32_t base = c0; base < c1; base += (uint32_t)ngi) {
                const uint32_t q = base + (uint32_t)gi;
                const bool on = active && q < c1;
                const uint32_t i = on ? G.class_sites[q] : 0u;
                // neighbour walk split over the 4 lanes, byte-SWAR accumulators
                uint32_t A[8];
#pragma unroll
                for (int m = 0; m < 8; ++m) A[m] = 0;
#if !TAPT_K2_HS
                int sumabs = 0;
#endif
                if (on) {
                    const uint32_t r1 = G.rowptr[i + 1];
                    for (uint32_t k = G.rowptr[i] + sub; k < r1; k += kTPS) {
                        const int J = G.J[k];
                        const uint32_t v = words[G.col[k]] ^ (J < 0 ? 0xFFFFFFFFu : 0u);
                        const uint32_t mag = (uint32_t)(J < 0 ? -J : J);
#if !TAPT_K2_HS
                        sumabs += (int)mag;
#endif
#pragma unroll
                        for (int m = 0; m < 8; ++m) {
#if TAPT_K2_WALKHI
                            // shifts as IMAD.HI by runtime powers of two: FMA pipe instead of ALU
                            const uint32_t vm = m == 0 ? v : __umulhi(v, a.mc.sh[m]);
#else
                            const uint32_t vm = v >> m;
#endif
                            A[m] += mag * (vm & 0x01010101u);
                        }
                    }
                }
                // 4-lane reduce-scatter: lane `sub` ends with A[2 sub] and A[2 sub + 1] summed
                uint32_t Bh[4];
                const bool h2 = (sub & 2) != 0, h1 = (sub & 1) != 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t send = h2 ? A[k] : A[k + 4];
                    Bh[k] = (h2 ? A[k + 4] : A[k]) + __shfl_xor_sync(0xFFFFFFFFu, send, 2);
                }
                uint32_t A0, A1;
                {
                    const uint32_t s0 = h1 ? Bh[0] : Bh[2], s1 = h1 ? Bh[1] : Bh[3];
                    const uint32_t r0 = __shfl_xor_sync(0xFFFFFFFFu, s0, 1);
                    const uint32_t r1 = __shfl_xor_sync(0xFFFFFFFFu, s1, 1);
                    A0 = (h1 ? Bh[2] : Bh[0]) + r0;
                    A1 = (h1 ? Bh[3] : Bh[1]) + r1;
                }
#if !TAPT_K2_HS
                sumabs += __shfl_xor_sync(0xFFFFFFFFu, sumabs, 1);
                sumabs += __shfl_xor_sync(0xFFFFFFFFu, sumabs, 2);
#endif
                uint32_t nw = 0, old = 0;
                if (on) {
#if TAPT_K2_HS
                    const int hs = G.hs[i];  // l_j = hs + 2*acc_j, table index l_j - lmin
#else
                    const int hs = G.hs[i] - sumabs;  // G.hs holds h here
#endif
                    old = words[i];
                    const uint64_t ph = (uint64_t)G.rank[i] * kPhi;
                    uint32_t tmin = 0xFFFFFFFFu, w = 0;
                    int l[8];
                    // descending j: the carry chain leaves NOT(up_j) in bit j of w.  Replicas past
                    // nv read a valid row and a spare stream slot; their bits are masked below.
#pragma unroll
                    for (int j = 7; j >= 0; --j) {
                        l[j] = hs + 2 * (int)prmt((j & 1) ? A1 : A0, 0u, 0x4440u | (uint32_t)(j >> 1));
                        const uint32_t thr = Uslot[trl[j] + l[j]];
                        const uint64_t z = S.sb[8 * (j >> 1) + m0 + (j & 1)] + ph;
                        const uint32_t hh = mix_pre_hi<TAPT_K2_MIXV>((uint32_t)z, (uint32_t)(z >> 32), a.mc);
                        tmin = min(tmin, decide_acc(hh, thr, w));
                    }
                    if (tmin > 2u) {
                        // bits j -> positions 8*(j>>1) + (j&1), then shift to this lane's replicas
                        const uint32_t u = ~w & 0xFFu;
                        const uint32_t y = (u | (u << 12)) & 0x000F000Fu;
                        nw = (((y | (y << 6)) & 0x03030303u) << m0) & mine;
                    } else {  // |h - U| <= 1 somewhere (p ~ 2^-31): exact 64-bit decisions
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int b = 8 * (j >> 1) + m0 + (j & 1);
                            if (b < nv && below(mix_final(S.sb[b] + ph), a.thr[(size_t)(trl[j] + l[j])])) nw |= 1u << b;
                        }
                    }
                    // flip energy 2 s_old l = 2 l (old - new) per replica: byte-wise old - new in
                    // {-1, 0, 1}, sign-extended by PRMT, times l (the factor 2 is applied at the end)
                    const uint32_t O = (old & mine) >> m0, N = nw >> m0;
                    const uint32_t X0 = (((O & 0x01010101u) | 0x80808080u) - (N & 0x01010101u)) ^ 0x80808080u;
                    const uint32_t X1 = ((((O >> 1) & 0x01010101u) | 0x80808080u) - ((N >> 1) & 0x01010101u)) ^ 0x80808080u;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        constexpr uint32_t kSx[4] = {0x8880u, 0x9991u, 0xAAA2u, 0xBBB3u};
                        dE[j] += l[j] * (int)prmt((j & 1) ? X1 : X0, 0u, kSx[j >> 1]);
                    }
                }
                nw |= __shfl_xor_sync(0xFFFFFFFFu, nw, 1);
                nw |= __shfl_xor_sync(0xFFFFFFFFu, nw, 2);
                if (on && sub == 0) words[i] = nw | (old & ~vmask);
            }
            __syncthreads();
        }
        // per-replica dE: reduce over the lanes of this warp that own the same (instance,
        // replicas) -- group ids equal mod ipb -- then over warps with shared atomics
        {
            const int gw = lane >> 2;  // group index inside the warp (0..7)
#pragma unroll
            for (int bit = 0; bit < 3; ++bit) {
                const int d = 1 << bit;  // partner group gw ^ d has the same instance iff d % ipb == 0
                if ((d % ipb) == 0) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) dE[j] += __shfl_xor_sync(0xFFFFFFFFu, dE[j], d * kTPS);
                }
            }
            if (active && gw < ipb) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int b = 8 * (j >> 1) + m0 + (j & 1);
                    if (b < nv) atomicAdd(&S.Ucnt[b], (uint32_t)(2 * dE[j]));
                }
            }
            __syncthreads();
            for (int e = tid; e < nin * nv; e += nt) {
                const int kin = e / nv, b = e - kin * nv;
                SS[kin].Eown[par][b] = SS[kin].Eown[prev][b] + (int32_t)SS[kin].Ucnt[b];
                SS[kin].Ucnt[b] = 0;
            }
        }
        uint64_t pass_k = pass;
        for (int kin = 0; kin < nin; ++kin) {
            pass_k = pass;
            pt_epilogue<CLU>(a, SS[kin], wbase + (size_t)kin * n, inst0 + kin, grp, t, pass_k);
        }
        pass = pass_k;
    }
    for (int kin = 0; kin < nin; ++kin) {
        const uint32_t* wk = wbase + (size_t)kin * n;
        for (int k = tid; k < n; k += nt) a.words[((size_t)(inst0 + kin) * a.G + grp) * n + k] = wk[k];
    }
    for (int kin = 0; kin < nin; ++kin) pt_finish<CLU>(a, SS[kin], inst0 + kin, grp, par);
    if (BAL && item.signal >= 0) pt_signal_flag<CLU>(a, item.signal, grp);
    if (BAL) __syncthreads();  // shared memory is reused by the next item
    }
}

size_t k2_smem_bytes(int n, int R, int nidx) {
    // dynamic part for one instance: per-slot threshold rows + spin words (control blocks are static)
    return (size_t)R * nidx * 4 + (size_t)n * 4;
}

size_t k2_smem_bytes_graph(int n, int R, int nidx, int nnz, int nfree) {
    return k2_smem_bytes(n, R, nidx) + k2_graph_bytes(n, nnz, nfree);
}

template <bool CLU, bool SMEMG, bool BAL>
static cudaError_t launch_k2_t(const PTArgs& a, const CsrArgs& g, int threads, int ipb, cudaStream_t st,
                               int* resident) {
    size_t smem = (size_t)a.R * a.nidx * 4 + (size_t)ipb * a.n * 4;
    if (SMEMG) smem += k2_graph_bytes(a.n, g.nnz, (int)g.n_free);
    auto fn = k2_csr_pt<CLU, SMEMG, BAL>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.sched ? (unsigned)(a.sched_clusters * a.G)
                               : (ipb > 1 ? (unsigned)((a.I + ipb - 1) / ipb) : (unsigned)(a.I * a.G)));
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
    if (resident) {  // co-resident clusters / CTAs of this shape (balanced schedule)
        if (CLU) return cudaOccupancyMaxActiveClusters(resident, (const void*)fn, &cfg);
        int per_sm = 0, dev = 0, nsm = 0;
        cudaError_t q = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
        if (q == cudaSuccess) q = cudaGetDevice(&dev);
        if (q == cudaSuccess) q = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        *resident = per_sm * nsm;
        return q;
    }
    return pt_launch(fn, cfg.gridDim.x, (unsigned)threads, smem, st, CLU ? (unsigned)a.G : 1u, a, g, ipb);
}

// Instances per CTA when one CTA holds a whole instance (G == 1, no cluster): 2 measured best
// on config 4 (tools/k2_shapes.sh, updates/s: 512 threads x {1,2,4} -> 2.93 / 3.20 / 2.90e11; 256 threads
// x {1,2,4} -> 2.81 / 2.93 / 2.17e11).
int k2_instances_per_cta(const PTArgs& a, const CsrArgs& g) {
    if (a.G != 1) return 1;
    if (const char* e = std::getenv("TAPT_K2_IPB")) return std::max(1, std::min(kIPB, std::atoi(e)));
    const size_t fixed = (size_t)a.R * a.nidx * 4 + (g.smem_graph ? k2_graph_bytes(a.n, g.nnz, (int)g.n_free) : 0);
    if (fixed + 2 * (size_t)a.n * 4 <= 110 * 1024 && a.I >= 2) return 2;
    return 1;
}

static cudaError_t k2_dispatch(const PTArgs& a, const CsrArgs& g, int threads, bool cluster, cudaStream_t st,
                               int* resident, bool bal) {
    // a balanced schedule runs one instance per CTA (its jobs are single instances)
    const int ipb = (cluster || bal) ? 1 : k2_instances_per_cta(a, g);
    if (bal) {
        if (g.smem_graph)
            return cluster ? launch_k2_t<true, true, true>(a, g, threads, 1, st, resident)
                           : launch_k2_t<false, true, true>(a, g, threads, 1, st, resident);
        return cluster ? launch_k2_t<true, false, true>(a, g, threads, 1, st, resident)
                       : launch_k2_t<false, false, true>(a, g, threads, 1, st, resident);
    }
    if (g.smem_graph)
        return cluster ? launch_k2_t<true, true, false>(a, g, threads, 1, st, resident)
                       : launch_k2_t<false, true, false>(a, g, threads, ipb, st, resident);
    return cluster ? launch_k2_t<true, false, false>(a, g, threads, 1, st, resident)
                   : launch_k2_t<false, false, false>(a, g, threads, ipb, st, resident);
}

cudaError_t launch_k2(const PTArgs& a, const CsrArgs& g, int threads, bool cluster, cudaStream_t st) {
    return k2_dispatch(a, g, threads, cluster, st, nullptr, a.sched != nullptr);
}

// Co-resident clusters (or single-instance CTAs) of the K2 launch shape (balanced schedule).
int k2_resident_units(const PTArgs& a, const CsrArgs& g, int threads, bool cluster) {
    int r = 0;
    return k2_dispatch(a, g, threads, cluster, nullptr, &r, true) == cudaSuccess ? r : 0;
}

}  // namespace tapt_dev
