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
// l - lmin.  Energies are tracked per replica by exact integer dE = 2*s_old*l on flips.
#include <cuda_runtime.h>

#include "pt_common.cuh"

namespace tapt_dev {

struct K2Smem {
    PTShared S;
};

template <bool CLU>
__global__ void __launch_bounds__(256) k2_csr_pt(const PTArgs a, const CsrArgs g) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    K2Smem& sm = *reinterpret_cast<K2Smem*>(smem_raw);
    uint32_t* Uhi = reinterpret_cast<uint32_t*>(smem_raw + ((sizeof(K2Smem) + 127) & ~size_t(127)));  // [R][nidx]
    uint32_t* words = Uhi + (size_t)a.R * a.nidx;                              // [n]
    const int tid = threadIdx.x, nt = blockDim.x;
    const int inst = blockIdx.x / a.G, grp = blockIdx.x % a.G;
    const int n = a.n, W = a.W, nv = own_count(a, grp);
    const int8_t* Jrow = g.J + (size_t)(g.nJ > 1 ? inst : 0) * g.nnz;

    for (int k = tid; k < n; k += nt) words[k] = a.words[((size_t)inst * a.G + grp) * n + k];
    for (int k = tid; k < a.R * a.nidx; k += nt) Uhi[k] = thr_hi(a.thr[k]);
    pt_load_perm(a, sm.S, inst);
    for (int b = tid; b < nv; b += nt) sm.S.Eown[(a.t0 + 1) & 1][b] = a.E[(size_t)inst * a.B + grp * W + b];
    __syncthreads();

    uint64_t pass = a.p0;
    int par = (int)((a.t0 + 1) & 1);
    for (int s = 0; s < a.n_sweeps; ++s) {
        const uint64_t t = a.t0 + (uint64_t)s;
        const int prev = par;
        par = (int)(t & 1);
        pt_stream_bases(a, sm.S, inst, grp, t);
        __syncthreads();
        int32_t dE[kW];
#pragma unroll
        for (int b = 0; b < kW; ++b) dE[b] = 0;

        for (int c = 0; c < g.n_classes; ++c) {
            const uint32_t c0 = g.class_ptr[c], c1 = g.class_ptr[c + 1];
            for (uint32_t q = c0 + tid; q < c1; q += nt) {
                const uint32_t i = g.class_sites[q];
                uint32_t A[8];
#pragma unroll
                for (int m = 0; m < 8; ++m) A[m] = 0;
                int sumabs = 0;
                for (uint32_t k = g.rowptr[i]; k < g.rowptr[i + 1]; ++k) {
                    const int J = Jrow[k];
                    const uint32_t v = words[g.col[k]] ^ (J < 0 ? 0xFFFFFFFFu : 0u);
                    const uint32_t mag = (uint32_t)(J < 0 ? -J : J);
                    sumabs += (int)mag;
#pragma unroll
                    for (int m = 0; m < 8; ++m) A[m] += mag * ((v >> m) & 0x01010101u);
                }
                const int l0 = g.h[i] - sumabs;            // l = l0 + 2*acc
                const uint32_t old = words[i];
                const uint64_t ph = (uint64_t)g.rank[i] * kPhi;
                uint32_t nw = 0;
#pragma unroll
                for (int b = 0; b < kW; ++b) {
                    if (b < nv) {
                        const int acc = (int)((A[b & 7] >> (8 * (b >> 3))) & 0xFFu);
                        const int l = l0 + 2 * acc;
                        const int slot = sm.S.slot_of[grp * W + b];
                        const int idx = l - g.lmin;
                        const uint64_t z = sm.S.sb[b] + ph;
                        const uint32_t xh = mix_final_hi(z);
                        const uint32_t U = Uhi[slot * a.nidx + idx];
                        bool up;
                        if (xh != U)
                            up = xh < U;
                        else
                            up = below(mix_final(z), a.thr[(size_t)slot * a.nidx + idx]);
                        const bool was = (old >> b) & 1u;
                        if (up) nw |= 1u << b;
                        if (up != was) dE[b] += was ? 2 * l : -2 * l;
                    }
                }
                words[i] = nw | (old & ~((nv >= 32) ? 0xFFFFFFFFu : ((1u << nv) - 1u)));
            }
            __syncthreads();
        }
        // per-replica dE summed over the CTA
        {
            const int32_t tot = warp_reduce_scatter32(dE);
            const int lane = tid & 31;
            if (lane < nv) atomicAdd(&sm.S.Ucnt[lane], (uint32_t)tot);
            __syncthreads();
            if (tid < nv) {
                sm.S.Eown[par][tid] = sm.S.Eown[prev][tid] + (int32_t)sm.S.Ucnt[tid];
                sm.S.Ucnt[tid] = 0;
            }
        }
        pt_epilogue<CLU>(a, sm.S, words, inst, grp, t, pass);
    }
    for (int k = tid; k < n; k += nt) a.words[((size_t)inst * a.G + grp) * n + k] = words[k];
    pt_finish<CLU>(a, sm.S, inst, grp, par);
}

size_t k2_smem_bytes(int n, int R, int nidx) {
    return ((sizeof(K2Smem) + 127) & ~size_t(127)) + (size_t)R * nidx * 4 + (size_t)n * 4;
}

template <bool CLU>
static cudaError_t launch_k2_t(const PTArgs& a, const CsrArgs& g, int threads, cudaStream_t st) {
    const size_t smem = k2_smem_bytes(a.n, a.R, a.nidx);
    auto fn = k2_csr_pt<CLU>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(a.I * a.G));
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
    return cudaLaunchKernelEx(&cfg, fn, a, g);
}

cudaError_t launch_k2(const PTArgs& a, const CsrArgs& g, int threads, bool cluster, cudaStream_t st) {
    return cluster ? launch_k2_t<true>(a, g, threads, st) : launch_k2_t<false>(a, g, threads, st);
}

}  // namespace tapt_dev
