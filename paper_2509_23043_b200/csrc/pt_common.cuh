// pt_common.cuh -- the per-sweep epilogue shared by the fused PT kernels:
// energy gather across the CTAs of an instance (thread-block cluster / DSMEM),
// replica-exchange pass (Eq. 1), best-energy tracking and the
// per-slot observables (magnetization() numerator, spin_model.cpp:109-114).
#pragma once
#include <cooperative_groups.h>

#include <type_traits>
#include <utility>

#include "kernels.h"

namespace tapt_dev {

namespace cg = cooperative_groups;

// Thread teams.  CtaTeam: the whole CTA (K1, K2).  SubTeam: a warp-aligned group of threads
// with its own named barrier, so several instances share one CTA (and its staged graph) while
// progressing independently (K3).
struct CtaTeam {
    __device__ __forceinline__ int tid() const { return (int)threadIdx.x; }
    __device__ __forceinline__ int nt() const { return (int)blockDim.x; }
    __device__ __forceinline__ void sync() const { __syncthreads(); }
};
struct SubTeam {
    int t, n, bar;  // thread index in the team, team size (multiple of 32), barrier id (>= 1)
    __device__ __forceinline__ int tid() const { return t; }
    __device__ __forceinline__ int nt() const { return n; }
    __device__ __forceinline__ void sync() const { asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(n) : "memory"); }
};

struct PTShared {
    uint64_t sb[kW];        // stream base of each own buffer for the current sweep
    int32_t Eown[2][kW];    // energies of own buffers, double-buffered by sweep parity
    uint32_t Ucnt[kW];      // per-buffer unsatisfied-bond (or energy) accumulators
    uint32_t Mcnt[kW];      // per-buffer up-spin counts (measurement)
    int32_t Eall[kMaxR];    // energies of all buffers of the instance
    uint8_t slot_of[kMaxR];
    uint8_t buf_of[kMaxR];
    uint32_t sacc[kMaxR];   // swap accepts of this launch by pair (flushed by pt_finish)
    uint64_t coord;         // the instance's coordinator stream state (swap draws)
    int best;
    int tie;
};

// Swap-table metadata of each ladder pair, staged in shared memory once per launch so that a
// swap decision costs one dependent global load (the threshold) instead of four.
struct SwapMeta {
    uint32_t off, K;
    int64_t kz;
    uint32_t always;
    double c;
};
constexpr int kSwm = 128;
__shared__ SwapMeta g_swm[kSwm];

__device__ __forceinline__ void pt_stage_swap(const PTArgs& a) {
    if (a.swap_every <= 0 || a.R - 1 > kSwm || !a.swap_tab.off) return;
    for (int r = threadIdx.x; r < a.R - 1; r += blockDim.x)
        g_swm[r] = SwapMeta{a.swap_tab.off[r], a.swap_tab.K[r], a.swap_tab.kz[r], a.swap_tab.always[r],
                            a.swap_tab.c ? a.swap_tab.c[r] : -1.0};
}

// metro_accept (common.cuh) for swap pair r with the staged metadata.  Inside the table the
// decision  uniform < p_host = exp(-c k)  (libm, tabulated as T = ceil(p 2^53)) is taken from the
// device exp when the draw is outside a relative band of 1e-12 around it (device and host exp differ
// by a few ulp, ~1e-16), so the table -- a dependent global load -- is read only inside the band.
__device__ __forceinline__ bool pt_swap_accept(const PTArgs& a, int r, int64_t dE, uint64_t x) {
    if (a.R - 1 > kSwm) return metro_accept(a.swap_tab, r, dE, x);
    const SwapMeta m = g_swm[r];
    if (dE >= 0 || m.always) return true;
    const int64_t k = -dE;
    if (k >= (int64_t)m.K) return below(x, k <= m.kz ? 1ull : 0ull);
    if (m.c >= 0.0) {
        const double p = exp(m.c * -(double)k);
        const double u = (double)(x >> 11) * 0x1.0p-53;
        if (u < p * (1.0 - 1e-12)) return true;
        if (u > p * (1.0 + 1e-12)) return false;
    }
    return below(x, a.swap_tab.tab[m.off + k]);
}

// Number of valid buffers owned by group `grp` (the last group of an instance may be partial).
__device__ __forceinline__ int own_count(const PTArgs& a, int grp) { return min(a.W, a.B - grp * a.W); }

// Load the permutation of instance `inst` into shared memory.
// (A SubTeam caller stages the swap metadata once per CTA itself: pt_stage_swap.)
template <class TM = CtaTeam>
__device__ __forceinline__ void pt_load_perm(const PTArgs& a, PTShared& S, int inst, const TM& tm = TM{}) {
    const int t0 = tm.tid(), nt = tm.nt();
    for (int k = t0; k < a.B; k += nt) S.slot_of[k] = a.slot_of[(size_t)inst * a.B + k];
    if (a.buf_of)
        for (int k = t0; k < a.R; k += nt) S.buf_of[k] = a.buf_of[(size_t)inst * a.R + k];
    if (t0 == 0) {
        S.best = a.best ? a.best[inst] : 0x7FFFFFFF;
        S.tie = 0;
        S.coord = a.coord ? a.coord[inst] : 0ull;
    }
    for (int k = t0; k < kW; k += nt) {
        S.Ucnt[k] = 0;
        S.Mcnt[k] = 0;
    }
    for (int k = t0; k < a.R; k += nt) S.sacc[k] = 0;
    if constexpr (std::is_same_v<TM, CtaTeam>) pt_stage_swap(a);
}

// Per-buffer stream base for sweep t: S_slot + (draw_base + t*n_free + 1)*phi.
template <class TM = CtaTeam>
__device__ __forceinline__ void pt_stream_bases(const PTArgs& a, PTShared& S, int inst, int grp, uint64_t t,
                                                const TM& tm = TM{}) {
    const int nv = own_count(a, grp);
    for (int b = tm.tid(); b < nv; b += tm.nt()) {
        const int slot = S.slot_of[grp * a.W + b];
        const uint64_t k0 = a.draw_base + t * (uint64_t)a.n_free + 1ull;
        S.sb[b] = a.streams[(size_t)inst * a.R + slot] + k0 * kPhi;
    }
}

// After Eown[par] is final for this CTA: gather, best, swap, measure.
// `words` = this CTA's group spins in shared memory (n words).
// pack > 1 (K1's packed narrow groups): a word holds `pack` sites of 32/pack replicas each.
template <bool CLU, class TM = CtaTeam, int PACK = 1>
__device__ void pt_epilogue(const PTArgs& a, PTShared& S, const uint32_t* words, int inst, int grp, uint64_t t,
                            uint64_t& pass, const TM& tm = TM{}) {
    constexpr int pack = PACK;
    const int tid = tm.tid(), nt = tm.nt(), lane = tid & 31;
    const int par = (int)(t & 1);
    if constexpr (CLU) {
        cg::cluster_group cl = cg::this_cluster();
        cl.sync();
        for (int gb = tid; gb < a.B; gb += nt) {
            const int r = gb / a.W;
            const int32_t* peer = cl.map_shared_rank(&S.Eown[par][0], r);
            S.Eall[gb] = peer[gb - r * a.W];
        }
    } else {
        // Without a cluster only this CTA's buffers are visible; the host never asks
        // for swaps or best-energy tracking when an instance spans several CTAs here.
        tm.sync();
        for (int b = tid; b < own_count(a, grp); b += nt) S.Eall[grp * a.W + b] = S.Eown[par][b];
    }
    tm.sync();
    const uint64_t T = t + 1;
    if (tid < 32 && a.best) {  // warp-wide min over the instance's energies
        int m = 0x7FFFFFFF;
        for (int b = lane; b < a.B; b += 32) m = min(m, S.Eall[b]);
        m = __reduce_min_sync(0xFFFFFFFFu, m);
        if (lane == 0) S.best = min(S.best, m);
    }
    if (a.swap_every > 0 && (T % (uint64_t)a.swap_every) == 0) {
        const int parity = (int)(pass & 1);
        const uint64_t c0 = S.coord;
        for (int r = parity + 2 * tid; r + 1 < a.R; r += 2 * nt) {
            const int b0 = S.buf_of[r], b1 = S.buf_of[r + 1];
            const int64_t dE = (int64_t)S.Eall[b1] - (int64_t)S.Eall[b0];
            const uint64_t x = draw(c0, pass * (uint64_t)a.R + (uint64_t)r + 1ull);
            const bool acc = pt_swap_accept(a, r, dE, x);
            // attempts are deterministic (pass parity) and counted by the host; accepts are
            // counted here and flushed once per launch
            if (acc) S.sacc[r] += 1;
            if (acc) {
                S.buf_of[r] = (uint8_t)b1;
                S.buf_of[r + 1] = (uint8_t)b0;
                S.slot_of[b1] = (uint8_t)r;
                S.slot_of[b0] = (uint8_t)(r + 1);
            }
        }
        ++pass;
        tm.sync();
    }
    if (a.measure_every > 0 && T > a.measure_from && (T % (uint64_t)a.measure_every) == 0) {
        uint32_t C[kCnt];
#pragma unroll
        for (int k = 0; k < kCnt; ++k) C[k] = 0;
        for (int i = tid; i < a.n / pack; i += nt) sliced_add1<kCnt>(C, words[i]);
        const uint32_t tot = warp_sliced_total<kCnt>(C);
        if (pack > 1)
            atomicAdd(&S.Mcnt[lane & (kW / pack - 1)], tot);  // every field of the word is one of the group's replicas
        else if (lane < own_count(a, grp))
            atomicAdd(&S.Mcnt[lane], tot);
        tm.sync();
        if (tid < own_count(a, grp)) {
            const int gb = grp * a.W + tid;
            const int slot = S.slot_of[gb];
            const long long e = S.Eall[gb];
            const long long m = 2ll * (long long)S.Mcnt[tid] - a.n;
            long long* o = a.obs + ((size_t)inst * a.R + slot) * 5;
            atomicAdd((unsigned long long*)&o[0], 1ull);
            atomicAdd((unsigned long long*)&o[1], (unsigned long long)e);
            atomicAdd((unsigned long long*)&o[2], (unsigned long long)(e * e));
            atomicAdd((unsigned long long*)&o[3], (unsigned long long)(m < 0 ? -m : m));
            atomicAdd((unsigned long long*)&o[4], (unsigned long long)(m * m));
            if (a.hist && a.nbins > 0) {
                long long bin = e < a.e_lo ? 0 : (e - a.e_lo) / a.width;
                if (bin >= a.nbins) bin = a.nbins - 1;
                atomicAdd(&a.hist[(size_t)slot * a.nbins + bin], 1ull);
            }
            S.Mcnt[tid] = 0;
        }
        tm.sync();
    }
}

// Launch a fused PT kernel with an optional thread-block cluster of `cluster_x` CTAs.
template <class... KArgs, class... Args>
__host__ cudaError_t pt_launch(void (*fn)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                               unsigned cluster_x, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    int na = 0;
    if (cluster_x > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = cluster_x;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = na ? attr : nullptr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, fn, std::forward<Args>(args)...);
}

// Balanced schedule: the unit (cluster / CTA / team) of the persistent grid that runs timeline `m` of
// McNaughton's rule is M - 1 - m.  A job cut between timelines m and m+1 runs its first sweeps at the
// start of m+1 and waits for them at the end of m, so with the reversed numbering every wait is on a
// LOWER-numbered unit: one the hardware dispatched earlier (units are dispatched in index order),
// already resident or finished, whose producing item comes first on its timeline and itself waits
// only on lower units.  No wait can depend on a unit that is not yet resident, so the schedule makes
// progress however many units fit at once (e.g. while another stream holds SMs).
__device__ __forceinline__ int pt_timeline(int unit, int n_units) { return n_units - 1 - unit; }

// Balanced schedule (SchedItem): wait for / publish the state of a split job.  The wait is
// bounded (~2 s of clock64 at 1.9 GHz); on timeout it flags an error instead of hanging.
template <class TM = CtaTeam>
__device__ __forceinline__ void pt_wait_flag(const PTArgs& a, int f, const TM& tm = TM{}) {
    if (tm.tid() == 0) {
        const long long t0 = clock64();
        while (atomicAdd(&a.flags[f], 0u) == 0u) {
            if (clock64() - t0 > 4000000000ll) {
                atomicExch(a.sched_err, 1u);
                break;
            }
            __nanosleep(256);
        }
        __threadfence();
    }
    tm.sync();
}

template <bool CLU, class TM = CtaTeam>
__device__ __forceinline__ void pt_signal_flag(const PTArgs& a, int f, int grp, const TM& tm = TM{}) {
    __threadfence();  // this team's stores (spins, permutation, energies) before the flag
    tm.sync();
    if constexpr (CLU) cg::this_cluster().sync();
    if (grp == 0 && tm.tid() == 0) atomicExch(&a.flags[f], 1u);
}

// End of launch: persist permutation, energies of own buffers and best energy.
template <bool CLU, class TM = CtaTeam>
__device__ void pt_finish(const PTArgs& a, PTShared& S, int inst, int grp, int last_par, const TM& tm = TM{}) {
    const int tid = tm.tid(), nt = tm.nt();
    tm.sync();
    if (a.E)
        for (int b = tid; b < own_count(a, grp); b += nt)
            a.E[(size_t)inst * a.B + grp * a.W + b] = S.Eown[last_par][b];
    if (grp == 0) {
        for (int r = tid; r + 1 < a.R; r += nt)
            if (S.sacc[r]) a.swap_acc[(size_t)inst * (a.R - 1) + r] += S.sacc[r];
        for (int k = tid; k < a.B; k += nt) a.slot_of[(size_t)inst * a.B + k] = S.slot_of[k];
        if (a.buf_of)
            for (int k = tid; k < a.R; k += nt) a.buf_of[(size_t)inst * a.R + k] = S.buf_of[k];
        if (tid == 0 && a.best) atomicMin(&a.best[inst], S.best);
    }
    if constexpr (CLU) cg::this_cluster().sync();  // peers may still read our Eown
}

}  // namespace tapt_dev
