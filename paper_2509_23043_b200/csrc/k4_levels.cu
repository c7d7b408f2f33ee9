// k4_levels.cu -- K4: the reference's index order (proj/src/mcmc.cpp:30-45, the bit-exact mode)
// on the dependency levels, with one warp per site word and one lane per replica.
//
// The level schedule (engine.cu: level(i) = 1 + max level of lower-index neighbours) reproduces the
// sequential index-ascending sweep; its levels are small (2D L=32: 63 levels of <= 32 sites; the
// 16-bit multiplier: 88 levels averaging 8 sites), so a sweep is a chain of short dependent steps.
// K2 gives a site word to four lanes that each make 8 decisions in sequence; here every lane owns
// one replica and makes one decision per site:
//   * local field: lane r walks the site's CSR row (entries col | J << 24, broadcast loads) and adds
//     J * bit_r(w_j); l = h - sum_j J_ij + 2 acc exactly;
//   * decision: K1's pre-xorshift high-word test against the slot's threshold row, with the
//     per-lane stream base held in a register for the whole sweep; ties (|h - U| <= 1) redo the
//     exact 64-bit test;
//   * the new word is one ballot; each lane keeps its replica's exact dE = 2 s_old l per flip in a
//     register (no transposes).
// Instance teams of 8 warps with named barriers, up to 2 per CTA, share one staged copy of the graph (as K3's teams do).  Bit-identical to K2's reference
// order and to the unmodified reference gibbs_sweep (tests/test_gpu_parity.py, golden vectors).
#include <cuda_runtime.h>

#include "pt_common.cuh"

namespace tapt_dev {

constexpr int kT4 = 256;   // threads per instance team (8 warps; 16-warp teams measured slower)
constexpr int kIPB4 = 2;   // instance teams per CTA

__host__ __device__ inline size_t k4_graph_words(int n, int nnz, int nfree, int nlev) {
    // rowptr [n+1] | adj [nnz] | hmJ [n] | rank [n] | level sites [nfree] | level ptr [nlev+1]
    return (size_t)(n + 1) + nnz + 2 * (size_t)n + nfree + (nlev + 1);
}

size_t k4_smem_bytes(int n, int R, int nidx, int nnz, int nfree, int nlev, int ipb) {
    return ((size_t)R * nidx + k4_graph_words(n, nnz, nfree, nlev) + (size_t)ipb * n) * 4;
}

template <bool BAL>
__global__ void __launch_bounds__(kT4 * kIPB4, 1) k4_levels_pt(const PTArgs a, const CsrArgs g) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __shared__ PTShared SS[kIPB4];
    __shared__ uint64_t str_sh[kIPB4][kW];
    const int n = a.n, nidx = a.nidx, nfree = (int)g.n_free, nlev = g.n_classes;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    const int ipb = nt / kT4, kin = tid / kT4, ti = tid - kin * kT4, wq = ti >> 5, nwq = kT4 >> 5;
    const SubTeam tm{ti, kT4, 1 + kin};
    const int nv = own_count(a, 0);
    const uint32_t vmask = nv >= 32 ? 0xFFFFFFFFu : ((1u << nv) - 1u);
    // shared memory: Uslot [R][nidx] | graph (k4_graph_words) | words [ipb][n]
    uint32_t* Uslot = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* rp = Uslot + (size_t)a.R * nidx;
    uint32_t* adj = rp + (n + 1);
    int32_t* hmJ = reinterpret_cast<int32_t*>(adj + g.nnz);
    uint32_t* rk = reinterpret_cast<uint32_t*>(hmJ + n);
    uint32_t* ls = rk + n;
    uint32_t* lp = ls + nfree;
    uint32_t* words = lp + (nlev + 1) + (size_t)kin * n;
    for (int k = tid; k < a.R * nidx; k += nt) Uslot[k] = thr_hi(a.thr[k]);
    for (int k = tid; k <= n; k += nt) rp[k] = g.rowptr[k];
    for (int k = tid; k < g.nnz; k += nt) adj[k] = g.col[k] | ((uint32_t)(uint8_t)g.J[k] << 24);
    for (int i = tid; i < n; i += nt) {
        int s = g.h[i];
        for (uint32_t k = g.rowptr[i]; k < g.rowptr[i + 1]; ++k) s -= g.J[k];
        hmJ[i] = s;  // l = h - sum_j J_ij + 2 sum_j J_ij [s_j = +1]
        rk[i] = g.rank[i];
    }
    for (int k = tid; k < nfree; k += nt) ls[k] = g.class_sites[k];
    for (int k = tid; k <= nlev; k += nt) lp[k] = g.class_ptr[k];
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
    PTShared& S = SS[kin];
    for (int it = it0; it < it1; ++it) {
        const SchedItem item = BAL ? a.sched[it] : SchedItem{unit, 0, a.n_sweeps, -1, -1};
        const int inst = item.inst;
        if (BAL && item.wait >= 0) pt_wait_flag(a, item.wait, tm);
        const uint64_t t0 = a.t0 + (uint64_t)item.s0;
        for (int k = ti; k < n; k += kT4) words[k] = a.words[(size_t)inst * n + k];
        pt_load_perm(a, S, inst, tm);
        for (int r = ti; r < a.R; r += kT4) str_sh[kin][r] = a.streams[(size_t)inst * a.R + r];
        for (int b = ti; b < nv; b += kT4) S.Eown[(t0 + 1) & 1][b] = a.E[(size_t)inst * a.B + b];
        tm.sync();

        uint64_t pass = a.p0;
        if (a.swap_every > 0 && item.s0 > 0) pass += t0 / (uint64_t)a.swap_every - a.t0 / (uint64_t)a.swap_every;
        int par = (int)((t0 + 1) & 1);
        for (int s = item.s0; s < item.s1; ++s) {
            const uint64_t t = a.t0 + (uint64_t)s;
            const int prev = par;
            par = (int)(t & 1);
            // this lane's replica: its slot's stream base and threshold row for the whole sweep
            const bool own = lane < nv;
            const int slot = own ? S.slot_of[lane] : 0;
            const uint64_t sb = str_sh[kin][slot] + (a.draw_base + t * (uint64_t)a.n_free + 1ull) * kPhi;
            const uint32_t* row = Uslot + (size_t)slot * nidx - g.lmin;
            int dE = 0;
            for (int c = 0; c < nlev; ++c) {
                const int c0 = (int)lp[c], c1 = (int)lp[c + 1];
                for (int q = c0 + wq; q < c1; q += nwq) {  // one site word per warp
                    const uint32_t i = ls[q];
                    const uint32_t r1 = rp[i + 1];
                    int acc = 0;
                    for (uint32_t k = rp[i]; k < r1; ++k) {
                        const uint32_t e = adj[k];
                        acc += ((int32_t)e >> 24) * (int)((words[e & 0xFFFFFFu] >> lane) & 1u);
                    }
                    const int l = hmJ[i] + 2 * acc;
                    const uint32_t old = words[i];
                    const uint64_t z = sb + (uint64_t)rk[i] * kPhi;
                    const uint32_t h = mix_pre_hi<TAPT_K1_VARIANT>((uint32_t)z, (uint32_t)(z >> 32), a.mc);
                    const uint32_t U = row[l];
                    bool up = h < U;
                    if (h - U + 1u <= 2u)  // |h - U| <= 1: the final xor-shift may decide (p ~ 2^-31)
                        up = below(mix_final(z), a.thr[(size_t)slot * nidx + (l - g.lmin)]);
                    const uint32_t nw = (__ballot_sync(0xFFFFFFFFu, up) & vmask) | (old & ~vmask);
                    const uint32_t ob = (old >> lane) & 1u;
                    if (own && ((nw >> lane) & 1u) != ob) dE += ob ? 2 * l : -2 * l;  // 2 s_old l
                    __syncwarp();
                    if (lane == 0) words[i] = nw;
                }
                tm.sync();
            }
            if (own) atomicAdd(&S.Ucnt[lane], (uint32_t)dE);
            tm.sync();
            for (int b = ti; b < nv; b += kT4) {
                S.Eown[par][b] = S.Eown[prev][b] + (int32_t)S.Ucnt[b];
                S.Ucnt[b] = 0;
            }
            pt_epilogue<false>(a, S, words, inst, 0, t, pass, tm);
        }
        for (int k = ti; k < n; k += kT4) a.words[(size_t)inst * n + k] = words[k];
        pt_finish<false>(a, S, inst, 0, par, tm);
        if (BAL && item.signal >= 0) pt_signal_flag<false>(a, item.signal, 0, tm);
        tm.sync();  // the team's shared memory is reused by the next item
    }
}

static cudaError_t k4_run(const PTArgs& a, const CsrArgs& g, int ipb, cudaStream_t st, int* resident) {
    const size_t smem = k4_smem_bytes(a.n, a.R, a.nidx, g.nnz, (int)g.n_free, g.n_classes, ipb);
    cudaError_t e = cudaFuncSetAttribute(k4_levels_pt<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k4_levels_pt<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (resident) {
        int per_sm = 0, dev = 0, nsm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k4_levels_pt<true>, kT4 * ipb, smem);
        if (e == cudaSuccess) e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        *resident = per_sm * nsm * ipb;
        return e;
    }
    const unsigned grid = a.sched ? (unsigned)((a.sched_clusters + ipb - 1) / ipb) : (unsigned)((a.I + ipb - 1) / ipb);
    if (a.sched)
        k4_levels_pt<true><<<grid, kT4 * ipb, smem, st>>>(a, g);
    else
        k4_levels_pt<false><<<grid, kT4 * ipb, smem, st>>>(a, g);
    return cudaGetLastError();
}

int k4_max_ipb() { return kIPB4; }

int k4_resident_units(const PTArgs& a, const CsrArgs& g, int ipb) {
    int r = 0;
    return k4_run(a, g, ipb, nullptr, &r) == cudaSuccess ? r : 0;
}

cudaError_t launch_k4(const PTArgs& a, const CsrArgs& g, int ipb, cudaStream_t st) {
    return k4_run(a, g, ipb, st, nullptr);
}

}  // namespace tapt_dev
