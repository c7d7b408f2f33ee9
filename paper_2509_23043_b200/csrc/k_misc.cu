// k_misc.cu -- the non-sweep device work of the TAPT verifier: replica initialisation
// (random_configuration), exact energies for arbitrary graphs, spin import/export,
// stand-alone swap passes, proposal conversion / Metropolis acceptance (Eq. 2) /
// application, the synthetic proposal generator and EA disorder generation.
#include <cuda_runtime.h>

#include "kernels.h"

namespace tapt_dev {

// ------------------------------------------------------------------ init --
// random_configuration (spin_model.cpp:116-121): site i takes coin draw i+1 of
// derive(seed, {kInit, gid, slot}); +1 iff the top bit is set; clamps override.
// At initialisation buffer b holds slot b.  grid: (ceil(n/256), G, I)
__global__ void k_init_random(uint32_t* words, int n, int G, int W, int B, const uint64_t* init_streams,
                              const int8_t* clampval, int n_clamp_sets) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int grp = blockIdx.y, inst = blockIdx.z;
    if (i >= n) return;
    const int8_t cv = clampval ? clampval[(size_t)(n_clamp_sets > 1 ? inst : 0) * n + i] : 0;
    uint32_t w = 0;
    for (int b = 0; b < W; ++b) {
        const int slot = grp * W + b;
        if (slot >= B) break;
        bool up;
        if (cv)
            up = cv > 0;
        else
            up = (draw(init_streams[(size_t)inst * B + slot], (uint64_t)i + 1) >> 63) != 0;
        if (up) w |= 1u << b;
    }
    words[((size_t)inst * G + grp) * n + i] = w;
}

// ----------------------------------------------------------------- energy --
// E = -sum_{i<j} J_ij s_i s_j - sum_i h_i s_i  (spin_model.cpp:79-89) for every buffer of
// a group.  grid: (G, I), block 256.  Per-replica partials in registers, reduced by a
// warp reduce-scatter then shared atomics.
__global__ void k_energy_csr(const uint32_t* words, int n, int G, int W, int B, const uint32_t* rowptr,
                             const uint32_t* col, const int8_t* J, int nJ, int nnz, const int32_t* h, int32_t* E) {
    __shared__ int32_t acc[kW];
    const int grp = blockIdx.x, inst = blockIdx.y;
    const uint32_t* w = words + ((size_t)inst * G + grp) * n;
    const int8_t* Jr = J + (size_t)(nJ > 1 ? inst : 0) * nnz;
    if (threadIdx.x < kW) acc[threadIdx.x] = 0;
    __syncthreads();
    int32_t e[kW];
#pragma unroll
    for (int b = 0; b < kW; ++b) e[b] = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t wi = w[i];
        const int hi = h ? h[i] : 0;
        // field: -h*s ; bond (i<j): -J*s_i*s_j = -J + 2J*[s_i != s_j]
        int jsum = 0;
        uint32_t mism_pos[1];
        (void)mism_pos;
        for (uint32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
            const uint32_t j = col[k];
            if (j <= (uint32_t)i) continue;
            const int Jk = Jr[k];
            jsum += Jk;
            const uint32_t x = wi ^ w[j];
#pragma unroll
            for (int b = 0; b < kW; ++b) e[b] += ((x >> b) & 1u) ? 2 * Jk : 0;
        }
#pragma unroll
        for (int b = 0; b < kW; ++b) e[b] += -jsum + (((wi >> b) & 1u) ? -hi : hi);
    }
    const int32_t tot = warp_reduce_scatter32(e);
    const int lane = threadIdx.x & 31;
    if (lane < W) atomicAdd(&acc[lane], tot);
    __syncthreads();
    if (threadIdx.x < W && grp * W + (int)threadIdx.x < B)
        E[(size_t)inst * B + grp * W + threadIdx.x] = acc[threadIdx.x];
}

// ------------------------------------------------------------- readout --
// spins [I][R][n] by slot  <-  words.  grid: (ceil(n/256), R, I)
__global__ void k_get_spins(const uint32_t* words, int n, int G, int W, int B, const uint8_t* buf_of, int R,
                            int8_t* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int slot = blockIdx.y, inst = blockIdx.z;
    if (i >= n) return;
    const int b = buf_of[(size_t)inst * R + slot];
    const uint32_t w = words[((size_t)inst * G + b / W) * n + i];
    out[((size_t)inst * R + slot) * n + i] = ((w >> (b % W)) & 1u) ? 1 : -1;
}

// packed [I][R][nbytes], LSB-first, +1 -> 1.  grid: (ceil(nbytes/256), R, I)
__global__ void k_get_packed(const uint32_t* words, int n, int G, int W, const uint8_t* buf_of, int R,
                             uint8_t* out) {
    const int nbytes = (n + 7) >> 3;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int slot = blockIdx.y, inst = blockIdx.z;
    if (k >= nbytes) return;
    const int b = buf_of[(size_t)inst * R + slot];
    const uint32_t* w = words + ((size_t)inst * G + b / W) * n;
    uint8_t v = 0;
    for (int q = 0; q < 8; ++q) {
        const int i = 8 * k + q;
        if (i < n && ((w[i] >> (b % W)) & 1u)) v |= (uint8_t)(1u << q);
    }
    out[((size_t)inst * R + slot) * nbytes + k] = v;
}

// words <- spins [I][S][n] (source index s = slot via slot_of for the main ensemble, or
// s = buffer for proposal sets when slot_of == nullptr); clamps forced.
// grid: (ceil(n/256), G, I)
__global__ void k_set_spins(uint32_t* words, int n, int G, int W, int B, const uint8_t* slot_of, const int8_t* in,
                            int S, const int8_t* clampval, int n_clamp_sets) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int grp = blockIdx.y, inst = blockIdx.z;
    if (i >= n) return;
    const int8_t cv = clampval ? clampval[(size_t)(n_clamp_sets > 1 ? inst : 0) * n + i] : 0;
    uint32_t w = 0;
    for (int b = 0; b < W; ++b) {
        const int gb = grp * W + b;
        if (gb >= B) break;
        const int src = slot_of ? slot_of[(size_t)inst * B + gb] : gb;
        const int8_t v = cv ? cv : in[((size_t)inst * S + src) * n + i];
        if (v > 0) w |= 1u << b;
    }
    words[((size_t)inst * G + grp) * n + i] = w;
}

// words <- packed [I][S][nbytes] (buffer = source index); clamps forced.
__global__ void k_set_packed(uint32_t* words, int n, int G, int W, int B, const uint8_t* in, int S,
                             const int8_t* clampval, int n_clamp_sets) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int grp = blockIdx.y, inst = blockIdx.z;
    if (i >= n) return;
    const int nbytes = (n + 7) >> 3;
    const int8_t cv = clampval ? clampval[(size_t)(n_clamp_sets > 1 ? inst : 0) * n + i] : 0;
    uint32_t w = 0;
    for (int b = 0; b < W; ++b) {
        const int gb = grp * W + b;
        if (gb >= B) break;
        bool up;
        if (cv)
            up = cv > 0;
        else
            up = (in[((size_t)inst * S + gb) * nbytes + (i >> 3)] >> (i & 7)) & 1u;
        if (up) w |= 1u << b;
    }
    words[((size_t)inst * G + grp) * n + i] = w;
}

// ------------------------------------------------------------- swap pass --
// One pass (Eq. 1) for every instance: pair (r, r+1), r = parity (mod 2), draw
// p*R + r + 1 of the coordinator stream.  grid: I, block >= R/2
__global__ void k_swap_pass(const int32_t* E, uint8_t* slot_of, uint8_t* buf_of, int R, const uint64_t* coord,
                            uint64_t p, int parity, MetroTable tab, uint64_t* att, uint64_t* acc) {
    const int inst = blockIdx.x;
    const int r = parity + 2 * (int)threadIdx.x;
    if (r + 1 >= R) return;
    uint8_t* bo = buf_of + (size_t)inst * R;
    uint8_t* so = slot_of + (size_t)inst * R;
    const int b0 = bo[r], b1 = bo[r + 1];
    const int64_t dE = (int64_t)E[(size_t)inst * R + b1] - (int64_t)E[(size_t)inst * R + b0];
    const bool a = metro_accept(tab, r, dE, draw(coord[inst], p * (uint64_t)R + (uint64_t)r + 1ull));
    att[(size_t)inst * (R - 1) + r] += 1;
    if (a) {
        acc[(size_t)inst * (R - 1) + r] += 1;
        bo[r] = (uint8_t)b1;
        bo[r + 1] = (uint8_t)b0;
        so[b1] = (uint8_t)r;
        so[b0] = (uint8_t)(r + 1);
    }
}

// ------------------------------------------------------------ proposals --
// Metropolis acceptance (Eq. 2) of proposal t for slot targets[t]: draw slot+1 of
// accept_streams[inst] (= derive(seed,{kCoordinator,gid,round+1})).  When `forced`
// is non-null the decision is taken from it (MH path decided on the host).
// grid: I, block >= n_targets
__global__ void k_accept_proposals(int32_t* E, const uint8_t* buf_of, int R, const int32_t* Eprop, int T,
                                   const uint32_t* targets, const uint64_t* accept_streams, MetroTable tab,
                                   const uint8_t* forced, uint8_t* accepted, uint64_t* att, uint64_t* accn) {
    const int inst = blockIdx.x, t = threadIdx.x;
    if (t >= T) return;
    const int slot = (int)targets[t];
    const int b = buf_of[(size_t)inst * R + slot];
    const int32_t ep = Eprop[(size_t)inst * T + t];
    const int64_t dE = (int64_t)E[(size_t)inst * R + b] - (int64_t)ep;
    bool a;
    if (forced)
        a = forced[(size_t)inst * T + t] != 0;
    else
        a = metro_accept(tab, slot, dE, draw(accept_streams[inst], (uint64_t)slot + 1ull));
    att[(size_t)inst * R + slot] += 1;
    if (a) {
        accn[(size_t)inst * R + slot] += 1;
        E[(size_t)inst * R + b] = ep;
    }
    accepted[(size_t)inst * T + t] = a ? 1 : 0;
}

// MH-corrected acceptance decided on the device:
//   a = exp(beta_r (E_r - E^T_r)) * exp(log q(cur) - log q(prop)),  accept iff uniform < a,
// with the device exp.  Device and glibc exp differ by a few ulp (~1e-16 relative), so a decision whose
// draw lies outside a relative band of 1e-12 around a is glibc's decision too; a draw inside the band
// (or a NaN) is counted in *n_ties and the host redoes the round's decisions with glibc (engine.cu).
// forced[i*T + t] receives the decision for k_accept_proposals.  grid: I, block >= n_targets
__global__ void k_decide_mh(const int32_t* E, const uint8_t* buf_of, int R, const int32_t* Eprop, int T,
                            const uint32_t* targets, const uint64_t* accept_streams, const double* betas,
                            const double* lq_cur, const double* lq_prop, uint8_t* forced, uint32_t* n_ties) {
    const int inst = blockIdx.x, t = threadIdx.x;
    if (t >= T) return;
    const int slot = (int)targets[t];
    const int b = buf_of[(size_t)inst * R + slot];
    const double ec = (double)E[(size_t)inst * R + b], ep = (double)Eprop[(size_t)inst * T + t];
    const size_t k = (size_t)inst * T + t;
    const double a = __dmul_rn(exp(__dmul_rn(betas[slot], ec - ep)), exp(lq_cur[k] - lq_prop[k]));
    const uint64_t x = draw(accept_streams[inst], (uint64_t)slot + 1ull);
    const double u = (double)(x >> 11) * 0x1.0p-53;
    const bool lo = u < a * (1.0 - 1e-12), hi = u > a * (1.0 + 1e-12);
    if (!lo && !hi) atomicAdd(n_ties, 1u);
    forced[k] = u < a ? 1 : 0;
}

// Copy accepted proposals into the ensemble: for every (instance, group, site), bit
// (b % W) of the group word takes bit t of the proposal word when proposal t (slot
// targets[t], buffer b) was accepted.  grid: (ceil(n/256), G, I)
__global__ void k_apply_proposals(uint32_t* words, int n, int G, int W, const uint8_t* buf_of, int R,
                                  const uint32_t* pwords, int GT, int WT, const uint32_t* targets, int T,
                                  const uint8_t* accepted) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int grp = blockIdx.y, inst = blockIdx.z;
    if (i >= n) return;
    uint32_t keep = 0xFFFFFFFFu, set = 0;
    for (int t = 0; t < T; ++t) {
        if (!accepted[(size_t)inst * T + t]) continue;
        const int b = buf_of[(size_t)inst * R + targets[t]];
        if (b / W != grp) continue;
        const uint32_t pw = pwords[((size_t)inst * GT + t / WT) * n + i];
        const int bit = b % W;
        keep &= ~(1u << bit);
        if ((pw >> (t % WT)) & 1u) set |= 1u << bit;
    }
    if (keep != 0xFFFFFFFFu) {
        uint32_t* w = words + ((size_t)inst * G + grp) * n + i;
        *w = (*w & keep) | set;
    }
}

// Synthetic generator initial states (stand-in for IsingFormer.sample): proposal t for
// slot targets[t] uses stream Q = derive(seed,{kReplica,gid,slot,round+1}); draw 1 is
// the sign coin, site i takes draw i+2: +1 iff (x>>11) < T_up[t][sign]; clamps forced.
// grid: (ceil(n/256), GT, I)
__global__ void k_gen_proposals(uint32_t* pwords, int n, int GT, int WT, int T, const uint64_t* qstreams,
                                const uint64_t* tup, const int8_t* clampval, int n_clamp_sets) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int grp = blockIdx.y, inst = blockIdx.z;
    if (i >= n) return;
    const int8_t cv = clampval ? clampval[(size_t)(n_clamp_sets > 1 ? inst : 0) * n + i] : 0;
    uint32_t w = 0;
    for (int b = 0; b < WT; ++b) {
        const int t = grp * WT + b;
        if (t >= T) break;
        const uint64_t q = qstreams[(size_t)inst * T + t];
        bool up;
        if (cv) {
            up = cv > 0;
        } else {
            const int sign = (int)(draw(q, 1) >> 63);
            up = below(draw(q, (uint64_t)i + 2), tup[2 * t + sign]);
        }
        if (up) w |= 1u << b;
    }
    pwords[((size_t)inst * GT + grp) * n + i] = w;
}

// ---------------------------------------------------------------- disorder --
// EA +-J bonds: bond k of the site-ordered bond list (site i,
// direction d in +x,+y[,+z]) takes coin k+1 of derive(seed, {0x88, gid}); +1 iff top bit.
// Periodic lattices with L > 2: bond k = dim*i + d.  grid: ceil(n/256), I
__global__ void k_ea_signs(int8_t* signs, int n, int dim, const uint64_t* streams) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int inst = blockIdx.y;
    if (i >= n) return;
    for (int d = 0; d < dim; ++d) {
        const uint64_t k = (uint64_t)dim * i + d;
        signs[(size_t)inst * dim * n + k] = (draw(streams[inst], k + 1) >> 63) ? 1 : -1;
    }
}

// Bond bytes for K1: bit 2d (+dir) / 2d+1 (-dir) set when that bond's J is negative.
__global__ void k_bond_bytes(const int8_t* signs, uint8_t* bytes, LatDims d, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int inst = blockIdx.y;
    if (i >= n) return;
    const int Lx = 1 << d.log2Lx, Ly = 1 << d.log2Ly;
    const int x = i & (Lx - 1);
    const int y = (i >> d.log2Lx) & (Ly - 1);
    const int z = i >> (d.log2Lx + d.log2Ly);
    const int8_t* s = signs + (size_t)inst * d.dim * n;
    int nb[3];
    nb[0] = (x == 0) ? i + Lx - 1 : i - 1;
    nb[1] = (y == 0) ? i + (Ly - 1) * Lx : i - Lx;
    nb[2] = (d.dim == 3) ? ((z == 0) ? i + (Ly - 1) * Lx * Ly : i - Lx * Ly) : 0;
    uint8_t v = 0;
    for (int k = 0; k < d.dim; ++k) {
        if (s[(size_t)d.dim * i + k] < 0) v |= (uint8_t)(1u << (2 * k));
        if (s[(size_t)d.dim * nb[k] + k] < 0) v |= (uint8_t)(1u << (2 * k + 1));
    }
    bytes[(size_t)inst * n + i] = v;
}

// Per-instance CSR couplings from bond signs: J[inst][k] = J0 * sign[bond_id[k]].
__global__ void k_csr_from_signs(const int8_t* signs, int nbonds, const uint32_t* bond_id, int nnz, int J0,
                                 int8_t* J) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int inst = blockIdx.y;
    if (k >= nnz) return;
    J[(size_t)inst * nnz + k] = (int8_t)(J0 * signs[(size_t)inst * nbonds + bond_id[k]]);
}

}  // namespace tapt_dev

namespace tapt_dev {

// RngStream::derive (proj/include/tapt/rng.hpp:21-27; include/tapt/rng.hpp derive_n) on the device:
// h = hash(root ^ phi), then h = hash(h ^ (p + phi)) for every path component, hash(v) = mix(v + phi).
__device__ __forceinline__ uint64_t d_hash64(uint64_t v) { return mix_final(v + kPhi); }

// Proposal-round streams: per (instance, target) {kReplica, gid, target, round} into qs [I][T] and
// full [I][R] (slot-indexed, for the refinement sweeps), and per instance the accept stream
// {kCoordinator, gid, round} into acc [I].  Grid: one block per instance.
__global__ void k_derive_round_streams(uint64_t seed, uint64_t gid0, const uint32_t* targets, int T, int R,
                                       uint64_t round, uint64_t* qs, uint64_t* full, uint64_t* acc) {
    const int i = blockIdx.x;
    const uint64_t h0 = d_hash64(seed ^ kPhi), gid = gid0 + (uint64_t)i;
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
        uint64_t h = d_hash64(h0 ^ (0x22ull + kPhi));
        h = d_hash64(h ^ (gid + kPhi));
        h = d_hash64(h ^ ((uint64_t)targets[t] + kPhi));
        h = d_hash64(h ^ (round + kPhi));
        if (qs) qs[(size_t)i * T + t] = h;
        if (full) full[(size_t)i * R + targets[t]] = h;
    }
    if (threadIdx.x == 0 && acc) {
        uint64_t h = d_hash64(h0 ^ (0x33ull + kPhi));
        h = d_hash64(h ^ (gid + kPhi));
        acc[i] = d_hash64(h ^ (round + kPhi));
    }
}

// best[i] = min(best[i], min_b E[i][b]) (one thread per instance)
__global__ void k_best_from_E(const int32_t* E, int I, int B, int* best) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= I) return;
    int m = best[i];
    for (int b = 0; b < B; ++b) m = min(m, E[(size_t)i * B + b]);
    best[i] = m;
}

}  // namespace tapt_dev
