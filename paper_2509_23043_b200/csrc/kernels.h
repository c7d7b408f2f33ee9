// kernels.h -- argument blocks shared by the host driver (engine.cpp) and the CUDA kernels.
//
// State layout in HBM (one ensemble = I instances x B buffers):
//   words [I][G][n] uint32  -- multi-replica spin coding: bit b of word (i, g, site)
//                              is the spin (1 = +1) of buffer g*W+b at that site.
//   E     [I][B]    int32   -- energy of each buffer (integer couplings, exact)
//   slot_of [I][B], buf_of [I][R]  uint8 -- the slot<->buffer permutation.  A swap
//                               exchanges two entries; no spins move.
// The dynamics stream and the beta of a buffer are those of the ladder slot it
// currently occupies.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace tapt_dev {

constexpr int kMaxR = 256;   // ladder slots per instance (uint8 permutation)
constexpr int kW = 32;       // replicas per group (bits per word)
constexpr int kCnt = 8;      // planes of the sliced per-thread counters
#ifndef TAPT_K1_NIB2
#define TAPT_K1_NIB2 1       // 1: 13-op nibble spread (measured +0.5..1%)
#endif
#ifndef TAPT_K1_IDX2
#define TAPT_K1_IDX2 1       // 1: masked-add periodic neighbour indices
#endif
#ifndef TAPT_K1_UM1
#define TAPT_K1_UM1 1        // 1: tables hold U - 1, so the tie band is d in {0, 1, 2} itself (needed by MIN3)
#endif
#ifndef TAPT_K1_MIN3
#define TAPT_K1_MIN3 1       // 1 (needs UM1): tie band of two sites folded by one 3-input min (VIMNMX3): +0.6..2 %
#endif
#ifndef TAPT_K1_IDXS
// Threshold offsets 4*q of a site's 32 replicas as bytes in a per-thread shared-memory scratch: one LDS.U8
// per decision replaces a shift and a mask on the ALU pipe (the binding pipe).  1: plain reads (ptxas may
// merge them into word loads + PRMT), 2: one LDS.U8 each.  Config-5 slice 900 -> 950 G/s.
#define TAPT_K1_IDXS 2
#endif
#ifndef TAPT_K1_PHOPQ
#define TAPT_K1_PHOPQ 1       // 1: stream base + counter as an explicit carry-chain add (IADD3 + IMAD.X, 4 pipe cycles) instead of
                             // ptxas's IMAD.WIDE + IMAD.IADD (6): config-5 slice +1 %, configs 1/2/3 +3.1 / +4.5 / +0.8 %
#endif
#ifndef TAPT_K1_XSEL
#define TAPT_K1_XSEL 1       // x-neighbour indices as one LOP3 bit-field select each (config-5 slice +2.0 %, config 3 +1.6 %)
#endif
#ifndef TAPT_K1_BLUT
#define TAPT_K1_BLUT 1       // bond sign masks from a 64-row shared-memory table (bulk shape only)
#endif
#ifndef TAPT_K1_PACK
#define TAPT_K1_PACK 1       // 1: narrow replica groups fold the lattice and pack 2 / 4 sites per word (k1_lattice.cu)
#endif
#ifndef TAPT_K1_PACK_SP1
#define TAPT_K1_PACK_SP1 1
#endif
#ifndef TAPT_K1_MINB256
#define TAPT_K1_MINB256 2    // CTAs per SM the 256-thread K1 shapes are compiled for (register cap 128 / 85)
#endif
#ifndef TAPT_K2_MIXV
#define TAPT_K2_MIXV TAPT_K1_VARIANT  // mix_pre_hi variant of the K2 decisions
#endif
#ifndef TAPT_K2_HS
#define TAPT_K2_HS 0         // 1: precomputed h - sum|J| per site (0: accumulate in the walk; 3% faster, config 4)
#endif
#ifndef TAPT_K2_WALKHI
#define TAPT_K2_WALKHI 0     // 1: neighbour-walk bit-plane shifts as IMAD.HI (FMA pipe)
#endif
#ifndef TAPT_K2_MAXT
#define TAPT_K2_MAXT 1024    // K2 launch bound (threads per CTA); 512 lifts the register cap to 128
#endif
#ifndef TAPT_K1_PIPE
#define TAPT_K1_PIPE 0       // 1: software-pipeline the stencil of the next site pair
#endif
#ifndef TAPT_K1_EPOST
#define TAPT_K1_EPOST 0      // 1: energies in a separate pass after the two colour halves
#endif
#ifndef TAPT_K1_VARIANT
#define TAPT_K1_VARIANT 6    // instruction-mix variant of the decision loop (common.cuh): 2D lattices
#endif
#ifndef TAPT_K1_VARIANT3
#define TAPT_K1_VARIANT3 6   // the same for 3D lattices (with IDXS the explicit 3-op first multiply, V & 2, adds 3 %)
#endif

struct LatDims {
    int dim;              // 2 or 3
    int log2Lx, log2Ly;   // 2D: Lx, Ly; 3D: L = Lx = Ly = Lz
    int log2hx;           // log2(Lx/2): colour sites per row
    int J0;               // |J|
};

// Balanced persistent schedule (McNaughton's wrap-around rule): cluster c runs items
// sched_ptr[c] .. sched_ptr[c+1]-1 in order; an item is sweeps [s0, s1) of the launch for
// one instance.  A job split over two clusters runs its first sweeps at the start of one
// timeline and its last sweeps at the end of the previous one; the later part waits for
// flags[wait] (set by the earlier part after its state is stored) -- by construction the
// earlier part has finished long before.
struct SchedItem {
    int inst, s0, s1, wait, signal;  // wait / signal: flag index or -1
};

// Everything one fused PT launch needs (lattice K1 and CSR K2 share it).
struct PTArgs {
    uint32_t* words;
    int I, G, W, B;            // instances, groups per instance, replicas per group, buffers
    int n;                     // sites per replica
    const uint8_t* bonds;      // [I][n] lattice bond-sign bytes (bit d: bond in direction d is -J0), or null
    uint32_t n_free;           // free sites (draw counter stride per sweep)
    int R;                     // ladder slots
    const uint64_t* streams;   // [I][R] dynamics stream state by ladder slot
    uint8_t* slot_of;          // [I][B]
    uint8_t* buf_of;           // [I][R]
    const uint64_t* thr;       // [R][nidx] heat-bath thresholds T = ceil(p*2^53)
    int nidx;                  // entries per slot
    uint64_t draw_base;        // extra offset of every dynamics draw counter
    uint64_t t0;               // global index of the first sweep of this launch
    int n_sweeps;
    int32_t* E;                // [I][B] out
    int energy_only;           // recompute energies, no sweeps
    // replica exchange
    int swap_every;            // 0: no swaps
    uint64_t p0;               // global index of the first swap pass in this launch
    const uint64_t* coord;     // [I] coordinator stream states
    MetroTable swap_tab;       // rows = pairs (r, r+1)
    uint64_t* swap_att;        // [I][R-1]
    uint64_t* swap_acc;
    // observables (by slot)
    int measure_every;
    uint64_t measure_from;
    long long* obs;            // [I][R][5]: count, sum E, sum E^2, sum |M|, sum M^2
    unsigned long long* hist;  // [R][nbins] (summed over instances)
    long long e_lo, width;
    int nbins;
    int* best;                 // [I] lowest energy seen (atomicMin)
    MixConsts mc;              // {4, 32}, opaque to the compiler (see common.cuh)
    // balanced persistent schedule (null: one instance per cluster, all launch sweeps)
    const int* sched_ptr;      // [n_clusters + 1]
    const SchedItem* sched;
    uint32_t* flags;           // [n_split] zeroed before the launch
    uint32_t* sched_err;       // set when a wait times out (the host raises)
    int sched_clusters;        // clusters of the persistent grid (with sched)
};

// CSR graph (K2): shared structure; couplings may be per instance.
struct CsrArgs {
    const uint32_t* rowptr;    // [n+1]
    const uint32_t* col;       // [nnz]
    const int8_t* J;           // [nJ][nnz]
    int nJ;                    // 1 (shared) or I (per instance)
    int nnz;
    const int32_t* h;          // [n]
    const int32_t* hs;         // [n] h_i - sum_k |J_ik| (per-instance couplings only flip signs)
    const uint32_t* rank;      // [n] position in the ascending free list
    const uint32_t* class_ptr; // [n_classes+1] into class_sites
    const uint32_t* class_sites;
    int n_classes;
    int lmin;                  // thresholds indexed by (l - lmin)
    int smem_graph;            // stage the CSR in shared memory (it fits)
    uint32_t n_free;
};

}  // namespace tapt_dev
