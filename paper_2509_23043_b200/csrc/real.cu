// real.cu -- K5, the FP64 sequential-order engine for real-valued couplings (see real.h), and its
// host driver RealEngine (the PT/TAPT operations of the C ABI for such models).
//
// Kernel layout.  One warp owns one 32-replica group of one instance (lane b = buffer 32g+b, its spin
// is bit b of the group's site words, as in every other kernel).  An instance's G = ceil(R/32) warps
// sit in one CTA, so the per-sweep swap pass and measurement need only __syncthreads; a CTA holds
// `ipc` instances.  Each warp visits the sites strictly in the sweep order (index order = the
// reference's gibbs_sweep; colour order = the colour classes), so the FP64 local-field sums and the
// per-sweep energy change are accumulated in exactly the reference's order.  Per site: the CSR row
// (warp-uniform broadcast loads) gives l = h_i + sum(+-J_ij) per lane, one counter-addressed
// splitmix64 draw per lane, the heat-bath decision, one ballot for the new site word.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"
#include "kernels.h"
#include "real.h"
#include "tapt/errors.hpp"
#include "tapt/rng.hpp"
#include "tapt_gpu.h"

namespace tapt_dev {
__global__ void k_init_random(uint32_t*, int, int, int, int, const uint64_t*, const int8_t*, int);
__global__ void k_get_spins(const uint32_t*, int, int, int, int, const uint8_t*, int, int8_t*);
__global__ void k_get_packed(const uint32_t*, int, int, int, const uint8_t*, int, uint8_t*);
__global__ void k_set_spins(uint32_t*, int, int, int, int, const uint8_t*, const int8_t*, int, const int8_t*, int);
__global__ void k_set_packed(uint32_t*, int, int, int, int, const uint8_t*, int, const int8_t*, int);
__global__ void k_apply_proposals(uint32_t*, int, int, int, const uint8_t*, int, const uint32_t*, int, int,
                                  const uint32_t*, int, const uint8_t*);
__global__ void k_gen_proposals(uint32_t*, int, int, int, int, const uint64_t*, const uint64_t*, const int8_t*, int);
__global__ void k_derive_round_streams(uint64_t, uint64_t, const uint32_t*, int, int, uint64_t, uint64_t*, uint64_t*,
                                       uint64_t*);
}  // namespace tapt_dev

namespace tapt_host {
void note_launches(unsigned n);
}

namespace tapt_real {

using namespace tapt_dev;

enum { kHeat = 0, kSwap = 1, kProp = 2, kRefine = 3 };

struct K5Args {
    // graph
    const uint32_t* rowptr;
    const uint32_t* col;
    const double* J;
    const double* h;
    const uint32_t* visit;  // sites in visiting order
    const uint32_t* vdraw;  // draw offset of each visited site (its rank among the free sites)
    int nv;
    uint32_t stride;  // draws per sweep
    int n;
    const uint64_t* thr;  // integer models: exact heat-bath rows [R][nidx] (null: FP64 + near-tie band)
    int lmin, nidx;
    // ensemble
    uint32_t* words;  // [I][G][n]
    int I, G, W, B, R, ipc;
    double* E;           // [I][B]
    uint8_t* slot_of;    // [I][B]
    uint8_t* buf_of;     // [I][R] (null for proposal groups)
    const uint64_t* streams;  // [I][R] by slot
    const double* betas;      // [R]
    unsigned long long draw_base, t0;
    int n_sweeps, hb_kind;
    unsigned long long key_t0;  // key time of the first sweep (kRefine: round * 2^20)
    double* dE_out;             // [n_sweeps] (drop-in, one buffer), nullable
    // swaps
    int swap_every, pass_only;  // pass_only >= 0: no sweeps, one pass of that parity
    unsigned long long p0;
    const uint64_t* coord;
    const double* swap_c;  // [R-1] b_{r+1} - b_r
    uint64_t* swap_att;
    uint64_t* swap_acc;
    // measurement
    int measure_every;
    unsigned long long measure_from;
    double* obs;  // [I][R][5]
    unsigned long long* hist;
    double e_lo, width;
    int nbins;
    double* best;  // [I]
    // near ties
    TieRec* ties;
    unsigned int* n_ties;
    unsigned int tie_cap;
    const TieKey* ovr;
    const uint32_t* ovr_dec;
    int n_ovr;
    double band, perturb;
};

__device__ __forceinline__ bool key_eq(const TieKey& a, const TieKey& b) {
    return a.kind == b.kind && a.inst == b.inst && a.slot == b.slot && a.site == b.site && a.t == b.t;
}

// uniform < p with the device p: decided outright outside the relative band, else a near tie
// (override if the host has resolved it, otherwise provisional + recorded).  x>>11 == 0 (u = 0) is
// always a tie: subnormal / underflowed p differ in absolute terms there.
__device__ bool decide_band(const K5Args& a, double p, unsigned long long x, double arg, double coef,
                            const TieKey& key) {
    if (a.perturb != 0.0) p *= 1.0 + a.perturb;
    const unsigned long long m = x >> 11;
    const double u = (double)m * 0x1.0p-53;
    if (m != 0ull && u < p * (1.0 - a.band)) return true;
    if (u > p * (1.0 + a.band)) return false;
    for (int k = 0; k < a.n_ovr; ++k)
        if (key_eq(a.ovr[k], key)) return a.ovr_dec[k] != 0;
    const bool d = u < p;
    const unsigned int idx = atomicAdd(a.n_ties, 1u);
    if (idx < a.tie_cap) {
        TieRec r;
        r.key = key;
        r.arg = arg;
        r.coef = coef;
        r.x = x;
        r.dec = d ? 1u : 0u;
        a.ties[idx] = r;
    }
    return d;
}

// One CTA = ipc instances x G warps.  Shared: words [ipc][G][n], E [ipc][B], slot_of [ipc][B],
// buf_of [ipc][R].
__global__ void __launch_bounds__(1024) k5_real_pt(const K5Args a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int loc = warp / a.G, g = warp % a.G;
    const int inst = blockIdx.x * a.ipc + loc;
    const bool live = loc < a.ipc && inst < a.I;
    uint32_t* Wall = reinterpret_cast<uint32_t*>(smem);
    double* Eall = reinterpret_cast<double*>(Wall + (size_t)a.ipc * a.G * a.n + ((size_t)a.ipc * a.G * a.n & 1));
    uint8_t* SOall = reinterpret_cast<uint8_t*>(Eall + (size_t)a.ipc * a.B);
    uint8_t* BOall = SOall + (size_t)a.ipc * a.B;
    uint32_t* Wd = Wall + ((size_t)loc * a.G + g) * a.n;
    double* Es = Eall + (size_t)loc * a.B;
    uint8_t* SO = SOall + (size_t)loc * a.B;
    uint8_t* BO = BOall + (size_t)loc * a.R;
    const int buf = g * a.W + lane;
    const bool own = live && lane < a.W && buf < a.B;
    // stage the instance
    if (live) {
        const uint32_t* src = a.words + ((size_t)inst * a.G + g) * a.n;
        for (int i = lane; i < a.n; i += 32) Wd[i] = src[i];
        if (g == 0) {
            for (int b = lane; b < a.B; b += 32) {
                Es[b] = a.E[(size_t)inst * a.B + b];
                SO[b] = a.slot_of[(size_t)inst * a.B + b];
            }
            if (a.buf_of)
                for (int r = lane; r < a.R; r += 32) BO[r] = a.buf_of[(size_t)inst * a.R + r];
        }
    }
    __syncthreads();
    const int nsw = a.pass_only >= 0 ? 1 : a.n_sweeps;
    for (int s = 0; s < nsw; ++s) {
        const unsigned long long t = a.t0 + (unsigned long long)s;
        if (a.pass_only < 0 && live) {
            const int slot = own ? SO[buf] : 0;
            const double beta = a.betas[slot];
            const double nb = -2.0 * beta;
            const uint64_t sb = own ? a.streams[(size_t)inst * a.R + slot] : 0ull;
            const unsigned long long k0 = a.draw_base + t * (unsigned long long)a.stride + 1ull;
            const uint64_t* trow = a.thr ? a.thr + (size_t)slot * a.nidx : nullptr;
            double dE = 0.0;
            for (int q = 0; q < a.nv; ++q) {
                const uint32_t i = __ldg(a.visit + q);
                const uint32_t rd = __ldg(a.vdraw + q);
                double l = __ldg(a.h + i);
                const uint32_t e0 = __ldg(a.rowptr + i), e1 = __ldg(a.rowptr + i + 1);
                for (uint32_t k = e0; k < e1; ++k) {
                    const uint32_t j = __ldg(a.col + k);
                    const double Jk = __ldg(a.J + k);
                    l = __dadd_rn(l, ((Wd[j] >> lane) & 1u) ? Jk : -Jk);
                }
                const uint64_t x = draw(sb, k0 + rd);
                bool up = false;
                if (own) {
                    if (trow) {
                        up = below(x, trow[(int)l - a.lmin]);
                    } else {
                        const double p = 1.0 / (1.0 + exp(__dmul_rn(nb, l)));
                        TieKey key{(uint32_t)a.hb_kind, (uint32_t)inst, (uint32_t)slot, i, a.key_t0 + (unsigned long long)s};
                        up = decide_band(a, p, x, l, beta, key);
                    }
                }
                const uint32_t wold = Wd[i];
                const bool old = ((wold >> lane) & 1u) != 0;
                if (own && up != old) dE = __dadd_rn(dE, old ? 2.0 * l : -2.0 * l);
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, up);
                const uint32_t ownm = __ballot_sync(0xFFFFFFFFu, own);  // lanes without a buffer keep their bit
                if (lane == 0) Wd[i] = (bal & ownm) | (wold & ~ownm);
                __syncwarp();
            }
            if (own) Es[buf] = __dadd_rn(Es[buf], dE);
            if (own && a.dE_out) a.dE_out[s] = dE;
        }
        __syncthreads();
        const unsigned long long T1 = t + 1;
        // best energy of the instance after the sweep
        if (live && g == 0 && a.best && a.pass_only < 0) {
            double m = INFINITY;
            for (int b = lane; b < a.B; b += 32) m = fmin(m, Es[b]);
            for (int o = 16; o; o >>= 1) m = fmin(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
            if (lane == 0 && m < a.best[inst]) a.best[inst] = m;
        }
        // replica exchange (Eq. 1): pairs (r, r+1) of the pass parity, coordinator draw p*R + r + 1
        const bool do_swap = a.pass_only >= 0 || (a.swap_every > 0 && (T1 % (unsigned long long)a.swap_every) == 0);
        if (do_swap && a.R >= 2) {
            const unsigned long long pass = a.p0 + (a.pass_only >= 0 ? 0ull : (T1 / a.swap_every - 1ull - (a.t0 / a.swap_every)));
            const int parity = a.pass_only >= 0 ? a.pass_only : (int)(pass & 1ull);
            if (live && g == 0) {
                const uint64_t c0 = a.coord[inst];
                for (int r = parity + 2 * lane; r + 1 < a.R; r += 64) {
                    const int b0 = BO[r], b1 = BO[r + 1];
                    const double dEs = Es[b1] - Es[b0];
                    const double c = a.swap_c[r];
                    const uint64_t x = draw(c0, pass * (unsigned long long)a.R + (unsigned long long)r + 1ull);
                    TieKey key{(uint32_t)kSwap, (uint32_t)inst, (uint32_t)r, 0u, pass};
                    const bool acc = decide_band(a, exp(__dmul_rn(c, dEs)), x, dEs, c, key);
                    a.swap_att[(size_t)inst * (a.R - 1) + r] += 1;
                    if (acc) {
                        a.swap_acc[(size_t)inst * (a.R - 1) + r] += 1;
                        BO[r] = (uint8_t)b1;
                        BO[r + 1] = (uint8_t)b0;
                        SO[b1] = (uint8_t)r;
                        SO[b0] = (uint8_t)(r + 1);
                    }
                }
            }
            __syncthreads();
        }
        // observables by slot (count, sum E, sum E^2, sum |M|, sum M^2) and the energy histogram
        if (a.pass_only < 0 && a.measure_every > 0 && T1 > a.measure_from &&
            (T1 % (unsigned long long)a.measure_every) == 0) {
            if (own) {
                int up = 0;
                for (int i = 0; i < a.n; ++i) up += (Wd[i] >> lane) & 1u;
                const double M = (double)(2 * up - a.n);
                const int slot = SO[buf];
                const double e = Es[buf];
                double* o = a.obs + ((size_t)inst * a.R + slot) * 5;
                o[0] += 1.0;
                o[1] += e;
                o[2] += e * e;
                o[3] += fabs(M);
                o[4] += M * M;
                if (a.hist && a.nbins > 0) {
                    long long bin = e < a.e_lo ? 0 : (long long)floor((e - a.e_lo) / a.width);
                    if (bin >= a.nbins) bin = a.nbins - 1;
                    atomicAdd(&a.hist[(size_t)slot * a.nbins + bin], 1ull);
                }
            }
            __syncthreads();
        }
    }
    // persist
    if (live) {
        uint32_t* dst = a.words + ((size_t)inst * a.G + g) * a.n;
        for (int i = lane; i < a.n; i += 32) dst[i] = Wd[i];
        if (g == 0) {
            for (int b = lane; b < a.B; b += 32) {
                a.E[(size_t)inst * a.B + b] = Es[b];
                a.slot_of[(size_t)inst * a.B + b] = SO[b];
            }
            if (a.buf_of)
                for (int r = lane; r < a.R; r += 32) a.buf_of[(size_t)inst * a.R + r] = BO[r];
        }
    }
}

// energy() (spin_model.cpp:79-89) of every buffer: couplings in (i<j) order, then the fields, one
// lane per buffer.  grid (G, I), block 32.
__global__ void k5_energy(const uint32_t* words, int n, int G, int W, int B, const uint32_t* ci,
                          const uint32_t* cj, const double* cJ, int nc, const double* h, double* E) {
    const int g = blockIdx.x, inst = blockIdx.y, lane = threadIdx.x;
    const int b = g * W + lane;
    if (lane >= W || b >= B) return;
    const uint32_t* w = words + ((size_t)inst * G + g) * n;
    double e = 0.0;
    for (int k = 0; k < nc; ++k) {
        const int si = ((w[ci[k]] >> lane) & 1u) ? 1 : -1, sj = ((w[cj[k]] >> lane) & 1u) ? 1 : -1;
        e = __dsub_rn(e, __dmul_rn(cJ[k], (double)(si * sj)));
    }
    for (int i = 0; i < n; ++i) e = __dsub_rn(e, __dmul_rn(h[i], ((w[i] >> lane) & 1u) ? 1.0 : -1.0));
    E[(size_t)inst * B + b] = e;
}

// Eq. 2 decisions (no state change): proposal t of instance i for slot r = targets[t] is accepted iff
// u < exp(beta_r (E_r - E^T_r)), u = draw r+1 of the round's accept stream; forced: host decisions
// (MH-corrected variant).  grid I, block >= T.
__global__ void k5_accept(K5Args a, const double* Ep, int T, const uint32_t* targets, const uint64_t* accs,
                          unsigned long long round, const uint8_t* forced, uint8_t* accepted) {
    const int inst = blockIdx.x, t = threadIdx.x;
    if (t >= T) return;
    bool acc;
    if (forced) {
        acc = forced[(size_t)inst * T + t] != 0;
    } else {
        const int r = (int)targets[t];
        const int b = a.buf_of[(size_t)inst * a.R + r];
        const double d = a.E[(size_t)inst * a.B + b] - Ep[(size_t)inst * T + t];
        const double beta = a.betas[r];
        const uint64_t x = draw(accs[inst], (uint64_t)r + 1ull);
        TieKey key{(uint32_t)kProp, (uint32_t)inst, (uint32_t)r, 0u, round};
        acc = decide_band(a, exp(__dmul_rn(beta, d)), x, d, beta, key);
    }
    accepted[(size_t)inst * T + t] = acc ? 1 : 0;
}

// Apply the decisions to energies and counters (words: k_apply_proposals), best energy.
__global__ void k5_apply_accept(double* E, const uint8_t* buf_of, int R, int B, const double* Ep, int T,
                                const uint32_t* targets, const uint8_t* accepted, uint64_t* att, uint64_t* accn,
                                double* best) {
    const int inst = blockIdx.x;
    if (threadIdx.x != 0) return;
    for (int t = 0; t < T; ++t) {
        const int r = (int)targets[t];
        att[(size_t)inst * R + r] += 1;
        if (accepted[(size_t)inst * T + t]) {
            accn[(size_t)inst * R + r] += 1;
            E[(size_t)inst * B + buf_of[(size_t)inst * R + r]] = Ep[(size_t)inst * T + t];
        }
    }
    double m = best[inst];
    for (int b = 0; b < B; ++b) m = fmin(m, E[(size_t)inst * B + b]);
    best[inst] = m;
}

__global__ void k5_best_from_E(const double* E, int I, int B, double* best) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= I) return;
    double m = best[i];
    for (int b = 0; b < B; ++b) m = fmin(m, E[(size_t)i * B + b]);
    best[i] = m;
}

// =================================================================== host ===

namespace {

#define K5_OK(expr)                                                                                      \
    do {                                                                                                 \
        cudaError_t e_ = (expr);                                                                         \
        if (e_ != cudaSuccess) throw tapt::CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

template <class T>
struct Buf {
    T* p = nullptr;
    size_t n = 0;
    Buf() = default;
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    ~Buf() {
        if (p) cudaFree(p);
    }
    void alloc(size_t c) {
        if (c == n && p) return;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        if (!c) return;
        K5_OK(cudaMalloc(&p, c * sizeof(T)));
        n = c;
    }
    void zero(cudaStream_t st) {
        if (p) K5_OK(cudaMemsetAsync(p, 0, n * sizeof(T), st));
    }
    void upload(const T* h, size_t c, cudaStream_t st) {
        alloc(c);
        if (c) K5_OK(cudaMemcpyAsync(p, h, c * sizeof(T), cudaMemcpyHostToDevice, st));
    }
    void upload(const std::vector<T>& h, cudaStream_t st) { upload(h.data(), h.size(), st); }
    std::vector<T> download(cudaStream_t st) const {
        std::vector<T> h(n);
        if (n) {
            K5_OK(cudaMemcpyAsync(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, st));
            K5_OK(cudaStreamSynchronize(st));
        }
        return h;
    }
    void copy_from(const Buf& o, cudaStream_t st) {
        alloc(o.n);
        if (n) K5_OK(cudaMemcpyAsync(p, o.p, n * sizeof(T), cudaMemcpyDeviceToDevice, st));
    }
};

double conditional_up(double beta, double l) { return 1.0 / (1.0 + std::exp(-2.0 * beta * l)); }

uint64_t threshold_of(double p) {
    if (!(p > 0.0)) return 0;
    if (p >= 1.0) return 1ull << 53;
    return static_cast<uint64_t>(std::ceil(p * 9007199254740992.0));
}

double env_double(const char* name, double dflt) {
    const char* v = std::getenv(name);
    return v ? std::atof(v) : dflt;
}

}  // namespace

struct RealEngineImpl {
    RealGraph g;
    uint32_t I = 0;
    uint64_t gid0 = 0, seed = 0;
    int R = 0, G = 0, W = 0, order = 0;
    std::vector<double> betas;
    cudaStream_t st = nullptr;
    unsigned long long T = 0, P = 0, Q = 0;
    bool ladder_decreasing = false;
    // graph on the device
    Buf<uint32_t> rowptr, col, visit, vdraw, ci, cj, upd_visit, upd_draw;
    Buf<double> J, h, cJ;
    Buf<int8_t> clamp;
    int nv = 0;
    // state
    Buf<uint32_t> words;
    Buf<double> E, d_betas, swap_c, obs, best;
    Buf<uint8_t> slot_of, buf_of;
    Buf<uint64_t> streams, coord, thr;
    Buf<uint64_t> swap_att, swap_acc, prop_att, prop_acc;
    Buf<unsigned long long> hist;
    double e_lo = 0, width = 1;
    int nbins = 0;
    // snapshot for tie replays
    Buf<uint32_t> s_words;
    Buf<double> s_E, s_obs, s_best;
    Buf<uint8_t> s_so, s_bo;
    Buf<uint64_t> s_satt, s_sacc;
    Buf<unsigned long long> s_hist;
    // near ties
    Buf<TieRec> ties;
    Buf<unsigned int> n_ties;
    Buf<TieKey> ovr;
    Buf<uint32_t> ovr_dec;
    std::vector<TieKey> h_ovr;
    std::vector<uint32_t> h_ovr_dec;
    unsigned int* h_nties = nullptr;  // pinned
    double band = 1e-12, perturb = 0.0;
    unsigned long long ties_seen = 0, replays = 0;
    unsigned tie_cap = 1u << 16;
    // proposal scratch
    Buf<uint32_t> pwords, ptargets, s_pwords;
    Buf<double> pE;
    Buf<uint8_t> pslot, pacc, pforced, pbytes;
    Buf<int8_t> pint8;
    Buf<uint64_t> pstreams, pfull, paccs, ptup;
    Buf<double> dE_dev;

    ~RealEngineImpl() {
        if (h_nties) cudaFreeHost(h_nties);
    }
    int n() const { return (int)g.n; }

    void upload_graph() {
        rowptr.upload(g.rowptr, st);
        col.upload(g.col, st);
        J.upload(g.J, st);
        h.upload(g.h, st);
        ci.upload(g.ci, st);
        cj.upload(g.cj, st);
        cJ.upload(g.cJ, st);
        clamp.upload(g.clamp, st);
        std::vector<uint32_t> v, d;
        if (order == TAPT_ORDER_REFERENCE) {
            v = g.free_sites;
        } else {
            v = g.colour_order;
        }
        for (uint32_t i : v) d.push_back(g.rank[i]);
        nv = (int)v.size();
        visit.upload(v, st);
        vdraw.upload(d, st);
        if (ci.n == 0) {  // keep valid pointers for empty graphs
            std::vector<uint32_t> z(1, 0);
            ci.upload(z, st);
            cj.upload(z, st);
            std::vector<double> zd(1, 0.0);
            cJ.upload(zd, st);
        }
        if (col.n == 0) {
            std::vector<uint32_t> z(1, 0);
            col.upload(z, st);
            std::vector<double> zd(1, 0.0);
            J.upload(zd, st);
        }
        if (visit.n == 0) {
            std::vector<uint32_t> z(1, 0);
            visit.upload(z, st);
            vdraw.upload(z, st);
        }
    }

    void build_tables() {
        d_betas.upload(betas, st);
        std::vector<double> c(std::max(R - 1, 1), 0.0);
        for (int r = 0; r + 1 < R; ++r) c[r] = betas[r + 1] - betas[r];
        swap_c.upload(c, st);
        if (g.integral) {  // exact heat-bath rows (conditional_up, mcmc.cpp:13-15) per slot
            const int nidx = g.lmax - g.lmin + 1;
            std::vector<uint64_t> th((size_t)R * nidx);
            for (int r = 0; r < R; ++r)
                for (int k = 0; k < nidx; ++k) th[(size_t)r * nidx + k] = threshold_of(conditional_up(betas[r], g.lmin + k));
            thr.upload(th, st);
        }
    }

    K5Args base() {
        K5Args a{};
        a.rowptr = rowptr.p;
        a.col = col.p;
        a.J = J.p;
        a.h = h.p;
        a.visit = visit.p;
        a.vdraw = vdraw.p;
        a.nv = nv;
        a.stride = (uint32_t)g.free_sites.size();
        a.n = n();
        a.thr = g.integral ? thr.p : nullptr;
        a.lmin = g.lmin;
        a.nidx = g.lmax - g.lmin + 1;
        a.words = words.p;
        a.I = (int)I;
        a.G = G;
        a.W = W;
        a.B = R;
        a.R = R;
        a.E = E.p;
        a.slot_of = slot_of.p;
        a.buf_of = buf_of.p;
        a.streams = streams.p;
        a.betas = d_betas.p;
        a.hb_kind = kHeat;
        a.swap_every = 0;
        a.pass_only = -1;
        a.coord = coord.p;
        a.swap_c = swap_c.p;
        a.swap_att = swap_att.p;
        a.swap_acc = swap_acc.p;
        a.obs = obs.p;
        a.hist = nbins ? hist.p : nullptr;
        a.e_lo = e_lo;
        a.width = width;
        a.nbins = nbins;
        a.best = best.p;
        a.ties = ties.p;
        a.n_ties = n_ties.p;
        a.tie_cap = tie_cap;
        a.band = band;
        a.perturb = perturb;
        return a;
    }

    void set_ovr(K5Args& a) {
        a.ovr = h_ovr.empty() ? nullptr : ovr.p;
        a.ovr_dec = h_ovr.empty() ? nullptr : ovr_dec.p;
        a.n_ovr = (int)h_ovr.size();
    }

    void launch_k5(K5Args a) {
        int ipc = a.G == 1 ? 4 : 1;
        const auto smem_of = [&](int k) {
            return (size_t)k * a.G * a.n * 4 + 8 + (size_t)k * a.B * 8 + (size_t)k * (a.B + a.R) + 16;
        };
        while (ipc > 1 && smem_of(ipc) > 200 * 1024) --ipc;
        const size_t smem = smem_of(ipc);
        if (smem > 227 * 1024) throw tapt::SizeError("K5: instance state exceeds shared memory");
        a.ipc = ipc;
        K5_OK(cudaFuncSetAttribute(k5_real_pt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const unsigned grid = (unsigned)((a.I + ipc - 1) / ipc);
        tapt_host::note_launches(1);
        k5_real_pt<<<grid, 32 * a.G * ipc, smem, st>>>(a);
        K5_OK(cudaGetLastError());
    }

    // Verify the recorded near ties with glibc exp; false (and new overrides) if any differs.
    bool verify_ties() {
        K5_OK(cudaMemcpyAsync(h_nties, n_ties.p, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        K5_OK(cudaStreamSynchronize(st));
        const unsigned cnt = *h_nties;
        if (cnt == 0) return true;
        if (cnt > tie_cap) throw tapt::NumericError("K5: more near-tie decisions than the tie buffer holds");
        ties_seen += cnt;
        std::vector<TieRec> rec(cnt);
        K5_OK(cudaMemcpyAsync(rec.data(), ties.p, cnt * sizeof(TieRec), cudaMemcpyDeviceToHost, st));
        K5_OK(cudaStreamSynchronize(st));
        bool ok = true;
        for (const TieRec& r : rec) {
            double p;
            if (r.key.kind == kHeat || r.key.kind == kRefine)
                p = conditional_up(r.coef, r.arg);  // mcmc.cpp:13-15
            else
                p = std::exp(r.coef * r.arg);  // Eq. 1 (coef = b_{r+1}-b_r, arg = dE) / Eq. 2 (beta, E - E^T)
            const double u = (double)(r.x >> 11) * 0x1.0p-53;
            const uint32_t d = u < p ? 1u : 0u;
            if (d != r.dec) {
                h_ovr.push_back(r.key);
                h_ovr_dec.push_back(d);
                ok = false;
            }
        }
        if (!ok) {
            ovr.upload(h_ovr, st);
            ovr_dec.upload(h_ovr_dec, st);
        }
        return ok;
    }

    void snapshot() {
        s_words.copy_from(words, st);
        s_E.copy_from(E, st);
        s_so.copy_from(slot_of, st);
        s_bo.copy_from(buf_of, st);
        s_satt.copy_from(swap_att, st);
        s_sacc.copy_from(swap_acc, st);
        s_obs.copy_from(obs, st);
        s_best.copy_from(best, st);
        if (nbins) s_hist.copy_from(hist, st);
    }
    void restore() {
        words.copy_from(s_words, st);
        E.copy_from(s_E, st);
        slot_of.copy_from(s_so, st);
        buf_of.copy_from(s_bo, st);
        swap_att.copy_from(s_satt, st);
        swap_acc.copy_from(s_sacc, st);
        obs.copy_from(s_obs, st);
        best.copy_from(s_best, st);
        if (nbins) hist.copy_from(s_hist, st);
    }

    // Launch a state-changing K5 run until every near tie agrees with glibc (snapshot / replay).
    template <class Launch, class Snap, class Rest>
    void exact(Launch&& launch, Snap&& snap, Rest&& rest) {
        const bool may_tie = true;  // swaps / Eq. 2 use the band even for integer models
        if (may_tie) snap();
        for (int round = 0;; ++round) {
            n_ties.zero(st);
            launch();
            if (!may_tie || verify_ties()) break;
            if (round > 10000) throw tapt::NumericError("K5: near-tie replay did not converge");
            ++replays;
            rest();
        }
        h_ovr.clear();
        h_ovr_dec.clear();
    }

    void recompute_energies(uint32_t* w, int GG, int WW, int BB, double* out) {
        tapt_host::note_launches(1);
        k5_energy<<<dim3(GG, I), 32, 0, st>>>(w, n(), GG, WW, BB, ci.p, cj.p, cJ.p, (int)g.ci.size(), h.p, out);
        K5_OK(cudaGetLastError());
    }
    void best_from_E() {
        tapt_host::note_launches(1);
        k5_best_from_E<<<(I + 127) / 128, 128, 0, st>>>(E.p, (int)I, R, best.p);
        K5_OK(cudaGetLastError());
    }

    void prepare_targets(const uint32_t* targets, uint32_t Tn) {
        if (Tn == 0 || Tn > (uint32_t)R) throw tapt::ConfigError("n_targets must be in [1, n_slots]");
        std::vector<uint8_t> seen(R, 0);
        for (uint32_t t = 0; t < Tn; ++t) {
            if (targets[t] >= (uint32_t)R) throw tapt::ConfigError("target slot out of range");
            if (seen[targets[t]]++) throw tapt::ConfigError("duplicate target slot");
        }
        const int GT = ((int)Tn + 31) / 32;
        pwords.alloc((size_t)I * GT * n());
        pE.alloc((size_t)I * Tn);
        std::vector<uint32_t> tg(targets, targets + Tn);
        ptargets.upload(tg, st);
        std::vector<uint8_t> ps((size_t)I * Tn);
        for (uint32_t i = 0; i < I; ++i)
            for (uint32_t t = 0; t < Tn; ++t) ps[(size_t)i * Tn + t] = (uint8_t)targets[t];
        pslot.upload(ps, st);
    }

    void derive_round(uint32_t Tn, bool slot_streams) {
        pstreams.alloc((size_t)I * Tn);
        if (pfull.n != (size_t)I * R) {
            pfull.alloc((size_t)I * R);
            pfull.zero(st);
        }
        paccs.alloc(I);
        tapt_host::note_launches(1);
        k_derive_round_streams<<<I, 64, 0, st>>>(seed, gid0, ptargets.p, slot_streams ? (int)Tn : 0, R, Q + 1,
                                                 pstreams.p, pfull.p, paccs.p);
        K5_OK(cudaGetLastError());
    }

    // refinement sweeps of the proposal groups at their target's beta (draws after the n + 1
    // generator draws of the round's slot stream), then exact proposal energies
    void refine_and_energy(uint32_t Tn, uint32_t refine) {
        const int WT = std::min<int>((int)Tn, 32), GT = ((int)Tn + 31) / 32;
        if (refine) {
            K5Args a = base();
            a.words = pwords.p;
            a.G = GT;
            a.W = WT;
            a.B = (int)Tn;
            a.E = pE.p;
            a.slot_of = pslot.p;
            a.buf_of = nullptr;
            a.streams = pfull.p;
            a.draw_base = (unsigned long long)n() + 1ull;
            a.t0 = 0;
            a.n_sweeps = (int)refine;
            a.hb_kind = kRefine;
            a.key_t0 = Q << 20;
            a.best = nullptr;
            a.obs = nullptr;
            a.hist = nullptr;
            pE.zero(st);
            exact([&] { set_ovr(a); launch_k5(a); }, [&] { s_pwords.copy_from(pwords, st); },
                  [&] { pwords.copy_from(s_pwords, st); });
        }
        recompute_energies(pwords.p, GT, WT, (int)Tn, pE.p);
    }

    void finish(uint32_t Tn, const uint32_t* targets, const double* lqc, const double* lqp, uint8_t* accepted) {
        const int WT = std::min<int>((int)Tn, 32), GT = ((int)Tn + 31) / 32;
        pacc.alloc((size_t)I * Tn);
        const uint8_t* forced = nullptr;
        if (lqc) {  // MH correction: decided on the host with libm exp from device energies
            std::vector<double> Ep = pE.download(st), Eb = E.download(st);
            std::vector<uint8_t> bo = buf_of.download(st);
            std::vector<uint8_t> f((size_t)I * Tn);
            for (uint32_t i = 0; i < I; ++i) {
                const auto as = tapt::RngStream::derive(seed, {tapt::stream::kCoordinator, gid0 + i, Q + 1});
                for (uint32_t t = 0; t < Tn; ++t) {
                    const uint32_t r = targets[t];
                    const double ec = Eb[(size_t)i * R + bo[(size_t)i * R + r]], ep = Ep[(size_t)i * Tn + t];
                    const double pa =
                        std::exp(betas[r] * (ec - ep)) * std::exp(lqc[(size_t)i * Tn + t] - lqp[(size_t)i * Tn + t]);
                    const uint64_t x = as.at(r + 1);
                    f[(size_t)i * Tn + t] = (double)(x >> 11) * 0x1.0p-53 < pa ? 1 : 0;
                }
            }
            pforced.upload(f, st);
            forced = pforced.p;
        }
        K5Args a = base();
        exact(
            [&] {
                set_ovr(a);
                tapt_host::note_launches(1);
                k5_accept<<<I, std::max(32, ((int)Tn + 31) / 32 * 32), 0, st>>>(a, pE.p, (int)Tn, ptargets.p, paccs.p,
                                                                               Q, forced, pacc.p);
                K5_OK(cudaGetLastError());
            },
            [] {}, [] {});
        tapt_host::note_launches(2);
        k5_apply_accept<<<I, 32, 0, st>>>(E.p, buf_of.p, R, R, pE.p, (int)Tn, ptargets.p, pacc.p, prop_att.p,
                                          prop_acc.p, best.p);
        K5_OK(cudaGetLastError());
        k_apply_proposals<<<dim3((n() + 255) / 256, G, I), 256, 0, st>>>(words.p, n(), G, W, buf_of.p, R, pwords.p, GT,
                                                                          WT, ptargets.p, (int)Tn, pacc.p);
        K5_OK(cudaGetLastError());
        if (accepted) {
            auto v = pacc.download(st);
            std::copy(v.begin(), v.end(), accepted);
        }
        Q += 1;
    }
};

RealEngine::RealEngine(const RealGraph& g, uint32_t I, uint64_t gid0, const std::vector<double>& betas, uint64_t seed,
                       int order, cudaStream_t st)
    : p_(std::make_unique<RealEngineImpl>()) {
    auto& e = *p_;
    e.g = g;
    e.I = I;
    e.gid0 = gid0;
    e.seed = seed;
    e.R = (int)betas.size();
    e.W = std::min(e.R, 32);
    e.G = (e.R + 31) / 32;
    e.order = order;
    e.betas = betas;
    e.st = st;
    e.band = env_double("TAPT_K5_BAND", 1e-12);
    e.perturb = env_double("TAPT_K5_PERTURB", 0.0);
    if (e.G > 8) throw tapt::ConfigError("at most 256 slots");
    K5_OK(cudaMallocHost(&e.h_nties, sizeof(unsigned)));
    e.upload_graph();
    e.build_tables();
    std::vector<uint64_t> s((size_t)I * e.R), c(I);
    for (uint32_t i = 0; i < I; ++i) {
        for (int r = 0; r < e.R; ++r)
            s[(size_t)i * e.R + r] = tapt::RngStream::derive(seed, {tapt::stream::kReplica, gid0 + i, (uint64_t)r}).state();
        c[i] = tapt::RngStream::derive(seed, {tapt::stream::kCoordinator, gid0 + i}).state();
    }
    e.streams.upload(s, st);
    e.coord.upload(c, st);
    e.words.alloc((size_t)I * e.G * e.n());
    e.words.zero(st);
    e.E.alloc((size_t)I * e.R);
    e.E.zero(st);
    std::vector<uint8_t> perm((size_t)I * e.R);
    for (uint32_t i = 0; i < I; ++i)
        for (int r = 0; r < e.R; ++r) perm[(size_t)i * e.R + r] = (uint8_t)r;
    e.slot_of.upload(perm, st);
    e.buf_of.upload(perm, st);
    const size_t np = (size_t)I * std::max(e.R - 1, 1);
    e.swap_att.alloc(np);
    e.swap_acc.alloc(np);
    e.prop_att.alloc((size_t)I * e.R);
    e.prop_acc.alloc((size_t)I * e.R);
    e.swap_att.zero(st);
    e.swap_acc.zero(st);
    e.prop_att.zero(st);
    e.prop_acc.zero(st);
    e.obs.alloc((size_t)I * e.R * 5);
    e.obs.zero(st);
    std::vector<double> b(I, INFINITY);
    e.best.upload(b, st);
    e.ties.alloc(e.tie_cap);
    e.n_ties.alloc(1);
    K5_OK(cudaStreamSynchronize(st));
}

RealEngine::~RealEngine() = default;

void RealEngine::set_stream(cudaStream_t st) { p_->st = st; }
cudaStream_t RealEngine::stream() const { return p_->st; }

void RealEngine::set_betas(const std::vector<double>& betas, bool decreasing) {
    auto& e = *p_;
    K5_OK(cudaStreamSynchronize(e.st));
    e.betas = betas;
    e.ladder_decreasing = decreasing;
    e.build_tables();
}

void RealEngine::set_streams(const uint64_t* states) { p_->streams.upload(states, (size_t)p_->I * p_->R, p_->st); }

void RealEngine::init_random() {
    std::vector<uint64_t> s((size_t)p_->I * p_->R);
    for (uint32_t i = 0; i < p_->I; ++i)
        for (int r = 0; r < p_->R; ++r)
            s[(size_t)i * p_->R + r] =
                tapt::RngStream::derive(p_->seed, {tapt::stream::kInit, p_->gid0 + i, (uint64_t)r}).state();
    init_from_streams(s.data());
}

void RealEngine::init_from_streams(const uint64_t* init_states) {
    auto& e = *p_;
    Buf<uint64_t> ds;
    ds.upload(init_states, (size_t)e.I * e.R, e.st);
    std::vector<uint8_t> perm((size_t)e.I * e.R);
    for (uint32_t i = 0; i < e.I; ++i)
        for (int r = 0; r < e.R; ++r) perm[(size_t)i * e.R + r] = (uint8_t)r;
    e.slot_of.upload(perm, e.st);
    e.buf_of.upload(perm, e.st);
    tapt_host::note_launches(1);
    k_init_random<<<dim3((e.n() + 255) / 256, e.G, e.I), 256, 0, e.st>>>(e.words.p, e.n(), e.G, e.W, e.R, ds.p,
                                                                         e.clamp.p, 1);
    K5_OK(cudaGetLastError());
    e.recompute_energies(e.words.p, e.G, e.W, e.R, e.E.p);
    e.best_from_E();
    K5_OK(cudaStreamSynchronize(e.st));
}

void RealEngine::set_spins(const int8_t* host, bool force_clamps) {
    auto& e = *p_;
    Buf<int8_t> d;
    d.upload(host, (size_t)e.I * e.R * e.n(), e.st);
    tapt_host::note_launches(1);
    k_set_spins<<<dim3((e.n() + 255) / 256, e.G, e.I), 256, 0, e.st>>>(e.words.p, e.n(), e.G, e.W, e.R, e.slot_of.p,
                                                                       d.p, e.R, force_clamps ? e.clamp.p : nullptr, 1);
    K5_OK(cudaGetLastError());
    e.recompute_energies(e.words.p, e.G, e.W, e.R, e.E.p);
    e.best_from_E();
    K5_OK(cudaStreamSynchronize(e.st));
}

void RealEngine::get_spins(int8_t* host) {
    auto& e = *p_;
    Buf<int8_t> d;
    d.alloc((size_t)e.I * e.R * e.n());
    tapt_host::note_launches(1);
    k_get_spins<<<dim3((e.n() + 255) / 256, e.R, e.I), 256, 0, e.st>>>(e.words.p, e.n(), e.G, e.W, e.R, e.buf_of.p,
                                                                       e.R, d.p);
    K5_OK(cudaGetLastError());
    K5_OK(cudaMemcpyAsync(host, d.p, d.n, cudaMemcpyDeviceToHost, e.st));
    K5_OK(cudaStreamSynchronize(e.st));
}

void RealEngine::get_spins_packed(uint8_t* host) {
    auto& e = *p_;
    const int nb = (e.n() + 7) / 8;
    Buf<uint8_t> d;
    d.alloc((size_t)e.I * e.R * nb);
    tapt_host::note_launches(1);
    k_get_packed<<<dim3((nb + 255) / 256, e.R, e.I), 256, 0, e.st>>>(e.words.p, e.n(), e.G, e.W, e.buf_of.p, e.R, d.p);
    K5_OK(cudaGetLastError());
    K5_OK(cudaMemcpyAsync(host, d.p, d.n, cudaMemcpyDeviceToHost, e.st));
    K5_OK(cudaStreamSynchronize(e.st));
}

void RealEngine::get_energies(double* host) {
    auto& e = *p_;
    auto E = e.E.download(e.st);
    auto bo = e.buf_of.download(e.st);
    for (uint32_t i = 0; i < e.I; ++i)
        for (int r = 0; r < e.R; ++r) host[(size_t)i * e.R + r] = E[(size_t)i * e.R + bo[(size_t)i * e.R + r]];
}

void RealEngine::get_permutation(uint8_t* host) {
    auto bo = p_->buf_of.download(p_->st);
    std::copy(bo.begin(), bo.end(), host);
}

void RealEngine::counters(uint64_t* T, uint64_t* P, uint64_t* Q) const {
    if (T) *T = p_->T;
    if (P) *P = p_->P;
    if (Q) *Q = p_->Q;
}

void RealEngine::acceptance(uint64_t* sa, uint64_t* sc, uint64_t* pa, uint64_t* pc) {
    auto& e = *p_;
    const size_t np = (size_t)e.I * (e.R - 1);
    if (sa && np) std::copy_n(e.swap_att.download(e.st).begin(), np, sa);
    if (sc && np) std::copy_n(e.swap_acc.download(e.st).begin(), np, sc);
    if (pa) {
        auto v = e.prop_att.download(e.st);
        std::copy(v.begin(), v.end(), pa);
    }
    if (pc) {
        auto v = e.prop_acc.download(e.st);
        std::copy(v.begin(), v.end(), pc);
    }
}

void RealEngine::observables(double* host) {
    auto v = p_->obs.download(p_->st);
    std::copy(v.begin(), v.end(), host);
}

void RealEngine::set_histogram(double e_lo, double width, uint32_t nbins) {
    auto& e = *p_;
    if (!(width > 0.0)) throw tapt::ConfigError("histogram bin width must be > 0");
    e.e_lo = e_lo;
    e.width = width;
    e.nbins = (int)nbins;
    e.hist.alloc((size_t)e.R * nbins);
    e.hist.zero(e.st);
    K5_OK(cudaStreamSynchronize(e.st));
}

void RealEngine::get_histogram(uint64_t* dst, bool on_device) {
    auto& e = *p_;
    if (!e.nbins) throw tapt::ConfigError("no histogram configured");
    K5_OK(cudaMemcpyAsync(dst, e.hist.p, e.hist.n * sizeof(uint64_t),
                          on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, e.st));
    K5_OK(cudaStreamSynchronize(e.st));
}

void RealEngine::best(double* host) {
    auto v = p_->best.download(p_->st);
    std::copy(v.begin(), v.end(), host);
}

void RealEngine::reset_observables() {
    p_->obs.zero(p_->st);
    p_->hist.zero(p_->st);
    K5_OK(cudaStreamSynchronize(p_->st));
}

void RealEngine::run(uint32_t n_sweeps, uint32_t swap_every, uint32_t measure_every, uint64_t measure_from) {
    auto& e = *p_;
    if (swap_every && e.R < 2) swap_every = 0;
    if (swap_every && e.ladder_decreasing)
        throw tapt::ConfigError("replica swaps need a non-decreasing beta ladder (SPEC.md:388)");
    const uint32_t chunk_max = 256;
    for (uint32_t done = 0; done < n_sweeps;) {
        const uint32_t chunk = std::min(chunk_max, n_sweeps - done);
        K5Args a = e.base();
        a.t0 = e.T;
        a.key_t0 = e.T;
        a.n_sweeps = (int)chunk;
        a.swap_every = (int)swap_every;
        a.p0 = e.P;
        a.measure_every = (int)measure_every;
        a.measure_from = measure_from;
        e.exact([&] { e.set_ovr(a); e.launch_k5(a); }, [&] { e.snapshot(); }, [&] { e.restore(); });
        if (swap_every) e.P += (e.T + chunk) / swap_every - e.T / swap_every;
        e.T += chunk;
        done += chunk;
    }
}

void RealEngine::swap_pass(int parity) {
    auto& e = *p_;
    if (e.ladder_decreasing) throw tapt::ConfigError("replica swaps need a non-decreasing beta ladder (SPEC.md:388)");
    if (e.R >= 2) {
        K5Args a = e.base();
        a.pass_only = parity;
        a.p0 = e.P;
        a.t0 = e.T;
        a.best = nullptr;
        e.exact([&] { e.set_ovr(a); e.launch_k5(a); }, [&] { e.snapshot(); }, [&] { e.restore(); });
    }
    e.P += 1;
}

void RealEngine::inject(const int8_t* props, bool on_device, const uint32_t* targets, uint32_t T, const double* lqc,
                        const double* lqp, uint8_t* accepted) {
    auto& e = *p_;
    if ((lqc == nullptr) != (lqp == nullptr)) throw tapt::ConfigError("log_q_cur and log_q_prop go together");
    e.prepare_targets(targets, T);
    const int WT = std::min<int>((int)T, 32), GT = ((int)T + 31) / 32;
    const int8_t* src = props;
    if (!on_device) {
        e.pint8.upload(props, (size_t)e.I * T * e.n(), e.st);
        src = e.pint8.p;
    }
    tapt_host::note_launches(1);
    k_set_spins<<<dim3((e.n() + 255) / 256, GT, e.I), 256, 0, e.st>>>(e.pwords.p, e.n(), GT, WT, (int)T, nullptr, src,
                                                                      (int)T, e.clamp.p, 1);
    K5_OK(cudaGetLastError());
    e.derive_round(T, false);
    e.refine_and_energy(T, 0);
    e.finish(T, targets, lqc, lqp, accepted);
    K5_OK(cudaStreamSynchronize(e.st));
}

void RealEngine::inject_packed(const uint8_t* props, bool on_device, const uint32_t* targets, uint32_t T,
                               uint32_t refine, uint8_t* accepted) {
    auto& e = *p_;
    e.prepare_targets(targets, T);
    const int WT = std::min<int>((int)T, 32), GT = ((int)T + 31) / 32;
    const int nb = (e.n() + 7) / 8;
    const uint8_t* src = props;
    if (!on_device) {
        e.pbytes.upload(props, (size_t)e.I * T * nb, e.st);
        src = e.pbytes.p;
    }
    tapt_host::note_launches(1);
    k_set_packed<<<dim3((e.n() + 255) / 256, GT, e.I), 256, 0, e.st>>>(e.pwords.p, e.n(), GT, WT, (int)T, src, (int)T,
                                                                       e.clamp.p, 1);
    K5_OK(cudaGetLastError());
    e.derive_round(T, refine > 0);
    e.refine_and_energy(T, refine);
    e.finish(T, targets, nullptr, nullptr, accepted);
    K5_OK(cudaStreamSynchronize(e.st));
}

void RealEngine::generate(const uint32_t* targets, uint32_t T, const double* m_bias, uint32_t refine,
                          uint8_t* accepted) {
    auto& e = *p_;
    e.prepare_targets(targets, T);
    const int WT = std::min<int>((int)T, 32), GT = ((int)T + 31) / 32;
    e.derive_round(T, true);
    std::vector<uint64_t> tup(2 * T);
    for (uint32_t t = 0; t < T; ++t) {
        const double mb = m_bias ? m_bias[t] : 0.0;
        tup[2 * t + 0] = threshold_of((1.0 + -1.0 * mb) / 2.0);
        tup[2 * t + 1] = threshold_of((1.0 + 1.0 * mb) / 2.0);
    }
    e.ptup.upload(tup, e.st);
    tapt_host::note_launches(1);
    k_gen_proposals<<<dim3((e.n() + 255) / 256, GT, e.I), 256, 0, e.st>>>(e.pwords.p, e.n(), GT, WT, (int)T,
                                                                          e.pstreams.p, e.ptup.p, e.clamp.p, 1);
    K5_OK(cudaGetLastError());
    e.refine_and_energy(T, refine);
    e.finish(T, targets, nullptr, nullptr, accepted);
    K5_OK(cudaStreamSynchronize(e.st));
}

void RealEngine::dropin_sweeps(int8_t* s, double beta, uint64_t state, uint32_t n_sweeps, double* dE,
                               const uint64_t*, int, int) {
    auto& e = *p_;
    if (e.I != 1 || e.R != 1) throw tapt::ConfigError("drop-in engine has one replica");
    if (e.betas[0] != beta) set_betas({beta}, false);
    e.streams.upload(&state, 1, e.st);
    Buf<int8_t> d;
    d.upload(s, e.n(), e.st);
    tapt_host::note_launches(1);
    k_set_spins<<<dim3((e.n() + 255) / 256, 1, 1), 256, 0, e.st>>>(e.words.p, e.n(), 1, 1, 1, e.slot_of.p, d.p, 1,
                                                                   nullptr, 1);
    K5_OK(cudaGetLastError());
    e.E.zero(e.st);
    e.dE_dev.alloc(std::max<uint32_t>(n_sweeps, 1));
    for (uint32_t done = 0; done < n_sweeps;) {
        const uint32_t chunk = std::min<uint32_t>(4096, n_sweeps - done);
        K5Args a = e.base();
        a.t0 = done;
        a.key_t0 = done;
        a.n_sweeps = (int)chunk;
        a.dE_out = e.dE_dev.p + done;
        a.best = nullptr;
        e.exact([&] { e.set_ovr(a); e.launch_k5(a); }, [&] { e.snapshot(); }, [&] { e.restore(); });
        done += chunk;
    }
    get_spins(s);
    if (dE) {
        K5_OK(cudaMemcpyAsync(dE, e.dE_dev.p, n_sweeps * sizeof(double), cudaMemcpyDeviceToHost, e.st));
        K5_OK(cudaStreamSynchronize(e.st));
    }
}

void RealEngine::dropin_update(int8_t* s, uint32_t site, double beta, uint64_t state, const uint64_t*, int, int) {
    auto& e = *p_;
    if (e.I != 1 || e.R != 1) throw tapt::ConfigError("drop-in engine has one replica");
    if (e.betas[0] != beta) set_betas({beta}, false);
    e.streams.upload(&state, 1, e.st);
    Buf<int8_t> d;
    d.upload(s, e.n(), e.st);
    tapt_host::note_launches(1);
    k_set_spins<<<dim3((e.n() + 255) / 256, 1, 1), 256, 0, e.st>>>(e.words.p, e.n(), 1, 1, 1, e.slot_of.p, d.p, 1,
                                                                   nullptr, 1);
    K5_OK(cudaGetLastError());
    const uint32_t zero = 0;
    e.upd_visit.upload(&site, 1, e.st);
    e.upd_draw.upload(&zero, 1, e.st);
    K5Args a = e.base();
    a.visit = e.upd_visit.p;
    a.vdraw = e.upd_draw.p;
    a.nv = 1;
    a.stride = 1;
    a.t0 = 0;
    a.key_t0 = 0;
    a.n_sweeps = 1;
    a.best = nullptr;
    e.exact([&] { e.set_ovr(a); e.launch_k5(a); }, [&] { e.snapshot(); }, [&] { e.restore(); });
    get_spins(s);
}

unsigned long long RealEngine::ties_seen() const { return p_->ties_seen; }
unsigned long long RealEngine::replays() const { return p_->replays; }
const char* RealEngine::kernel_name() const { return "k5_real_pt"; }

}  // namespace tapt_real
