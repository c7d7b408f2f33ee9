// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the UNMODIFIED reference sources
// (/root/reference/proj/src/{spin_model,lattice,mcmc}.cpp, compiled by
// oracle/Makefile into oracle/_ref/libtapt_ref.so).  Used to pin the C
// restatement in oracle/tapt_oracle.c, to produce tests/golden/, and as the
// CPU baseline ("kind": "reference") timed by bench.py.
//
// The reference has no parallel-tempering driver (proj/src/tempering.cpp:1 is a
// placeholder), so ref_pt_run restates SPEC.md:400-441 on top of the
// reference's own gibbs_sweep (mcmc.cpp:30-45), energy (spin_model.cpp:79-89),
// random_configuration (spin_model.cpp:116-121) and RngStream (rng.hpp), with
// the stream/draw conventions of DESIGN.md section 3.  Everything that draws
// random numbers or sweeps spins is the reference's code.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "tapt/lattice.hpp"
#include "tapt/mcmc.hpp"
#include "tapt/rng.hpp"
#include "tapt/spin_model.hpp"
#include "tapt/threading.hpp"

using namespace tapt;

namespace {

RngStream derive_path(std::uint64_t root, const std::uint64_t* p, int n) {
    switch (n) {
        case 0: return RngStream::derive(root, {});
        case 1: return RngStream::derive(root, {p[0]});
        case 2: return RngStream::derive(root, {p[0], p[1]});
        case 3: return RngStream::derive(root, {p[0], p[1], p[2]});
        case 4: return RngStream::derive(root, {p[0], p[1], p[2], p[3]});
        default: return RngStream::derive(root, {p[0], p[1], p[2], p[3], p[4]});
    }
}

}  // namespace

extern "C" {

void ref_draws(std::uint64_t root, const std::uint64_t* path, int n, std::uint64_t count, std::uint64_t* out) {
    RngStream r = derive_path(root, path, n);
    for (std::uint64_t k = 0; k < count; ++k) out[k] = r.next_u64();
}

std::uint64_t ref_derive_state(std::uint64_t root, const std::uint64_t* path, int n) {
    return derive_path(root, path, n).state();
}

void* ref_graph_build(std::uint32_t n, std::uint32_t nc, const std::uint32_t* ci, const std::uint32_t* cj,
                      const double* J, const double* h, const std::int8_t* clamp) {
    CouplingGraph::Builder b(n);
    for (std::uint32_t k = 0; k < nc; ++k) b.add_coupling(ci[k], cj[k], J[k]);
    if (h)
        for (std::uint32_t i = 0; i < n; ++i)
            if (h[i] != 0.0) b.add_field(i, h[i]);
    if (clamp)
        for (std::uint32_t i = 0; i < n; ++i)
            if (clamp[i]) b.set_clamp(i, clamp[i]);
    return new CouplingGraph(b.build());
}

void* ref_graph_lattice(int kind, int ly, int lx, int l, double J, int periodic) {
    auto bnd = periodic ? LatticeSpec::Boundary::periodic : LatticeSpec::Boundary::open;
    LatticeSpec s = kind == 2 ? LatticeSpec::grid2d(ly, lx, J, bnd) : LatticeSpec::grid3d(l, J, bnd);
    return new CouplingGraph(s.graph());
}

// The reference tests' random graph (proj/tests/test_spin_model.cpp:24-32): for each i, an edge
// (i, j > i) with probability edge_prob and a standard-normal coupling (RngStream::normal), then a
// normal field if `fields`; draws from RngStream(seed) in that order.  Writes the Builder input
// (ci, cj, J: up to n(n-1)/2 entries; h: n) and returns the coupling count.
std::uint32_t ref_random_graph(std::uint32_t n, double edge_prob, int fields, std::uint64_t seed, std::uint32_t* ci,
                               std::uint32_t* cj, double* J, double* h) {
    RngStream rng(seed);
    std::uint32_t m = 0;
    for (std::uint32_t i = 0; i < n; ++i) {
        for (std::uint32_t j = i + 1; j < n; ++j)
            if (rng.uniform() < edge_prob) {
                ci[m] = i;
                cj[m] = j;
                J[m] = rng.normal();
                ++m;
            }
        h[i] = fields ? rng.normal() : 0.0;
    }
    return m;
}

void ref_graph_free(void* g) { delete static_cast<CouplingGraph*>(g); }

std::uint32_t ref_graph_n(void* g) { return static_cast<std::uint32_t>(static_cast<CouplingGraph*>(g)->n_spins()); }
std::uint32_t ref_graph_ncoup(void* g) {
    return static_cast<std::uint32_t>(static_cast<CouplingGraph*>(g)->couplings().size());
}
void ref_graph_couplings(void* gp, std::uint32_t* ci, std::uint32_t* cj, double* J) {
    const auto& c = static_cast<CouplingGraph*>(gp)->couplings();
    for (std::size_t k = 0; k < c.size(); ++k) {
        ci[k] = c[k].i;
        cj[k] = c[k].j;
        J[k] = c[k].value;
    }
}
std::uint64_t ref_graph_digest(void* g) { return static_cast<CouplingGraph*>(g)->digest(); }

double ref_energy(void* g, const std::int8_t* s) {
    auto* G = static_cast<CouplingGraph*>(g);
    return energy(*G, std::span<const std::int8_t>(s, G->n_spins()));
}

double ref_local_field(void* g, const std::int8_t* s, std::uint32_t i) {
    auto* G = static_cast<CouplingGraph*>(g);
    return local_field(*G, std::span<const std::int8_t>(s, G->n_spins()), i);
}

void ref_random_configuration(void* g, std::uint64_t root, const std::uint64_t* path, int n, std::int8_t* out) {
    auto* G = static_cast<CouplingGraph*>(g);
    RngStream r = derive_path(root, path, n);
    SpinConfiguration s = random_configuration(*G, r);
    std::memcpy(out, s.data(), s.size());
}

// gibbs_update (mcmc.cpp:24-28) at site i with stream derive(root, path); *clamped = 1 when the
// reference throws ClampedSiteError.  Returns the stream state afterwards.
std::uint64_t ref_gibbs_update(void* g, std::int8_t* spins, std::uint32_t i, double beta, std::uint64_t root,
                               const std::uint64_t* path, int n, int* clamped) {
    auto* G = static_cast<CouplingGraph*>(g);
    RngStream r = derive_path(root, path, n);
    SpinConfiguration s(spins, spins + G->n_spins());
    *clamped = 0;
    try {
        gibbs_update(*G, s, i, beta, r);
    } catch (const ClampedSiteError&) {
        *clamped = 1;
    }
    std::memcpy(spins, s.data(), s.size());
    return r.state();
}

// n_sweeps consecutive reference gibbs_sweep calls on one stream; dE per sweep.
void ref_gibbs_sweeps(void* g, std::int8_t* spins, double beta, std::uint64_t root, const std::uint64_t* path,
                      int n, std::uint64_t n_sweeps, double* dE) {
    auto* G = static_cast<CouplingGraph*>(g);
    RngStream r = derive_path(root, path, n);
    SpinConfiguration s(spins, spins + G->n_spins());
    for (std::uint64_t k = 0; k < n_sweeps; ++k) {
        double d = gibbs_sweep(*G, s, beta, r);
        if (dE) dE[k] = d;
    }
    std::memcpy(spins, s.data(), s.size());
}

// run_chain output (mcmc.cpp:47-65): records [n_records][n].
void ref_run_chain(void* g, double beta, std::uint64_t mixing, std::uint64_t thinning, std::uint64_t seed,
                   std::uint64_t n_records, std::int8_t* out) {
    auto* G = static_cast<CouplingGraph*>(g);
    ChainConfig c;
    c.beta = beta;
    c.mixing_sweeps = mixing;
    c.thinning = thinning;
    c.seed = seed;
    SampleDataset d = run_chain(*G, c, n_records);
    for (std::size_t r = 0; r < d.records.size(); ++r)
        std::memcpy(out + r * G->n_spins(), d.records[r].spins.data(), G->n_spins());
}

// generate_training_corpus (mcmc.cpp:67-84): records [n_betas * per_beta][n] in reference order.
void ref_generate_corpus(void* g, const double* betas, int nb, std::uint64_t per_beta, std::uint64_t mixing,
                         std::uint64_t thinning, std::uint64_t seed, std::int8_t* out) {
    auto* G = static_cast<CouplingGraph*>(g);
    ChainConfig c;
    c.mixing_sweeps = mixing;
    c.thinning = thinning;
    c.seed = seed;
    std::vector<double> b(betas, betas + nb);
    SampleDataset d = generate_training_corpus(*G, b, per_beta, c, 1);
    for (std::size_t r = 0; r < d.records.size(); ++r)
        std::memcpy(out + r * G->n_spins(), d.records[r].spins.data(), G->n_spins());
}

// Restated PT/TAPT schedule over the reference's sweep, for
// n_inst instances (gids gid0..gid0+n_inst-1), each with its own graph graphs[k].
// Per global sweep T (1-based): every slot sweeps; if swap_every | T a swap pass
// with parity (pass & 1); if prop_every | T a synthetic proposal round for slots
// r < n_targets (i.i.d. with bias m_bias[r], then `refine` reference sweeps,
// then Eq. 2).  Outputs are by slot: spins [I][R][n], E [I][R], swap
// accept counts [I][R-1], proposal accept counts [I][R].  Threads: parallel_for
// over instances (threading.hpp:14-35), results independent of thread count.
void ref_pt_run(void** graphs, int n_inst, std::uint64_t gid0, int R, const double* beta, std::uint64_t seed,
                std::uint64_t n_sweeps, std::uint64_t swap_every, std::uint64_t prop_every, int n_targets,
                const double* m_bias, int refine, unsigned n_threads, std::int8_t* spins_out, double* E_out,
                std::uint64_t* swap_acc, std::uint64_t* prop_acc) {
    parallel_for(static_cast<std::size_t>(n_inst), n_threads, [&](std::size_t k) {
        const CouplingGraph& g = *static_cast<CouplingGraph*>(graphs[k]);
        const std::size_t n = g.n_spins();
        const std::uint64_t gid = gid0 + k;
        std::vector<SpinConfiguration> S(R);
        std::vector<double> E(R);
        std::vector<RngStream> dyn(R);
        for (int r = 0; r < R; ++r) {
            RngStream init = RngStream::derive(seed, {stream::kInit, gid, static_cast<std::uint64_t>(r)});
            S[r] = random_configuration(g, init);
            E[r] = energy(g, S[r]);
            dyn[r] = RngStream::derive(seed, {stream::kReplica, gid, static_cast<std::uint64_t>(r)});
        }
        RngStream coord = RngStream::derive(seed, {stream::kCoordinator, gid});
        std::uint64_t pass = 0, round = 0;
        std::vector<double> u(R);
        for (std::uint64_t T = 1; T <= n_sweeps; ++T) {
            for (int r = 0; r < R; ++r) E[r] += gibbs_sweep(g, S[r], beta[r], dyn[r]);
            if (swap_every && T % swap_every == 0) {
                for (int r = 0; r < R; ++r) u[r] = coord.uniform();
                for (int r = static_cast<int>(pass & 1); r + 1 < R; r += 2) {
                    if (u[r] < std::exp((beta[r + 1] - beta[r]) * (E[r + 1] - E[r]))) {
                        std::swap(S[r], S[r + 1]);
                        std::swap(E[r], E[r + 1]);
                        if (swap_acc) swap_acc[k * (R - 1) + r] += 1;
                    }
                }
                ++pass;
            }
            if (prop_every && T % prop_every == 0) {
                RngStream acc = RngStream::derive(seed, {stream::kCoordinator, gid, round + 1});
                for (int r = 0; r < R; ++r) u[r] = acc.uniform();
                for (int r = 0; r < n_targets && r < R; ++r) {
                    RngStream q = RngStream::derive(seed, {stream::kReplica, gid, static_cast<std::uint64_t>(r), round + 1});
                    const double sign = q.coin() ? 1.0 : -1.0;
                    const double p_up = (1.0 + sign * m_bias[r]) / 2.0;
                    SpinConfiguration P(n);
                    for (std::size_t i = 0; i < n; ++i) P[i] = q.uniform() < p_up ? 1 : -1;
                    apply_clamps(g, P);
                    for (int m = 0; m < refine; ++m) gibbs_sweep(g, P, beta[r], q);
                    const double EP = energy(g, P);
                    if (u[r] < std::exp(beta[r] * (E[r] - EP))) {
                        S[r] = std::move(P);
                        E[r] = EP;
                        if (prop_acc) prop_acc[k * R + r] += 1;
                    }
                }
                ++round;
            }
        }
        for (int r = 0; r < R; ++r) {
            if (spins_out) std::memcpy(spins_out + (k * R + r) * n, S[r].data(), n);
            if (E_out) E_out[k * R + r] = E[r];
        }
    });
}

}  // extern "C"
