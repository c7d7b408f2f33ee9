// C++ drop-in API test driver (compiled and run by tests/test_cpp_api.py).
// Re-expresses the reference's own doctest assertions (proj/tests/test_spin_model.cpp) against
// include/tapt/*.hpp, and exercises the device paths (gibbs_sweep, run_chain, run_pt/run_tapt).
#include <cassert>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <sstream>

#include "tapt/distributed.hpp"
#include "tapt/generator.hpp"
#include "tapt/lattice.hpp"
#include "tapt/mcmc.hpp"
#include "tapt/tempering.hpp"

using namespace tapt;

#define CHECK(c)                                                              \
    do {                                                                      \
        if (!(c)) {                                                           \
            std::fprintf(stderr, "CHECK failed: %s (line %d)\n", #c, __LINE__); \
            return 1;                                                         \
        }                                                                     \
    } while (0)

template <class E, class F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static CouplingGraph and_gate() {
    CouplingGraph::Builder b(3);
    b.add_coupling(0, 1, -1.0).add_coupling(0, 2, 2.0).add_coupling(1, 2, 2.0);
    b.add_field(0, 1.0).add_field(1, 1.0).add_field(2, -2.0);
    return b.build();
}

static int cpu_tests() {
    // test_spin_model.cpp:36-65
    auto g22 = LatticeSpec::grid2d(2, 2).graph();
    CHECK(energy(g22, SpinConfiguration(4, 1)) == -4.0);
    CouplingGraph::Builder b1(1);
    b1.add_field(0, 2.0);
    CHECK(energy(b1.build(), SpinConfiguration{1}) == -2.0);
    CHECK(energy(and_gate(), SpinConfiguration{1, 1, 1}) == -3.0);
    CHECK(throws<DimensionError>([&] { energy(g22, SpinConfiguration(3, 1)); }));
    // :67-97 local field
    auto g33 = LatticeSpec::grid2d(3, 3).graph();
    SpinConfiguration s3(9, 1);
    CHECK(local_field(g33, s3, 4) == 4.0);
    CouplingGraph::Builder bc(2);
    bc.add_coupling(0, 1, 1.0).set_clamp(0, 1);
    CHECK(throws<ClampedSiteError>([&] { local_field(bc.build(), SpinConfiguration{1, 1}, 0); }));
    // :99-122 flip delta
    for (std::uint32_t i = 0; i < 4; ++i) CHECK(flip_delta(g22, SpinConfiguration(4, 1), i) == 4.0);
    CHECK(flip_delta(and_gate(), SpinConfiguration{1, 1, 1}, 2) == 4.0);
    // :124-137 flip identity on random graphs
    RngStream rng(12345);
    for (int trial = 0; trial < 20; ++trial) {
        CouplingGraph::Builder b(10);
        for (std::uint32_t i = 0; i < 10; ++i) {
            for (std::uint32_t j = i + 1; j < 10; ++j)
                if (rng.uniform() < 0.4) b.add_coupling(i, j, rng.normal());
            if (trial % 2 == 0) b.add_field(i, rng.normal());
        }
        auto g = b.build();
        auto s = random_configuration(g, rng);
        const double e0 = energy(g, s);
        for (std::uint32_t i = 0; i < 10; ++i) {
            auto f = s;
            f[i] = static_cast<std::int8_t>(-f[i]);
            CHECK(std::fabs(energy(g, f) - e0 - flip_delta(g, s, i)) < 1e-12);
        }
    }
    // :189-233 instance file round trip and parse errors
    {
        std::ostringstream os;
        and_gate().save(os);
        std::istringstream is(os.str());
        auto g = CouplingGraph::load(is);
        CHECK(g.digest() == and_gate().digest());
        std::istringstream bad("isingmodel v2\nn 2\n");
        CHECK(throws<FormatError>([&] { CouplingGraph::load(bad); }));
        std::istringstream dup("isingmodel v1\nn 3\nc 0 1 1\nc 1 0 2\n");
        CHECK(throws<FormatError>([&] { CouplingGraph::load(dup); }));
        std::istringstream self("isingmodel v1\nn 2\nc 0 0 1.0\n");
        CHECK(throws<ConfigError>([&] { CouplingGraph::load(self); }));
    }
    // :235-242 builder merges duplicates
    CouplingGraph::Builder bm(3);
    bm.add_coupling(0, 1, 1.5).add_coupling(1, 0, 0.5);
    auto gm = bm.build();
    CHECK(gm.couplings().size() == 1 && gm.couplings()[0].value == 2.0);
    // :244-259 lattice counts and bijection
    auto s2 = LatticeSpec::grid2d(4, 5);
    CHECK(s2.n_sites() == 20 && s2.n_edges() == 4 * 4 + 5 * 3 && s2.graph().couplings().size() == s2.n_edges());
    CHECK(s2.index2d(1, 0) == 5);
    auto sp = LatticeSpec::grid3d(3);
    CHECK(sp.n_sites() == 27 && sp.n_edges() == 54 && sp.graph().couplings().size() == 54);
    CHECK(sp.index3d(0, 1, 0) == 3 && sp.index3d(0, 0, 1) == 9);
    // ISFD1 round trip
    SampleDataset d;
    d.records.push_back({0.5, SpinConfiguration{1, -1, 1, 1, -1, -1, 1, -1, 1}});
    std::ostringstream os;
    d.save(os);
    std::istringstream is(os.str());
    auto d2 = SampleDataset::load(is);
    CHECK(d2.records.size() == 1 && d2.records[0].spins == d.records[0].spins && d2.records[0].beta == 0.5);
    {   // mcmc.cpp:142: a trailing partial beta is a clean end of file; a cut inside a record throws
        std::istringstream tail(os.str() + std::string(3, '\x01'));
        CHECK(SampleDataset::load(tail).records.size() == 1);
        std::istringstream cut(os.str().substr(0, os.str().size() - 1));
        CHECK(throws<FormatError>([&] { SampleDataset::load(cut); }));
    }
    // C ABI digest matches
    std::uint64_t dig = 0;
    CHECK(tapt_model_digest(and_gate().device(), &dig) == TAPT_OK && dig == and_gate().digest());
    // IsingFormer host side: default parameter count, ISFW1 round trip
    {
        GeneratorConfig gc;
        CHECK(gc.parameter_count() == 68353);
        auto gl = LatticeSpec::grid2d(4, 4, 1.0, LatticeSpec::Boundary::periodic).graph();
        IsingFormer f(gl, gc, IsingFormer::init_params(gc, 1));
        const std::string path = "tests/cpp/build/former_cpu.isfw";
        f.save_checkpoint(path);
        auto f2 = IsingFormer::load_checkpoint(gl, path);
        CHECK(f2.config().max_sequence_length == gc.max_sequence_length && f2.prefix_length() == 0);
        CHECK(throws<DimensionError>([&] { IsingFormer(gl, gc, ParameterSet(10)); }));
    }
    // residual_energy: mean over runs of the coldest replica's energy, minus E_gnd, / N
    {
        auto chain = [](double e_cold, double e_best) {
            RunTrace t;
            t.energies = {{0.0, 5.0, e_cold}, {1.0, e_cold}};
            t.best_energy = {e_best, e_best};
            return t;
        };
        const double eg = -9.0;  // open ferromagnetic chain, N = 10 spins, J = 1: E_gnd = -9
        auto r0 = residual_energy(chain(eg, eg), eg, 10);
        CHECK(r0.size() == 2 && r0[0] == 0.0 && r0[1] == 0.0);                 // trace at the ground state
        auto r1 = residual_energy(chain(eg + 2.0, eg + 2.0), eg, 10);          // one excited bond, dE = 2J
        CHECK(std::fabs(r1[0] - 0.2) < 1e-15 && std::fabs(r1[1] - 0.2) < 1e-15);
        auto r2 = residual_energy(std::vector<RunTrace>{chain(eg, eg), chain(eg + 4.0, eg + 4.0)}, eg, 10);
        CHECK(std::fabs(r2[0] - 0.2) < 1e-15);                                 // mean over runs
        auto r3 = residual_energy(std::vector<RunTrace>{chain(eg + 4.0, eg)}, eg, 10, true);
        CHECK(r3[0] == 0.0);                                                   // best-so-far variant
        RunTrace shorter = chain(eg, eg);
        shorter.energies.pop_back();
        CHECK(throws<DimensionError>([&] { residual_energy(std::vector<RunTrace>{chain(eg, eg), shorter}, eg, 10); }));
        CHECK(throws<ConfigError>([&] { residual_energy(std::vector<RunTrace>{}, eg, 10); }));
    }
    std::printf("cpu ok\n");
    return 0;
}

// Synthetic proposal source (stand-in for the IsingFormer): fair i.i.d. spins.
struct IidSource : ProposalSource {
    SpinConfiguration sample(std::size_t, double, std::span<const std::int8_t> ctx, std::size_t, RngStream& rng) override {
        SpinConfiguration s(ctx.size());
        for (auto& v : s) v = rng.coin() ? 1 : -1;
        return s;
    }
};

static int gpu_tests() {
    // gibbs_sweep drop-in: same result as the sequential host restatement of mcmc.cpp:30-45
    auto g = LatticeSpec::grid2d(16, 16, 1.0, LatticeSpec::Boundary::periodic).graph();
    RngStream init(7);
    auto s = random_configuration(g, init);
    auto h = s;
    RngStream r1 = RngStream::derive(1, {stream::kChain});
    RngStream r2 = r1;
    for (int k = 0; k < 5; ++k) {
        const double d = gibbs_sweep(g, s, 0.6, r1);
        double dh = 0.0;  // host restatement
        for (std::uint32_t i : g.free_sites()) {
            const double l = local_field(g, h, i);
            const std::int8_t nx = r2.uniform() < 1.0 / (1.0 + std::exp(-2.0 * 0.6 * l)) ? 1 : -1;
            if (nx != h[i]) {
                dh += 2.0 * h[i] * l;
                h[i] = nx;
            }
        }
        CHECK(d == dh && s == h && r1.state() == r2.state());
    }
    // real-valued couplings (the reference tests' Gaussian random graphs, test_spin_model.cpp:24-32):
    // the drop-in gibbs_sweep / gibbs_update run on K5 and equal the host restatement bit for bit
    {
        RngStream gr(4242);
        CouplingGraph::Builder b(30);
        for (std::uint32_t i = 0; i < 30; ++i) {
            for (std::uint32_t j = i + 1; j < 30; ++j)
                if (gr.uniform() < 0.2) b.add_coupling(i, j, gr.normal());
            b.add_field(i, gr.normal());
        }
        b.set_clamp(7, -1);
        auto gg = b.build();
        RngStream ri(5);
        auto sd = random_configuration(gg, ri), sh = sd;
        RngStream d1 = RngStream::derive(3, {stream::kChain}), d2 = d1;
        for (int k = 0; k < 10; ++k) {
            const double dd = gibbs_sweep(gg, sd, 0.9, d1);
            double dh = 0.0;
            for (std::uint32_t i : gg.free_sites()) {
                const double l = local_field(gg, sh, i);
                const std::int8_t nx = d2.uniform() < 1.0 / (1.0 + std::exp(-2.0 * 0.9 * l)) ? 1 : -1;
                if (nx != sh[i]) {
                    dh += 2.0 * sh[i] * l;
                    sh[i] = nx;
                }
            }
            CHECK(dd == dh && sd == sh && d1.state() == d2.state());
        }
        for (std::uint32_t i = 0; i < 30; ++i) {
            if (i == 7) {
                CHECK(throws<ClampedSiteError>([&] { gibbs_update(gg, sd, i, 1.1, d1); }));
                continue;
            }
            const double l = local_field(gg, sh, i);
            sh[i] = d2.uniform() < 1.0 / (1.0 + std::exp(-2.0 * 1.1 * l)) ? 1 : -1;
            gibbs_update(gg, sd, i, 1.1, d1);
            CHECK(sd == sh && d1.state() == d2.state());
        }
        // PT on it: energies stay the reference's doubles (E += gibbs_sweep's return)
        auto lad = BetaLadder::geometric(0.3, 2.0, 6);
        TAPTConfig c;
        c.n_swap = 20;
        c.M = 2;
        c.seed = 6;
        auto tr = run_pt(gg, lad, c);
        CHECK(std::fabs(energy(gg, tr.final_state) - tr.final_energy) < 1e-9);
    }
    // run_chain: deterministic per seed, records distinct
    ChainConfig cc;
    cc.beta = 0.4;
    cc.mixing_sweeps = 10;
    cc.thinning = 2;
    cc.seed = 3;
    auto ds = run_chain(g, cc, 4);
    CHECK(ds.records.size() == 4 && ds.graph_digest == g.digest());
    auto ds2 = run_chain(g, cc, 4);
    for (int k = 0; k < 4; ++k) CHECK(ds.records[k].spins == ds2.records[k].spins);
    // batched corpus == per-beta run_chain (mcmc.cpp:67-84 semantics, two device paths)
    {
        ChainConfig c2;
        c2.mixing_sweeps = 5;
        c2.thinning = 3;
        c2.seed = 11;
        std::vector<double> bs{0.3, 0.9, 0.5};
        auto corpus = generate_training_corpus(g, bs, 2, c2);
        CHECK(corpus.records.size() == 6);
        for (std::size_t bi = 0; bi < bs.size(); ++bi) {
            ChainConfig c = c2;
            c.beta = bs[bi];
            c.seed = RngStream::derive(c2.seed, {stream::kChain, bi}).state();
            auto one = run_chain(g, c, 2);
            for (int k = 0; k < 2; ++k) CHECK(one.records[k].spins == corpus.records[bi * 2 + k].spins);
        }
    }
    // run_pt / run_tapt move audit and best-energy monotonicity
    auto ladder = BetaLadder::geometric(0.2, 1.0, 8);
    TAPTConfig cfg;
    cfg.n_swap = 30;
    cfg.M = 2;
    cfg.seed = 9;
    auto tr = run_pt(g, ladder, cfg);
    for (std::size_t m = 0; m < tr.move_kind.size(); ++m) CHECK(tr.move_kind[m] == int(m % 3) + 1);
    for (std::size_t m = 1; m < tr.best_energy.size(); ++m) CHECK(tr.best_energy[m] <= tr.best_energy[m - 1]);
    CHECK(energy(g, tr.final_state) == tr.final_energy);
    cfg.N_T = 4;
    IidSource src;
    auto tt = run_tapt(g, ladder, cfg, &src);
    std::uint64_t att = 0;
    for (auto v : tt.gen_attempts) att += v;
    CHECK(att == 4 * 10);
    cfg.n_swap = 0;
    auto t0 = run_pt(g, ladder, cfg);
    CHECK(t0.move_kind.empty());
    auto rho = residual_energy(tr, -2.0 * 256, 256);
    CHECK(rho.size() == tr.energies.size() && rho.back() >= 0.0);
    // IsingFormer as run_tapt's proposal source with the MH-corrected move
    {
        GeneratorConfig gc;
        gc.max_sequence_length = 256;
        IsingFormer gen(g, gc, IsingFormer::init_params(gc, 5, 1.0));
        RngStream rr(3);
        auto p = gen.sample(0, 0.5, {}, 0, rr);
        CHECK(std::fabs(gen.last_log_q() - gen.log_prob(p, 0.5)) < 1e-4);
        CHECK(rr.state() == RngStream(3).state() + 256 * 0x9E3779B97F4A7C15ull);
        const std::string path = "tests/cpp/build/former_gpu.isfw";
        gen.save_checkpoint(path);
        auto g2 = IsingFormer::load_checkpoint(g, path);
        CHECK(g2.forward_logits(p, 0.5) == gen.forward_logits(p, 0.5));
        TAPTConfig c3 = cfg;
        c3.n_swap = 30;
        c3.N_T = 4;
        c3.mh_corrected = true;
        c3.context_fraction = 0.25;
        auto tf = run_tapt(g, ladder, c3, &gen);
        std::uint64_t a3 = 0;
        for (auto v : tf.gen_attempts) a3 += v;
        CHECK(a3 == 4 * 10 && energy(g, tf.final_state) == tf.final_energy);
    }
    auto al = adaptive_ladder(g, 0.2, 1.0, 0.5, 50, 1);
    for (std::size_t r = 1; r < al.betas.size(); ++r) CHECK(al.betas[r] > al.betas[r - 1]);
    CHECK(al.betas.front() == 0.2 && al.betas.back() == 1.0);
    // adaptive_ladder's SPEC.md:447-449 examples, measured with run_pt on the ladder it returns
    auto pair_acceptance = [](const CouplingGraph& gg, const BetaLadder& lad, std::uint64_t moves) {
        TAPTConfig c;
        c.n_swap = moves;
        c.M = 1;
        c.seed = 21;
        auto t = run_pt(gg, lad, c);
        std::vector<double> acc;
        for (std::size_t r = 0; r + 1 < lad.betas.size(); ++r)
            acc.push_back(double(t.swap_accepts[r]) / double(std::max<std::uint64_t>(t.swap_attempts[r], 1)));
        return acc;
    };
    {  // zero-coupling graph (E constant): geometric fallback, still strictly increasing to beta_max
        CouplingGraph::Builder bz(4);
        auto z = adaptive_ladder(bz.build(), 0.1, 2.0, 0.5, 20, 3);
        CHECK(z.betas.size() >= 3 && z.betas.front() == 0.1 && z.betas.back() == 2.0);
        for (std::size_t r = 1; r < z.betas.size(); ++r) CHECK(z.betas[r] > z.betas[r - 1]);
        CHECK(throws<ConfigError>([&] { adaptive_ladder(bz.build(), 0.1, 2.0, 1.0, 20, 3); }));
        CHECK(throws<ConfigError>([&] { adaptive_ladder(bz.build(), 0.1, 2.0, 0.0, 20, 3); }));
    }
    {  // target 0.99 on a 3x3 ferromagnet -> dense ladder, every neighbour pair accepts >= 0.8
        auto g3 = LatticeSpec::grid2d(3, 3).graph();
        auto lad = adaptive_ladder(g3, 0.1, 1.0, 0.99, 4000, 5);
        CHECK(lad.betas.size() > 10 && lad.betas.size() <= 256);
        auto acc = pair_acceptance(g3, lad, 6000);
        for (double a : acc) CHECK(a >= 0.8);
    }
    {  // target 0.3 on a 3D EA instance, L = 4 -> >= 80 % of pairs accept within [0.1, 0.6]
        auto spec = LatticeSpec::grid3d(4, 1.0, LatticeSpec::Boundary::periodic);
        auto base = spec.graph();
        CouplingGraph::Builder be(base.n_spins());
        RngStream dr(77);
        for (const auto& c : base.couplings()) be.add_coupling(c.i, c.j, dr.coin() ? 1.0 : -1.0);
        auto ea = be.build();
        auto lad = adaptive_ladder(ea, 0.2, 3.0, 0.3, 4000, 6);
        auto acc = pair_acceptance(ea, lad, 6000);
        std::size_t ok = 0;
        for (double a : acc) ok += (a >= 0.1 && a <= 0.6);
        std::printf("adaptive ladder EA L=4: %zu betas, %zu/%zu pairs in [0.1,0.6]\n", lad.betas.size(), ok, acc.size());
        CHECK(ok * 5 >= acc.size() * 4);
        // residual energy in the best-so-far sense is non-increasing
        TAPTConfig c;
        c.n_swap = 300;
        c.M = 2;
        c.seed = 4;
        std::vector<RunTrace> runs{run_pt(ea, lad, c)};
        c.seed = 5;
        runs.push_back(run_pt(ea, lad, c));
        auto rho = residual_energy(runs, -200.0, ea.n_spins(), true);
        for (std::size_t t = 1; t < rho.size(); ++t) CHECK(rho[t] <= rho[t - 1]);
    }
    // multi-GPU plumbing from C++: shards cover every instance once; a one-rank NCCL communicator's
    // reductions equal the local sums (the only collectives of a sharded run)
    {
        for (int world : {1, 2, 3, 8}) {
            std::uint64_t next = 0;
            for (int r = 0; r < world; ++r) {
                auto sh = Shard::of(4096, world, r);
                CHECK(sh.offset == next);
                next += sh.count;
            }
            CHECK(next == 4096);
        }
        Communicator comm(Communicator::unique_id(), 1, 0);
        CHECK(comm.size() == 1);
        Replicas reps(g, BetaLadder::geometric(0.2, 1.0, 6), 5);
        throw_status(tapt_set_histogram(reps.handle(), -600, 8, 160));
        tapt_schedule sc{40, 1, 4, 0};
        throw_status(tapt_run(reps.handle(), &sc));
        auto red = comm.allreduce_observables(reps.handle(), 6, 160);
        std::vector<std::int64_t> local(6 * 5);
        throw_status(tapt_get_observables(reps.handle(), local.data()));
        CHECK(red.obs == local && red.obs[0] == 10);
        std::uint64_t tot = 0;
        for (auto v : red.hist) tot += v;
        CHECK(tot == 6 * 10);
    }
    std::printf("gpu ok\n");
    return 0;
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "cpu";
    try {
        if (mode == "cpu") return cpu_tests();
        if (mode == "gpu") return gpu_tests();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "exception: %s\n", e.what());
        return 2;
    }
    return 3;
}
