// tapt/mcmc.hpp -- drop-in for the reference's local-MCMC API (proj/include/tapt/mcmc.hpp:15-56,
// proj/src/mcmc.cpp) with every sweep executed on the B200 (index-ascending schedule, bit-exact
// with the reference's gibbs_sweep for integer couplings: same heat-bath conditional, same
// per-site draw of the caller's RngStream, same returned energy change).
#pragma once

#include <cstring>
#include <memory>
#include <iosfwd>
#include <istream>
#include <ostream>

#include "tapt/spin_model.hpp"

namespace tapt {

struct ChainConfig {
    double beta = 1.0;
    std::uint64_t mixing_sweeps = 0;
    std::uint64_t thinning = 1;
    std::uint64_t seed = 0;
};

struct SampleRecord {
    double beta;
    SpinConfiguration spins;
};

struct SampleDataset {
    std::vector<SampleRecord> records;
    std::uint64_t graph_digest = 0;

    // binary `ISFD1`: magic, then per record f64 beta, u32 count, spins bit-packed LSB-first
    // (+1 -> 1), little-endian (mcmc.cpp:86-162 format).
    void save(std::ostream& os) const {
        os.write("ISFD1", 5);
        for (const auto& r : records) {
            os.write(reinterpret_cast<const char*>(&r.beta), 8);
            const std::uint32_t n = static_cast<std::uint32_t>(r.spins.size());
            os.write(reinterpret_cast<const char*>(&n), 4);
            std::vector<unsigned char> p((n + 7) / 8, 0);
            for (std::uint32_t i = 0; i < n; ++i)
                if (r.spins[i] > 0) p[i / 8] |= static_cast<unsigned char>(1u << (i % 8));
            os.write(reinterpret_cast<const char*>(p.data()), static_cast<std::streamsize>(p.size()));
        }
    }
    void save_file(const std::string& path) const {
        std::ofstream os(path, std::ios::binary);
        if (!os) throw FormatError("cannot open " + path + " for writing");
        save(os);
    }
    static SampleDataset load(std::istream& is) {
        char magic[5];
        is.read(magic, 5);
        if (is.gcount() != 5 || std::memcmp(magic, "ISFD1", 5) != 0) throw FormatError("bad dataset magic (expected ISFD1)");
        SampleDataset out;
        for (;;) {
            double beta;
            is.read(reinterpret_cast<char*>(&beta), 8);
            if (is.gcount() != 8) break;  // clean EOF; a partial beta ends the file too (mcmc.cpp:142)
            std::uint32_t n;
            is.read(reinterpret_cast<char*>(&n), 4);
            if (is.gcount() != 4) throw FormatError("truncated dataset record");
            std::vector<unsigned char> p((n + 7) / 8);
            is.read(reinterpret_cast<char*>(p.data()), static_cast<std::streamsize>(p.size()));
            if (is.gcount() != static_cast<std::streamsize>(p.size())) throw FormatError("truncated dataset record");
            SpinConfiguration s(n);
            for (std::uint32_t i = 0; i < n; ++i) s[i] = (p[i / 8] >> (i % 8)) & 1u ? 1 : -1;
            out.records.push_back({beta, std::move(s)});
        }
        return out;
    }
    static SampleDataset load_file(const std::string& path) {
        std::ifstream is(path, std::ios::binary);
        if (!is) throw FormatError("cannot open " + path);
        return load(is);
    }
};

// One device sweep (or n): updates s in place, advances rng by n_free draws per sweep,
// returns the total energy change.
inline double gibbs_sweeps(const CouplingGraph& g, SpinConfiguration& s, double beta, RngStream& rng,
                           std::uint32_t n_sweeps, std::vector<double>* per_sweep = nullptr) {
    if (s.size() != g.n_spins()) throw DimensionError("configuration length mismatch");
    if (n_sweeps == 0 || g.n_free() == 0) return 0.0;
    std::uint64_t st = rng.state();
    if (!per_sweep && n_sweeps > 1) {  // one device launch for all sweeps; total from the energies
        const double e0 = energy(g, s);
        throw_status(tapt_gibbs_sweep(g.device(), s.data(), s.size(), beta, &st, n_sweeps, nullptr));
        rng = RngStream::from_state(st);
        return energy(g, s) - e0;
    }
    std::vector<double> d(n_sweeps);
    throw_status(tapt_gibbs_sweep(g.device(), s.data(), s.size(), beta, &st, n_sweeps, d.data()));
    rng = RngStream::from_state(st);
    double tot = 0.0;
    for (double v : d) tot += v;
    if (per_sweep) *per_sweep = std::move(d);
    return tot;
}

inline double gibbs_sweep(const CouplingGraph& g, SpinConfiguration& s, double beta, RngStream& rng) {
    return gibbs_sweeps(g, s, beta, rng, 1);
}

// Single-site heat-bath update (mcmc.cpp:24-28) on the device (tapt_gibbs_update: K5 with a one-site
// visit list): one draw of rng; ClampedSiteError for a clamped i, DimensionError on a length mismatch.
inline void gibbs_update(const CouplingGraph& g, SpinConfiguration& s, std::uint32_t i, double beta, RngStream& rng) {
    std::uint64_t st = rng.state();
    throw_status(tapt_gibbs_update(g.device(), s.data(), s.size(), i, beta, &st));
    rng = RngStream::from_state(st);
}

inline void check_chain_config(const ChainConfig& c) {
    if (c.beta < 0.0) throw ConfigError("beta must be >= 0");
    if (c.thinning < 1) throw ConfigError("thinning must be >= 1");
}

// run_chain (mcmc.cpp:47-65): init from derive(seed,{kInit,kChain}), dynamics
// derive(seed,{kChain}); mixing sweeps, then a record every `thinning` sweeps.
inline SampleDataset run_chain(const CouplingGraph& g, const ChainConfig& config, std::uint64_t n_records) {
    check_chain_config(config);
    SampleDataset out;
    out.graph_digest = g.digest();
    if (n_records == 0) return out;
    RngStream init = RngStream::derive(config.seed, {stream::kInit, stream::kChain});
    RngStream dyn = RngStream::derive(config.seed, {stream::kChain});
    SpinConfiguration s = random_configuration(g, init);
    if (config.mixing_sweeps) gibbs_sweeps(g, s, config.beta, dyn, static_cast<std::uint32_t>(config.mixing_sweeps));
    for (std::uint64_t r = 0; r < n_records; ++r) {
        gibbs_sweeps(g, s, config.beta, dyn, static_cast<std::uint32_t>(config.thinning));
        out.records.push_back({config.beta, s});
    }
    return out;
}

// generate_training_corpus (mcmc.cpp:67-84): per beta a chain seeded by
// derive(seed,{kChain, index}).state(); records concatenated in beta order.  All chains run
// together as the slots of one device ensemble (index-ascending sweeps, per-slot streams
// overridden to run_chain's), so the corpus is bit-identical to the reference's.
inline SampleDataset generate_training_corpus(const CouplingGraph& g, const std::vector<double>& betas,
                                              std::uint64_t per_beta, const ChainConfig& config,
                                              unsigned /*n_threads: the device replaces the thread pool*/ = 1) {
    check_chain_config(config);
    for (double b : betas)
        if (b < 0.0) throw ConfigError("beta must be >= 0");
    SampleDataset out;
    out.graph_digest = g.digest();
    const std::size_t n = g.n_spins();
    std::vector<std::vector<SpinConfiguration>> rec(betas.size());
    for (std::size_t c0 = 0; c0 < betas.size(); c0 += 256) {
        const std::size_t R = std::min<std::size_t>(256, betas.size() - c0);
        std::vector<double> dummy(R), bs(betas.begin() + c0, betas.begin() + c0 + R);
        for (std::size_t r = 0; r < R; ++r) dummy[r] = 0.5 + double(r);
        tapt_ensemble_desc d{1, 0, static_cast<std::uint32_t>(R), dummy.data(), 0, TAPT_ORDER_REFERENCE};
        tapt_ensemble_t e = nullptr;
        throw_status(tapt_ensemble_create(g.device(), &d, &e));
        std::unique_ptr<tapt_ensemble_s, tapt_status (*)(tapt_ensemble_t)> hold(e, tapt_ensemble_destroy);
        throw_status(tapt_ensemble_set_betas(e, bs.data(), 2));
        std::vector<std::uint64_t> init(R), dyn(R);
        for (std::size_t r = 0; r < R; ++r) {
            const std::uint64_t cs = RngStream::derive(config.seed, {stream::kChain, c0 + r}).state();
            init[r] = RngStream::derive(cs, {stream::kInit, stream::kChain}).state();
            dyn[r] = RngStream::derive(cs, {stream::kChain}).state();
        }
        throw_status(tapt_ensemble_init_from_streams(e, init.data()));
        throw_status(tapt_ensemble_set_streams(e, dyn.data()));
        tapt_schedule sch{0, 0, 0, 0};
        if (config.mixing_sweeps) {
            sch.n_sweeps = static_cast<std::uint32_t>(config.mixing_sweeps);
            throw_status(tapt_run(e, &sch));
        }
        std::vector<std::int8_t> flat(R * n);
        for (std::uint64_t k = 0; k < per_beta; ++k) {
            sch.n_sweeps = static_cast<std::uint32_t>(config.thinning);
            throw_status(tapt_run(e, &sch));
            throw_status(tapt_ensemble_get_spins(e, flat.data()));
            for (std::size_t r = 0; r < R; ++r)
                rec[c0 + r].emplace_back(flat.begin() + r * n, flat.begin() + (r + 1) * n);
        }
    }
    for (std::size_t bi = 0; bi < betas.size(); ++bi)
        for (auto& s : rec[bi]) out.records.push_back({betas[bi], std::move(s)});
    return out;
}

}  // namespace tapt
