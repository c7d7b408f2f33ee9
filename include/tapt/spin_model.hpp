// tapt/spin_model.hpp -- drop-in for the reference's CouplingGraph API
// (proj/include/tapt/spin_model.hpp:30-113, proj/src/spin_model.cpp) on the B200 engine.
//
// The graph is an immutable host value (couplings merged and sorted, ascending CSR, free-site
// list, FNV-1a digest -- identical to the reference's Builder semantics) that lazily owns a
// device model (tapt_model_t) the first time a sweep kernel needs it.  energy / local_field /
// flip_delta / magnetization are host arithmetic on one configuration, as in the reference;
// every sweep, swap and proposal decision runs on the device (tapt/mcmc.hpp, tapt/tempering.hpp).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <map>
#include <memory>
#include <span>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "tapt/errors.hpp"
#include "tapt/rng.hpp"
#include "tapt_gpu.h"

namespace tapt {

using SpinConfiguration = std::vector<std::int8_t>;

struct Coupling {
    std::uint32_t i;  // i < j
    std::uint32_t j;
    double value;
};

// tapt_status -> the reference's exception types (errors.hpp).
inline void throw_status(tapt_status st, const char* msg = nullptr) {
    if (st == TAPT_OK) return;
    const std::string m = msg ? msg : tapt_last_error();
    switch (st) {
        case TAPT_ERR_CONFIG: throw ConfigError(m);
        case TAPT_ERR_DIMENSION: throw DimensionError(m);
        case TAPT_ERR_CLAMPED_SITE: throw ClampedSiteError(m);
        case TAPT_ERR_SIZE: throw SizeError(m);
        case TAPT_ERR_GEOMETRY: throw GeometryError(m);
        case TAPT_ERR_NUMERIC: throw NumericError(m);
        case TAPT_ERR_FORMAT: throw FormatError(m);
        case TAPT_ERR_TRAINING_DIVERGED: throw TrainingDivergedError(m);
        case TAPT_ERR_NCCL: throw NcclError(m);
        case TAPT_ERR_CUDA: throw CudaError(m);
        default: throw std::runtime_error(m);
    }
}

class CouplingGraph {
  public:
    class Builder {
      public:
        explicit Builder(std::size_t n_spins) : n_(n_spins), h_(n_spins, 0.0), x_(n_spins, 0) {}
        Builder& add_coupling(std::uint32_t i, std::uint32_t j, double value) {
            if (i == j) throw ConfigError("self-coupling on spin " + std::to_string(i));
            if (i >= n_ || j >= n_) throw ConfigError("coupling index out of range");
            pending_.push_back({std::min(i, j), std::max(i, j), value});
            return *this;
        }
        Builder& add_field(std::uint32_t i, double value) {
            if (i >= n_) throw ConfigError("field index out of range");
            h_[i] += value;
            return *this;
        }
        Builder& set_clamp(std::uint32_t i, int value) {
            if (i >= n_) throw ConfigError("clamp index out of range");
            if (value != 1 && value != -1) throw ConfigError("clamp value must be ±1");
            x_[i] = static_cast<std::int8_t>(value);
            return *this;
        }
        CouplingGraph build() const {
            CouplingGraph g;
            g.n_ = n_;
            g.fields_ = h_;
            g.clamps_ = x_;
            std::map<std::pair<std::uint32_t, std::uint32_t>, double> acc;
            for (const auto& c : pending_) acc[{c.i, c.j}] += c.value;
            for (const auto& [k, v] : acc) g.couplings_.push_back({k.first, k.second, v});
            g.finish();
            return g;
        }

      private:
        std::size_t n_;
        std::vector<Coupling> pending_;
        std::vector<double> h_;
        std::vector<std::int8_t> x_;
    };

    struct Neighbor {
        std::uint32_t index;
        double value;
    };

    std::size_t n_spins() const { return n_; }
    std::size_t n_free() const { return free_.size(); }
    const std::vector<Coupling>& couplings() const { return couplings_; }
    const std::vector<double>& fields() const { return fields_; }
    double field(std::uint32_t i) const { return fields_[i]; }
    bool is_clamped(std::uint32_t i) const { return clamps_[i] != 0; }
    std::int8_t clamp_value(std::uint32_t i) const { return clamps_[i]; }
    const std::vector<std::uint32_t>& free_sites() const { return free_; }
    bool has_clamps() const { return free_.size() != n_; }
    std::span<const Neighbor> neighbors(std::uint32_t i) const {
        return {adj_.data() + off_[i], off_[i + 1] - off_[i]};
    }
    std::uint64_t digest() const { return digest_; }

    // `isingmodel v1` text format (spin_model.cpp:123-226 semantics).
    void save(std::ostream& os) const {
        char buf[64];
        os << "isingmodel v1\n" << "n " << n_ << "\n";
        for (const auto& c : couplings_) {
            std::snprintf(buf, sizeof buf, "%.17g", c.value);
            os << "c " << c.i << " " << c.j << " " << buf << "\n";
        }
        for (std::size_t i = 0; i < n_; ++i)
            if (fields_[i] != 0.0) {
                std::snprintf(buf, sizeof buf, "%.17g", fields_[i]);
                os << "f " << i << " " << buf << "\n";
            }
        for (std::size_t i = 0; i < n_; ++i)
            if (clamps_[i]) os << "x " << i << " " << (clamps_[i] > 0 ? "+1" : "-1") << "\n";
    }
    void save_file(const std::string& path) const {
        std::ofstream os(path, std::ios::binary);
        if (!os) throw FormatError("cannot open " + path + " for writing");
        save(os);
    }
    static CouplingGraph load(std::istream& is) {
        std::string line;
        if (!std::getline(is, line)) throw FormatError("empty instance file");
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line != "isingmodel v1") throw FormatError("bad header: expected 'isingmodel v1'");
        std::size_t n = 0, lineno = 1;
        bool have_n = false;
        std::vector<std::tuple<std::uint32_t, std::uint32_t, double>> cs;
        std::vector<std::pair<std::uint32_t, double>> fs;
        std::vector<std::pair<std::uint32_t, int>> xs;
        while (std::getline(is, line)) {
            ++lineno;
            if (!line.empty() && line.back() == '\r') line.pop_back();
            std::istringstream ls(line);
            std::string tag;
            if (!(ls >> tag) || tag[0] == '#') continue;
            const std::string where = "line " + std::to_string(lineno) + ": ";
            if (tag == "n") {
                if (have_n) throw FormatError(where + "duplicate n line");
                if (!(ls >> n)) throw FormatError(where + "bad n line");
                have_n = true;
            } else if (tag == "c") {
                std::uint32_t i, j;
                double v;
                if (!(ls >> i >> j >> v)) throw FormatError(where + "bad coupling line");
                cs.emplace_back(i, j, v);
            } else if (tag == "f") {
                std::uint32_t i;
                double v;
                if (!(ls >> i >> v)) throw FormatError(where + "bad field line");
                fs.emplace_back(i, v);
            } else if (tag == "x") {
                std::uint32_t i;
                std::string v;
                if (!(ls >> i >> v)) throw FormatError(where + "bad clamp line");
                if (v != "+1" && v != "1" && v != "-1") throw FormatError(where + "clamp value must be +1 or -1");
                xs.emplace_back(i, v == "-1" ? -1 : 1);
            } else {
                throw FormatError(where + "unknown record tag '" + tag + "'");
            }
        }
        if (!have_n) throw FormatError("missing n line");
        Builder b(n);
        std::map<std::pair<std::uint32_t, std::uint32_t>, bool> seen;
        for (auto [i, j, v] : cs) {
            const auto key = std::minmax(i, j);
            if (seen.count({key.first, key.second}))
                throw FormatError("duplicate coupling (" + std::to_string(i) + "," + std::to_string(j) + ")");
            seen[{key.first, key.second}] = true;
            b.add_coupling(i, j, v);
        }
        for (auto [i, v] : fs) b.add_field(i, v);
        for (auto [i, v] : xs) b.set_clamp(i, v);
        return b.build();
    }
    static CouplingGraph load_file(const std::string& path) {
        std::ifstream is(path, std::ios::binary);
        if (!is) throw FormatError("cannot open " + path);
        return load(is);
    }

    // Device model (created on first use; shared by copies of this graph).
    tapt_model_t device() const {
        if (!dev_) {
            tapt_model_t m = nullptr;
            if (lattice_) {
                throw_status(tapt_model_create_lattice(lattice_->dim, lattice_->ly, lattice_->lx, lattice_->l,
                                                       lattice_->J, lattice_->periodic ? 1 : 0, &m));
                if (has_clamps()) {  // clamped lattices go through the general CSR model
                    tapt_model_destroy(m);
                    m = nullptr;
                }
            }
            if (!m) {
                std::vector<std::uint32_t> ci, cj;
                std::vector<double> J;
                for (const auto& c : couplings_) {
                    ci.push_back(c.i);
                    cj.push_back(c.j);
                    J.push_back(c.value);
                }
                throw_status(tapt_model_create_graph(static_cast<std::uint32_t>(n_), static_cast<std::uint32_t>(ci.size()),
                                                     ci.data(), cj.data(), J.data(), fields_.data(), clamps_.data(), &m));
            }
            dev_ = std::shared_ptr<tapt_model_s>(m, [](tapt_model_t p) { tapt_model_destroy(p); });
        }
        return dev_.get();
    }

    // Lattice provenance (set by LatticeSpec) so the device picks the stencil kernel.
    struct LatticeTag {
        int dim, ly, lx, l;
        double J;
        bool periodic;
    };
    void tag_lattice(const LatticeTag& t) { lattice_ = std::make_shared<LatticeTag>(t); }

  private:
    CouplingGraph() = default;
    void finish() {
        off_.assign(n_ + 1, 0);
        std::vector<std::vector<Neighbor>> adj(n_);
        for (const auto& c : couplings_) {
            adj[c.i].push_back({c.j, c.value});
            adj[c.j].push_back({c.i, c.value});
        }
        for (std::size_t i = 0; i < n_; ++i) {
            std::sort(adj[i].begin(), adj[i].end(), [](const Neighbor& a, const Neighbor& b) { return a.index < b.index; });
            off_[i + 1] = off_[i] + adj[i].size();
            adj_.insert(adj_.end(), adj[i].begin(), adj[i].end());
        }
        for (std::uint32_t i = 0; i < n_; ++i)
            if (!clamps_[i]) free_.push_back(i);
        auto fnv = [](const void* p, std::size_t k, std::uint64_t h) {
            const unsigned char* c = static_cast<const unsigned char*>(p);
            for (std::size_t q = 0; q < k; ++q) h = (h ^ c[q]) * 0x100000001B3ull;
            return h;
        };
        const std::uint64_t n64 = n_;
        std::uint64_t d = fnv(&n64, sizeof n64, 0xCBF29CE484222325ull);
        if (!couplings_.empty()) d = fnv(couplings_.data(), couplings_.size() * sizeof(Coupling), d);
        if (!fields_.empty()) d = fnv(fields_.data(), fields_.size() * sizeof(double), d);
        if (!clamps_.empty()) d = fnv(clamps_.data(), clamps_.size(), d);
        digest_ = d;
    }

    std::size_t n_ = 0;
    std::vector<Coupling> couplings_;
    std::vector<double> fields_;
    std::vector<std::int8_t> clamps_;
    std::vector<std::uint32_t> free_;
    std::vector<Neighbor> adj_;
    std::vector<std::size_t> off_;
    std::uint64_t digest_ = 0;
    std::shared_ptr<LatticeTag> lattice_;
    mutable std::shared_ptr<tapt_model_s> dev_;
};

// --- energy arithmetic on one host configuration (spin_model.cpp:79-121) -----------

inline double energy(const CouplingGraph& g, std::span<const std::int8_t> s) {
    if (s.size() != g.n_spins())
        throw DimensionError("configuration length " + std::to_string(s.size()) + " != n_spins " +
                             std::to_string(g.n_spins()));
    double e = 0.0;
    for (const auto& c : g.couplings()) e -= c.value * static_cast<double>(s[c.i] * s[c.j]);
    for (std::size_t i = 0; i < g.n_spins(); ++i) e -= g.field(static_cast<std::uint32_t>(i)) * s[i];
    return e;
}

inline double local_field(const CouplingGraph& g, std::span<const std::int8_t> s, std::uint32_t i) {
    if (s.size() != g.n_spins()) throw DimensionError("configuration length mismatch");
    if (g.is_clamped(i)) throw ClampedSiteError("spin " + std::to_string(i) + " is clamped");
    double l = g.field(i);
    for (const auto& nb : g.neighbors(i)) l += nb.value * static_cast<double>(s[nb.index]);
    return l;
}

inline double flip_delta(const CouplingGraph& g, std::span<const std::int8_t> s, std::uint32_t i) {
    return 2.0 * static_cast<double>(s[i]) * local_field(g, s, i);
}

inline void apply_clamps(const CouplingGraph& g, SpinConfiguration& s) {
    if (s.size() != g.n_spins()) throw DimensionError("configuration length mismatch");
    for (std::uint32_t i = 0; i < g.n_spins(); ++i)
        if (g.is_clamped(i)) s[i] = g.clamp_value(i);
}

inline double magnetization(std::span<const std::int8_t> s) {
    if (s.empty()) return 0.0;
    long m = 0;
    for (auto v : s) m += v;
    return static_cast<double>(m) / static_cast<double>(s.size());
}

// One coin per site (clamped sites too), then clamps -- identical draw sequence.
inline SpinConfiguration random_configuration(const CouplingGraph& g, RngStream& rng) {
    SpinConfiguration s(g.n_spins());
    for (auto& v : s) v = rng.coin() ? 1 : -1;
    apply_clamps(g, s);
    return s;
}

}  // namespace tapt
