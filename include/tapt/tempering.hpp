// tapt/tempering.hpp -- the tempering module of SPEC.md:381-484 (the reference's
// proj/src/tempering.cpp:1 is a placeholder) on the B200 engine: BetaLadder, TAPTConfig,
// RunTrace, swap_pass (Eq. 1), generator_move / mh_corrected_move (Eq. 2), run_pt,
// run_tapt (Algorithm 1), adaptive_ladder, residual_energy.
//
// Replicas is the device-resident verifier state of one instance.  Sweeps, swaps and
// proposal acceptance all run on the GPU; the host only drives Algorithm 1's move cycle
// and talks to the proposal source.  Stream conventions: slot r of
// instance 0 sweeps with derive(seed,{kReplica,0,r}); swap pass p draws p*R+r+1 of
// derive(seed,{kCoordinator,0}); generator round q draws slot+1 of
// derive(seed,{kCoordinator,0,q+1}); the proposal source for slot r in round q receives
// derive(seed,{kReplica,0,r,q+1}).
#pragma once

#include <functional>
#include <limits>
#include <memory>
#include <ostream>

#include "tapt/mcmc.hpp"

namespace tapt {

struct BetaLadder {
    std::vector<double> betas;  // strictly increasing, index 0 hottest

    void validate() const {
        if (betas.empty()) throw ConfigError("empty beta ladder");
        for (std::size_t r = 0; r < betas.size(); ++r) {
            if (!(betas[r] >= 0.0)) throw ConfigError("beta must be >= 0");
            if (r && !(betas[r] > betas[r - 1])) throw ConfigError("beta ladder must be strictly increasing");
        }
    }
    static BetaLadder geometric(double b0, double b1, std::size_t R) {
        BetaLadder l;
        for (std::size_t r = 0; r < R; ++r)
            l.betas.push_back(R == 1 ? b0 : b0 * std::pow(b1 / b0, double(r) / double(R - 1)));
        return l;
    }
    static BetaLadder linear(double b0, double b1, std::size_t R) {
        BetaLadder l;
        for (std::size_t r = 0; r < R; ++r) l.betas.push_back(R == 1 ? b0 : b0 + (b1 - b0) * double(r) / double(R - 1));
        return l;
    }
};

struct TAPTConfig {
    std::uint64_t n_swap = 0;       // global moves
    std::uint64_t M = 1;            // local sweeps after each global move
    std::size_t N_T = 0;            // hottest replicas receiving generator proposals
    double context_fraction = 0.0;  // Appendix C prefix length / n_free
    bool mh_corrected = false;
    std::uint64_t seed = 0;

    void validate(std::size_t R) const {
        if (N_T > R) throw ConfigError("N_T must be <= number of replicas");
        if (!(context_fraction >= 0.0 && context_fraction <= 1.0)) throw ConfigError("context_fraction in [0,1]");
    }
};

enum class MoveKind : int { generator = 1, swap_even = 2, swap_odd = 3 };

struct RunTrace {
    std::vector<int> move_kind;                  // per global move (Alg. 1 move variable)
    std::vector<std::vector<double>> energies;   // per move, per replica (after the M sweeps)
    std::vector<std::vector<std::uint8_t>> accepted;  // per move, per replica / pair (1 = accepted)
    std::vector<std::uint64_t> swap_attempts, swap_accepts;  // per pair (r, r+1)
    std::vector<std::uint64_t> gen_attempts, gen_accepts;    // per replica
    std::vector<double> best_energy;             // best so far after each move (non-increasing)
    double best = std::numeric_limits<double>::infinity();
    SpinConfiguration best_state;
    SpinConfiguration final_state;               // coldest replica at the end (Alg. 1 output)
    double final_energy = 0.0;

    // CSV columns of SPEC.md:476: move_index, move_kind, replica, beta, energy, accepted
    void write_csv(std::ostream& os, const BetaLadder& ladder) const {
        os << "move_index,move_kind,replica,beta,energy,accepted\n";
        for (std::size_t m = 0; m < energies.size(); ++m)
            for (std::size_t r = 0; r < energies[m].size(); ++r)
                os << m << "," << move_kind[m] << "," << r << "," << ladder.betas[r] << "," << energies[m][r] << ","
                   << int(r < accepted[m].size() ? accepted[m][r] : 0) << "\n";
    }
};

// Proposal source (stands in for IsingFormer.sample / log_prob).
class ProposalSource {
  public:
    virtual ~ProposalSource() = default;
    // A full configuration for replica `replica` at inverse temperature `beta`; `context` holds the
    // current state and `context_len` the number of leading free spins given as prefix.
    virtual SpinConfiguration sample(std::size_t replica, double beta, std::span<const std::int8_t> context,
                                     std::size_t context_len, RngStream& rng) = 0;
    virtual double log_prob(std::span<const std::int8_t> /*s*/, double /*beta*/) { return 0.0; }
};

class Replicas {
  public:
    Replicas(const CouplingGraph& g, const BetaLadder& ladder, std::uint64_t seed,
             int order = TAPT_ORDER_REFERENCE)
        : g_(&g), ladder_(ladder), seed_(seed) {
        ladder_.validate();
        tapt_ensemble_desc d{};
        d.n_instances = 1;
        d.instance_offset = 0;
        d.n_slots = static_cast<std::uint32_t>(ladder_.betas.size());
        d.betas = ladder_.betas.data();
        d.seed = seed;
        d.order = order;
        tapt_ensemble_t e = nullptr;
        throw_status(tapt_ensemble_create(g.device(), &d, &e));
        e_ = std::shared_ptr<tapt_ensemble_s>(e, [](tapt_ensemble_t p) { tapt_ensemble_destroy(p); });
        throw_status(tapt_ensemble_init_random(e));
    }
    std::size_t size() const { return ladder_.betas.size(); }
    const BetaLadder& ladder() const { return ladder_; }
    tapt_ensemble_t handle() const { return e_.get(); }

    void sweep(std::uint64_t M) { throw_status(tapt_sweep(e_.get(), static_cast<std::uint32_t>(M))); }

    // swap_pass: pairs (r, r+1), r = parity (mod 2); returns per-pair accept flags.
    std::vector<std::uint8_t> swap_pass(int parity) {
        const std::size_t P = size() > 1 ? size() - 1 : 0;
        std::vector<std::uint64_t> a0(P), a1(P);
        if (P) throw_status(tapt_get_acceptance(e_.get(), nullptr, a0.data(), nullptr, nullptr));
        throw_status(tapt_swap_pass(e_.get(), parity));
        if (P) throw_status(tapt_get_acceptance(e_.get(), nullptr, a1.data(), nullptr, nullptr));
        std::vector<std::uint8_t> acc(P);
        for (std::size_t r = 0; r < P; ++r) acc[r] = static_cast<std::uint8_t>(a1[r] - a0[r]);
        return acc;
    }

    // generator_move / mh_corrected_move for the listed slots (Eq. 2).
    std::vector<std::uint8_t> inject(const std::vector<SpinConfiguration>& proposals,
                                     const std::vector<std::uint32_t>& slots, const std::vector<double>* lq_cur = nullptr,
                                     const std::vector<double>* lq_prop = nullptr) {
        const std::size_t n = g_->n_spins();
        std::vector<std::int8_t> flat(slots.size() * n);
        for (std::size_t t = 0; t < slots.size(); ++t) {
            if (proposals[t].size() != n) throw DimensionError("proposal length mismatch");
            std::copy(proposals[t].begin(), proposals[t].end(), flat.begin() + t * n);
        }
        std::vector<std::uint8_t> acc(slots.size());
        throw_status(tapt_inject_proposals(e_.get(), flat.data(), 0, slots.data(), static_cast<std::uint32_t>(slots.size()),
                                           lq_cur ? lq_cur->data() : nullptr, lq_prop ? lq_prop->data() : nullptr,
                                           acc.data()));
        return acc;
    }

    std::vector<double> energies() const {  // doubles: exact for integer and real-valued couplings
        std::vector<double> e(size());
        throw_status(tapt_ensemble_get_energies_f64(e_.get(), e.data()));
        return e;
    }
    std::vector<SpinConfiguration> states() const {
        const std::size_t n = g_->n_spins();
        std::vector<std::int8_t> flat(size() * n);
        throw_status(tapt_ensemble_get_spins(e_.get(), flat.data()));
        std::vector<SpinConfiguration> out(size());
        for (std::size_t r = 0; r < size(); ++r) out[r].assign(flat.begin() + r * n, flat.begin() + (r + 1) * n);
        return out;
    }
    std::uint64_t rounds() const {
        std::uint64_t q = 0;
        throw_status(tapt_ensemble_counters(e_.get(), nullptr, nullptr, &q));
        return q;
    }
    std::uint64_t seed() const { return seed_; }

  private:
    const CouplingGraph* g_;
    BetaLadder ladder_;
    std::uint64_t seed_;
    std::shared_ptr<tapt_ensemble_s> e_;
};

// Algorithm 1: move 1 -> generator proposals into replicas 0..N_T-1,
// move 2 -> even swaps, move 3 -> odd swaps; M sweeps of every replica after each move.
inline RunTrace run_tapt(const CouplingGraph& g, const BetaLadder& ladder, const TAPTConfig& cfg, ProposalSource* gen,
                         int order = TAPT_ORDER_REFERENCE) {
    cfg.validate(ladder.betas.size());
    if (cfg.N_T > 0 && !gen) throw ConfigError("N_T > 0 needs a proposal source");
    Replicas reps(g, ladder, cfg.seed, order);
    const std::size_t R = reps.size();
    RunTrace tr;
    tr.swap_attempts.assign(R > 1 ? R - 1 : 0, 0);
    tr.swap_accepts.assign(R > 1 ? R - 1 : 0, 0);
    tr.gen_attempts.assign(R, 0);
    tr.gen_accepts.assign(R, 0);
    int move = 1;
    for (std::uint64_t step = 0; step < cfg.n_swap; ++step) {
        std::vector<std::uint8_t> acc;
        if (move == 1) {
            if (cfg.N_T > 0) {
                const auto cur = reps.states();
                const std::size_t ctx = static_cast<std::size_t>(std::floor(cfg.context_fraction * double(g.n_free())));
                std::vector<SpinConfiguration> props;
                std::vector<std::uint32_t> slots;
                std::vector<double> lqc, lqp;
                const std::uint64_t q = reps.rounds();
                for (std::size_t r = 0; r < cfg.N_T; ++r) {
                    RngStream rng = RngStream::derive(cfg.seed, {stream::kReplica, 0, r, q + 1});
                    SpinConfiguration p = gen->sample(r, ladder.betas[r], cur[r], ctx, rng);
                    apply_clamps(g, p);
                    if (cfg.mh_corrected) {
                        lqc.push_back(gen->log_prob(cur[r], ladder.betas[r]));
                        lqp.push_back(gen->log_prob(p, ladder.betas[r]));
                    }
                    props.push_back(std::move(p));
                    slots.push_back(static_cast<std::uint32_t>(r));
                }
                const auto a = reps.inject(props, slots, cfg.mh_corrected ? &lqc : nullptr, cfg.mh_corrected ? &lqp : nullptr);
                acc.assign(R, 0);
                for (std::size_t t = 0; t < slots.size(); ++t) {
                    acc[slots[t]] = a[t];
                    tr.gen_attempts[slots[t]] += 1;
                    tr.gen_accepts[slots[t]] += a[t];
                }
            }
        } else {
            acc = reps.swap_pass(move == 2 ? 0 : 1);
            for (std::size_t r = (move == 2 ? 0 : 1); r + 1 < R; r += 2) {
                tr.swap_attempts[r] += 1;
                tr.swap_accepts[r] += acc[r];
            }
        }
        reps.sweep(cfg.M);
        auto E = reps.energies();
        tr.move_kind.push_back(move);
        for (std::size_t r = 0; r < R; ++r)
            if (E[r] < tr.best) {
                tr.best = E[r];
                tr.best_state = reps.states()[r];
            }
        tr.best_energy.push_back(tr.best);
        tr.energies.push_back(std::move(E));
        tr.accepted.push_back(std::move(acc));
        move = move % 3 + 1;
    }
    auto S = reps.states();
    auto E = reps.energies();
    tr.final_state = S.back();
    tr.final_energy = E.back();
    if (tr.best_state.empty()) {
        for (std::size_t r = 0; r < R; ++r)
            if (E[r] < tr.best) {
                tr.best = E[r];
                tr.best_state = S[r];
            }
    }
    return tr;
}

// run_pt = Algorithm 1 with N_T = 0.
inline RunTrace run_pt(const CouplingGraph& g, const BetaLadder& ladder, const TAPTConfig& cfg,
                       int order = TAPT_ORDER_REFERENCE) {
    TAPTConfig c = cfg;
    c.N_T = 0;
    return run_tapt(g, ladder, c, nullptr, order);
}

// residual_energy: rho(t) = (<E_coldest(t)>_runs - E_gnd) / N, the
// coldest replica's energy after global move t averaged over independent runs.  best_so_far: use each
// run's best energy up to move t instead (the "best-so-far sense" of SPEC.md:456; non-increasing).
// Runs must have the same number of moves (DimensionError otherwise).
inline std::vector<double> residual_energy(const std::vector<RunTrace>& runs, double e_gnd, std::size_t n_spins,
                                           bool best_so_far = false) {
    if (runs.empty()) throw ConfigError("residual_energy needs at least one run");
    if (n_spins == 0) throw ConfigError("n_spins must be > 0");
    const std::size_t T = best_so_far ? runs[0].best_energy.size() : runs[0].energies.size();
    std::vector<double> rho(T, 0.0);
    for (const auto& tr : runs) {
        const std::size_t Tk = best_so_far ? tr.best_energy.size() : tr.energies.size();
        if (Tk != T) throw DimensionError("residual_energy: runs differ in their number of global moves");
        for (std::size_t t = 0; t < T; ++t) {
            if (!best_so_far && tr.energies[t].empty()) throw DimensionError("residual_energy: empty energy record");
            rho[t] += best_so_far ? tr.best_energy[t] : tr.energies[t].back();
        }
    }
    for (double& v : rho) v = (v / double(runs.size()) - e_gnd) / double(n_spins);
    return rho;
}

inline std::vector<double> residual_energy(const RunTrace& tr, double e_gnd, std::size_t n_spins) {
    return residual_energy(std::vector<RunTrace>{tr}, e_gnd, n_spins);
}

// adaptive_ladder: greedy from beta_min; probe chains (device sweeps, stream
// kProbe) estimate sigma_E, and the next beta is placed where the Gaussian-approximated swap
// acceptance erfc(dbeta*sigma/2) equals the target, sigma being the mean of the probe estimates at
// both ends of the gap (refined twice); degenerate variance falls back to geometric spacing.
inline BetaLadder adaptive_ladder(const CouplingGraph& g, double beta_min, double beta_max, double target,
                                  std::uint64_t probe_budget, std::uint64_t seed) {
    if (!(target > 0.0 && target < 1.0)) throw ConfigError("target acceptance must be in (0, 1)");
    if (!(beta_max > beta_min) || beta_min < 0.0) throw ConfigError("need 0 <= beta_min < beta_max");
    auto erfcinv = [](double y) {  // bisection on erfc (monotone decreasing)
        double lo = 0.0, hi = 10.0;
        for (int k = 0; k < 200; ++k) {
            const double mid = 0.5 * (lo + hi);
            if (std::erfc(mid) > y) lo = mid; else hi = mid;
        }
        return 0.5 * (lo + hi);
    };
    BetaLadder out;
    double b = beta_min;
    std::uint64_t k = 0;
    const std::uint64_t sweeps = std::max<std::uint64_t>(probe_budget, 8);
    // sigma_E at beta from a fresh probe chain (own streams {kProbe, k, 0|1}, second half of the run)
    auto sigma = [&](double beta) {
        RngStream init = RngStream::derive(seed, {stream::kProbe, k, 0});
        RngStream dyn = RngStream::derive(seed, {stream::kProbe, k, 1});
        ++k;
        SpinConfiguration s = random_configuration(g, init);
        std::vector<double> dE;
        const double e0 = energy(g, s);
        gibbs_sweeps(g, s, beta, dyn, static_cast<std::uint32_t>(sweeps), &dE);
        std::vector<double> E;
        double cur = e0;
        for (double d : dE) E.push_back(cur += d);
        const std::size_t from = E.size() / 2;
        double mu = 0, var = 0;
        for (std::size_t t = from; t < E.size(); ++t) mu += E[t];
        mu /= double(E.size() - from);
        for (std::size_t t = from; t < E.size(); ++t) var += (E[t] - mu) * (E[t] - mu);
        var /= double(E.size() - from);
        return std::sqrt(var);
    };
    const double x = 2.0 * erfcinv(target);  // erfc(dbeta * sigma / 2) = target  <=>  dbeta * sigma = x
    // at most 255 probe points + beta_max (the engine's 256-slot limit)
    while (b < beta_max && out.betas.size() < 255) {
        out.betas.push_back(b);
        const double s0 = sigma(b);
        double step;
        if (s0 <= 0.0) {
            step = b * (std::pow(beta_max / std::max(beta_min, 1e-3), 1.0 / 15.0) - 1.0) + 1e-3;
        } else {
            // sigma_E changes across the gap: place the next beta with the mean of sigma at both ends
            // (two fixed-point refinements, each probing the candidate), not sigma at b alone
            step = x / s0;
            for (int it = 0; it < 2 && b + step < beta_max; ++it) {
                const double s1 = sigma(b + step);
                step = x / (0.5 * (s0 + s1) > 0.0 ? 0.5 * (s0 + s1) : s0);
            }
        }
        b += std::max(step, 1e-4);
    }
    // close at beta_max; a last gap below the minimum step would make the swap tables oversize
    // ("beta spacing too fine"), so beta_max then replaces the last probe point instead
    if (out.betas.size() > 1 && beta_max - out.betas.back() < 1e-4)
        out.betas.back() = beta_max;
    else if (out.betas.back() < beta_max)
        out.betas.push_back(beta_max);
    return out;
}

}  // namespace tapt
