// tapt/generator.hpp -- the generator module of SPEC.md:275-379 (the IsingFormer; the
// reference's proj/src/generator.cpp:1 is a placeholder), inference on the B200 through
// tapt_former_* (tapt_gpu.h).  GeneratorConfig / ParameterSet / forward_logits / sample /
// log_prob / save/load_checkpoint (ISFW1).  Training is out of scope.
//
// Token order (SPEC design decision): the clamped sites in ascending index
// form the prefix, then the free sites in ascending index (for an unclamped lattice this is
// raster order).  Token 1 = spin +1.  As a ProposalSource for run_tapt, the prefix is the
// clamps plus the first context_len free spins of the current state (Appendix C);
// log_prob then scores the positions after that prefix, which is the proposal density the
// MH-corrected move needs.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "tapt/tempering.hpp"

namespace tapt {

struct GeneratorConfig {
    std::uint32_t d_model = 64, heads = 2, ffn = 128, layers = 2, max_sequence_length = 1024, beta_features = 16;

    tapt_former_config c() const {
        return tapt_former_config{d_model, heads, ffn, layers, max_sequence_length, beta_features};
    }
    std::size_t parameter_count() const {
        const auto x = c();
        return tapt_former_param_count(&x);
    }
};

using ParameterSet = std::vector<float>;  // canonical ISFW1 order

class IsingFormer : public ProposalSource {
  public:
    IsingFormer(const CouplingGraph& g, const GeneratorConfig& cfg, const ParameterSet& params) : g_(&g) {
        const auto c = cfg.c();
        if (params.size() != cfg.parameter_count()) throw DimensionError("parameter count does not match the config");
        tapt_former_t f = nullptr;
        throw_status(tapt_former_create(&c, params.data(), &f));
        adopt(f);
    }
    static IsingFormer load_checkpoint(const CouplingGraph& g, const std::string& path) {
        tapt_former_t f = nullptr;
        throw_status(tapt_former_load(path.c_str(), &f));
        return IsingFormer(g, f);
    }
    void save_checkpoint(const std::string& path) const { throw_status(tapt_former_save(f_.get(), path.c_str())); }
    // K/V cache precision of the device model: bf16 storage halves the sampling-bound K/V stream
    // (fp32 attention math).  Default fp32.
    void set_kv_bf16(bool on) { throw_status(tapt_former_set_kv_bf16(f_.get(), on ? 1 : 0)); }
    static ParameterSet init_params(const GeneratorConfig& cfg, std::uint64_t seed, double scale = 1.0) {
        const auto c = cfg.c();
        ParameterSet p(cfg.parameter_count());
        throw_status(tapt_former_init_params(&c, seed, scale, p.data()));
        return p;
    }
    GeneratorConfig config() const {
        tapt_former_config c{};
        throw_status(tapt_former_get(f_.get(), &c, nullptr));
        return GeneratorConfig{c.d_model, c.heads, c.ffn, c.layers, c.max_len, c.beta_features};
    }

    // Token sequence of a configuration (clamps first, then free sites).
    std::vector<std::uint8_t> tokens(std::span<const std::int8_t> s) const {
        if (s.size() != g_->n_spins()) throw DimensionError("configuration length mismatch");
        std::vector<std::uint8_t> t(order_.size());
        for (std::size_t k = 0; k < order_.size(); ++k) t[k] = s[order_[k]] > 0 ? 1 : 0;
        return t;
    }
    std::size_t prefix_length() const { return n_clamped_; }

    // forward_logits: one logit per token position.
    std::vector<float> forward_logits(std::span<const std::int8_t> s, double beta) const {
        const auto t = tokens(s);
        std::vector<float> z(t.size());
        double lq = 0.0;
        throw_status(tapt_former_log_prob(f_.get(), t.data(), 1, (std::uint32_t)t.size(), &beta, 0, &lq, z.data()));
        return z;
    }
    // log q of s: positions after the clamps and the current context.
    double log_prob(std::span<const std::int8_t> s, double beta) override {
        const auto t = tokens(s);
        double lq = 0.0;
        throw_status(tapt_former_log_prob(f_.get(), t.data(), 1, (std::uint32_t)t.size(), &beta,
                                          (std::uint32_t)(n_clamped_ + ctx_), &lq, nullptr));
        return lq;
    }
    // Ancestral sample: position t >= prefix draws draw t+1 of rng's state;
    // rng is advanced past the sequence.
    SpinConfiguration sample(std::size_t /*replica*/, double beta, std::span<const std::int8_t> context,
                             std::size_t context_len, RngStream& rng) override {
        const std::size_t T = order_.size();
        ctx_ = std::min(context_len, T - n_clamped_);
        std::vector<std::uint8_t> pre(n_clamped_ + ctx_);
        for (std::size_t k = 0; k < n_clamped_; ++k) pre[k] = g_->clamp_value(order_[k]) > 0 ? 1 : 0;
        if (ctx_) {
            if (context.size() != g_->n_spins()) throw DimensionError("context length mismatch");
            for (std::size_t k = n_clamped_; k < pre.size(); ++k) pre[k] = context[order_[k]] > 0 ? 1 : 0;
        }
        const std::uint64_t st = rng.state();
        std::vector<std::uint8_t> tok(T);
        double lq = 0.0;
        throw_status(tapt_former_sample(f_.get(), 1, (std::uint32_t)T, &beta, pre.empty() ? nullptr : pre.data(),
                                        (std::uint32_t)pre.size(), &st, tok.data(), &lq));
        rng.advance(T);
        SpinConfiguration s(g_->n_spins());
        for (std::size_t k = 0; k < T; ++k) s[order_[k]] = tok[k] ? 1 : -1;
        last_log_q_ = lq;
        return s;
    }
    double last_log_q() const { return last_log_q_; }

  private:
    IsingFormer(const CouplingGraph& g, tapt_former_t f) : g_(&g) { adopt(f); }
    void adopt(tapt_former_t f) {
        f_ = std::shared_ptr<tapt_former_s>(f, [](tapt_former_t p) { tapt_former_destroy(p); });
        for (std::uint32_t i = 0; i < g_->n_spins(); ++i)
            if (g_->is_clamped(i)) order_.push_back(i);
        n_clamped_ = order_.size();
        for (std::uint32_t i : g_->free_sites()) order_.push_back(i);
        if (order_.size() > config().max_sequence_length) throw SizeError("graph longer than the model's max_len");
    }
    const CouplingGraph* g_;
    std::shared_ptr<tapt_former_s> f_;
    std::vector<std::uint32_t> order_;
    std::size_t n_clamped_ = 0, ctx_ = 0;
    double last_log_q_ = 0.0;
};

}  // namespace tapt
