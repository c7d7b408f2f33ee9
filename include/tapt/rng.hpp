// tapt/rng.hpp -- counter-based RNG streams, API-compatible with the reference
// (proj/include/tapt/rng.hpp:14-79): splitmix64 increment + finalizer, streams derived
// by hashing a path of integers under a root seed.
//
// B200 note: because draw k of a stream is mix_final(state + k*phi), the device
// kernels address any draw directly from (stream state, counter); this class keeps
// the sequential interface the reference's callers use and adds the random-access
// helpers (at / advance / from_state) the drop-in wrappers need.
#pragma once

#include <cmath>
#include <cstdint>
#include <initializer_list>
#include <numbers>

namespace tapt {

namespace detail {
inline constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ull;

constexpr std::uint64_t finalize64(std::uint64_t v) {
    v ^= v >> 30;
    v *= 0xBF58476D1CE4E5B9ull;
    v ^= v >> 27;
    v *= 0x94D049BB133111EBull;
    v ^= v >> 31;
    return v;
}
constexpr std::uint64_t hash64(std::uint64_t v) { return finalize64(v + kGolden); }
}  // namespace detail

class RngStream {
  public:
    RngStream() = default;
    explicit RngStream(std::uint64_t seed) : s_(detail::hash64(seed ^ detail::kGolden)) {}

    // derive(root, {tag, a, b, ...}): hash the path components one after another.
    static RngStream derive(std::uint64_t root, std::initializer_list<std::uint64_t> path) {
        return derive_n(root, path.begin(), path.size());
    }
    static RngStream derive_n(std::uint64_t root, const std::uint64_t* path, std::size_t n) {
        std::uint64_t h = detail::hash64(root ^ detail::kGolden);
        for (std::size_t k = 0; k < n; ++k) h = detail::hash64(h ^ (path[k] + detail::kGolden));
        return from_state(h);
    }
    static RngStream from_state(std::uint64_t s) {
        RngStream r;
        r.s_ = s;
        return r;
    }

    std::uint64_t next_u64() {
        s_ += detail::kGolden;
        return detail::finalize64(s_);
    }
    double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double normal() {  // Box-Muller, two uniforms per call
        double a = uniform();
        const double b = uniform();
        if (a <= 0.0) a = 0x1.0p-53;
        return std::sqrt(-2.0 * std::log(a)) * std::cos(2.0 * std::numbers::pi * b);
    }
    std::uint64_t below(std::uint64_t n) {
        return static_cast<std::uint64_t>((static_cast<unsigned __int128>(next_u64()) * n) >> 64);
    }
    bool coin() { return (next_u64() >> 63) != 0; }
    std::uint64_t state() const { return s_; }

    // Random access: draw k (1-based) relative to the current state, without advancing.
    std::uint64_t at(std::uint64_t k) const { return detail::finalize64(s_ + k * detail::kGolden); }
    void advance(std::uint64_t k) { s_ += k * detail::kGolden; }

  private:
    std::uint64_t s_ = 0;
};

namespace stream {
constexpr std::uint64_t kInit = 0x11;
constexpr std::uint64_t kReplica = 0x22;
constexpr std::uint64_t kCoordinator = 0x33;
constexpr std::uint64_t kChain = 0x44;
constexpr std::uint64_t kAnneal = 0x55;
constexpr std::uint64_t kTrain = 0x66;
constexpr std::uint64_t kProbe = 0x77;
constexpr std::uint64_t kDisorder = 0x88;  // B200 build: EA bond signs
}  // namespace stream

}  // namespace tapt
