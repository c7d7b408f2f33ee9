// problems.cu -- host-side problem suite (the reference's
// proj/src/problems.cpp:1 is a placeholder): invertible AND / full-adder gate
// Hamiltonians, the 3n^2+n array multiplier with spin identification, product clamping,
// decoding, semiprimes.  Instance construction only -- never on the timed path.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "tapt/errors.hpp"
#include "tapt/rng.hpp"
#include "tapt_gpu.h"

namespace {

thread_local std::string g_prob_err;

template <class F>
tapt_status pguard(F&& f) {
    try {
        f();
        return TAPT_OK;
    } catch (const tapt::ConfigError& e) {
        g_prob_err = e.what();
        return TAPT_ERR_CONFIG;
    } catch (const tapt::SizeError& e) {
        g_prob_err = e.what();
        return TAPT_ERR_SIZE;
    } catch (const tapt::DimensionError& e) {
        g_prob_err = e.what();
        return TAPT_ERR_DIMENSION;
    } catch (const std::exception& e) {
        g_prob_err = e.what();
        return TAPT_ERR_INTERNAL;
    }
}

struct Gate {
    std::vector<uint32_t> ci, cj;
    std::vector<double> J, h;
};

// AND(A, B) = C: J_AB = -1, J_AC = J_BC = 2, h = (1, 1, -2)
void add_and(Gate& g, uint32_t a, uint32_t b, uint32_t c) {
    const uint32_t s[3] = {a, b, c};
    const double hv[3] = {1, 1, -2};
    g.ci.insert(g.ci.end(), {a, a, b});
    g.cj.insert(g.cj.end(), {b, c, c});
    g.J.insert(g.J.end(), {-1, 2, 2});
    for (int k = 0; k < 3; ++k) g.h[s[k]] += hv[k];
}

// FA(A, B, Cin) = (S, Cout): J_AB = J_ACin = J_BCin = -1; J_AS = J_BS = J_CinS = 1;
// J_ACout = J_BCout = J_CinCout = 2; J_SCout = -2 (the couplings of SPEC.md:525-532) and NO
// fields.  With x = (1+s)/2 these are E = 2 (a+b+c-s-2o)^2 - 4, so the 8 valid rows sit at
// E = -4 and every invalid row at E >= -2.  The fields h = (1,1,1,-1,-2) listed in SPEC.md
// add -2(a+b+c-s-2o), which puts the L = +1 rows (e.g. 0+0+1 -> S=0, Cout=0) at -4 too:
// enumeration rejects them (tests/test_problems_cpu.py), so they are not used.
void add_fa(Gate& g, uint32_t a, uint32_t b, uint32_t cin, uint32_t s, uint32_t cout) {
    const uint32_t v[5] = {a, b, cin, s, cout};
    const double hv[5] = {0, 0, 0, 0, 0};
    const int pairs[10][2] = {{0, 1}, {0, 2}, {1, 2}, {0, 3}, {1, 3}, {2, 3}, {0, 4}, {1, 4}, {2, 4}, {3, 4}};
    const double jv[10] = {-1, -1, -1, 1, 1, 1, 2, 2, 2, -2};
    for (int k = 0; k < 10; ++k) {
        g.ci.push_back(v[pairs[k][0]]);
        g.cj.push_back(v[pairs[k][1]]);
        g.J.push_back(jv[k]);
    }
    for (int k = 0; k < 5; ++k) g.h[v[k]] += hv[k];
}

// Spin layout of the n-bit array multiplier (3n^2 + n spins):
//   A_i = i, B_j = n + j, p_ij = 2n + i + n*j,
//   FA (row j = 1..n-1, column i = 0..n-1): S = 2n + n^2 + 2((j-1) n + i), Cout = S + 1,
//   carry-in k = 2n + n^2 + 2n(n-1) + k   (clamped to logical 0).
struct Mult {
    uint32_t n;
    uint32_t A(uint32_t i) const { return i; }
    uint32_t B(uint32_t j) const { return n + j; }
    uint32_t P(uint32_t i, uint32_t j) const { return 2 * n + i + n * j; }
    uint32_t S(uint32_t j, uint32_t i) const { return 2 * n + n * n + 2 * ((j - 1) * n + i); }
    uint32_t Co(uint32_t j, uint32_t i) const { return S(j, i) + 1; }
    uint32_t Cin(uint32_t k) const { return 2 * n + n * n + 2 * n * (n - 1) + k; }
    uint32_t size() const { return 3 * n * n + n; }
    // row j, column i: inputs (partial product, running-sum bit, carry)
    uint32_t fa_b(uint32_t j, uint32_t i) const {
        if (i + 1 < n) return j == 1 ? P(i + 1, 0) : S(j - 1, i + 1);
        return j == 1 ? Cin(n - 1) : Co(j - 1, n - 1);  // weight j+n-1 of the running sum
    }
    uint32_t fa_cin(uint32_t j, uint32_t i) const { return i == 0 ? Cin(j - 1) : Co(j, i - 1); }
    // product bit k
    uint32_t C(uint32_t k) const {
        if (k == 0) return P(0, 0);
        if (n == 1) return Cin(0);
        if (k < n - 1) return S(k, 0);
        if (k < 2 * n - 1) return S(n - 1, k - (n - 1));
        return Co(n - 1, n - 1);
    }
};

bool is_prime(uint64_t v) {
    if (v < 2) return false;
    for (uint64_t d = 2; d * d <= v; ++d)
        if (v % d == 0) return false;
    return true;
}

}  // namespace

extern "C" {

const char* tapt_problem_last_error(void) { return g_prob_err.c_str(); }

uint32_t tapt_multiplier_spins(uint32_t n) { return 3 * n * n + n; }

// Couplings (before merging) and fields of the n-bit multiplier; ci/cj/J need
// 3n^2 + 10 n(n-1) entries, h and clamp need 3n^2+n; wires (nullable): A[n], B[n], C[2n], carry-in[n].
tapt_status tapt_multiplier_build(uint32_t n, uint32_t* n_couplings, uint32_t* ci, uint32_t* cj, double* J, double* h,
                                  int8_t* clamp, uint32_t* wires) {
    return pguard([&] {
        if (n < 2 || n > 31) throw tapt::ConfigError("multiplier width must be in [2, 31]");
        Mult m{n};
        Gate g;
        g.h.assign(m.size(), 0.0);
        for (uint32_t j = 0; j < n; ++j)
            for (uint32_t i = 0; i < n; ++i) add_and(g, m.A(i), m.B(j), m.P(i, j));
        for (uint32_t j = 1; j < n; ++j)
            for (uint32_t i = 0; i < n; ++i) add_fa(g, m.P(i, j), m.fa_b(j, i), m.fa_cin(j, i), m.S(j, i), m.Co(j, i));
        if (n_couplings) *n_couplings = (uint32_t)g.ci.size();
        if (ci) std::memcpy(ci, g.ci.data(), g.ci.size() * 4);
        if (cj) std::memcpy(cj, g.cj.data(), g.cj.size() * 4);
        if (J) std::memcpy(J, g.J.data(), g.J.size() * 8);
        if (h) std::memcpy(h, g.h.data(), g.h.size() * 8);
        if (clamp) {
            std::memset(clamp, 0, m.size());
            for (uint32_t k = 0; k < 2 * n; ++k) clamp[m.C(k)] = -1;  // product 0 until clamp_product
            for (uint32_t k = 0; k < n; ++k) clamp[m.Cin(k)] = -1;
        }
        if (wires) {
            for (uint32_t i = 0; i < n; ++i) wires[i] = m.A(i);
            for (uint32_t i = 0; i < n; ++i) wires[n + i] = m.B(i);
            for (uint32_t k = 0; k < 2 * n; ++k) wires[2 * n + k] = m.C(k);
            for (uint32_t k = 0; k < n; ++k) wires[4 * n + k] = m.Cin(k);
        }
    });
}

// Forward evaluation: the fully consistent wire assignment for inputs (a, b) (+1 = logical 1).
tapt_status tapt_multiplier_forward(uint32_t n, uint64_t a, uint64_t b, int8_t* s) {
    return pguard([&] {
        if (n < 2 || n > 31) throw tapt::ConfigError("multiplier width must be in [2, 31]");
        Mult m{n};
        std::vector<int> v(m.size(), 0);
        for (uint32_t i = 0; i < n; ++i) {
            v[m.A(i)] = (a >> i) & 1;
            v[m.B(i)] = (b >> i) & 1;
            v[m.Cin(i)] = 0;
        }
        for (uint32_t j = 0; j < n; ++j)
            for (uint32_t i = 0; i < n; ++i) v[m.P(i, j)] = v[m.A(i)] & v[m.B(j)];
        for (uint32_t j = 1; j < n; ++j)
            for (uint32_t i = 0; i < n; ++i) {
                const int t = v[m.P(i, j)] + v[m.fa_b(j, i)] + v[m.fa_cin(j, i)];
                v[m.S(j, i)] = t & 1;
                v[m.Co(j, i)] = t >> 1;
            }
        for (uint32_t k = 0; k < m.size(); ++k) s[k] = v[k] ? 1 : -1;
    });
}

// clamp_product: product bits to the binary expansion of C (LSB at C_0),
// carry-ins to logical 0, everything else free.
tapt_status tapt_multiplier_clamps(uint32_t n, uint64_t C, int8_t* clamp) {
    return pguard([&] {
        if (n < 2 || n > 31) throw tapt::ConfigError("multiplier width must be in [2, 31]");
        if (C >> (2 * n)) throw tapt::ConfigError("product does not fit 2n bits");
        Mult m{n};
        std::memset(clamp, 0, m.size());
        for (uint32_t k = 0; k < 2 * n; ++k) clamp[m.C(k)] = ((C >> k) & 1) ? 1 : -1;
        for (uint32_t k = 0; k < n; ++k) clamp[m.Cin(k)] = -1;
    });
}

// decode_and_check: A, B from their wires; success iff A*B == C.
tapt_status tapt_multiplier_decode(uint32_t n, const int8_t* s, uint64_t C, uint64_t* a, uint64_t* b, int* success) {
    return pguard([&] {
        if (n < 2 || n > 31) throw tapt::ConfigError("multiplier width must be in [2, 31]");
        Mult m{n};
        uint64_t x = 0, y = 0;
        for (uint32_t i = 0; i < n; ++i) {
            if (s[m.A(i)] > 0) x |= 1ull << i;
            if (s[m.B(i)] > 0) y |= 1ull << i;
        }
        if (a) *a = x;
        if (b) *b = y;
        if (success) *success = (x * y == C) ? 1 : 0;
    });
}

// enumerate_semiprimes: all p*q, p <= q primes < 2^n, ascending.
tapt_status tapt_enumerate_semiprimes(uint32_t n, uint64_t* out, uint32_t cap, uint32_t* count) {
    return pguard([&] {
        if (n < 1 || n > 20) throw tapt::ConfigError("semiprime enumeration supports n in [1, 20]");
        std::vector<uint64_t> pr, v;
        for (uint64_t x = 2; x < (1ull << n); ++x)
            if (is_prime(x)) pr.push_back(x);
        for (size_t i = 0; i < pr.size(); ++i)
            for (size_t j = i; j < pr.size(); ++j) v.push_back(pr[i] * pr[j]);
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
        if (count) *count = (uint32_t)v.size();
        if (out)
            for (size_t k = 0; k < v.size() && k < cap; ++k) out[k] = v[k];
    });
}

// Random semiprime of instance gid: p then q, each the first prime among
// candidates 2^(bits-1) + below(2^(bits-1)) drawn from derive(seed, {0x99, gid}).
tapt_status tapt_random_semiprime(uint64_t seed, uint64_t gid, uint32_t bits, uint64_t* p, uint64_t* q) {
    return pguard([&] {
        if (bits < 2 || bits > 31) throw tapt::ConfigError("prime width must be in [2, 31]");
        tapt::RngStream r = tapt::RngStream::derive(seed, {0x99, gid});
        const uint64_t base = 1ull << (bits - 1);
        auto next = [&] {
            for (;;) {
                const uint64_t c = base + r.below(base);
                if (is_prime(c)) return c;
            }
        };
        *p = next();
        *q = next();
    });
}

}  // extern "C"
