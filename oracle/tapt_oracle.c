/*
 * oracle/tapt_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the TAPT verifier path (parallel-tempering
 * sweeps, Metropolis replica swaps, Metropolis acceptance of whole-configuration
 * proposals).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this file's shared object; the
 * product (paper_2509_23043_b200/, include/) never links or calls it.
 *
 * Parity status: PINNED.  The restated pieces that exist in the reference are
 * checked bit-for-bit against the unmodified reference sources compiled into
 * oracle/_ref (see oracle/Makefile, oracle/ref_shim.cpp, tests/test_oracle_cpu.py)
 * and against the committed golden vectors in tests/golden/ that were produced
 * from oracle/_ref by tests/golden/make_golden.py.
 *
 * What each function follows (paths relative to /root/reference):
 *   oc_mix_final / oc_derive / oc_draw  proj/include/tapt/rng.hpp:21-32,58-65
 *       draw k (1-based) of a stream with state s0 is mix_final(s0 + k*phi)
 *   oc_uniform / coin                   rng.hpp:35 (53-bit uniform), rng.hpp:53 (top bit)
 *   oc_conditional_up                   proj/src/mcmc.cpp:13-15
 *   oc_energy                           proj/src/spin_model.cpp:79-89
 *   oc_random_configuration             proj/src/spin_model.cpp:116-121 (+ apply_clamps 103-107)
 *   oc_sweep (index order)              proj/src/mcmc.cpp:30-45 (gibbs_sweep)
 *   oc_sweep (colour order)             same update rule and the same per-site draw
 *                                       index, visiting colour classes in order
 *   oc_pt_swap_pass                     SPEC.md:400-408, PAPER.md:131 (Eq. 1)
 *   oc_pt_inject                        SPEC.md:409-417, PAPER.md:137 (Eq. 2)
 *   oc_pt_synthetic_proposals           BASELINE.json configs[1], configs[4] (stand-in generator)
 * The stream/draw-address conventions for the spec-only pieces (swap, proposal,
 * generator) are the ones written down in DESIGN.md section 3.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OC_PHI 0x9E3779B97F4A7C15ull
#define OC_TAG_INIT 0x11ull
#define OC_TAG_REPLICA 0x22ull
#define OC_TAG_COORD 0x33ull

/* ---------------------------------------------------------------- RNG ---- */

uint64_t oc_mix_final(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint64_t oc_mix(uint64_t z) { return oc_mix_final(z + OC_PHI); }

uint64_t oc_derive(uint64_t root, const uint64_t* path, int n) {
    uint64_t s = oc_mix(root ^ OC_PHI);
    for (int k = 0; k < n; ++k) s = oc_mix(s ^ (path[k] + OC_PHI));
    return s;
}

uint64_t oc_draw(uint64_t s0, uint64_t k) { return oc_mix_final(s0 + k * OC_PHI); }

double oc_uniform(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

double oc_conditional_up(double beta, double l) { return 1.0 / (1.0 + exp(-2.0 * beta * l)); }

static uint64_t derive2(uint64_t seed, uint64_t a, uint64_t b) {
    uint64_t p[2] = {a, b};
    return oc_derive(seed, p, 2);
}
static uint64_t derive3(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
    uint64_t p[3] = {a, b, c};
    return oc_derive(seed, p, 3);
}
static uint64_t derive4(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    uint64_t p[4] = {a, b, c, d};
    return oc_derive(seed, p, 4);
}

/* -------------------------------------------------------------- graph ---- */

/* CSR graph with integer couplings and fields.  Neighbour lists are ascending
 * by index (the reference's CSR order, spin_model.cpp:52-63). */
typedef struct {
    uint32_t n;
    uint32_t n_free;
    const uint32_t* rowptr; /* n+1 */
    const uint32_t* col;    /* rowptr[n] */
    const int32_t* J;       /* rowptr[n] */
    const int32_t* h;       /* n */
    const int8_t* clamp;    /* n: 0 free, +-1 clamped */
    const uint32_t* rank;   /* n: position in ascending free list (clamped: unused) */
} oc_graph;

int64_t oc_energy(const oc_graph* g, const int8_t* s) {
    double e = 0.0;
    for (uint32_t i = 0; i < g->n; ++i)
        for (uint32_t k = g->rowptr[i]; k < g->rowptr[i + 1]; ++k) {
            uint32_t j = g->col[k];
            if (j > i) e -= (double)g->J[k] * (double)(s[i] * s[j]);
        }
    for (uint32_t i = 0; i < g->n; ++i) e -= (double)g->h[i] * (double)s[i];
    return (int64_t)e;
}

double oc_local_field(const oc_graph* g, const int8_t* s, uint32_t i) {
    double l = (double)g->h[i];
    for (uint32_t k = g->rowptr[i]; k < g->rowptr[i + 1]; ++k) l += (double)g->J[k] * (double)s[g->col[k]];
    return l;
}

/* random_configuration: one coin per site (clamped sites too), then clamps. */
void oc_random_configuration(const oc_graph* g, uint64_t s0, int8_t* s) {
    for (uint32_t i = 0; i < g->n; ++i) s[i] = (oc_draw(s0, (uint64_t)i + 1) >> 63) ? 1 : -1;
    for (uint32_t i = 0; i < g->n; ++i)
        if (g->clamp[i]) s[i] = g->clamp[i];
}

/* One heat-bath sweep over the free sites listed in `order` (n_free entries).
 * Site i uses draw  draw_base + rank[i] + 1  of stream s0 regardless of when
 * it is visited, so index order reproduces gibbs_sweep exactly and colour
 * order is the same chain with a different (parallel) visiting schedule.
 * Returns the energy change (exact for integer couplings). */
int64_t oc_sweep(const oc_graph* g, const uint32_t* order, int8_t* s, double beta, uint64_t s0,
                 uint64_t draw_base) {
    double delta = 0.0;
    for (uint32_t q = 0; q < g->n_free; ++q) {
        uint32_t i = order[q];
        double l = oc_local_field(g, s, i);
        uint64_t x = oc_draw(s0, draw_base + g->rank[i] + 1);
        int8_t next = oc_uniform(x) < oc_conditional_up(beta, l) ? 1 : -1;
        if (next != s[i]) {
            delta += 2.0 * (double)s[i] * l;
            s[i] = next;
        }
    }
    return (int64_t)delta;
}

/* ----------------------------------------------------------- PT state ---- */
/* State is stored BY SLOT: configurations and energies move on a swap, the
 * inverse temperature and the dynamics stream stay with the slot
 * (SPEC.md:403,466). */

uint64_t oc_stream_init(uint64_t seed, uint64_t gid, uint64_t slot) {
    return derive3(seed, OC_TAG_INIT, gid, slot);
}
uint64_t oc_stream_replica(uint64_t seed, uint64_t gid, uint64_t slot) {
    return derive3(seed, OC_TAG_REPLICA, gid, slot);
}
uint64_t oc_stream_coord(uint64_t seed, uint64_t gid) { return derive2(seed, OC_TAG_COORD, gid); }
uint64_t oc_stream_accept(uint64_t seed, uint64_t gid, uint64_t round) {
    return derive3(seed, OC_TAG_COORD, gid, round + 1);
}
uint64_t oc_stream_proposal(uint64_t seed, uint64_t gid, uint64_t slot, uint64_t round) {
    return derive4(seed, OC_TAG_REPLICA, gid, slot, round + 1);
}

void oc_pt_init(const oc_graph* g, int R, uint64_t seed, uint64_t gid, int8_t* spins, int64_t* E) {
    for (int r = 0; r < R; ++r) {
        int8_t* s = spins + (size_t)r * g->n;
        oc_random_configuration(g, oc_stream_init(seed, gid, (uint64_t)r), s);
        E[r] = oc_energy(g, s);
    }
}

/* One sweep of every slot; sweep index t (0-based) uses draws t*n_free+rank+1. */
void oc_pt_sweep_all(const oc_graph* g, const uint32_t* order, int R, const double* beta, uint64_t seed,
                     uint64_t gid, uint64_t t, int8_t* spins, int64_t* E) {
    for (int r = 0; r < R; ++r) {
        uint64_t s0 = oc_stream_replica(seed, gid, (uint64_t)r);
        E[r] += oc_sweep(g, order, spins + (size_t)r * g->n, beta[r], s0, t * (uint64_t)g->n_free);
    }
}

static void swap_slots(int8_t* spins, size_t n, int64_t* E, int a, int b, int8_t* tmp) {
    memcpy(tmp, spins + (size_t)a * n, n);
    memcpy(spins + (size_t)a * n, spins + (size_t)b * n, n);
    memcpy(spins + (size_t)b * n, tmp, n);
    int64_t e = E[a];
    E[a] = E[b];
    E[b] = e;
}

/* Swap pass number p (0-based) over pairs (r, r+1), r = parity, parity+2, ...
 * Pair r uses draw p*R + r + 1 of the instance's coordinator stream; accept iff
 * uniform < exp((beta[r+1]-beta[r]) * (E[r+1]-E[r])) (= min[1, exp(.)], Eq. 1). */
void oc_pt_swap_pass(int R, const double* beta, uint64_t seed, uint64_t gid, uint64_t p, int parity,
                     int8_t* spins, size_t n, int64_t* E, uint64_t* att, uint64_t* acc, uint8_t* dec) {
    uint64_t c0 = oc_stream_coord(seed, gid);
    int8_t* tmp = (int8_t*)malloc(n ? n : 1);
    if (dec)
        for (int r = 0; r + 1 < R; ++r) dec[r] = 0;
    for (int r = parity; r + 1 < R; r += 2) {
        uint64_t x = oc_draw(c0, p * (uint64_t)R + (uint64_t)r + 1);
        double dbeta = beta[r + 1] - beta[r];
        double dE = (double)E[r + 1] - (double)E[r];
        int accept = oc_uniform(x) < exp(dbeta * dE);
        if (att) att[r] += 1;
        if (accept) {
            if (acc) acc[r] += 1;
            swap_slots(spins, n, E, r, r + 1, tmp);
        }
        if (dec) dec[r] = (uint8_t)(accept ? 1 : 2);
    }
    free(tmp);
}

/* Metropolis acceptance of externally supplied proposals (Eq. 2) for slots with
 * mask[r] != 0.  Round n uses draw r+1 of stream derive(seed,{kCoordinator,gid,n+1});
 * accept iff uniform < exp(beta[r] * (E[r] - Eprop[r])). */
void oc_pt_inject(int R, const double* beta, uint64_t seed, uint64_t gid, uint64_t round, const uint8_t* mask,
                  const int8_t* props, const int64_t* Eprop, int8_t* spins, size_t n, int64_t* E, uint64_t* att,
                  uint64_t* acc, uint8_t* dec) {
    uint64_t a0 = oc_stream_accept(seed, gid, round);
    for (int r = 0; r < R; ++r) {
        if (dec) dec[r] = 0;
        if (!mask[r]) continue;
        uint64_t x = oc_draw(a0, (uint64_t)r + 1);
        double dE = (double)E[r] - (double)Eprop[r];
        int accept = oc_uniform(x) < exp(beta[r] * dE);
        if (att) att[r] += 1;
        if (accept) {
            if (acc) acc[r] += 1;
            memcpy(spins + (size_t)r * n, props + (size_t)r * n, n);
            E[r] = Eprop[r];
        }
        if (dec) dec[r] = (uint8_t)(accept ? 1 : 2);
    }
}

/* MH-corrected variant: accept iff
 * uniform < exp(beta[r]*(E[r]-Eprop[r])) * exp(logq_cur[r] - logq_prop[r]). */
void oc_pt_inject_mh(int R, const double* beta, uint64_t seed, uint64_t gid, uint64_t round, const uint8_t* mask,
                     const int8_t* props, const int64_t* Eprop, const double* lq_cur, const double* lq_prop,
                     int8_t* spins, size_t n, int64_t* E, uint64_t* att, uint64_t* acc, uint8_t* dec) {
    uint64_t a0 = oc_stream_accept(seed, gid, round);
    for (int r = 0; r < R; ++r) {
        if (dec) dec[r] = 0;
        if (!mask[r]) continue;
        uint64_t x = oc_draw(a0, (uint64_t)r + 1);
        double dE = (double)E[r] - (double)Eprop[r];
        double a = exp(beta[r] * dE) * exp(lq_cur[r] - lq_prop[r]);
        int accept = oc_uniform(x) < a;
        if (att) att[r] += 1;
        if (accept) {
            if (acc) acc[r] += 1;
            memcpy(spins + (size_t)r * n, props + (size_t)r * n, n);
            E[r] = Eprop[r];
        }
        if (dec) dec[r] = (uint8_t)(accept ? 1 : 2);
    }
}

/* Stand-in generator (BASELINE configs 2 and 5): for each slot with mask[r],
 * stream Q = derive(seed,{kReplica,gid,r,round+1}); draw 1 picks the sign of the
 * bias (top bit set -> +), draws 2..n+1 give i.i.d. spins (+1 iff uniform < p_up,
 * p_up = (1 + sign*m_bias[r])/2), clamps are applied, then `refine` sweeps at
 * beta[r] in `order` use draws (n+1) + m*n_free + rank + 1. */
void oc_pt_synthetic_proposals(const oc_graph* g, const uint32_t* order, int R, const double* beta,
                               const double* m_bias, uint64_t seed, uint64_t gid, uint64_t round,
                               const uint8_t* mask, int refine, int8_t* props, int64_t* Eprop) {
    for (int r = 0; r < R; ++r) {
        if (!mask[r]) continue;
        int8_t* s = props + (size_t)r * g->n;
        uint64_t q = oc_stream_proposal(seed, gid, (uint64_t)r, round);
        double sign = (oc_draw(q, 1) >> 63) ? 1.0 : -1.0;
        double p_up = (1.0 + sign * m_bias[r]) / 2.0;
        for (uint32_t i = 0; i < g->n; ++i) s[i] = oc_uniform(oc_draw(q, (uint64_t)i + 2)) < p_up ? 1 : -1;
        for (uint32_t i = 0; i < g->n; ++i)
            if (g->clamp[i]) s[i] = g->clamp[i];
        for (int m = 0; m < refine; ++m)
            oc_sweep(g, order, s, beta[r], q, (uint64_t)g->n + 1 + (uint64_t)m * g->n_free);
        Eprop[r] = oc_energy(g, s);
    }
}

/* Per-slot observables: count, sum E, sum E^2, sum |M|, sum M^2 (M = sum of all
 * spins, clamped included, magnetization() numerator spin_model.cpp:109-114),
 * and an energy histogram with bins of `width` starting at e_lo. */
void oc_pt_measure(const int8_t* spins, size_t n, int R, const int64_t* E, int64_t* cnt, int64_t* sumE,
                   int64_t* sumE2, int64_t* sumAbsM, int64_t* sumM2, int64_t e_lo, int64_t width, int nbins,
                   int64_t* hist) {
    for (int r = 0; r < R; ++r) {
        int64_t m = 0;
        const int8_t* s = spins + (size_t)r * n;
        for (size_t i = 0; i < n; ++i) m += s[i];
        cnt[r] += 1;
        sumE[r] += E[r];
        sumE2[r] += E[r] * E[r];
        sumAbsM[r] += m < 0 ? -m : m;
        sumM2[r] += m * m;
        if (hist && nbins > 0) {
            int64_t b = (E[r] - e_lo) / width;
            if (E[r] < e_lo) b = 0;
            if (b >= nbins) b = nbins - 1;
            hist[(size_t)r * nbins + b] += 1;
        }
    }
}

/* ======================================================= real couplings ==== */
/* The same path for real-valued couplings and fields (the reference's CouplingGraph
 * takes any double J, spin_model.cpp:18-24, and gibbs_sweep works in FP64,
 * mcmc.cpp:30-45).  Energies are doubles: the initial energy is energy()
 * (spin_model.cpp:79-89: couplings in (i<j) order, then fields), after a sweep
 * E += the sweep's return value (the sum, in visiting order, of 2*s_old*l over the
 * flipped sites, mcmc.cpp:38-42), and a proposal's energy is energy() of it.  Swap and
 * proposal decisions are the expressions of ref_shim.cpp's restated driver (Eq. 1, 2)
 * on these doubles.  Index order reproduces the reference bit for bit (pinned by
 * tests/golden/pt_real*.npz from oracle/_ref). */

typedef struct {
    uint32_t n;
    uint32_t n_free;
    const uint32_t* rowptr;
    const uint32_t* col;
    const double* J;      /* rowptr[n], merged coupling value per CSR entry */
    const double* h;      /* n */
    const int8_t* clamp;
    const uint32_t* rank;
} oc_rgraph;

double oc_renergy(const oc_rgraph* g, const int8_t* s) {
    double e = 0.0;
    for (uint32_t i = 0; i < g->n; ++i)
        for (uint32_t k = g->rowptr[i]; k < g->rowptr[i + 1]; ++k) {
            uint32_t j = g->col[k];
            if (j > i) e -= g->J[k] * (double)(s[i] * s[j]);
        }
    for (uint32_t i = 0; i < g->n; ++i) e -= g->h[i] * (double)s[i];
    return e;
}

double oc_rlocal_field(const oc_rgraph* g, const int8_t* s, uint32_t i) {
    double l = g->h[i];
    for (uint32_t k = g->rowptr[i]; k < g->rowptr[i + 1]; ++k) l += g->J[k] * (double)s[g->col[k]];
    return l;
}

/* One sweep over `order` (n_free sites); site i takes draw draw_base + rank[i] + 1. */
double oc_rsweep(const oc_rgraph* g, const uint32_t* order, int8_t* s, double beta, uint64_t s0, uint64_t draw_base) {
    double delta = 0.0;
    for (uint32_t q = 0; q < g->n_free; ++q) {
        uint32_t i = order[q];
        double l = oc_rlocal_field(g, s, i);
        uint64_t x = oc_draw(s0, draw_base + g->rank[i] + 1);
        int8_t next = oc_uniform(x) < oc_conditional_up(beta, l) ? 1 : -1;
        if (next != s[i]) {
            delta += 2.0 * (double)s[i] * l;
            s[i] = next;
        }
    }
    return delta;
}

/* gibbs_update (mcmc.cpp:24-28): one site, the stream's next draw (draw 1 of s0). */
int8_t oc_rupdate(const oc_rgraph* g, const int8_t* s, uint32_t i, double beta, uint64_t s0) {
    double l = oc_rlocal_field(g, s, i);
    return oc_uniform(oc_draw(s0, 1)) < oc_conditional_up(beta, l) ? 1 : -1;
}

void oc_rpt_init(const oc_rgraph* g, int R, uint64_t seed, uint64_t gid, int8_t* spins, double* E) {
    for (int r = 0; r < R; ++r) {
        int8_t* s = spins + (size_t)r * g->n;
        uint64_t s0 = oc_stream_init(seed, gid, (uint64_t)r);
        for (uint32_t i = 0; i < g->n; ++i) s[i] = (oc_draw(s0, (uint64_t)i + 1) >> 63) ? 1 : -1;
        for (uint32_t i = 0; i < g->n; ++i)
            if (g->clamp[i]) s[i] = g->clamp[i];
        E[r] = oc_renergy(g, s);
    }
}

void oc_rpt_sweep_all(const oc_rgraph* g, const uint32_t* order, int R, const double* beta, uint64_t seed,
                      uint64_t gid, uint64_t t, int8_t* spins, double* E) {
    for (int r = 0; r < R; ++r) {
        uint64_t s0 = oc_stream_replica(seed, gid, (uint64_t)r);
        E[r] += oc_rsweep(g, order, spins + (size_t)r * g->n, beta[r], s0, t * (uint64_t)g->n_free);
    }
}

void oc_rpt_swap_pass(int R, const double* beta, uint64_t seed, uint64_t gid, uint64_t p, int parity, int8_t* spins,
                      size_t n, double* E, uint64_t* att, uint64_t* acc, uint8_t* dec) {
    uint64_t c0 = oc_stream_coord(seed, gid);
    int8_t* tmp = (int8_t*)malloc(n ? n : 1);
    if (dec)
        for (int r = 0; r + 1 < R; ++r) dec[r] = 0;
    for (int r = parity; r + 1 < R; r += 2) {
        uint64_t x = oc_draw(c0, p * (uint64_t)R + (uint64_t)r + 1);
        int accept = oc_uniform(x) < exp((beta[r + 1] - beta[r]) * (E[r + 1] - E[r]));
        if (att) att[r] += 1;
        if (accept) {
            if (acc) acc[r] += 1;
            memcpy(tmp, spins + (size_t)r * n, n);
            memcpy(spins + (size_t)r * n, spins + (size_t)(r + 1) * n, n);
            memcpy(spins + (size_t)(r + 1) * n, tmp, n);
            double e = E[r];
            E[r] = E[r + 1];
            E[r + 1] = e;
        }
        if (dec) dec[r] = (uint8_t)(accept ? 1 : 2);
    }
    free(tmp);
}

void oc_rpt_inject(int R, const double* beta, uint64_t seed, uint64_t gid, uint64_t round, const uint8_t* mask,
                   const int8_t* props, const double* Eprop, int8_t* spins, size_t n, double* E, uint64_t* att,
                   uint64_t* acc, uint8_t* dec) {
    uint64_t a0 = oc_stream_accept(seed, gid, round);
    for (int r = 0; r < R; ++r) {
        if (dec) dec[r] = 0;
        if (!mask[r]) continue;
        uint64_t x = oc_draw(a0, (uint64_t)r + 1);
        int accept = oc_uniform(x) < exp(beta[r] * (E[r] - Eprop[r]));
        if (att) att[r] += 1;
        if (accept) {
            if (acc) acc[r] += 1;
            memcpy(spins + (size_t)r * n, props + (size_t)r * n, n);
            E[r] = Eprop[r];
        }
        if (dec) dec[r] = (uint8_t)(accept ? 1 : 2);
    }
}

void oc_rpt_synthetic_proposals(const oc_rgraph* g, const uint32_t* order, int R, const double* beta,
                                const double* m_bias, uint64_t seed, uint64_t gid, uint64_t round,
                                const uint8_t* mask, int refine, int8_t* props, double* Eprop) {
    for (int r = 0; r < R; ++r) {
        if (!mask[r]) continue;
        int8_t* s = props + (size_t)r * g->n;
        uint64_t q = oc_stream_proposal(seed, gid, (uint64_t)r, round);
        double sign = (oc_draw(q, 1) >> 63) ? 1.0 : -1.0;
        double p_up = (1.0 + sign * m_bias[r]) / 2.0;
        for (uint32_t i = 0; i < g->n; ++i) s[i] = oc_uniform(oc_draw(q, (uint64_t)i + 2)) < p_up ? 1 : -1;
        for (uint32_t i = 0; i < g->n; ++i)
            if (g->clamp[i]) s[i] = g->clamp[i];
        for (int m = 0; m < refine; ++m)
            oc_rsweep(g, order, s, beta[r], q, (uint64_t)g->n + 1 + (uint64_t)m * g->n_free);
        Eprop[r] = oc_renergy(g, s);
    }
}

/* MH-corrected variant with FP64 energies: accept iff
 * uniform < exp(beta[r]*(E[r]-Eprop[r])) * exp(lq_cur[r] - lq_prop[r]). */
void oc_rpt_inject_mh(int R, const double* beta, uint64_t seed, uint64_t gid, uint64_t round, const uint8_t* mask,
                      const int8_t* props, const double* Eprop, const double* lq_cur, const double* lq_prop,
                      int8_t* spins, size_t n, double* E, uint64_t* att, uint64_t* acc, uint8_t* dec) {
    uint64_t a0 = oc_stream_accept(seed, gid, round);
    for (int r = 0; r < R; ++r) {
        if (dec) dec[r] = 0;
        if (!mask[r]) continue;
        uint64_t x = oc_draw(a0, (uint64_t)r + 1);
        double a = exp(beta[r] * (E[r] - Eprop[r])) * exp(lq_cur[r] - lq_prop[r]);
        int accept = oc_uniform(x) < a;
        if (att) att[r] += 1;
        if (accept) {
            if (acc) acc[r] += 1;
            memcpy(spins + (size_t)r * n, props + (size_t)r * n, n);
            E[r] = Eprop[r];
        }
        if (dec) dec[r] = (uint8_t)(accept ? 1 : 2);
    }
}
