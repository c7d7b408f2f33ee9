// real.h -- K5: the FP64 sequential-order engine (real-valued couplings and fields).
//
// The reference's CouplingGraph takes any double J and h (spin_model.cpp:18-24) and gibbs_sweep
// computes the local field in FP64 in CSR order and decides with libm exp (mcmc.cpp:13-15,30-45).
// For such graphs no exact threshold table exists, so K5 reproduces the reference arithmetic:
//   * local field l = h_i, then l += (+-J_ij) over the CSR row in ascending neighbour order -- the
//     same IEEE additions as `l += nb.value * (double)s_j` (the product by +-1 is exact);
//   * heat-bath p = 1 / (1 + exp(-2*beta*l)), Eq. 1 exp((b_{r+1}-b_r)(E_{r+1}-E_r)) and Eq. 2
//     exp(b_r (E_r - E^T_r)) with the device exp, which differs from glibc's by a few ulp;
//   * a decision whose draw u lies within a relative band (1e-12) of the device probability is a
//     NEAR TIE: the kernel takes the device decision provisionally and records (event key, argument,
//     draw).  The host re-evaluates every recorded tie with glibc exp; if any provisional decision
//     differs, it restores the launch's state snapshot and relaunches with that decision as an
//     override (keyed by instance, time, slot, site), until every tie agrees.  Results are therefore
//     bit-identical to the reference while glibc is only ever consulted for near ties (~1e-12 of
//     the decisions);
//   * energies: E = energy() after init / set_spins / for proposals (couplings in (i<j) order, then
//     fields, spin_model.cpp:79-89), and E += the sweep's return value (the visiting-order sum of
//     2*s_old*l over flipped sites) after every sweep, as the restated driver does.
// Integer-valued models may use K5 too (the drop-in gibbs_sweep / gibbs_update): they pass the exact
// heat-bath tables and decide without ties.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

namespace tapt_real {

// A near-tie event (or an override of one).  kind: 0 heat-bath (t = global sweep, slot, site),
// 1 swap (t = pass, slot = pair r), 2 proposal (t = round, slot = target slot).
struct TieKey {
    uint32_t kind, inst, slot, site;
    unsigned long long t;
};
struct TieRec {
    TieKey key;
    double arg;   // l (heat-bath), E_{r+1}-E_r (swap), E_r - E^T_r (proposal)
    double coef;  // beta (heat-bath / proposal), b_{r+1}-b_r (swap)
    unsigned long long x;
    uint32_t dec;  // provisional device decision
};

// Host description of the graph (CouplingGraph semantics: merged couplings sorted (i<j), CSR rows
// ascending, free sites ascending).
struct RealGraph {
    uint32_t n = 0;
    std::vector<uint32_t> rowptr, col, ci, cj, free_sites, rank;
    std::vector<double> J, h, cJ;  // J per CSR entry; cJ per merged coupling
    std::vector<int8_t> clamp;
    std::vector<uint32_t> colour_order;  // free sites by colour class (ascending inside a class)
    // integer models: exact heat-bath threshold rows are supplied per ensemble (lmin, nidx)
    bool integral = false;
    int lmin = 0, lmax = 0;
};

struct RealEngineImpl;

// Device-resident ensemble state for K5 (I instances x R slots, multi-replica spin words
// [I][G][n], G = ceil(R/32), as the integer engine), with the PT/TAPT operations of the C ABI.
class RealEngine {
  public:
    RealEngine(const RealGraph& g, uint32_t I, uint64_t gid0, const std::vector<double>& betas, uint64_t seed,
               int order, cudaStream_t st);
    ~RealEngine();
    void set_stream(cudaStream_t st);
    cudaStream_t stream() const;
    void set_betas(const std::vector<double>& betas, bool decreasing);
    void set_streams(const uint64_t* states);            // [I][R] dynamics stream states by slot
    void init_random();
    void init_from_streams(const uint64_t* init_states);  // random_configuration from given streams
    void set_spins(const int8_t* host, bool force_clamps);  // [I][R][n] by slot; E = energy()
    void get_spins(int8_t* host);
    void get_spins_packed(uint8_t* host);
    void get_energies(double* host);                     // [I][R] by slot
    void get_permutation(uint8_t* host);                 // buf_of [I][R]
    void counters(uint64_t* T, uint64_t* P, uint64_t* Q) const;
    void acceptance(uint64_t* sa, uint64_t* sc, uint64_t* pa, uint64_t* pc);
    void observables(double* host);                      // [I][R][5] count, sum E, sum E^2, sum |M|, sum M^2
    void set_histogram(double e_lo, double width, uint32_t nbins);
    void get_histogram(uint64_t* dst, bool on_device);
    void best(double* host);
    void reset_observables();
    void run(uint32_t n_sweeps, uint32_t swap_every, uint32_t measure_every, uint64_t measure_from);
    void swap_pass(int parity);
    // proposals: int8 [I][T][n] / packed [I][T][ceil(n/8)] (host or device), or the synthetic
    // generator; `refine` sweeps at the target's beta, then Eq. 2 (MH-corrected with log q)
    void inject(const int8_t* props, bool on_device, const uint32_t* targets, uint32_t T, const double* lqc,
                const double* lqp, uint8_t* accepted);
    void inject_packed(const uint8_t* props, bool on_device, const uint32_t* targets, uint32_t T, uint32_t refine,
                       uint8_t* accepted);
    void generate(const uint32_t* targets, uint32_t T, const double* m_bias, uint32_t refine, uint8_t* accepted);
    // drop-in gibbs_sweep (single replica, caller's stream state, per-sweep dE) and gibbs_update
    void dropin_sweeps(int8_t* s, double beta, uint64_t state, uint32_t n_sweeps, double* dE,
                       const uint64_t* int_thr, int lmin, int nidx);
    void dropin_update(int8_t* s, uint32_t site, double beta, uint64_t state, const uint64_t* int_thr, int lmin,
                       int nidx);
    // test knobs: relative tie band and a perturbation of the device probabilities (TAPT_K5_BAND,
    // TAPT_K5_PERTURB) -- a perturbed device exp must still give reference-exact results
    unsigned long long ties_seen() const;
    unsigned long long replays() const;
    const char* kernel_name() const;

  private:
    std::unique_ptr<RealEngineImpl> p_;
};

}  // namespace tapt_real
