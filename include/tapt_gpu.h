/*
 * tapt_gpu.h -- C ABI of the B200-native TAPT verifier (parallel-tempering engine).
 *
 * The reference (/root/reference) is a C++20 library whose parallel-tempering
 * layer exists only as a specification; this header is the flat, exception-free
 * boundary a reference-side binding (C++ wrapper, ctypes, cgo, JNI ...) calls.
 * Every entry point below names the reference interface it replaces:
 *
 *   tapt_model_create_lattice   LatticeSpec::grid2d / grid3d + graph()      proj/include/tapt/lattice.hpp:25-35, proj/src/lattice.cpp:5-24,55-87
 *   tapt_model_create_graph     CouplingGraph::Builder(...).build()          proj/include/tapt/spin_model.hpp:32-48, proj/src/spin_model.cpp:15-77
 *   tapt_gibbs_sweep            gibbs_sweep(g, s, beta, rng)                 proj/include/tapt/mcmc.hpp:43-45, proj/src/mcmc.cpp:30-45
 *   tapt_gibbs_update           gibbs_update(g, s, i, beta, rng)             proj/include/tapt/mcmc.hpp:40-41, proj/src/mcmc.cpp:24-28
 *   tapt_ensemble_create        BetaLadder / TAPTConfig / replica state
 *   tapt_ensemble_init_random   random_configuration per replica             proj/src/spin_model.cpp:116-121, PAPER.md:89-90 (Alg. 1 l.1-2)
 *   tapt_sweep                  M x gibbs_sweep of every replica             PAPER.md:107-111 (Alg. 1)
 *   tapt_swap_pass              swap_pass(replicas, ladder, parity, rng)     SPEC.md:400-408, PAPER.md:131 (Eq. 1)
 *   tapt_run                    run_pt / run_tapt inner loop (fused)
 *   tapt_inject_proposals       generator_move / mh_corrected_move           SPEC.md:409-425, PAPER.md:137 (Eq. 2)
 *   tapt_generate_proposals     stand-in for IsingFormer.sample (synthetic)  BASELINE.json configs[1], configs[4]
 *   tapt_get_energies/_spins    energy(g, s) / magnetization(s) readout      proj/src/spin_model.cpp:79-89,109-114
 *   tapt_get_observables        RunTrace accumulators
 *   tapt_last_error / status    tapt::*Error exceptions                      proj/include/tapt/errors.hpp:11-41
 *   tapt_former_*               IsingFormer forward_logits / sample /        SPEC.md:275-379 (generator module;
 *                               log_prob / save/load_checkpoint (ISFW1)      proj/src/generator.cpp:1 is a placeholder)
 *
 * Conventions
 *   - Every function returns a tapt_status (0 = OK); no C++ exception crosses this
 *     boundary.  The message of the last failure on the calling thread is
 *     returned by tapt_last_error().  Status codes map 1:1 onto the reference's
 *     eight exception types (errors.hpp) plus CUDA / NCCL / internal failures.
 *   - Host buffers are caller-owned and copied synchronously.  Handles own all
 *     device memory; destroy them explicitly.  Calls on one handle are stream-ordered
 *     on the handle's CUDA stream (tapt_ensemble_set_stream).
 *   - Slots are ladder positions (index 0 = hottest); a swap moves the
 *     configuration, beta and dynamics stream stay with the slot.
 *     All per-replica inputs/outputs are ordered BY SLOT.
 *   - Spin arrays are int8 +-1, [instance][slot][site], row-major.
 *   - Results depend only on (seed, global instance id, slot), never on the number
 *     of GPUs, the grid shape or the kernel choice.
 */
#ifndef TAPT_GPU_H
#define TAPT_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TAPT_OK = 0,
    TAPT_ERR_CONFIG = 1,            /* ConfigError          errors.hpp:13 */
    TAPT_ERR_DIMENSION = 2,         /* DimensionError       errors.hpp:17 */
    TAPT_ERR_CLAMPED_SITE = 3,      /* ClampedSiteError     errors.hpp:21 */
    TAPT_ERR_SIZE = 4,              /* SizeError            errors.hpp:25 */
    TAPT_ERR_GEOMETRY = 5,          /* GeometryError        errors.hpp:29 */
    TAPT_ERR_NUMERIC = 6,           /* NumericError         errors.hpp:33 */
    TAPT_ERR_FORMAT = 7,            /* FormatError          errors.hpp:37 */
    TAPT_ERR_TRAINING_DIVERGED = 8, /* TrainingDivergedError errors.hpp:41 */
    TAPT_ERR_CUDA = 9,
    TAPT_ERR_NCCL = 10,
    TAPT_ERR_INTERNAL = 11
} tapt_status;

typedef struct tapt_model_s* tapt_model_t;
typedef struct tapt_ensemble_s* tapt_ensemble_t;

/* Sweep orders. */
enum {
    TAPT_ORDER_COLOUR = 0,    /* colour classes (checkerboard / greedy colouring): the parallel chain */
    TAPT_ORDER_REFERENCE = 1  /* index-ascending, bit-exact with the reference gibbs_sweep (mcmc.cpp:34) */
};

enum { TAPT_BOUNDARY_OPEN = 0, TAPT_BOUNDARY_PERIODIC = 1 };

const char* tapt_last_error(void);
const char* tapt_version(void);
/* Number of CUDA devices visible (0 without a GPU); never fails. */
int tapt_device_count(void);
/* Make `device` the current device of this library's CUDA runtime on the calling thread (one process
 * per GPU: call it once per rank; handles live on the device current at their creation). */
tapt_status tapt_set_device(int device);
/* Kernels this library has launched so far (benchmark evidence); never fails. */
unsigned long long tapt_launch_count(void);
/* Measured ceiling of the per-update ALU work (one splitmix64 draw + threshold lookup +
 * compare + bit insert, no stencil, no memory traffic), in decisions per second. */
tapt_status tapt_probe_decision_rate(int blocks_per_sm, int threads, uint32_t iters, double* decisions_per_s,
                                     double* seconds);

/* ----------------------------------------------------------------- models -- */

/* LatticeSpec::grid2d(ly, lx, J, boundary) for dim == 2 (lz ignored),
 * LatticeSpec::grid3d(l = lx, J, boundary) for dim == 3.  Any double J, as the reference:
 * integer-valued couplings take the exact-table kernels (K1-K4), real-valued ones K5 (see below). */
tapt_status tapt_model_create_lattice(int dim, int ly, int lx, int lz, double J, int boundary, tapt_model_t* out);

/* CouplingGraph::Builder: n spins, n_couplings (i, j, J) triples (duplicates summed,
 * i != j), per-spin fields h (nullable), clamp values (nullable; 0 free, +-1 clamped).
 * Any double J and h, as CouplingGraph::Builder (spin_model.cpp:18-24).  Integer-valued couplings
 * (|J| <= 127) and fields run on the exact-table kernels K1-K4.  Real-valued ones run on K5: FP64 local
 * fields in the reference's order, device exp, and every decision whose draw falls within a relative
 * 1e-12 of the probability (a near tie) re-evaluated with the host's glibc exp -- with a state replay
 * if the device's provisional decision differed -- so results stay bit-identical to the reference.
 * Such ensembles report energies and observables as doubles (the *_f64 getters). */
tapt_status tapt_model_create_graph(uint32_t n, uint32_t n_couplings, const uint32_t* ci, const uint32_t* cj,
                                    const double* J, const double* h, const int8_t* clamp, tapt_model_t* out);
tapt_status tapt_model_destroy(tapt_model_t m);
/* CouplingGraph::load_file / save_file: the `isingmodel v1` text format (spin_model.cpp:123-226);
 * parse errors -> TAPT_ERR_FORMAT, invalid records -> TAPT_ERR_CONFIG, as the reference throws. */
tapt_status tapt_model_load_file(const char* path, tapt_model_t* out);
tapt_status tapt_model_save_file(tapt_model_t m, const char* path);
tapt_status tapt_model_info(tapt_model_t m, uint32_t* n_spins, uint32_t* n_free, uint32_t* n_couplings,
                            int32_t* lmin, int32_t* lmax, uint32_t* n_colours, uint32_t* n_levels);
/* Couplings after merging/sorting (CouplingGraph::couplings(), spin_model.hpp:57). */
tapt_status tapt_model_couplings(tapt_model_t m, uint32_t* ci, uint32_t* cj, double* J);
/* Greedy colour of each site (clamped: -1) and dependency level (index-order schedule). */
tapt_status tapt_model_schedule(tapt_model_t m, int32_t* colour, int32_t* level);
/* FNV-1a content digest identical to CouplingGraph::digest() (spin_model.cpp:68-75). */
tapt_status tapt_model_digest(tapt_model_t m, uint64_t* digest);

/* Host-side energy of one configuration (spin_model.cpp:79-89), for API parity. */
tapt_status tapt_model_energy(tapt_model_t m, const int8_t* s, size_t len, double* out);

/* -------------------------------------------------------- drop-in sweeps -- */

/* gibbs_update(g, s, i, beta, rng) (mcmc.cpp:24-28) on the device: s[i] <- heat-bath draw with the
 * stream's next draw; *rng_state advances by one draw.  Clamped i -> TAPT_ERR_CLAMPED_SITE,
 * len != n_spins -> TAPT_ERR_DIMENSION, as the reference throws. */
tapt_status tapt_gibbs_update(tapt_model_t m, int8_t* s, size_t len, uint32_t site, double beta, uint64_t* rng_state);

/* gibbs_sweep(g, s, beta, rng) on the device: updates s (host, n_spins entries) in
 * place with n_sweeps consecutive index-ascending heat-bath sweeps starting at
 * stream state *rng_state, advances *rng_state by n_sweeps*n_free draws and
 * writes each sweep's energy change to dE (nullable).  Bit-exact with the
 * reference for integer couplings. */
tapt_status tapt_gibbs_sweep(tapt_model_t m, int8_t* s, size_t len, double beta, uint64_t* rng_state,
                             uint32_t n_sweeps, double* dE);

/* ------------------------------------------------------------- ensembles -- */

typedef struct {
    uint32_t n_instances;     /* instances on this device                              */
    uint64_t instance_offset; /* global id of the first local instance (sharding)      */
    uint32_t n_slots;         /* R: ladder length (1..256)                              */
    const double* betas;      /* R values, strictly increasing, >= 0      */
    uint64_t seed;            /* root seed of every stream        */
    int order;                /* TAPT_ORDER_COLOUR or TAPT_ORDER_REFERENCE              */
} tapt_ensemble_desc;

tapt_status tapt_ensemble_create(tapt_model_t m, const tapt_ensemble_desc* d, tapt_ensemble_t* out);
tapt_status tapt_ensemble_destroy(tapt_ensemble_t e);
/* cudaStream_t to enqueue on (NULL: the handle's own non-blocking stream). */
tapt_status tapt_ensemble_set_stream(tapt_ensemble_t e, void* cuda_stream);
tapt_status tapt_ensemble_synchronize(tapt_ensemble_t e);
/* Kernel that serves sweeps of this ensemble: "lattice" (K1), "bitcsr" (K3), "levels" (K4) or "csr" (K2). */
const char* tapt_ensemble_kernel(tapt_ensemble_t e);
/* Distinct sweep-kernel instantiations this ensemble has launched, one per line, in first-launch
 * order ("k1_lattice_pt<3,1,1,2,512,1,1,0> balanced M=74" = template arguments, plus the persistent
 * grid's co-resident units when the balanced schedule ran).  Test evidence of which path ran. */
tapt_status tapt_ensemble_launch_log(tapt_ensemble_t e, char* buf, size_t cap);

/* Edwards-Anderson +-J disorder for lattice models, one sign per bond:
 * signs [n_instances][n_bonds] (+-1, bond order of LatticeSpec::graph), or generate
 * them on the device from (seed, global instance id). */
tapt_status tapt_ensemble_set_bond_signs(tapt_ensemble_t e, const int8_t* signs, size_t n_bonds);
tapt_status tapt_ensemble_generate_ea_disorder(tapt_ensemble_t e, uint64_t disorder_seed);
tapt_status tapt_ensemble_get_bond_signs(tapt_ensemble_t e, int8_t* signs, size_t n_bonds);
/* Per-instance clamp values [n_instances][n_spins] (only sites clamped in the model
 * may be non-zero; they override the model's clamp values). */
tapt_status tapt_ensemble_set_clamps(tapt_ensemble_t e, const int8_t* clamps);

/* random_configuration(g, derive(seed, {kInit, gid, slot})) for every slot. */
tapt_status tapt_ensemble_init_random(tapt_ensemble_t e);
tapt_status tapt_ensemble_set_spins(tapt_ensemble_t e, const int8_t* spins);
tapt_status tapt_ensemble_get_spins(tapt_ensemble_t e, int8_t* spins);
/* Same, bit-packed: [instance][slot][ceil(n/8)] bytes, LSB-first, +1 -> 1 (ISFD1 order, mcmc.cpp:86-90). */
tapt_status tapt_ensemble_get_spins_packed(tapt_ensemble_t e, uint8_t* packed);
tapt_status tapt_ensemble_get_energies(tapt_ensemble_t e, int64_t* E);      /* [I][R] by slot  */
tapt_status tapt_ensemble_get_permutation(tapt_ensemble_t e, uint8_t* buffer_of_slot); /* [I][R] */
tapt_status tapt_ensemble_counters(tapt_ensemble_t e, uint64_t* sweeps, uint64_t* passes, uint64_t* rounds);
/* [I][R-1] swap attempts / accepts by pair; [I][R] proposal attempts / accepts by slot (nullable). */
tapt_status tapt_get_acceptance(tapt_ensemble_t e, uint64_t* swap_att, uint64_t* swap_acc, uint64_t* prop_att,
                                uint64_t* prop_acc);

/* Observables: per (instance, slot): count, sum E, sum E^2, sum |M|, sum M^2 (M = sum of
 * all spins), accumulated at measurement points of tapt_run. */
tapt_status tapt_get_observables(tapt_ensemble_t e, int64_t* obs /* [I][R][5] */);
/* Energy histograms per slot summed over local instances: bins of `width` from e_lo. */
tapt_status tapt_set_histogram(tapt_ensemble_t e, int64_t e_lo, int64_t width, uint32_t nbins);
/* dst: [R][nbins] uint64, host (dst_on_device = 0) or device pointer. */
tapt_status tapt_get_histogram(tapt_ensemble_t e, uint64_t* dst, int dst_on_device);
tapt_status tapt_get_best(tapt_ensemble_t e, int64_t* best /* [I] */);
tapt_status tapt_reset_observables(tapt_ensemble_t e);

/* Replace the ladder values (thresholds re-tabulated); allow_flat = 1 permits equal neighbours
 * (annealing stages), 2 any order (independent chains, e.g. a training corpus); swaps must then
 * stay disabled. */
tapt_status tapt_ensemble_set_betas(tapt_ensemble_t e, const double* betas, int allow_flat);
/* Override the per-slot dynamics stream states [I][R] (e.g. run_chain's derive(seed,{kChain})). */
tapt_status tapt_ensemble_set_streams(tapt_ensemble_t e, const uint64_t* states);
/* random_configuration of every slot from the given init stream states [I][R]. */
tapt_status tapt_ensemble_init_from_streams(tapt_ensemble_t e, const uint64_t* init_states);

/* n_sweeps sweeps of every slot, no swaps (Alg. 1 lines 21-25). */
tapt_status tapt_sweep(tapt_ensemble_t e, uint32_t n_sweeps);
/* One swap pass over pairs (r, r+1), r = parity, parity+2, ... (Eq. 1). */
tapt_status tapt_swap_pass(tapt_ensemble_t e, int parity);

typedef struct {
    uint32_t n_sweeps;      /* sweeps to run                                           */
    uint32_t swap_every;    /* swap pass after every k-th global sweep (0: none);
                               parity alternates with the global pass counter        */
    uint32_t measure_every; /* accumulate observables every k-th global sweep (0: none) */
    uint64_t measure_from;  /* ... only once the global sweep count exceeds this       */
} tapt_schedule;

/* Fused PT loop (run_pt inner loop): per global sweep T: sweep all slots; swap pass
 * if swap_every | T; measure if due.  Runs device-resident with no host round trips. */
tapt_status tapt_run(tapt_ensemble_t e, const tapt_schedule* s);

/* Proposal injection (generator_move, Eq. 2).  proposals: [I][n_targets][n_spins] int8
 * for slots targets[0..n_targets) (host pointer, or device pointer if on_device).
 * Clamped sites are forced to their clamp values.  Round q uses accept draw slot+1 of
 * derive(seed, {kCoordinator, gid, q+1}).  log_q_cur / log_q_prop ([I][n_targets],
 * nullable): MH-corrected acceptance.  accepted: [I][n_targets]
 * (nullable). */
tapt_status tapt_inject_proposals(tapt_ensemble_t e, const int8_t* proposals, int on_device, const uint32_t* targets,
                                  uint32_t n_targets, const double* log_q_cur, const double* log_q_prop,
                                  uint8_t* accepted);
/* Same, bit-packed proposals [I][n_targets][ceil(n/8)] (ISFD1 bit order). */
tapt_status tapt_inject_proposals_packed(tapt_ensemble_t e, const uint8_t* proposals, int on_device,
                                         const uint32_t* targets, uint32_t n_targets, uint8_t* accepted);
/* Same, with `refine` heat-bath sweeps of each proposal at its target slot's beta before Eq. 2
 * (BASELINE.json configs[4]: "i.i.d. +-1 spins, then 5 Gibbs sweeps at the target beta").  The
 * refinement of slot r in round q draws from derive(seed, {kReplica, gid, r, q+1}) starting at
 * draw n+2, exactly as tapt_generate_proposals does after its own n+1 generator draws, so
 * host-generated proposals equal to the synthetic generator's give identical results. */
tapt_status tapt_inject_proposals_packed_refined(tapt_ensemble_t e, const uint8_t* proposals, int on_device,
                                                 const uint32_t* targets, uint32_t n_targets, uint32_t refine,
                                                 uint8_t* accepted);

/* Synthetic stand-in generator + Eq. 2 in one call (BASELINE configs 2 and 5): for each
 * target slot r, i.i.d. spins with P(+1) = (1 + sign*m_bias[r])/2 (sign: coin), clamps,
 * then `refine` sweeps at beta_r, then Metropolis acceptance.  m_bias: [n_targets]
 * (nullable = fair coin). */
tapt_status tapt_generate_proposals(tapt_ensemble_t e, const uint32_t* targets, uint32_t n_targets,
                                    const double* m_bias, uint32_t refine, uint8_t* accepted);

/* ------------------------------------------------------- real couplings -- */
/* Energies by slot [I][R] as doubles (every model; required for real-valued couplings, where
 * tapt_ensemble_get_energies returns TAPT_ERR_NUMERIC). */
tapt_status tapt_ensemble_get_energies_f64(tapt_ensemble_t e, double* out);
/* Observables [I][R][5] (count, sum E, sum E^2, sum |M|, sum M^2) and best energies [I] as doubles. */
tapt_status tapt_get_observables_f64(tapt_ensemble_t e, double* obs);
tapt_status tapt_get_best_f64(tapt_ensemble_t e, double* best);
/* Near-tie decisions K5 re-evaluated with glibc exp so far, and the state replays they caused. */
tapt_status tapt_ensemble_near_ties(tapt_ensemble_t e, uint64_t* ties, uint64_t* replays);

/* ------------------------------------------------------------ multi-GPU -- */
/* One process per GPU; rank g owns a contiguous block of global instance ids (instance_offset), so a
 * sharded run equals the single-GPU run instance by instance.  Replicas never span GPUs: the only
 * collectives are these end-of-run reductions over NCCL (SPEC.md:472-473 concurrency contract,
 * proj/include/tapt/threading.hpp:14-35 parallel_for over instances).  NCCL is loaded at run time;
 * its failures return TAPT_ERR_NCCL.  comm is an ncclComm_t (created here or by the caller). */
tapt_status tapt_nccl_unique_id(uint8_t* id, size_t len); /* rank 0 creates, broadcasts 128 bytes */
tapt_status tapt_nccl_comm_create(const uint8_t* id, int n_ranks, int rank, void** comm);
tapt_status tapt_nccl_comm_destroy(void* comm);
tapt_status tapt_nccl_comm_size(void* comm, int* n_ranks);
/* All-reduce over the communicator (every rank receives the result; each nullable):
 *   obs  [R][5]      per-slot count, sum E, sum E^2, sum |M|, sum M^2 over all ranks' instances
 *   hist [R][nbins]  per-slot energy histograms summed over ranks (the ensemble's own stays local)
 *   best [1]         lowest energy seen by any instance on any rank
 * Integer-coupling ensembles. */
tapt_status tapt_allreduce_observables(tapt_ensemble_t e, void* comm, int64_t* obs, uint64_t* hist, int64_t* best);
/* Per-instance best energies of all ranks in global instance order, out[total] (ncclAllGather of each
 * rank's (instance_offset, count) and of its best energies padded to the largest shard). */
tapt_status tapt_allgather_best(tapt_ensemble_t e, void* comm, uint64_t total, int64_t* out);

/* ------------------------------------------------------ problem suite -- */
/* Instance construction for BASELINE config 4 (proj/src/problems.cpp:1 is a
 * placeholder).  Host-only, never on the timed path.  Spin +1 = logical 1. */

const char* tapt_problem_last_error(void);
/* 3n^2 + n. */
uint32_t tapt_multiplier_spins(uint32_t n);
/* build_multiplier(n): AND gates + n-1 ripple rows of full adders with spin identification.
 * Outputs the un-merged coupling list (3n^2 + 10n(n-1) entries; CouplingGraph::Builder sums
 * shared wire pairs), fields [3n^2+n], the clamp set (product bits and carry-ins, values for
 * C = 0) and wires (nullable): A[n], B[n], C[2n], carry-in[n]. */
tapt_status tapt_multiplier_build(uint32_t n, uint32_t* n_couplings, uint32_t* ci, uint32_t* cj, double* J,
                                  double* h, int8_t* clamp, uint32_t* wires);
/* Consistent wire assignment for inputs (a, b) (forward evaluation). */
tapt_status tapt_multiplier_forward(uint32_t n, uint64_t a, uint64_t b, int8_t* spins);
/* clamp_product: clamp values for product C ([3n^2+n], 0 = free). */
tapt_status tapt_multiplier_clamps(uint32_t n, uint64_t C, int8_t* clamp);
/* decode_and_check. */
tapt_status tapt_multiplier_decode(uint32_t n, const int8_t* spins, uint64_t C, uint64_t* a, uint64_t* b,
                                   int* success);
/* enumerate_semiprimes. */
tapt_status tapt_enumerate_semiprimes(uint32_t n, uint64_t* out, uint32_t cap, uint32_t* count);
/* p, q: first primes among 2^(bits-1) + below(2^(bits-1)) draws of derive(seed, {0x99, gid}). */
tapt_status tapt_random_semiprime(uint64_t seed, uint64_t gid, uint32_t bits, uint64_t* p, uint64_t* q);

/* ------------------------------------------------ IsingFormer generator -- */
/* Decoder-only autoregressive proposal model over spin tokens conditioned on beta
 * (Appendix F), inference on the device.  Token 1 = spin +1.
 * Architecture and the SPEC's open choices are fixed in DESIGN.md section 10 (pre-LN blocks,
 * sinusoidal positions, sinusoidal beta features + linear map added at every position, GELU
 * (tanh), one Bernoulli logit per position).  Parameters are fp32 in the canonical ISFW1
 * order.  The device kernels support d_model = 64 with 32-wide heads and ffn = 128 (the
 * SPEC default); layers, beta_features and max_len are free. */
typedef struct tapt_former_s* tapt_former_t;

typedef struct {
    uint32_t d_model;       /* 64 */
    uint32_t heads;         /* 2 */
    uint32_t ffn;           /* 128 */
    uint32_t layers;        /* 2 */
    uint32_t max_len;       /* longest token sequence */
    uint32_t beta_features; /* even, sin/cos pairs */
} tapt_former_config;

/* Number of fp32 parameters of a configuration (68 353 at the SPEC default). */
size_t tapt_former_param_count(const tapt_former_config* c);
/* Seeded initialisation (host): matrices N(0, scale^2 / fan_in) from derive(seed, {0x77}),
 * biases 0, LayerNorm gains 1.  params: [tapt_former_param_count]. */
tapt_status tapt_former_init_params(const tapt_former_config* c, uint64_t seed, double scale, float* params);
tapt_status tapt_former_create(const tapt_former_config* c, const float* params, tapt_former_t* out);
tapt_status tapt_former_destroy(tapt_former_t f);
tapt_status tapt_former_get(tapt_former_t f, tapt_former_config* c, float* params /* nullable */);
/* save/load_checkpoint: magic "ISFW1", u32 version (1), u32 config block (d_model, heads,
 * ffn, layers, max_len, beta_features), u32 parameter count, then little-endian fp32
 * parameters.  Bad magic / truncation -> TAPT_ERR_FORMAT. */
tapt_status tapt_former_save(tapt_former_t f, const char* path);
tapt_status tapt_former_load(const char* path, tapt_former_t* out);
/* K/V cache precision: 0 (default) fp32; 1 bf16 storage with fp32 attention math (half the bytes
 * of the sampling-bound K/V stream; logits then agree with the fp32 path to ~1e-2, and sampling
 * and log_prob stay mutually consistent).  No reference counterpart (the generator is a
 * placeholder there). */
tapt_status tapt_former_set_kv_bf16(tapt_former_t f, int bf16);
/* log_prob engine: 1 (default) the dense products (QKV, out-projection, FFN) on the 5th-generation
 * tensor cores -- tcgen05.mma with TMEM accumulators, operands split bf16 hi + lo ("bf16x3", fp32
 * accuracy); 0 the fp32 CUDA-core row engine.  Attention runs on CUDA cores in both. */
tapt_status tapt_former_set_tensor_cores(tapt_former_t f, int on);
/* forward_logits / log_prob: tokens [B][T] (0/1, host), betas [B]; log_q [B] sums the
 * Bernoulli log-probabilities of positions >= n_prefix; logits [B][T] (nullable). */
tapt_status tapt_former_log_prob(tapt_former_t f, const uint8_t* tokens, uint32_t B, uint32_t T, const double* betas,
                                 uint32_t n_prefix, double* log_q, float* logits);
/* sample: B sequences of T tokens; positions < n_prefix are forced to prefix[b][t]
 * (prefix [B][n_prefix], nullable when n_prefix = 0); position t >= n_prefix draws
 * u = (x >> 11) 2^-53 with x = draw t+1 of stream state streams[b] and takes token 1 iff
 * u < sigmoid(logit_t).  tokens [B][T] and log_q [B] out (host). */
tapt_status tapt_former_sample(tapt_former_t f, uint32_t B, uint32_t T, const double* betas, const uint8_t* prefix,
                               uint32_t n_prefix, const uint64_t* streams, uint8_t* tokens, double* log_q);

#ifdef __cplusplus
}
#endif
#endif /* TAPT_GPU_H */
