// engine.cu -- host driver of the B200 TAPT verifier and the C ABI of include/tapt_gpu.h.
//
// Responsibilities: build the device model (the reference's CouplingGraph semantics,
// spin_model.cpp:15-77, and LatticeSpec, lattice.cpp:55-87), turn every probability
// the reference evaluates with libm exp into an exact integer threshold table on the
// host (heat-bath: mcmc.cpp:13-15; swaps: Eq. 1; proposals: Eq. 2), derive the RNG
// stream states (rng.hpp:21-27), choose the kernel (K1 lattice / K2 CSR), and keep the
// global sweep / pass / round counters that address every random draw.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "kernels.h"
#include "real.h"
#include "tapt/spin_model.hpp"

#ifndef TAPT_K1_DEFAULT_THREADS
#define TAPT_K1_DEFAULT_THREADS 512
#endif
#include "tapt/errors.hpp"
#include "tapt/rng.hpp"
#include "tapt_gpu.h"

namespace tapt_dev {
cudaError_t launch_k1(const PTArgs& a, const LatDims& d, int threads, bool cluster, cudaStream_t st);
int k1_resident_units(const PTArgs& a, const LatDims& d, int threads, bool cluster);
void k1_variant_name(const PTArgs& a, const LatDims& d, int threads, bool cluster, char* out);
int k2_resident_units(const PTArgs& a, const CsrArgs& g, int threads, bool cluster);
struct Csr3 {
    const uint4* meta;
    const uint32_t* adj;
    const uint32_t* class_ptr;
    int n_classes;
    int nadj;
    int n2;
    int nidx4;
};
size_t k3_smem_bytes(int R, int nidx, int nadj, int nfree, int n, int ncls, int ipb);
int k3_row_stride();
// shape: instance teams per CTA (1..4), or -Q for split sites (Q = 2, 4 lanes per site, one team per CTA)
int k3_resident_units(const PTArgs& a, const Csr3& g, int shape);
cudaError_t launch_k3(const PTArgs& a, const Csr3& g, int shape, cudaStream_t st);
cudaError_t launch_k2(const PTArgs& a, const CsrArgs& g, int threads, bool cluster, cudaStream_t st);
size_t k4_smem_bytes(int n, int R, int nidx, int nnz, int nfree, int nlev, int ipb);
int k4_max_ipb();
int k4_resident_units(const PTArgs& a, const CsrArgs& g, int ipb);
cudaError_t launch_k4(const PTArgs& a, const CsrArgs& g, int ipb, cudaStream_t st);
size_t k1_smem_bytes(int n, bool dis, int R);
size_t k2_smem_bytes(int n, int R, int nidx);
size_t k2_smem_bytes_graph(int n, int R, int nidx, int nnz, int nfree);
cudaError_t launch_decision_probe(int blocks, int threads, uint32_t iters, uint32_t* sink, cudaStream_t st,
                                  int variant);
__global__ void k_init_random(uint32_t*, int, int, int, int, const uint64_t*, const int8_t*, int);
__global__ void k_energy_csr(const uint32_t*, int, int, int, int, const uint32_t*, const uint32_t*, const int8_t*, int,
                             int, const int32_t*, int32_t*);
__global__ void k_get_spins(const uint32_t*, int, int, int, int, const uint8_t*, int, int8_t*);
__global__ void k_get_packed(const uint32_t*, int, int, int, const uint8_t*, int, uint8_t*);
__global__ void k_set_spins(uint32_t*, int, int, int, int, const uint8_t*, const int8_t*, int, const int8_t*, int);
__global__ void k_set_packed(uint32_t*, int, int, int, int, const uint8_t*, int, const int8_t*, int);
__global__ void k_swap_pass(const int32_t*, uint8_t*, uint8_t*, int, const uint64_t*, uint64_t, int, MetroTable,
                            uint64_t*, uint64_t*);
__global__ void k_accept_proposals(int32_t*, const uint8_t*, int, const int32_t*, int, const uint32_t*,
                                   const uint64_t*, MetroTable, const uint8_t*, uint8_t*, uint64_t*, uint64_t*);
__global__ void k_decide_mh(const int32_t*, const uint8_t*, int, const int32_t*, int, const uint32_t*, const uint64_t*,
                            const double*, const double*, const double*, uint8_t*, uint32_t*);
__global__ void k_apply_proposals(uint32_t*, int, int, int, const uint8_t*, int, const uint32_t*, int, int,
                                  const uint32_t*, int, const uint8_t*);
__global__ void k_gen_proposals(uint32_t*, int, int, int, int, const uint64_t*, const uint64_t*, const int8_t*, int);
__global__ void k_ea_signs(int8_t*, int, int, const uint64_t*);
__global__ void k_derive_round_streams(uint64_t, uint64_t, const uint32_t*, int, int, uint64_t, uint64_t*, uint64_t*,
                                       uint64_t*);
__global__ void k_best_from_E(const int32_t*, int, int, int*);
__global__ void k_bond_bytes(const int8_t*, uint8_t*, LatDims, int);
__global__ void k_csr_from_signs(const int8_t*, int, const uint32_t*, int, int, int8_t*);
}  // namespace tapt_dev

using namespace tapt_dev;

namespace {

thread_local std::string g_last_error;
std::atomic<unsigned long long> g_launches{0};  // kernels launched by this library (bench evidence)

#define CUDA_OK(expr)                                                                                    \
    do {                                                                                                 \
        cudaError_t e_ = (expr);                                                                         \
        if (e_ != cudaSuccess) throw tapt::CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

template <class F>
tapt_status guard(F&& f) {
    try {
        f();
        return TAPT_OK;
    } catch (const tapt::ConfigError& e) {
        g_last_error = e.what();
        return TAPT_ERR_CONFIG;
    } catch (const tapt::DimensionError& e) {
        g_last_error = e.what();
        return TAPT_ERR_DIMENSION;
    } catch (const tapt::ClampedSiteError& e) {
        g_last_error = e.what();
        return TAPT_ERR_CLAMPED_SITE;
    } catch (const tapt::SizeError& e) {
        g_last_error = e.what();
        return TAPT_ERR_SIZE;
    } catch (const tapt::GeometryError& e) {
        g_last_error = e.what();
        return TAPT_ERR_GEOMETRY;
    } catch (const tapt::NumericError& e) {
        g_last_error = e.what();
        return TAPT_ERR_NUMERIC;
    } catch (const tapt::FormatError& e) {
        g_last_error = e.what();
        return TAPT_ERR_FORMAT;
    } catch (const tapt::CudaError& e) {
        g_last_error = e.what();
        return TAPT_ERR_CUDA;
    } catch (const tapt::NcclError& e) {
        g_last_error = e.what();
        return TAPT_ERR_NCCL;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return TAPT_ERR_INTERNAL;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return TAPT_ERR_INTERNAL;
    }
}

}  // namespace

// Hooks for the other translation units of the library (former.cu): shared last-error
// message and launch counter.
namespace tapt_host {
void set_last_error(const std::string& m) { g_last_error = m; }
void note_launches(unsigned n) { g_launches += n; }
}  // namespace tapt_host

namespace {

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t count) {
        if (count == n && p) return;
        release();
        if (count == 0) return;
        CUDA_OK(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void zero(cudaStream_t st) {
        if (p) CUDA_OK(cudaMemsetAsync(p, 0, n * sizeof(T), st));
    }
    void upload(const std::vector<T>& h, cudaStream_t st) {
        alloc(h.size());
        if (n) CUDA_OK(cudaMemcpyAsync(p, h.data(), n * sizeof(T), cudaMemcpyHostToDevice, st));
    }
    void upload(const T* h, size_t count, cudaStream_t st) {
        alloc(count);
        if (n) CUDA_OK(cudaMemcpyAsync(p, h, n * sizeof(T), cudaMemcpyHostToDevice, st));
    }
    std::vector<T> download(cudaStream_t st) const {
        std::vector<T> h(n);
        if (n) {
            CUDA_OK(cudaMemcpyAsync(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, st));
            CUDA_OK(cudaStreamSynchronize(st));
        }
        return h;
    }
};

bool is_integer(double v) { return std::isfinite(v) && std::nearbyint(v) == v && std::fabs(v) < 1e9; }

int ilog2_exact(int v) {
    if (v <= 0 || (v & (v - 1))) return -1;
    int k = 0;
    while ((1 << k) < v) ++k;
    return k;
}

// ceil(p * 2^53): uniform() < p  <=>  (x >> 11) < threshold  (uniform = (x>>11) 2^-53, rng.hpp:35)
uint64_t threshold_of(double p) {
    if (!(p > 0.0)) return 0;
    if (p >= 1.0) return 1ull << 53;
    return static_cast<uint64_t>(std::ceil(p * 9007199254740992.0));
}

// The reference heat-bath conditional, evaluated exactly as mcmc.cpp:13-15 does.
double conditional_up(double beta, double local) { return 1.0 / (1.0 + std::exp(-2.0 * beta * local)); }

uint64_t fnv1a(const void* data, size_t n, uint64_t h) {
    const unsigned char* c = static_cast<const unsigned char*>(data);
    for (size_t k = 0; k < n; ++k) {
        h ^= c[k];
        h *= 0x100000001B3ull;
    }
    return h;
}

// Host table for the Metropolis rule  accept iff uniform < exp(c * dE)  (dE integer <= 0).
struct HostMetro {
    bool oversize = false;
    std::vector<uint64_t> tab;
    std::vector<uint32_t> off, K;
    std::vector<int64_t> kz;
    std::vector<uint8_t> always;
    std::vector<double> coef;
    void add_row(double c) {
        coef.push_back(c > 0.0 ? c : 0.0);
        off.push_back(static_cast<uint32_t>(tab.size()));
        if (!(c > 0.0)) {  // c == 0: exp(0) = 1 > uniform always
            always.push_back(1);
            K.push_back(1);
            kz.push_back(-1);
            tab.push_back(1ull << 53);
            return;
        }
        uint32_t k = 0;
        for (;; ++k) {
            const double e = std::exp(c * -static_cast<double>(k));
            const uint64_t T = threshold_of(e);
            tab.push_back(T);
            if (T <= 1) break;
            if (tab.size() > (64u << 20)) {
                oversize = true;  // reported when a swap / proposal actually needs this table
                tab.resize(off.back());
                always.push_back(0);
                K.push_back(0);
                kz.push_back(-1);
                return;
            }
        }
        always.push_back(0);
        K.push_back(k + 1);
        // largest k with exp(-c k) > 0 (threshold 1 between K and kz, 0 beyond)
        int64_t lo = k, hi = int64_t(1) << 40;
        if (std::exp(c * -static_cast<double>(lo)) == 0.0) {
            kz.push_back(lo - 1);
            return;
        }
        while (hi - lo > 1) {
            const int64_t mid = lo + (hi - lo) / 2;
            if (std::exp(c * -static_cast<double>(mid)) > 0.0)
                lo = mid;
            else
                hi = mid;
        }
        kz.push_back(lo);
    }
};

struct DevMetro {
    DevBuf<uint64_t> tab;
    DevBuf<uint32_t> off, K;
    DevBuf<int64_t> kz;
    DevBuf<uint8_t> always;
    DevBuf<double> coef;
    void upload(const HostMetro& h, cudaStream_t st) {
        coef.upload(h.coef, st);
        tab.upload(h.tab, st);
        off.upload(h.off, st);
        K.upload(h.K, st);
        kz.upload(h.kz, st);
        always.upload(h.always, st);
    }
    MetroTable view() const { return MetroTable{tab.p, off.p, K.p, kz.p, always.p, coef.p}; }
};

}  // namespace

// =================================================================== model ===

struct tapt_model_s {
    // single-replica ensemble reused by the drop-in tapt_gibbs_sweep (created lazily)
    tapt_ensemble_t dropin = nullptr;
    std::mutex dropin_mu;
    // real-valued couplings or fields (or |J| > 127): every ensemble of the model runs on K5 (real.h)
    bool real = false;
    std::vector<double> Jcsr;  // merged coupling value of every CSR entry
    // single-replica K5 engine of the drop-in gibbs_sweep (per-sweep dE) / gibbs_update (created lazily)
    std::unique_ptr<tapt_real::RealEngine> dropin_real;
    cudaStream_t dropin_stream = nullptr;

    tapt_real::RealGraph real_graph() const {
        tapt_real::RealGraph g;
        g.n = n;
        g.rowptr = rowptr;
        g.col = col;
        g.ci = ci;
        g.cj = cj;
        g.free_sites = free_sites;
        g.rank = rank;
        g.J = Jcsr;
        g.h = h;
        g.cJ = J;
        g.clamp = clamp;
        g.colour_order = col_sites;
        g.integral = !real;
        g.lmin = lmin;
        g.lmax = lmax;
        return g;
    }
    ~tapt_model_s();
    uint32_t n = 0;
    std::vector<uint32_t> ci, cj;  // merged, sorted (i<j)
    std::vector<double> J;
    std::vector<uint32_t> bond_of;  // per merged coupling: index in the add order (lattices)
    std::vector<double> h;
    std::vector<int8_t> clamp;
    std::vector<uint32_t> rowptr, col, adj_bond;
    std::vector<int8_t> adjJ;
    std::vector<int32_t> hi;
    std::vector<uint32_t> free_sites, rank;
    std::vector<int32_t> colour, level;
    std::vector<uint32_t> col_ptr, col_sites, lev_ptr, lev_sites;
    int lmin = 0, lmax = 0, max_sumabs = 0;
    uint64_t digest = 0;
    // lattice
    bool lattice = false, k1 = false;
    int dim = 0, ly = 0, lx = 0, lz = 0, boundary = 0, J0 = 0, Jsign = 1;
    uint32_t nbonds = 0;
    LatDims ld{};
    // device copies
    bool on_device = false;
    DevBuf<uint32_t> d_rowptr, d_col, d_rank, d_colptr, d_colsites, d_levptr, d_levsites, d_adjbond;
    DevBuf<int8_t> d_J, d_clamp;
    DevBuf<int32_t> d_h, d_hs;
    // K3 (bit-sliced CSR, colour order; k3_bitcsr.cu): unit-weight padded adjacency (byte offsets
    // into the instance word image [w | ~w | ONES | ZEROS]) and per-position site metadata, class
    // positions sorted by (chunks desc, threshold offset, site); built on first use (build_k3)
    int k3_state = 0;  // 0 unbuilt, 1 eligible, -1 not eligible
    int k3_nadj = 0, k3_max_per_thread = 0;
    DevBuf<uint32_t> d_adj3;
    DevBuf<uint4> d_meta3;

    void build_k3(cudaStream_t st) {
        if (k3_state) return;
        k3_state = -1;
        const uint32_t nf = (uint32_t)free_sites.size();
        if (nf == 0 || (size_t)(2 * n + 2) * 4 >= (1u << 31)) return;
        // Rows with S' <= 15 ("light"): unit entries (a coupling |J| times, a field |h| times, zeros
        // padding) in one 16-entry chunk, counted into 4 planes.  Heavier rows: the field is the constant
        // hc = max(h, 0) (its entries would all read ONES or ZEROS), and each coupling is split into
        // |J| = 2q + r: q entries in weight-2 chunks (their count enters one plane up) and r in weight-1
        // chunks, counted into 7 planes.  Multiplier inputs (16 x J=1, 16 x J=2, h=16): 2 chunks, not 4.
        std::vector<int> nch_of(n, 0), off_of(n, 0), sp_of(n, 0), key_of(n, 0);
        std::vector<std::vector<uint32_t>> rows_of(n);
        std::vector<uint32_t> w2_of(n, 0), hc_of(n, 0);
        const uint32_t ONES = 2 * n, ZEROS = 2 * n + 1;
        if (nf >= (1u << 24)) return;
        for (uint32_t i = 0; i < n; ++i) {
            if (clamp[i]) continue;
            int sp = std::abs(hi[i]);
            for (uint32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) sp += std::abs((int)adjJ[k]);
            if (sp > 127) return;
            sp_of[i] = sp;
            off_of[i] = -sp - lmin;
            auto& e = rows_of[i];
            if (sp <= 15) {
                for (uint32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
                    const int Jk = adjJ[k];
                    for (int r = 0; r < std::abs(Jk); ++r) e.push_back(4u * (Jk > 0 ? col[k] : n + col[k]));
                }
                for (int r = 0; r < std::abs(hi[i]); ++r) e.push_back(4u * (hi[i] > 0 ? ONES : ZEROS));
                while (e.size() < 16) e.push_back(4u * ZEROS);
                nch_of[i] = 1;
                key_of[i] = 1;
                continue;
            }
            std::vector<uint32_t> l1, l2;
            for (uint32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
                const int Jk = adjJ[k];
                const uint32_t ent = 4u * (Jk > 0 ? col[k] : n + col[k]);
                for (int r = 0; r < std::abs(Jk) / 2; ++r) l2.push_back(ent);
                if (std::abs(Jk) & 1) l1.push_back(ent);
            }
            const int c1 = (int)((l1.size() + 15) / 16), c2 = (int)((l2.size() + 15) / 16);
            if (c1 + c2 <= 4) {
                e = l1;
                e.resize(16 * (size_t)c1, 4u * ZEROS);
                e.insert(e.end(), l2.begin(), l2.end());
                e.resize(16 * (size_t)(c1 + c2), 4u * ZEROS);
                nch_of[i] = c1 + c2;
                for (int ch = c1; ch < c1 + c2; ++ch) w2_of[i] |= 1u << ch;
            } else {  // unit weights
                for (uint32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
                    const int Jk = adjJ[k];
                    for (int r = 0; r < std::abs(Jk); ++r) e.push_back(4u * (Jk > 0 ? col[k] : n + col[k]));
                }
                nch_of[i] = (int)((e.size() + 15) / 16);
                e.resize(16 * (size_t)nch_of[i], 4u * ZEROS);
            }
            hc_of[i] = hi[i] > 0 ? (uint32_t)hi[i] : 0u;
            key_of[i] = 16 + nch_of[i];  // heavy rows first, then by chunk count
        }
        std::vector<uint32_t> adj;
        std::vector<uint4> meta;
        int per_thread = 0;
        for (size_t c = 0; c + 1 < col_ptr.size(); ++c) {
            std::vector<uint32_t> v(col_sites.begin() + col_ptr[c], col_sites.begin() + col_ptr[c + 1]);
            std::stable_sort(v.begin(), v.end(), [&](uint32_t x, uint32_t y) {
                if (key_of[x] != key_of[y]) return key_of[x] > key_of[y];
                if (off_of[x] != off_of[y]) return off_of[x] < off_of[y];
                return x < y;
            });
            per_thread += (int)((v.size() + 127) / 128);
            for (uint32_t i : v) {
                const size_t start = adj.size();
                adj.insert(adj.end(), rows_of[i].begin(), rows_of[i].end());
                if (off_of[i] + 32768 < 0 || off_of[i] + 32768 > 0xFFFF) return;
                // x: site; y: rank | hc << 24; z: first entry; w: off+32768 | nch << 16 | S' << 20 |
                // heavy << 27 | weight-2 chunk flags << 28
                meta.push_back(make_uint4(i, rank[i] | (hc_of[i] << 24), (uint32_t)start,
                                          (uint32_t)(off_of[i] + 32768) | ((uint32_t)nch_of[i] << 16) |
                                              ((uint32_t)sp_of[i] << 20) | ((uint32_t)(sp_of[i] > 15) << 27) |
                                              (w2_of[i] << 28)));
            }
        }
        // Bank-aware entry order.  A warp gathers entry k of 32 rows (32 lanes = 32 consecutive class
        // positions) in one LDS per k; lanes reading different words of one bank serialise.  Each row's
        // entries are a multiset that the carry-save count sums in any order, so per warp, chunk and
        // entry column a greedy pick (most-constrained lane first) takes a word already chosen in the
        // column (broadcast) or one in an unused bank.  Config 4: 1616 -> 886 wavefronts per sweep for
        // 576 gathers; the counts, and so every result, are unchanged.
        if (std::getenv("TAPT_K3_BANKS") == nullptr || std::atoi(std::getenv("TAPT_K3_BANKS")) != 0) {
            for (size_t c = 0; c + 1 < col_ptr.size(); ++c) {
                const uint32_t p0 = col_ptr[c], p1 = col_ptr[c + 1];
                for (uint32_t w0 = p0; w0 < p1; w0 += 32) {
                    const uint32_t w1 = std::min(p1, w0 + 32);
                    int maxch = 0;
                    for (uint32_t q = w0; q < w1; ++q) maxch = std::max(maxch, (int)((meta[q].w >> 16) & 15u));
                    for (int ch = 0; ch < maxch; ++ch) {
                        std::vector<uint32_t> lanes;
                        for (uint32_t q = w0; q < w1; ++q)
                            if ((int)((meta[q].w >> 16) & 15u) > ch) lanes.push_back(q);
                        std::vector<std::vector<uint32_t>> rem(lanes.size()), out(lanes.size());
                        for (size_t l = 0; l < lanes.size(); ++l) {
                            const uint32_t st = meta[lanes[l]].z + 16u * ch;
                            rem[l].assign(adj.begin() + st, adj.begin() + st + 16);
                        }
                        for (int k = 0; k < 16; ++k) {
                            std::vector<size_t> order(lanes.size());
                            std::iota(order.begin(), order.end(), 0);
                            auto distinct = [](const std::vector<uint32_t>& v) {
                                std::vector<uint32_t> u(v);
                                std::sort(u.begin(), u.end());
                                return (size_t)(std::unique(u.begin(), u.end()) - u.begin());
                            };
                            std::vector<size_t> nd(lanes.size());
                            for (size_t l = 0; l < lanes.size(); ++l) nd[l] = distinct(rem[l]);
                            std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) { return nd[x] < nd[y]; });
                            std::vector<std::vector<uint32_t>> bank(32);
                            for (size_t l : order) {
                                size_t bi = 0;
                                int bc0 = 1 << 30, bc1 = 0;
                                for (size_t e = 0; e < rem[l].size(); ++e) {
                                    const uint32_t wd = rem[l][e] / 4;
                                    const auto& bk = bank[wd % 32];
                                    const bool shared = std::find(bk.begin(), bk.end(), wd) != bk.end();
                                    const int c0 = shared ? 0 : (int)bk.size();
                                    const int c1 = (int)std::count(rem[l].begin(), rem[l].end(), rem[l][e]);
                                    if (c0 < bc0 || (c0 == bc0 && c1 > bc1)) {
                                        bi = e;
                                        bc0 = c0;
                                        bc1 = c1;
                                    }
                                }
                                const uint32_t pick = rem[l][bi];
                                rem[l].erase(rem[l].begin() + bi);
                                out[l].push_back(pick);
                                auto& bk = bank[(pick / 4) % 32];
                                if (std::find(bk.begin(), bk.end(), pick / 4) == bk.end()) bk.push_back(pick / 4);
                            }
                        }
                        for (size_t l = 0; l < lanes.size(); ++l)
                            std::copy(out[l].begin(), out[l].end(), adj.begin() + meta[lanes[l]].z + 16u * ch);
                    }
                }
            }
        }
        k3_nadj = (int)adj.size();
        k3_max_per_thread = per_thread;
        d_adj3.upload(adj, st);
        d_meta3.upload(meta, st);
        CUDA_OK(cudaStreamSynchronize(st));  // shared by every ensemble of the model, on any stream
        k3_state = 1;
    }

    void ensure_device(cudaStream_t st) {
        if (on_device) return;
        d_rowptr.upload(rowptr, st);
        d_col.upload(col, st);
        d_rank.upload(rank, st);
        d_colptr.upload(col_ptr, st);
        d_colsites.upload(col_sites, st);
        d_levptr.upload(lev_ptr, st);
        d_levsites.upload(lev_sites, st);
        d_adjbond.upload(adj_bond, st);
        d_J.upload(adjJ, st);
        d_clamp.upload(clamp, st);
        d_h.upload(hi, st);
        {  // h_i - sum_k |J_ik|: the local field of the all-down neighbourhood (K2 adds 2*acc)
            std::vector<int32_t> hs(hi);
            for (size_t i = 0; i + 1 < rowptr.size(); ++i)
                for (uint32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) hs[i] -= std::abs((int)adjJ[k]);
            d_hs.upload(hs, st);
        }
        CUDA_OK(cudaStreamSynchronize(st));
        on_device = true;
    }
};

namespace {

// CouplingGraph::Builder::build semantics (spin_model.cpp:15-77) plus the schedules.
void build_model(tapt_model_s& m, uint32_t n, const std::vector<uint32_t>& ai, const std::vector<uint32_t>& aj,
                 const std::vector<double>& aJ, const double* h, const int8_t* clamp) {
    m.n = n;
    std::map<std::pair<uint32_t, uint32_t>, std::pair<double, uint32_t>> merged;
    for (size_t k = 0; k < ai.size(); ++k) {
        uint32_t i = ai[k], j = aj[k];
        if (i == j) throw tapt::ConfigError("self-coupling on spin " + std::to_string(i));
        if (i >= n || j >= n) throw tapt::ConfigError("coupling index out of range");
        if (i > j) std::swap(i, j);
        auto it = merged.find({i, j});
        if (it == merged.end())
            merged.emplace(std::make_pair(i, j), std::make_pair(aJ[k], static_cast<uint32_t>(k)));
        else
            it->second.first += aJ[k];
    }
    m.h.assign(n, 0.0);
    m.clamp.assign(n, 0);
    for (uint32_t i = 0; i < n; ++i) {
        if (h) m.h[i] = h[i];
        if (clamp && clamp[i]) {
            if (clamp[i] != 1 && clamp[i] != -1) throw tapt::ConfigError("clamp value must be ±1");
            m.clamp[i] = clamp[i];
        }
    }
    for (const auto& [key, v] : merged) {
        m.ci.push_back(key.first);
        m.cj.push_back(key.second);
        m.J.push_back(v.first);
        m.bond_of.push_back(v.second);
    }
    // digest: FNV-1a over (n, couplings {u32,u32,f64}, fields, clamps) as spin_model.cpp:68-75
    {
        uint64_t d = fnv1a(&m.n, 0, 0xCBF29CE484222325ull);
        const uint64_t n64 = n;
        d = fnv1a(&n64, sizeof(n64), 0xCBF29CE484222325ull);
        struct Rec {
            uint32_t i, j;
            double v;
        };
        static_assert(sizeof(Rec) == 16, "layout");
        for (size_t k = 0; k < m.ci.size(); ++k) {
            Rec r{m.ci[k], m.cj[k], m.J[k]};
            d = fnv1a(&r, sizeof(r), d);
        }
        if (n) d = fnv1a(m.h.data(), n * sizeof(double), d);
        if (n) d = fnv1a(m.clamp.data(), n, d);
        m.digest = d;
    }
    // CSR, neighbours ascending (spin_model.cpp:52-63 yields this order)
    std::vector<std::vector<std::pair<uint32_t, size_t>>> adj(n);
    for (size_t k = 0; k < m.ci.size(); ++k) {
        adj[m.ci[k]].push_back({m.cj[k], k});
        adj[m.cj[k]].push_back({m.ci[k], k});
    }
    m.rowptr.assign(n + 1, 0);
    m.hi.assign(n, 0);
    bool integral = true;
    for (uint32_t i = 0; i < n; ++i) {
        std::sort(adj[i].begin(), adj[i].end());
        m.rowptr[i + 1] = m.rowptr[i] + static_cast<uint32_t>(adj[i].size());
        for (auto& [j, k] : adj[i]) {
            m.col.push_back(j);
            const double v = m.J[k];
            m.Jcsr.push_back(v);
            if (!is_integer(v) || std::fabs(v) > 127) integral = false;
            m.adjJ.push_back(static_cast<int8_t>(integral ? v : 0));
            m.adj_bond.push_back(m.bond_of[k]);
        }
        if (!is_integer(m.h[i])) integral = false;
        m.hi[i] = integral ? static_cast<int32_t>(m.h[i]) : 0;
    }
    // Real-valued (or large) couplings and fields: no exact threshold tables exist; such models run on
    // K5 (real.h: FP64 fields in the reference's order, device exp with near ties resolved by glibc).
    m.real = !integral;
    if (m.real) {
        std::fill(m.adjJ.begin(), m.adjJ.end(), (int8_t)0);
        std::fill(m.hi.begin(), m.hi.end(), 0);
    }
    for (uint32_t i = 0; i < n; ++i)
        if (!m.clamp[i]) m.free_sites.push_back(i);
    m.rank.assign(n, 0);
    for (uint32_t q = 0; q < m.free_sites.size(); ++q) m.rank[m.free_sites[q]] = q;
    // local-field range over free sites; byte-SWAR capacity check is done when K2 is chosen
    m.lmin = 0;
    m.lmax = 0;
    bool first = true;
    for (uint32_t i : m.free_sites) {
        int sa = 0;
        for (uint32_t k = m.rowptr[i]; k < m.rowptr[i + 1]; ++k) sa += std::abs((int)m.adjJ[k]);
        m.max_sumabs = std::max(m.max_sumabs, sa);
        const int lo = m.hi[i] - sa, hi = m.hi[i] + sa;
        if (first || lo < m.lmin) m.lmin = lo;
        if (first || hi > m.lmax) m.lmax = hi;
        first = false;
    }
    // greedy colouring (ascending order) and dependency levels of the index order
    m.colour.assign(n, -1);
    m.level.assign(n, -1);
    int ncol = 0, nlev = 0;
    std::vector<int> mark;
    for (uint32_t i : m.free_sites) {
        mark.assign(ncol + 2, 0);
        int lv = 0;
        for (uint32_t k = m.rowptr[i]; k < m.rowptr[i + 1]; ++k) {
            const uint32_t j = m.col[k];
            if (m.colour[j] >= 0) mark[m.colour[j]] = 1;
            if (j < i && m.level[j] >= 0) lv = std::max(lv, m.level[j] + 1);
        }
        int c = 0;
        while (mark[c]) ++c;
        m.colour[i] = c;
        m.level[i] = lv;
        ncol = std::max(ncol, c + 1);
        nlev = std::max(nlev, lv + 1);
    }
    // equitable rebalancing: move sites (ascending index, repeated passes) out of classes larger
    // than T = ceil(n_free / ncol) into the smallest class below T that no neighbour uses.  The
    // sweep processes a class in rounds of one site per lane group, so the round count
    // sum_c ceil(|c| / groups) is what a sweep costs (multiplier 16: 15 -> 12 rounds at 64 groups).
    if (ncol > 1) {
        std::vector<uint32_t> size(ncol, 0);
        for (uint32_t i : m.free_sites) ++size[m.colour[i]];
        const uint32_t T = (uint32_t)((m.free_sites.size() + ncol - 1) / ncol);
        for (bool changed = true; changed;) {
            changed = false;
            for (uint32_t i : m.free_sites) {
                const int c = m.colour[i];
                if (size[c] <= T) continue;
                mark.assign(ncol, 0);
                for (uint32_t k = m.rowptr[i]; k < m.rowptr[i + 1]; ++k)
                    if (m.colour[m.col[k]] >= 0) mark[m.colour[m.col[k]]] = 1;
                int best = -1;
                for (int d = 0; d < ncol; ++d)
                    if (d != c && size[d] < T && !mark[d] && (best < 0 || size[d] < size[best])) best = d;
                if (best >= 0) {
                    m.colour[i] = best;
                    --size[c];
                    ++size[best];
                    changed = true;
                }
            }
        }
    }
    auto classes = [&](const std::vector<int32_t>& cls, int nc, std::vector<uint32_t>& ptr,
                       std::vector<uint32_t>& sites) {
        ptr.assign(nc + 1, 0);
        for (uint32_t i : m.free_sites) ++ptr[cls[i] + 1];
        for (int c = 0; c < nc; ++c) ptr[c + 1] += ptr[c];
        sites.assign(m.free_sites.size(), 0);
        std::vector<uint32_t> cur(ptr.begin(), ptr.end() - 1);
        for (uint32_t i : m.free_sites) sites[cur[cls[i]]++] = i;
    };
    classes(m.colour, ncol, m.col_ptr, m.col_sites);
    classes(m.level, nlev, m.lev_ptr, m.lev_sites);
}

}  // namespace

// ========================================================= balanced schedule ===

namespace {

// McNaughton's wrap-around rule for I equal jobs of S sweeps on M co-resident clusters:
// lay the jobs end to end, cut the line into M segments of C = ceil(I*S/M) sweeps.  A job
// cut between machines k and k+1 runs its FIRST sweeps at the start of k+1's timeline
// (signalling a flag when its state is stored) and its LAST sweeps at the end of k's timeline
// (waiting for the flag); C >= S guarantees the first part ends before the second starts.
struct HostSched {
    std::vector<int> ptr;
    std::vector<SchedItem> items;
    int nflags = 0;
};

HostSched mcnaughton(int I, int S, int M) {
    HostSched h;
    const long long total = (long long)I * S, C = (total + M - 1) / M;
    h.ptr.assign(M + 1, 0);
    int pending = -1;
    for (int k = 0; k < M; ++k) {
        const long long a = k * C, b = std::min(total, (k + 1) * C);
        for (long long pos = a; pos < b;) {
            const int j = (int)(pos / S), s_in = (int)(pos % S);
            const long long end = std::min(b, (long long)(j + 1) * S);
            const int len = (int)(end - (long long)j * S) - s_in;
            if (s_in > 0) {  // continuation of the job cut at this segment's start: its first sweeps
                h.items.push_back({j, 0, len, -1, pending});
            } else if (len < S) {  // cut at this segment's end: its last sweeps, after the flag
                pending = h.nflags++;
                h.items.push_back({j, S - len, S, pending, -1});
            } else {
                h.items.push_back({j, 0, S, -1, -1});
            }
            pos = end;
        }
        h.ptr[k + 1] = (int)h.items.size();
    }
    return h;
}

}  // namespace

// ================================================================ ensemble ===

struct tapt_ensemble_s {
    tapt_model_s* m = nullptr;
    // real-valued models: the whole ensemble lives in K5's engine (real.h); the fields below are unused
    std::unique_ptr<tapt_real::RealEngine> rx;
    uint32_t I = 0;
    uint64_t gid0 = 0;
    int R = 0, W = 0, G = 0, order = 0;
    std::vector<double> betas;
    uint64_t seed = 0;
    bool use_k1 = false;
    int k1_threads = 0, k2_threads = 512;
    // K3 (bit-sliced CSR, k3_bitcsr.cu) for colour-order runs of graphs with small integer
    // couplings and fields; instance teams per CTA (k3_ipb), 0 = not eligible / not decided
    int k3_ipb = -1;
    int k3_q = 1;  // lanes per site (k3_bitcsr.cu split sites)
    int k3_shape() const { return k3_q > 1 ? -k3_q : k3_ipb; }

    Csr3 k3_args() const {
        Csr3 g{};
        g.meta = m->d_meta3.p;
        g.adj = m->d_adj3.p;
        g.class_ptr = m->d_colptr.p;
        g.n_classes = (int)(m->col_ptr.size() - 1);
        g.nadj = m->k3_nadj;
        g.n2 = (2 * n() + 2 + 3) & ~3;
        g.nidx4 = (nidx + 3) & ~3;
        return g;
    }

    bool k3_eligible() {
        if (k3_ipb >= 0) return k3_ipb > 0;
        k3_ipb = 0;
        if (use_k1 || order != TAPT_ORDER_COLOUR || G != 1 || csrJ.p || nidx > k3_row_stride()) return false;
        // TAPT_K3=0 selects K2 (the byte-SWAR kernel) for every CSR run
        if (const char* e = std::getenv("TAPT_K3"); e && std::atoi(e) == 0) return false;
        m->build_k3(stream);
        if (m->k3_state != 1) return false;
        // energy counters: at most 2 x 127 per site and thread per sweep into 12 planes
        if (m->k3_max_per_thread * 254 > 4095) return false;
        // Instance teams per CTA (the graph is staged once per CTA).  Modelled throughput, with the
        // per-team rate r(k) for k teams on an SM measured on config 4 (tools/k3_ipb_shards.py:
        // 1.64 / 1.32 / 1.00 / 0.83 G updates/s for k = 1..4):
        //   balanced:   co-resident teams M(ipb) <= I, every SM busy  -> M x r(teams per SM)
        //   one CTA/SM: ipb = ceil(I / SMs) <= 4                      -> I x r(ipb)
        // (config 4 at 512 / 256 / 128 / 64 instances -> 3 / 2 / 1 / 1 teams per CTA)
        int fit = 0;
        for (int ipb = 4; ipb >= 1 && !fit; --ipb)
            if (k3_smem_bytes(R, nidx, m->k3_nadj, (int)m->free_sites.size(), n(), (int)m->col_ptr.size() - 1, ipb) <=
                200 * 1024)
                fit = ipb;
        if (!fit) return false;
        auto rate = [](int k) { return k <= 1 ? 1.64 : k == 2 ? 1.32 : k == 3 ? 1.0 : 0.83 * 4.0 / k; };
        int dev = 0, nsm = 148;
        CUDA_OK(cudaGetDevice(&dev));
        CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        PTArgs a = base_args();
        double best = -1.0;
        k3_ipb = 1;
        for (int ipb = 1; ipb <= fit; ++ipb) {
            const int M = k3_resident_units(a, k3_args(), ipb);
            double v = -1.0;
            if (M > 0 && M <= (int)I) v = M * rate(M / nsm);
            if (((int)I + ipb - 1) / ipb <= nsm)
                v = std::max(v, (double)I * rate(ipb));
            if (v > best) {
                best = v;
                k3_ipb = ipb;
            }
        }
        if (const char* e = std::getenv("TAPT_K3_IPB"))
            k3_ipb = std::max(1, std::min(fit, std::atoi(e)));
        // Split sites (4 lanes per site, one 512-thread team per CTA) when every instance has an SM
        // to itself: a lone team is bound by its per-site dependency chains, and splitting the
        // replicas over 4 lanes raises its rate to ~1.9 G updates/s (config 4 at 64 / 148
        // instances: +11 / +14 %, tools/k3_q_shards.py); with two or more teams per SM one lane per
        // site wins (no replicated site work).
        k3_q = 1;
        if ((int)I <= nsm && I * 1.9 > best) k3_q = 4;
        if (const char* e = std::getenv("TAPT_K3_Q")) {
            const int q = std::atoi(e);
            k3_q = q >= 4 ? 4 : q >= 2 ? 2 : 1;
        }
        if (k3_q > 1) k3_ipb = 1;
        return k3_ipb > 0;
    }

    // K4 (k4_levels.cu): the reference's index order on the dependency levels, one warp per site
    // word; shared couplings, <= 32 slots.  TAPT_K4=0 selects K2.
    int k4_ipb = -1;
    bool k4_eligible() {
        if (k4_ipb >= 0) return k4_ipb > 0;
        k4_ipb = 0;
        if (use_k1 || order != TAPT_ORDER_REFERENCE || G != 1 || csrJ.p || m->n >= (1u << 24)) return false;
        if (const char* e = std::getenv("TAPT_K4"); e && std::atoi(e) == 0) return false;
        const int nlev = (int)m->lev_ptr.size() - 1;
        for (int ipb = std::min(k4_max_ipb(), (int)std::max(1u, I)); ipb >= 1; --ipb)
            if (k4_smem_bytes(n(), R, nidx, (int)m->col.size(), (int)m->free_sites.size(), nlev, ipb) <= 200 * 1024) {
                k4_ipb = ipb;
                break;
            }
        return k4_ipb > 0;
    }

    // balanced persistent K1 schedule (McNaughton), cached per launch length
    int k1_units = -1;  // co-resident clusters (or CTAs) of the sweep kernel's launch shape
    int sched_S = -1, sched_M = 0, sched_nflags = 0;
    DevBuf<int> sched_ptr;
    DevBuf<SchedItem> sched_items;
    DevBuf<uint32_t> sched_flags, sched_err;  // sched_err is sticky until checked
    uint32_t* sched_err_host = nullptr;        // pinned copy, read once the stream has passed it
    cudaEvent_t sched_ev = nullptr;
    bool sched_pending = false;
    ~tapt_ensemble_s() {
        if (sched_ev) cudaEventDestroy(sched_ev);
        if (sched_err_host) cudaFreeHost(sched_err_host);
    }

    // Report a timed-out wait of a balanced launch (set by the kernel, copied asynchronously after
    // the launch).  force: wait for the copy (getters and synchronize, which sync anyway);
    // otherwise only if the stream has already passed it (no host stall on the launch path).
    void poll_sched(bool force) {
        if (!sched_pending) return;
        if (force)
            CUDA_OK(cudaEventSynchronize(sched_ev));
        else if (cudaEventQuery(sched_ev) != cudaSuccess)
            return;
        sched_pending = false;
        if (*sched_err_host) {
            *sched_err_host = 0;
            sched_err.zero(stream);
            throw tapt::CudaError("balanced sweep schedule: a split job waited > 2 s for its first part "
                                  "(another kernel holding SMs?); results of that run are invalid; set TAPT_BALANCE=0");
        }
    }
    int nidx = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    uint64_t T = 0, P = 0, Q = 0;  // sweeps, swap passes, proposal rounds (global)
    // swap passes run inside the fused kernel, by parity: pair r is attempted once per pass of
    // parity r & 1 (the kernel counts only accepts; tapt_get_acceptance adds these attempts)
    uint64_t fused_passes[2] = {0, 0};
    int clamp_sets = 1;
    bool have_disorder = false;
    uint32_t launch_chunk = 2000;
    bool swap_oversize = false, prop_oversize = false;  // exact tables too large for this ladder
    bool ladder_unordered = false;  // set_betas accepted a decreasing neighbour pair: swaps refused

    DevBuf<uint32_t> words;
    DevBuf<int32_t> E;
    DevBuf<uint8_t> slot_of, buf_of;
    DevBuf<uint64_t> streams, coord, thr;
    DevMetro swap_tab, prop_tab;
    DevBuf<uint64_t> swap_att, swap_acc, prop_att, prop_acc;
    DevBuf<long long> obs;
    DevBuf<unsigned long long> hist;
    long long e_lo = 0, width = 1;
    int nbins = 0;
    DevBuf<int> best;
    DevBuf<int8_t> signs, csrJ, clampval;
    DevBuf<uint8_t> bonds;
    // proposal scratch
    DevBuf<uint32_t> pwords;
    DevBuf<int32_t> pE;
    DevBuf<uint8_t> pslot, pacc, pforced, pbytes;
    DevBuf<double> plq, dbetas;      // MH correction: log q (cur | prop) of the round, the ladder
    std::vector<double> dbetas_host;  // the ladder dbetas holds
    DevBuf<uint32_t> pties;
    uint64_t mh_tie_rounds = 0;       // MH rounds that fell back to the host decisions
    DevBuf<int8_t> pint8;
    DevBuf<uint64_t> pstreams, paccs, ptup, pfull;
    std::vector<uint32_t> last_targets;  // prepare_targets: device copies are current for these
    DevBuf<uint32_t> ptargets;

    int n() const { return (int)m->n; }
    int group_words() const { return G; }

    const int8_t* clamp_ptr() const { return clampval.p ? clampval.p : m->d_clamp.p; }
    int clamp_count() const { return clampval.p ? (int)I : 1; }
    bool has_clamps() const { return m->free_sites.size() != m->n; }

    CsrArgs csr_args(bool level_order) const {
        CsrArgs g{};
        g.rowptr = m->d_rowptr.p;
        g.col = m->d_col.p;
        g.J = csrJ.p ? csrJ.p : m->d_J.p;
        g.nJ = csrJ.p ? (int)I : 1;
        g.nnz = (int)m->col.size();
        g.h = m->d_h.p;
        g.hs = m->d_hs.p;
        g.rank = m->d_rank.p;
        g.class_ptr = level_order ? m->d_levptr.p : m->d_colptr.p;
        g.class_sites = level_order ? m->d_levsites.p : m->d_colsites.p;
        g.n_classes = (int)((level_order ? m->lev_ptr.size() : m->col_ptr.size()) - 1);
        g.lmin = m->lmin;
        g.n_free = (uint32_t)m->free_sites.size();
        g.smem_graph = k2_smem_bytes_graph(n(), R, nidx, g.nnz, (int)g.n_free) <= 200 * 1024 ? 1 : 0;
        return g;
    }

    PTArgs base_args() {
        PTArgs a{};
        a.words = words.p;
        a.I = (int)I;
        a.G = G;
        a.W = W;
        a.B = R;
        a.n = n();
        a.bonds = bonds.p;
        a.n_free = (uint32_t)m->free_sites.size();
        a.R = R;
        a.streams = streams.p;
        a.slot_of = slot_of.p;
        a.buf_of = buf_of.p;
        a.thr = thr.p;
        a.nidx = nidx;
        a.E = E.p;
        a.coord = coord.p;
        a.swap_tab = swap_tab.view();
        a.swap_att = swap_att.p;
        a.swap_acc = swap_acc.p;
        a.obs = obs.p;
        a.hist = nbins ? hist.p : nullptr;
        a.e_lo = e_lo;
        a.width = width;
        a.nbins = nbins;
        a.best = best.p;
        a.mc = make_mix_consts();
        return a;
    }

    int k2_nt() const {
        int nt = k2_threads;
        if (const char* env = std::getenv("TAPT_K2_THREADS")) nt = std::max(128, std::min(TAPT_K2_MAXT, std::atoi(env)));
        return nt;
    }

    // Distinct sweep-kernel instantiations this ensemble launched ("name" or "name balanced M=<units>"),
    // in first-launch order: test evidence of which code path ran (tapt_ensemble_launch_log).
    std::vector<std::string> launch_log;
    void log_launch(std::string name, const PTArgs& a) {
        if (a.sched) name += " balanced M=" + std::to_string(a.sched_clusters);
        if (std::find(launch_log.begin(), launch_log.end(), name) == launch_log.end() && launch_log.size() < 64)
            launch_log.push_back(std::move(name));
    }

    void launch(const PTArgs& a, bool cluster, int k1_nt = 0) {
        ++g_launches;
        cudaError_t e;
        if (use_k1) {
            const int nt = k1_nt > 0 ? k1_nt : k1_threads;
            char name[96];
            k1_variant_name(a, m->ld, nt, cluster, name);
            log_launch(name, a);
            e = launch_k1(a, m->ld, nt, cluster, stream);
        } else if (!a.energy_only && a.G == 1 && k3_eligible()) {
            log_launch("k3_bitcsr_pt<" + std::string(a.sched ? "1," : "0,") + std::to_string(k3_ipb) + "," +
                           std::to_string(k3_q) + ">",
                       a);
            e = launch_k3(a, k3_args(), k3_shape(), stream);
        } else if (!a.energy_only && a.G == 1 && k4_eligible()) {
            log_launch(std::string("k4_levels_pt<") + (a.sched ? "1>" : "0>"), a);
            e = launch_k4(a, csr_args(true), k4_ipb, stream);
        } else {
            log_launch(std::string("k2_csr_pt") + (cluster ? "<cluster>" : ""), a);
            e = launch_k2(a, csr_args(order == TAPT_ORDER_REFERENCE), k2_nt(), cluster, stream);
        }
        if (e != cudaSuccess) throw tapt::CudaError(std::string("sweep kernel launch: ") + cudaGetErrorString(e));
        CUDA_OK(cudaGetLastError());
    }

    // Exact energies of every buffer from the spins.
    void recompute_energies() {
        if (use_k1) {
            PTArgs a = base_args();
            a.energy_only = 1;
            a.n_sweeps = 0;
            a.swap_every = 0;
            a.measure_every = 0;
            a.best = nullptr;
            launch(a, false);
        } else {
            CsrArgs g = csr_args(false);
            ++g_launches;
            k_energy_csr<<<dim3(G, I), 256, 0, stream>>>(words.p, n(), G, W, R, g.rowptr, g.col, g.J, g.nJ, g.nnz,
                                                          g.h, E.p);
            CUDA_OK(cudaGetLastError());
        }
    }

    void update_best_from_E() {  // best = min(best, min over buffers), stream-ordered
        ++g_launches;
        k_best_from_E<<<(I + 127) / 128, 128, 0, stream>>>(E.p, (int)I, R, best.p);
        CUDA_OK(cudaGetLastError());
    }

    // Heat-bath thresholds [R][nidx] and the swap (rows = pairs) / proposal (rows = slots)
    // Metropolis tables for the current ladder.
    void build_tables() {
        std::vector<uint64_t> th((size_t)R * nidx);
        for (int r = 0; r < R; ++r)
            for (int k = 0; k < nidx; ++k) {
                const double l = use_k1 ? (double)(m->J0 * (2 * k - 2 * m->dim)) : (double)(m->lmin + k);
                th[(size_t)r * nidx + k] = threshold_of(conditional_up(betas[r], l));
            }
        thr.upload(th, stream);
        HostMetro sw, pr;
        for (int r = 0; r + 1 < R; ++r) sw.add_row(betas[r + 1] - betas[r]);
        if (R < 2) sw.add_row(0.0);
        for (int r = 0; r < R; ++r) pr.add_row(betas[r]);
        swap_tab.upload(sw, stream);
        prop_tab.upload(pr, stream);
        swap_oversize = sw.oversize;
        prop_oversize = pr.oversize;
    }

    // When the instances (one cluster each) do not fill whole waves of co-resident clusters,
    // launch a persistent grid that runs McNaughton's balanced schedule.
    // TAPT_BALANCE=0 disables it.
    bool balance(PTArgs& a, bool cluster) {
        if (a.energy_only) return false;
        if (const char* e = std::getenv("TAPT_BALANCE"); e && std::atoi(e) == 0) return false;
        if (k1_units < 0)
            k1_units = use_k1           ? k1_resident_units(a, m->ld, k1_threads, cluster)
                       : k3_eligible() ? k3_resident_units(a, k3_args(), k3_shape())
                       : k4_eligible() ? k4_resident_units(a, csr_args(true), k4_ipb)
                                       : k2_resident_units(a, csr_args(order == TAPT_ORDER_REFERENCE), k2_nt(), cluster);
        const int M = k1_units;
        if (M <= 0 || (int)I <= M) return false;
        const double waves = (double)I / M;
        if (waves / std::ceil(waves) > 0.999) return false;
        if (!sched_err_host) {
            CUDA_OK(cudaMallocHost(&sched_err_host, 4));
            *sched_err_host = 0;
            CUDA_OK(cudaEventCreateWithFlags(&sched_ev, cudaEventDisableTiming));
            sched_err.alloc(1);
            sched_err.zero(stream);
        }
        if (sched_S != a.n_sweeps || sched_M != M) {
            const HostSched h = mcnaughton((int)I, a.n_sweeps, M);
            sched_ptr.upload(h.ptr, stream);
            sched_items.upload(h.items, stream);
            sched_flags.alloc(std::max(1, h.nflags));
            sched_S = a.n_sweeps;
            sched_M = M;
            sched_nflags = h.nflags;
        }
        sched_flags.zero(stream);
        a.sched_ptr = sched_ptr.p;
        a.sched = sched_items.p;
        a.flags = sched_flags.p;
        a.sched_err = sched_err.p;
        a.sched_clusters = M;
        return true;
    }

    void run(uint32_t n_sweeps, uint32_t swap_every, uint32_t measure_every, uint64_t measure_from) {
        if (n_sweeps == 0) return;
        if (swap_every && R < 2) swap_every = 0;
        if (swap_every && swap_oversize)
            throw tapt::ConfigError("beta spacing too fine for exact swap tables (adjacent betas closer than ~1e-5)");
        if (swap_every && ladder_unordered)
            throw tapt::ConfigError("replica swaps need a non-decreasing beta ladder (SPEC.md:388); the "
                                    "current ladder (set with allow_flat=2) has a decreasing neighbour pair");
        const bool cluster = G > 1;
        uint32_t done = 0;
        while (done < n_sweeps) {
            const uint32_t chunk = std::min(launch_chunk, n_sweeps - done);
            PTArgs a = base_args();
            a.t0 = T;
            a.n_sweeps = (int)chunk;
            a.swap_every = (int)swap_every;
            a.p0 = P;
            a.measure_every = (int)measure_every;
            a.measure_from = measure_from;
            const bool balanced = balance(a, cluster);
            launch(a, cluster);
            if (balanced) {
                CUDA_OK(cudaMemcpyAsync(sched_err_host, sched_err.p, 4, cudaMemcpyDeviceToHost, stream));
                CUDA_OK(cudaEventRecord(sched_ev, stream));
                sched_pending = true;
            }
            if (swap_every) {
                const uint64_t P1 = P + (T + chunk) / swap_every - T / swap_every;
                const uint64_t even = (P1 + 1) / 2 - (P + 1) / 2;  // passes p in [P, P1) with p even
                fused_passes[0] += even;
                fused_passes[1] += (P1 - P) - even;
                P = P1;
            }
            T += chunk;
            done += chunk;
        }
    }
};

namespace {

void check_model(const tapt_model_s* m) {
    if (!m) throw tapt::ConfigError("null model handle");
}
void check_ens(tapt_ensemble_s* e) {
    if (!e) throw tapt::ConfigError("null ensemble handle");
    e->poll_sched(false);
}

// LatticeSpec::graph_clamped bond list (lattice.cpp:55-87): per site, +x then +y (then +z);
// wrap bonds only when periodic and the extent is > 2.
void lattice_bonds(int dim, int ly, int lx, int l, bool periodic, std::vector<uint32_t>& ci,
                   std::vector<uint32_t>& cj) {
    if (dim == 2) {
        for (int r = 0; r < ly; ++r)
            for (int c = 0; c < lx; ++c) {
                const uint32_t i = (uint32_t)(r * lx + c);
                if (c + 1 < lx) {
                    ci.push_back(i);
                    cj.push_back((uint32_t)(r * lx + c + 1));
                } else if (periodic && lx > 2) {
                    ci.push_back(i);
                    cj.push_back((uint32_t)(r * lx));
                }
                if (r + 1 < ly) {
                    ci.push_back(i);
                    cj.push_back((uint32_t)((r + 1) * lx + c));
                } else if (periodic && ly > 2) {
                    ci.push_back(i);
                    cj.push_back((uint32_t)c);
                }
            }
        return;
    }
    auto idx = [l](int x, int y, int z) { return (uint32_t)(x + l * (y + (long)l * z)); };
    for (int z = 0; z < l; ++z)
        for (int y = 0; y < l; ++y)
            for (int x = 0; x < l; ++x) {
                const uint32_t i = idx(x, y, z);
                if (x + 1 < l) {
                    ci.push_back(i);
                    cj.push_back(idx(x + 1, y, z));
                } else if (periodic && l > 2) {
                    ci.push_back(i);
                    cj.push_back(idx(0, y, z));
                }
                if (y + 1 < l) {
                    ci.push_back(i);
                    cj.push_back(idx(x, y + 1, z));
                } else if (periodic && l > 2) {
                    ci.push_back(i);
                    cj.push_back(idx(x, 0, z));
                }
                if (z + 1 < l) {
                    ci.push_back(i);
                    cj.push_back(idx(x, y, z + 1));
                } else if (periodic && l > 2) {
                    ci.push_back(i);
                    cj.push_back(idx(x, y, 0));
                }
            }
}

void sync_if(cudaStream_t st) { CUDA_OK(cudaStreamSynchronize(st)); }

}  // namespace

// ==================================================================== C ABI ===

extern "C" {

const char* tapt_last_error(void) { return g_last_error.c_str(); }
const char* tapt_version(void) { return "tapt-b200 0.1 (sm_100a)"; }
unsigned long long tapt_launch_count(void) { return g_launches.load(); }

tapt_status tapt_probe_decision_rate(int blocks_per_sm, int threads, uint32_t iters, double* decisions_per_s,
                                     double* seconds) {
    return guard([&] {
        if (tapt_device_count() == 0) throw tapt::CudaError("no CUDA device");
        cudaStream_t st;
        CUDA_OK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        int dev = 0, nsm = 0;
        CUDA_OK(cudaGetDevice(&dev));
        CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        const int blocks = nsm * std::max(1, blocks_per_sm);
        DevBuf<uint32_t> sink;
        sink.alloc((size_t)blocks * threads);
        cudaEvent_t a, b;
        CUDA_OK(cudaEventCreate(&a));
        CUDA_OK(cudaEventCreate(&b));
        ++g_launches;
        const char* ve = std::getenv("TAPT_PROBE_VARIANT");
        const int variant = ve ? std::atoi(ve) : -1;
        CUDA_OK(launch_decision_probe(blocks, threads, iters, sink.p, st, variant));  // warm-up
        CUDA_OK(cudaEventRecord(a, st));
        ++g_launches;
        CUDA_OK(launch_decision_probe(blocks, threads, iters, sink.p, st, variant));
        CUDA_OK(cudaEventRecord(b, st));
        CUDA_OK(cudaEventSynchronize(b));
        float ms = 0;
        CUDA_OK(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaStreamDestroy(st);
        const double n = (double)blocks * threads * iters * 64.0;
        if (seconds) *seconds = ms * 1e-3;
        if (decisions_per_s) *decisions_per_s = n / (ms * 1e-3);
    });
}
// Make `device` current for this library's CUDA runtime on the calling thread (the library links
// cudart statically, so a caller's cudaSetDevice through another runtime -- e.g. torch's -- is only
// seen through the thread's current context; one process per GPU should call this explicitly).
tapt_status tapt_set_device(int device) {
    return guard([&] {
        const int n = tapt_device_count();
        if (device < 0 || device >= n) throw tapt::ConfigError("device index out of range");
        CUDA_OK(cudaSetDevice(device));
    });
}

int tapt_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return c;
}

tapt_status tapt_model_create_lattice(int dim, int ly, int lx, int lz, double J, int boundary, tapt_model_t* out) {
    return guard([&] {
        if (!out) throw tapt::ConfigError("null output handle");
        if (dim != 2 && dim != 3) throw tapt::ConfigError("lattice dim must be 2 or 3");
        if (dim == 2 && (ly < 1 || lx < 1)) throw tapt::ConfigError("grid2d dimensions must be >= 1");
        if (dim == 3 && lx < 1) throw tapt::ConfigError("grid3d size must be >= 1");
        (void)lz;
        auto m = std::make_unique<tapt_model_s>();
        std::vector<uint32_t> ci, cj;
        const bool per = boundary == TAPT_BOUNDARY_PERIODIC;
        const int l = lx;
        lattice_bonds(dim, ly, lx, l, per, ci, cj);
        const uint32_t n = dim == 2 ? (uint32_t)(ly * lx) : (uint32_t)(l * l * l);
        std::vector<double> Jv(ci.size(), J);
        build_model(*m, n, ci, cj, Jv, nullptr, nullptr);
        m->lattice = true;
        m->dim = dim;
        m->ly = dim == 2 ? ly : l;
        m->lx = lx;
        m->lz = dim == 2 ? 1 : l;
        m->boundary = boundary;
        m->J0 = (int)std::fabs(J);
        m->Jsign = J < 0 ? -1 : 1;
        m->nbonds = (uint32_t)ci.size();
        const int a = ilog2_exact(lx), b = ilog2_exact(m->ly);
        m->k1 = !m->real && per && a >= 2 && b >= 2 && (dim == 2 || a == b) && n <= 40000 && m->J0 <= 127;
        m->ld.dim = dim;
        m->ld.log2Lx = a;
        m->ld.log2Ly = b;
        m->ld.log2hx = a - 1;
        m->ld.J0 = m->J0;
        *out = m.release();
    });
}

tapt_status tapt_model_create_graph(uint32_t n, uint32_t nc, const uint32_t* ci, const uint32_t* cj, const double* J,
                                    const double* h, const int8_t* clamp, tapt_model_t* out) {
    return guard([&] {
        if (!out) throw tapt::ConfigError("null output handle");
        if (nc && (!ci || !cj || !J)) throw tapt::ConfigError("null coupling arrays");
        auto m = std::make_unique<tapt_model_s>();
        std::vector<uint32_t> a(ci, ci + nc), b(cj, cj + nc);
        std::vector<double> v(J, J + nc);
        build_model(*m, n, a, b, v, h, clamp);
        *out = m.release();
    });
}

// `isingmodel v1` text files (spin_model.cpp:123-226 format and errors).
tapt_status tapt_model_load_file(const char* path, tapt_model_t* out) {
    return guard([&] {
        if (!path || !out) throw tapt::ConfigError("null path / output");
        const tapt::CouplingGraph g = tapt::CouplingGraph::load_file(path);
        std::vector<uint32_t> ci, cj;
        std::vector<double> J;
        for (const auto& c : g.couplings()) {
            ci.push_back(c.i);
            cj.push_back(c.j);
            J.push_back(c.value);
        }
        std::vector<int8_t> cl(g.n_spins());
        for (uint32_t i = 0; i < g.n_spins(); ++i) cl[i] = g.clamp_value(i);
        auto m = std::make_unique<tapt_model_s>();
        build_model(*m, (uint32_t)g.n_spins(), ci, cj, J, g.fields().data(), cl.data());
        *out = m.release();
    });
}

tapt_status tapt_model_save_file(tapt_model_t m, const char* path) {
    return guard([&] {
        check_model(m);
        if (!path) throw tapt::ConfigError("null path");
        tapt::CouplingGraph::Builder b(m->n);
        for (size_t k = 0; k < m->ci.size(); ++k) b.add_coupling(m->ci[k], m->cj[k], m->J[k]);
        for (uint32_t i = 0; i < m->n; ++i) {
            if (m->h[i] != 0.0) b.add_field(i, m->h[i]);
            if (m->clamp[i]) b.set_clamp(i, m->clamp[i]);
        }
        b.build().save_file(path);
    });
}

tapt_status tapt_model_destroy(tapt_model_t m) {
    return guard([&] { delete m; });
}

}  // extern "C"

tapt_model_s::~tapt_model_s() {
    if (dropin) tapt_ensemble_destroy(dropin);
    dropin_real.reset();
    if (dropin_stream) cudaStreamDestroy(dropin_stream);
}

extern "C" {

tapt_status tapt_model_info(tapt_model_t m, uint32_t* n_spins, uint32_t* n_free, uint32_t* n_couplings, int32_t* lmin,
                            int32_t* lmax, uint32_t* n_colours, uint32_t* n_levels) {
    return guard([&] {
        check_model(m);
        if (n_spins) *n_spins = m->n;
        if (n_free) *n_free = (uint32_t)m->free_sites.size();
        if (n_couplings) *n_couplings = (uint32_t)m->ci.size();
        if (lmin) *lmin = m->lmin;
        if (lmax) *lmax = m->lmax;
        if (n_colours) *n_colours = (uint32_t)(m->col_ptr.size() - 1);
        if (n_levels) *n_levels = (uint32_t)(m->lev_ptr.size() - 1);
    });
}

tapt_status tapt_model_couplings(tapt_model_t m, uint32_t* ci, uint32_t* cj, double* J) {
    return guard([&] {
        check_model(m);
        for (size_t k = 0; k < m->ci.size(); ++k) {
            if (ci) ci[k] = m->ci[k];
            if (cj) cj[k] = m->cj[k];
            if (J) J[k] = m->J[k];
        }
    });
}

tapt_status tapt_model_schedule(tapt_model_t m, int32_t* colour, int32_t* level) {
    return guard([&] {
        check_model(m);
        if (colour) std::copy(m->colour.begin(), m->colour.end(), colour);
        if (level) std::copy(m->level.begin(), m->level.end(), level);
    });
}

tapt_status tapt_model_digest(tapt_model_t m, uint64_t* digest) {
    return guard([&] {
        check_model(m);
        *digest = m->digest;
    });
}

tapt_status tapt_model_energy(tapt_model_t m, const int8_t* s, size_t len, double* out) {
    return guard([&] {
        check_model(m);
        if (len != m->n)
            throw tapt::DimensionError("configuration length " + std::to_string(len) + " != n_spins " +
                                       std::to_string(m->n));
        double e = 0.0;
        for (size_t k = 0; k < m->ci.size(); ++k) e -= m->J[k] * (double)(s[m->ci[k]] * s[m->cj[k]]);
        for (uint32_t i = 0; i < m->n; ++i) e -= m->h[i] * (double)s[i];
        *out = e;
    });
}

// ---------------------------------------------------------------- ensembles

tapt_status tapt_ensemble_create(tapt_model_t m, const tapt_ensemble_desc* d, tapt_ensemble_t* out) {
    return guard([&] {
        check_model(m);
        if (!d || !out) throw tapt::ConfigError("null descriptor / output");
        if (d->n_instances == 0) throw tapt::ConfigError("n_instances must be >= 1");
        if (m->n == 0) throw tapt::ConfigError("model has no spins");
        if (d->n_slots < 1 || d->n_slots > (uint32_t)kMaxR) throw tapt::ConfigError("n_slots must be in [1, 256]");
        if (!d->betas) throw tapt::ConfigError("null beta ladder");
        for (uint32_t r = 0; r < d->n_slots; ++r) {
            if (!(d->betas[r] >= 0.0) || !std::isfinite(d->betas[r])) throw tapt::ConfigError("beta must be >= 0");
            if (r && !(d->betas[r] > d->betas[r - 1]))
                throw tapt::ConfigError("beta ladder must be strictly increasing (SPEC.md:388)");
        }
        if (d->order != TAPT_ORDER_COLOUR && d->order != TAPT_ORDER_REFERENCE)
            throw tapt::ConfigError("unknown sweep order");
        if (tapt_device_count() == 0) throw tapt::CudaError("no CUDA device: the TAPT engine has no CPU fallback");
        auto e = std::make_unique<tapt_ensemble_s>();
        e->m = m;
        e->I = d->n_instances;
        e->gid0 = d->instance_offset;
        e->R = (int)d->n_slots;
        e->betas.assign(d->betas, d->betas + d->n_slots);
        e->seed = d->seed;
        e->order = d->order;
        e->W = std::min(e->R, kW);
        e->G = (e->R + kW - 1) / kW;
        CUDA_OK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
        e->own_stream = true;
        if (m->real) {
            e->rx = std::make_unique<tapt_real::RealEngine>(m->real_graph(), e->I, e->gid0, e->betas, e->seed, e->order,
                                                            e->stream);
            *out = e.release();
            return;
        }
        m->ensure_device(e->stream);
        const int n = (int)m->n;
        e->use_k1 = m->k1 && d->order == TAPT_ORDER_COLOUR && !e->has_clamps();
        if (e->use_k1) {
            // Replica-group width: with fewer instance-groups than SMs (e.g. configs 2/3 sharded over
            // 8 GPUs), narrower groups (16 or 8 replicas per CTA, clusters of up to 8 CTAs) spread each
            // instance over more SMs.  Results do not depend on the grouping (streams and tables are
            // keyed by slot; tests/test_gpu_parity.py::test_k1_group_width_does_not_change_the_chain).
            int dev = 0, nsm = 148;
            CUDA_OK(cudaGetDevice(&dev));
            CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
            // Model: throughput ~ eff(W) x min(1, CTAs / SMs) with one 512-thread CTA per SM; eff measured
            // on config 3 (tools/narrow_groups.py: 32 / 16 / 8 replicas -> 975 / 727 / 600 G/s at 256
            // instances, with the narrow groups' lattice folded so that a word holds 2 / 4 sites).  Small lattices (several 128-thread CTAs per SM) keep 32-replica groups.
            int w = e->W;
            if (n / 4 >= TAPT_K1_DEFAULT_THREADS) {
                auto score = [&](int cand) {
                    const double eff = cand >= 32 ? 1.0 : (cand >= 16 ? 0.745 : 0.615);
                    const double ctas = (double)e->I * ((e->R + cand - 1) / cand);
                    return eff * std::min(1.0, ctas / nsm);
                };
                double best = score(w);
                for (int cand : {16, 8})
                    if (e->R > cand && (e->R + cand - 1) / cand <= 8 && score(cand) > 1.05 * best) {
                        best = score(cand);
                        w = cand;
                    }
            }
            if (const char* env = std::getenv("TAPT_K1_W")) w = std::max(1, std::min(kW, std::atoi(env)));
            w = std::min(w, e->R);
            if ((e->R + w - 1) / w > 8) throw tapt::ConfigError("TAPT_K1_W: at most 8 replica groups per instance");
            e->W = w;
            e->G = (e->R + w - 1) / w;
            e->nidx = 2 * m->dim + 1;
            int nt = TAPT_K1_DEFAULT_THREADS;
            if (n / 4 < TAPT_K1_DEFAULT_THREADS) {
                // small lattices: one whole-SM CTA per instance-group while they do not exceed the
                // SMs, else 256-thread CTAs (2 site words per thread, registers capped for 2 CTAs per
                // SM) so that several share an SM (config 1, 1024 sites: 16 seeds 42 -> 51 G/s; 296
                // seeds: 128-thread CTAs 627, 256-thread CTAs 674 G/s; tools/cfg1_shapes.sh)
                int dev = 0, nsm = 148;
                CUDA_OK(cudaGetDevice(&dev));
                CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
                nt = (long long)e->I * e->G >= 2ll * nsm ? 256 : TAPT_K1_DEFAULT_THREADS;
            } else if (k1_smem_bytes(n, true, e->R) <= (100 - (TAPT_K1_IDXS ? 18 : 0)) * 1024) {
                // mid-size lattices with at least two instance-groups per SM: two independent 256-thread
                // CTAs per SM (barriers decoupled) instead of one 512-thread CTA (config 3: 803 -> 840
                // G/s; config 2's 256 groups on 296 slots lose 7 % and keep 512 threads)
                int dev = 0, nsm = 148;
                CUDA_OK(cudaGetDevice(&dev));
                CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
                if ((long long)e->I * e->G >= 2ll * nsm) nt = 256;
            }
            // large lattices (config 5): 640 threads (5 warps per scheduler at <= 102 registers, now that the
            // threshold offsets live in the shared-memory scratch) when the site pairs still divide evenly enough
            if (nt == 512 && TAPT_K1_IDXS && n / 4 >= 8 * 640 &&
                (double)(n / 4) / (double)(((n / 4 + 639) / 640) * 640) >= 0.97 &&
                k1_smem_bytes(n, true, e->R) + 640 * 64 + 11 * 1024 <= 227 * 1024)
                nt = 640;
            if (const char* env = std::getenv("TAPT_K1_THREADS")) nt = std::max(32, std::min(1024, std::atoi(env)));
            nt = (nt / 32) * 32;
            // the per-thread bit-sliced counters hold < 256: unsatisfied bonds of this thread's
            // colour-1 sites (2*dim each) and up-spins of its share of all sites
            while (nt < 1024 && ((n / 2 + nt - 1) / nt * 2 * m->dim >= 256 || (n + nt - 1) / nt >= 256)) nt *= 2;
            e->k1_threads = nt;
            // dynamic part + the kernel's static block (control block ~6 KB, index scratch 32 KB with TAPT_K1_IDXS)
            if (k1_smem_bytes(n, true, e->R) > (221 - (TAPT_K1_IDXS ? 32 : 0)) * 1024) throw tapt::SizeError("lattice too large for shared memory");
        } else {
            if (m->max_sumabs > 255) throw tapt::SizeError("sum of |J| at a site exceeds 255 (byte-SWAR fields)");
            e->nidx = m->lmax - m->lmin + 1;
            if (k2_smem_bytes(n, e->R, e->nidx) > 227 * 1024) throw tapt::SizeError("graph too large for shared memory");
        }
        if (e->G > 8) throw tapt::ConfigError("at most 256 slots");
        e->build_tables();
        // streams
        std::vector<uint64_t> st((size_t)e->I * e->R), co(e->I);
        for (uint32_t i = 0; i < e->I; ++i) {
            const uint64_t gid = e->gid0 + i;
            for (int r = 0; r < e->R; ++r)
                st[(size_t)i * e->R + r] = tapt::RngStream::derive(e->seed, {tapt::stream::kReplica, gid, (uint64_t)r}).state();
            co[i] = tapt::RngStream::derive(e->seed, {tapt::stream::kCoordinator, gid}).state();
        }
        e->streams.upload(st, e->stream);
        e->coord.upload(co, e->stream);
        // state
        e->words.alloc((size_t)e->I * e->G * n);
        e->words.zero(e->stream);
        e->E.alloc((size_t)e->I * e->R);
        e->E.zero(e->stream);
        std::vector<uint8_t> perm((size_t)e->I * e->R);
        for (uint32_t i = 0; i < e->I; ++i)
            for (int r = 0; r < e->R; ++r) perm[(size_t)i * e->R + r] = (uint8_t)r;
        e->slot_of.upload(perm, e->stream);
        e->buf_of.upload(perm, e->stream);
        const size_t np = (size_t)e->I * std::max(e->R - 1, 1);
        e->swap_att.alloc(np);
        e->swap_acc.alloc(np);
        e->prop_att.alloc((size_t)e->I * e->R);
        e->prop_acc.alloc((size_t)e->I * e->R);
        e->swap_att.zero(e->stream);
        e->fused_passes[0] = e->fused_passes[1] = 0;
        e->swap_acc.zero(e->stream);
        e->prop_att.zero(e->stream);
        e->prop_acc.zero(e->stream);
        e->obs.alloc((size_t)e->I * e->R * 5);
        e->obs.zero(e->stream);
        std::vector<int> b(e->I, 0x7FFFFFFF);
        e->best.upload(b, e->stream);
        sync_if(e->stream);
        *out = e.release();
        if (m->lattice && !m->real && m->Jsign < 0 && m->J0 != 0) {  // antiferromagnet: every bond negative
            std::vector<int8_t> sg((size_t)(*out)->I * m->nbonds, -1);
            if (tapt_ensemble_set_bond_signs(*out, sg.data(), m->nbonds) != TAPT_OK) {
                const std::string msg = g_last_error;
                tapt_ensemble_destroy(*out);
                *out = nullptr;
                throw tapt::CudaError(msg);
            }
        }
    });
}

// New ladder values for the same slots (e.g. a simulated-annealing stage).  A ladder that is
// not strictly increasing is accepted only with allow_flat (swaps must then stay disabled:
// equal neighbours have c = 0 rows that accept every swap).
tapt_status tapt_ensemble_set_betas(tapt_ensemble_t e, const double* betas, int allow_flat) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            e->rx->set_betas(std::vector<double>(betas, betas + e->R), [&] {
                for (int r = 0; r < e->R; ++r) {
                    if (!(betas[r] >= 0.0) || !std::isfinite(betas[r])) throw tapt::ConfigError("beta must be >= 0");
                    if (r && !(betas[r] > betas[r - 1]) && !(allow_flat == 1 && betas[r] >= betas[r - 1]) && allow_flat != 2)
                        throw tapt::ConfigError("beta ladder must be strictly increasing (SPEC.md:388)");
                }
                bool dec = false;
                for (int r = 1; r < e->R; ++r) dec = dec || betas[r] < betas[r - 1];
                return dec;
            }());
            e->betas.assign(betas, betas + e->R);
            return;
        }
        for (int r = 0; r < e->R; ++r) {
            if (!(betas[r] >= 0.0) || !std::isfinite(betas[r])) throw tapt::ConfigError("beta must be >= 0");
            if (r && !(betas[r] > betas[r - 1]) && !(allow_flat == 1 && betas[r] >= betas[r - 1]) && allow_flat != 2)
                throw tapt::ConfigError("beta ladder must be strictly increasing (SPEC.md:388)");
        }
        // Eq. 1 with equal neighbours accepts every swap (exp(0) = 1), which the c = 0 rows do; a
        // decreasing pair would need exp(c dE) with c < 0, which the tables clamp to "always"
        bool decreasing = false;
        for (int r = 1; r < e->R; ++r) decreasing = decreasing || betas[r] < betas[r - 1];
        CUDA_OK(cudaStreamSynchronize(e->stream));
        e->betas.assign(betas, betas + e->R);
        e->ladder_unordered = decreasing;
        e->build_tables();
        sync_if(e->stream);
    });
}

tapt_status tapt_ensemble_set_streams(tapt_ensemble_t e, const uint64_t* states) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            if (!states) throw tapt::ConfigError("null stream states");
            e->rx->set_streams(states);
            sync_if(e->stream);
            return;
        }
        if (!states) throw tapt::ConfigError("null stream states");
        e->streams.upload(states, (size_t)e->I * e->R, e->stream);
        sync_if(e->stream);
    });
}

tapt_status tapt_ensemble_init_from_streams(tapt_ensemble_t e, const uint64_t* init_states) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            if (!init_states) throw tapt::ConfigError("null stream states");
            e->rx->init_from_streams(init_states);
            return;
        }
        if (!init_states) throw tapt::ConfigError("null stream states");
        DevBuf<uint64_t> ds;
        ds.upload(init_states, (size_t)e->I * e->R, e->stream);
        std::vector<uint8_t> perm((size_t)e->I * e->R);
        for (uint32_t i = 0; i < e->I; ++i)
            for (int r = 0; r < e->R; ++r) perm[(size_t)i * e->R + r] = (uint8_t)r;
        e->slot_of.upload(perm, e->stream);
        e->buf_of.upload(perm, e->stream);
        const int n = e->n();
        ++g_launches;
        k_init_random<<<dim3((n + 255) / 256, e->G, e->I), 256, 0, e->stream>>>(e->words.p, n, e->G, e->W, e->R, ds.p,
                                                                                e->clamp_ptr(), e->clamp_count());
        CUDA_OK(cudaGetLastError());
        e->recompute_energies();
        e->update_best_from_E();
        sync_if(e->stream);
    });
}

tapt_status tapt_ensemble_destroy(tapt_ensemble_t e) {
    return guard([&] {
        if (!e) return;
        cudaStreamSynchronize(e->stream);
        if (e->own_stream) cudaStreamDestroy(e->stream);
        delete e;
    });
}

tapt_status tapt_ensemble_set_stream(tapt_ensemble_t e, void* s) {
    return guard([&] {
        check_ens(e);
        CUDA_OK(cudaStreamSynchronize(e->stream));
        if (e->own_stream) cudaStreamDestroy(e->stream);
        if (s) {
            e->stream = static_cast<cudaStream_t>(s);
            e->own_stream = false;
        } else {
            CUDA_OK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
            e->own_stream = true;
        }
        if (e->rx) e->rx->set_stream(e->stream);
    });
}

tapt_status tapt_ensemble_synchronize(tapt_ensemble_t e) {
    return guard([&] {
        check_ens(e);
        e->poll_sched(true);
        CUDA_OK(cudaStreamSynchronize(e->stream));
    });
}

tapt_status tapt_ensemble_launch_log(tapt_ensemble_t e, char* buf, size_t cap) {
    return guard([&] {
        check_ens(e);
        if (!buf || cap == 0) throw tapt::ConfigError("null buffer");
        std::string all;
        for (const auto& s : e->launch_log) all += s + "\n";
        if (e->rx) all += std::string(e->rx->kernel_name()) + "\n";
        if (all.size() + 1 > cap) throw tapt::SizeError("launch log buffer too small");
        std::memcpy(buf, all.c_str(), all.size() + 1);
    });
}

const char* tapt_ensemble_kernel(tapt_ensemble_t e) {
    if (!e) return "csr";
    if (e->rx) return "real";
    if (e->use_k1) return "lattice";
    try {
        return e->k3_eligible() ? "bitcsr" : e->k4_eligible() ? "levels" : "csr";
    } catch (...) {
        return "csr";
    }
}

tapt_status tapt_ensemble_set_bond_signs(tapt_ensemble_t e, const int8_t* signs, size_t n_bonds) {
    return guard([&] {
        check_ens(e);
        if (e->rx) throw tapt::ConfigError("bond signs apply to integer lattice models (this model has real-valued couplings)");
        tapt_model_s* m = e->m;
        if (!m->lattice) throw tapt::ConfigError("bond signs apply to lattice models only");
        if (n_bonds != m->nbonds) throw tapt::DimensionError("bond count mismatch");
        for (size_t k = 0; k < (size_t)e->I * n_bonds; ++k)
            if (signs[k] != 1 && signs[k] != -1) throw tapt::ConfigError("bond signs must be +-1");
        e->signs.upload(signs, (size_t)e->I * n_bonds, e->stream);
        e->have_disorder = true;
        const int n = (int)m->n;
        if (e->use_k1) {
            e->bonds.alloc((size_t)e->I * n);
            ++g_launches;
            k_bond_bytes<<<dim3((n + 255) / 256, e->I), 256, 0, e->stream>>>(e->signs.p, e->bonds.p, m->ld, n);
            CUDA_OK(cudaGetLastError());
        } else {
            const int nnz = (int)m->col.size();
            e->csrJ.alloc((size_t)e->I * nnz);
            e->k3_ipb = -1;  // per-instance couplings: K2 only
            e->k4_ipb = -1;
            e->k1_units = -1;
            ++g_launches;
            k_csr_from_signs<<<dim3((nnz + 255) / 256, e->I), 256, 0, e->stream>>>(
                e->signs.p, (int)n_bonds, m->d_adjbond.p, nnz, m->J0, e->csrJ.p);
            CUDA_OK(cudaGetLastError());
        }
        e->recompute_energies();
        sync_if(e->stream);
    });
}

tapt_status tapt_ensemble_generate_ea_disorder(tapt_ensemble_t e, uint64_t disorder_seed) {
    return guard([&] {
        check_ens(e);
        if (e->rx) throw tapt::ConfigError("EA disorder applies to integer lattice models (this model has real-valued couplings)");
        tapt_model_s* m = e->m;
        if (!m->lattice || m->boundary != TAPT_BOUNDARY_PERIODIC || m->lx <= 2 || m->ly <= 2)
            throw tapt::ConfigError("EA disorder generation needs a periodic lattice with L > 2");
        if (m->nbonds != (uint32_t)m->dim * m->n) throw tapt::GeometryError("unexpected bond count");
        std::vector<uint64_t> st(e->I);
        for (uint32_t i = 0; i < e->I; ++i)
            st[i] = tapt::RngStream::derive(disorder_seed, {tapt::stream::kDisorder, e->gid0 + i}).state();
        DevBuf<uint64_t> ds;
        ds.upload(st, e->stream);
        DevBuf<int8_t> sg;
        sg.alloc((size_t)e->I * m->nbonds);
        const int n = (int)m->n;
        ++g_launches;
        k_ea_signs<<<dim3((n + 255) / 256, e->I), 256, 0, e->stream>>>(sg.p, n, m->dim, ds.p);
        CUDA_OK(cudaGetLastError());
        std::vector<int8_t> h = sg.download(e->stream);
        if (m->J0 != 0 && m->Jsign < 0)
            for (auto& v : h) v = (int8_t)-v;
        tapt_status s = tapt_ensemble_set_bond_signs(e, h.data(), m->nbonds);
        if (s != TAPT_OK) throw tapt::CudaError(g_last_error);
    });
}

tapt_status tapt_ensemble_get_bond_signs(tapt_ensemble_t e, int8_t* signs, size_t n_bonds) {
    return guard([&] {
        check_ens(e);
        if (e->rx) throw tapt::ConfigError("bond signs apply to integer lattice models");
        if (n_bonds != e->m->nbonds) throw tapt::DimensionError("bond count mismatch");
        if (!e->signs.p) {
            std::fill(signs, signs + (size_t)e->I * n_bonds, (int8_t)1);
            return;
        }
        auto h = e->signs.download(e->stream);
        std::copy(h.begin(), h.end(), signs);
    });
}

tapt_status tapt_ensemble_set_clamps(tapt_ensemble_t e, const int8_t* clamps) {
    return guard([&] {
        check_ens(e);
        if (e->rx) throw tapt::ConfigError("per-instance clamps need integer couplings; clamp the model instead");
        const uint32_t n = e->m->n;
        for (uint32_t i = 0; i < e->I; ++i)
            for (uint32_t s = 0; s < n; ++s) {
                const int8_t v = clamps[(size_t)i * n + s];
                if (v != 0 && v != 1 && v != -1) throw tapt::ConfigError("clamp value must be ±1");
                if ((v != 0) != (e->m->clamp[s] != 0))
                    throw tapt::ClampedSiteError("per-instance clamps must cover exactly the model's clamped sites");
            }
        e->clampval.upload(clamps, (size_t)e->I * n, e->stream);
        sync_if(e->stream);
    });
}

tapt_status tapt_ensemble_init_random(tapt_ensemble_t e) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            e->rx->init_random();
            return;
        }
        std::vector<uint64_t> st((size_t)e->I * e->R);
        for (uint32_t i = 0; i < e->I; ++i)
            for (int r = 0; r < e->R; ++r)
                st[(size_t)i * e->R + r] =
                    tapt::RngStream::derive(e->seed, {tapt::stream::kInit, e->gid0 + i, (uint64_t)r}).state();
        DevBuf<uint64_t> ds;
        ds.upload(st, e->stream);
        std::vector<uint8_t> perm((size_t)e->I * e->R);
        for (uint32_t i = 0; i < e->I; ++i)
            for (int r = 0; r < e->R; ++r) perm[(size_t)i * e->R + r] = (uint8_t)r;
        e->slot_of.upload(perm, e->stream);
        e->buf_of.upload(perm, e->stream);
        const int n = e->n();
        ++g_launches;
        k_init_random<<<dim3((n + 255) / 256, e->G, e->I), 256, 0, e->stream>>>(e->words.p, n, e->G, e->W, e->R, ds.p,
                                                                                e->clamp_ptr(), e->clamp_count());
        CUDA_OK(cudaGetLastError());
        e->recompute_energies();
        e->update_best_from_E();
        sync_if(e->stream);
    });
}

static void set_spins_impl(tapt_ensemble_t e, const int8_t* spins, bool force_clamps) {
    const int n = e->n();
    DevBuf<int8_t> d;
    d.upload(spins, (size_t)e->I * e->R * n, e->stream);
    ++g_launches;
    k_set_spins<<<dim3((n + 255) / 256, e->G, e->I), 256, 0, e->stream>>>(
        e->words.p, n, e->G, e->W, e->R, e->slot_of.p, d.p, e->R, force_clamps ? e->clamp_ptr() : nullptr,
        e->clamp_count());
    CUDA_OK(cudaGetLastError());
    e->recompute_energies();
    e->update_best_from_E();
    sync_if(e->stream);
}

tapt_status tapt_ensemble_set_spins(tapt_ensemble_t e, const int8_t* spins) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            e->rx->set_spins(spins, true);
            return;
        }
        set_spins_impl(e, spins, true);
    });
}

tapt_status tapt_ensemble_get_spins(tapt_ensemble_t e, int8_t* spins) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            e->rx->get_spins(spins);
            return;
        }
        e->poll_sched(true);
        const int n = e->n();
        DevBuf<int8_t> d;
        d.alloc((size_t)e->I * e->R * n);
        ++g_launches;
        k_get_spins<<<dim3((n + 255) / 256, e->R, e->I), 256, 0, e->stream>>>(e->words.p, n, e->G, e->W, e->R,
                                                                             e->buf_of.p, e->R, d.p);
        CUDA_OK(cudaGetLastError());
        CUDA_OK(cudaMemcpyAsync(spins, d.p, d.n, cudaMemcpyDeviceToHost, e->stream));
        sync_if(e->stream);
    });
}

tapt_status tapt_ensemble_get_spins_packed(tapt_ensemble_t e, uint8_t* packed) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            e->rx->get_spins_packed(packed);
            return;
        }
        e->poll_sched(true);
        const int n = e->n(), nb = (n + 7) / 8;
        DevBuf<uint8_t> d;
        d.alloc((size_t)e->I * e->R * nb);
        ++g_launches;
        k_get_packed<<<dim3((nb + 255) / 256, e->R, e->I), 256, 0, e->stream>>>(e->words.p, n, e->G, e->W,
                                                                               e->buf_of.p, e->R, d.p);
        CUDA_OK(cudaGetLastError());
        CUDA_OK(cudaMemcpyAsync(packed, d.p, d.n, cudaMemcpyDeviceToHost, e->stream));
        sync_if(e->stream);
    });
}

tapt_status tapt_ensemble_get_energies(tapt_ensemble_t e, int64_t* out) {
    return guard([&] {
        check_ens(e);
        if (e->rx) throw tapt::NumericError("energies are real-valued for this model: use tapt_ensemble_get_energies_f64");
        e->poll_sched(true);
        auto E = e->E.download(e->stream);
        auto bo = e->buf_of.download(e->stream);
        for (uint32_t i = 0; i < e->I; ++i)
            for (int r = 0; r < e->R; ++r)
                out[(size_t)i * e->R + r] = E[(size_t)i * e->R + bo[(size_t)i * e->R + r]];
    });
}

tapt_status tapt_ensemble_get_permutation(tapt_ensemble_t e, uint8_t* out) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            e->rx->get_permutation(out);
            return;
        }
        e->poll_sched(true);
        auto bo = e->buf_of.download(e->stream);
        std::copy(bo.begin(), bo.end(), out);
    });
}

tapt_status tapt_ensemble_counters(tapt_ensemble_t e, uint64_t* sweeps, uint64_t* passes, uint64_t* rounds) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            e->rx->counters(sweeps, passes, rounds);
            return;
        }
        if (sweeps) *sweeps = e->T;
        if (passes) *passes = e->P;
        if (rounds) *rounds = e->Q;
    });
}

tapt_status tapt_get_acceptance(tapt_ensemble_t e, uint64_t* sa, uint64_t* sc, uint64_t* pa, uint64_t* pc) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            e->rx->acceptance(sa, sc, pa, pc);
            return;
        }
        e->poll_sched(true);
        const size_t np = (size_t)e->I * (e->R - 1);
        if (sa && np) {
            std::copy_n(e->swap_att.download(e->stream).begin(), np, sa);
            for (size_t q = 0; q < np; ++q) sa[q] += e->fused_passes[(q % (e->R - 1)) & 1];
        }
        if (sc && np) std::copy_n(e->swap_acc.download(e->stream).begin(), np, sc);
        if (pa) {
            auto v = e->prop_att.download(e->stream);
            std::copy(v.begin(), v.end(), pa);
        }
        if (pc) {
            auto v = e->prop_acc.download(e->stream);
            std::copy(v.begin(), v.end(), pc);
        }
    });
}

tapt_status tapt_get_observables(tapt_ensemble_t e, int64_t* obs) {
    return guard([&] {
        check_ens(e);
        if (e->rx) throw tapt::NumericError("observables are real-valued for this model: use tapt_get_observables_f64");
        e->poll_sched(true);
        auto v = e->obs.download(e->stream);
        std::copy(v.begin(), v.end(), obs);
    });
}

tapt_status tapt_set_histogram(tapt_ensemble_t e, int64_t e_lo, int64_t width, uint32_t nbins) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            if (width < 1) throw tapt::ConfigError("histogram bin width must be >= 1");
            e->rx->set_histogram((double)e_lo, (double)width, nbins);
            return;
        }
        if (width < 1) throw tapt::ConfigError("histogram bin width must be >= 1");
        e->e_lo = e_lo;
        e->width = width;
        e->nbins = (int)nbins;
        e->hist.alloc((size_t)e->R * nbins);
        e->hist.zero(e->stream);
        sync_if(e->stream);
    });
}

tapt_status tapt_get_histogram(tapt_ensemble_t e, uint64_t* dst, int on_device) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            e->rx->get_histogram(dst, on_device != 0);
            return;
        }
        e->poll_sched(true);
        if (!e->nbins) throw tapt::ConfigError("no histogram configured");
        CUDA_OK(cudaMemcpyAsync(dst, e->hist.p, e->hist.n * sizeof(uint64_t),
                                on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, e->stream));
        sync_if(e->stream);
    });
}

tapt_status tapt_get_best(tapt_ensemble_t e, int64_t* best) {
    return guard([&] {
        check_ens(e);
        if (e->rx) throw tapt::NumericError("energies are real-valued for this model: use tapt_get_best_f64");
        e->poll_sched(true);
        auto v = e->best.download(e->stream);
        for (uint32_t i = 0; i < e->I; ++i) best[i] = v[i];
    });
}

tapt_status tapt_reset_observables(tapt_ensemble_t e) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            e->rx->reset_observables();
            return;
        }
        e->obs.zero(e->stream);
        e->hist.zero(e->stream);
        sync_if(e->stream);
    });
}

tapt_status tapt_ensemble_get_energies_f64(tapt_ensemble_t e, double* out) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            e->rx->get_energies(out);
            return;
        }
        std::vector<int64_t> v((size_t)e->I * e->R);
        if (tapt_ensemble_get_energies(e, v.data()) != TAPT_OK) throw tapt::CudaError(g_last_error);
        for (size_t k = 0; k < v.size(); ++k) out[k] = (double)v[k];
    });
}

tapt_status tapt_get_observables_f64(tapt_ensemble_t e, double* obs) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            e->rx->observables(obs);
            return;
        }
        e->poll_sched(true);
        auto v = e->obs.download(e->stream);
        for (size_t k = 0; k < v.size(); ++k) obs[k] = (double)v[k];
    });
}

tapt_status tapt_get_best_f64(tapt_ensemble_t e, double* best) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            e->rx->best(best);
            return;
        }
        e->poll_sched(true);
        auto v = e->best.download(e->stream);
        for (uint32_t i = 0; i < e->I; ++i) best[i] = v[i];
    });
}

tapt_status tapt_ensemble_near_ties(tapt_ensemble_t e, uint64_t* ties, uint64_t* replays) {
    return guard([&] {
        check_ens(e);
        if (ties) *ties = e->rx ? e->rx->ties_seen() : 0;
        if (replays) *replays = e->rx ? e->rx->replays() : 0;
    });
}

tapt_status tapt_sweep(tapt_ensemble_t e, uint32_t n_sweeps) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            e->rx->run(n_sweeps, 0, 0, 0);
            return;
        }
        e->run(n_sweeps, 0, 0, 0);
    });
}

tapt_status tapt_swap_pass(tapt_ensemble_t e, int parity) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            if (parity != 0 && parity != 1) throw tapt::ConfigError("parity must be 0 or 1");
            e->rx->swap_pass(parity);
            return;
        }
        if (parity != 0 && parity != 1) throw tapt::ConfigError("parity must be 0 or 1");
        if (e->swap_oversize) throw tapt::ConfigError("beta spacing too fine for exact swap tables");
        if (e->ladder_unordered)
            throw tapt::ConfigError("replica swaps need a non-decreasing beta ladder (SPEC.md:388); the "
                                    "current ladder (set with allow_flat=2) has a decreasing neighbour pair");
        if (e->R >= 2) {
            ++g_launches;
            k_swap_pass<<<e->I, std::max(32, (e->R / 2 + 31) / 32 * 32), 0, e->stream>>>(
                e->E.p, e->slot_of.p, e->buf_of.p, e->R, e->coord.p, e->P, parity, e->swap_tab.view(), e->swap_att.p,
                e->swap_acc.p);
            CUDA_OK(cudaGetLastError());
        }
        e->P += 1;
    });
}

tapt_status tapt_run(tapt_ensemble_t e, const tapt_schedule* s) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            if (!s) throw tapt::ConfigError("null schedule");
            e->rx->run(s->n_sweeps, s->swap_every, s->measure_every, s->measure_from);
            return;
        }
        if (!s) throw tapt::ConfigError("null schedule");
        if (s->measure_every && !e->obs.p) throw tapt::ConfigError("observables not allocated");
        e->run(s->n_sweeps, s->swap_every, s->measure_every, s->measure_from);
    });
}

}  // extern "C"

// ------------------------------------------------------------- proposals ---

namespace {

// Energies of the proposal set (buffers t = 0..T-1 at slots targets[t]), then
// Metropolis (Eq. 2) and application.  pwords holds the proposals.
void finish_proposals(tapt_ensemble_s* e, const uint32_t* targets, uint32_t T, bool have_energies,
                      const double* lqc, const double* lqp, uint8_t* accepted) {
    const int n = e->n();
    const int WT = std::min<int>((int)T, kW), GT = ((int)T + kW - 1) / kW;
    // proposal energies
    if (!have_energies) {
        if (e->use_k1) {
            PTArgs a = e->base_args();
            a.words = e->pwords.p;
            a.G = GT;
            a.W = WT;
            a.B = (int)T;
            a.slot_of = e->pslot.p;
            a.buf_of = nullptr;
            a.E = e->pE.p;
            a.energy_only = 1;
            a.n_sweeps = 0;
            a.swap_every = 0;
            a.measure_every = 0;
            a.best = nullptr;
            ++g_launches;
            cudaError_t err = launch_k1(a, e->m->ld, e->k1_threads, false, e->stream);
            if (err != cudaSuccess) throw tapt::CudaError(cudaGetErrorString(err));
        } else {
            CsrArgs g = e->csr_args(false);
            ++g_launches;
            k_energy_csr<<<dim3(GT, e->I), 256, 0, e->stream>>>(e->pwords.p, n, GT, WT, (int)T, g.rowptr, g.col, g.J,
                                                                 g.nJ, g.nnz, g.h, e->pE.p);
        }
        CUDA_OK(cudaGetLastError());
    }
    // accept streams for this round (derived on the device: {kCoordinator, gid, round})
    e->paccs.alloc(e->I);
    ++g_launches;
    k_derive_round_streams<<<e->I, 32, 0, e->stream>>>(e->seed, e->gid0, e->ptargets.p, 0, e->R, e->Q + 1, nullptr,
                                                       nullptr, e->paccs.p);
    CUDA_OK(cudaGetLastError());
    e->pacc.alloc((size_t)e->I * T);
    const uint8_t* forced = nullptr;
    if (lqc) {
        // MH correction: decided on the device (k_decide_mh); only a draw within 1e-12 (relative) of the
        // acceptance probability -- where the device exp could disagree with glibc -- sends the round to
        // the host path below, so the usual round reads back four bytes instead of three arrays.
        const size_t IT = (size_t)e->I * T;
        e->plq.alloc(2 * IT);
        CUDA_OK(cudaMemcpyAsync(e->plq.p, lqc, IT * sizeof(double), cudaMemcpyHostToDevice, e->stream));
        CUDA_OK(cudaMemcpyAsync(e->plq.p + IT, lqp, IT * sizeof(double), cudaMemcpyHostToDevice, e->stream));
        if (e->dbetas.n != (size_t)e->R || e->dbetas_host != e->betas) {
            e->dbetas.upload(e->betas, e->stream);
            e->dbetas_host = e->betas;
        }
        e->pforced.alloc(IT);
        e->pties.alloc(1);
        e->pties.zero(e->stream);
        ++g_launches;
        k_decide_mh<<<e->I, std::max(32, ((int)T + 31) / 32 * 32), 0, e->stream>>>(
            e->E.p, e->buf_of.p, e->R, e->pE.p, (int)T, e->ptargets.p, e->paccs.p, e->dbetas.p, e->plq.p,
            e->plq.p + IT, e->pforced.p, e->pties.p);
        CUDA_OK(cudaGetLastError());
        uint32_t ties = e->pties.download(e->stream)[0];
        if (std::getenv("TAPT_MH_HOST")) ties = 1;  // tests: force the glibc path
        e->mh_tie_rounds += ties ? 1 : 0;
        if (ties) {  // decide the whole round on the host with glibc exp (bit-exact with the oracle)
            std::vector<uint64_t> as(e->I);
            for (uint32_t i = 0; i < e->I; ++i)
                as[i] = tapt::RngStream::derive(e->seed, {tapt::stream::kCoordinator, e->gid0 + i, e->Q + 1}).state();
            std::vector<int32_t> Ep = e->pE.download(e->stream);
            std::vector<int32_t> Eb = e->E.download(e->stream);
            std::vector<uint8_t> bo = e->buf_of.download(e->stream);
            std::vector<uint8_t> f(IT);
            for (uint32_t i = 0; i < e->I; ++i)
                for (uint32_t t = 0; t < T; ++t) {
                    const uint32_t r = targets[t];
                    const double ec = Eb[(size_t)i * e->R + bo[(size_t)i * e->R + r]];
                    const double ep = Ep[(size_t)i * T + t];
                    const double a = std::exp(e->betas[r] * (ec - ep)) *
                                     std::exp(lqc[(size_t)i * T + t] - lqp[(size_t)i * T + t]);
                    const uint64_t x = tapt::RngStream::from_state(as[i]).at(r + 1);
                    const double u = (double)(x >> 11) * 0x1.0p-53;
                    f[(size_t)i * T + t] = u < a ? 1 : 0;
                }
            e->pforced.upload(f, e->stream);
        }
        forced = e->pforced.p;
    }
    ++g_launches;
    k_accept_proposals<<<e->I, std::max(32, ((int)T + 31) / 32 * 32), 0, e->stream>>>(
        e->E.p, e->buf_of.p, e->R, e->pE.p, (int)T, e->ptargets.p, e->paccs.p, e->prop_tab.view(), forced, e->pacc.p,
        e->prop_att.p, e->prop_acc.p);
    CUDA_OK(cudaGetLastError());
    ++g_launches;
    k_apply_proposals<<<dim3((n + 255) / 256, e->G, e->I), 256, 0, e->stream>>>(
        e->words.p, n, e->G, e->W, e->buf_of.p, e->R, e->pwords.p, GT, WT, e->ptargets.p, (int)T, e->pacc.p);
    CUDA_OK(cudaGetLastError());
    e->update_best_from_E();
    if (accepted) {  // synchronous copy into the caller's buffer; otherwise the round stays stream-ordered
        auto a = e->pacc.download(e->stream);
        std::copy(a.begin(), a.end(), accepted);
    }
    e->Q += 1;
}

void prepare_targets(tapt_ensemble_s* e, const uint32_t* targets, uint32_t T) {
    if (e->prop_oversize) throw tapt::ConfigError("beta too small for exact proposal tables");
    if (T == 0 || T > (uint32_t)e->R) throw tapt::ConfigError("n_targets must be in [1, n_slots]");
    std::vector<uint8_t> seen(e->R, 0);
    for (uint32_t t = 0; t < T; ++t) {
        if (targets[t] >= (uint32_t)e->R) throw tapt::ConfigError("target slot out of range");
        if (seen[targets[t]]++) throw tapt::ConfigError("duplicate target slot");
    }
    const int n = e->n();
    const int GT = ((int)T + kW - 1) / kW;
    e->pwords.alloc((size_t)e->I * GT * n);
    e->pE.alloc((size_t)e->I * T);
    std::vector<uint32_t> tg(targets, targets + T);
    if (tg == e->last_targets && e->ptargets.n == T && e->pslot.n == (size_t)e->I * T) return;
    e->last_targets = tg;
    e->ptargets.upload(tg, e->stream);
    std::vector<uint8_t> ps((size_t)e->I * T);
    for (uint32_t i = 0; i < e->I; ++i)
        for (uint32_t t = 0; t < T; ++t) ps[(size_t)i * T + t] = (uint8_t)targets[t];
    e->pslot.upload(ps, e->stream);
}

}  // namespace

extern "C" {

tapt_status tapt_inject_proposals(tapt_ensemble_t e, const int8_t* proposals, int on_device, const uint32_t* targets,
                                  uint32_t T, const double* lqc, const double* lqp, uint8_t* accepted) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            e->rx->inject(proposals, on_device != 0, targets, T, lqc, lqp, accepted);
            return;
        }
        if ((lqc == nullptr) != (lqp == nullptr)) throw tapt::ConfigError("log_q_cur and log_q_prop go together");
        prepare_targets(e, targets, T);
        const int n = e->n();
        const int WT = std::min<int>((int)T, kW), GT = ((int)T + kW - 1) / kW;
        const int8_t* src = proposals;
        if (!on_device) {
            e->pint8.upload(proposals, (size_t)e->I * T * n, e->stream);
            src = e->pint8.p;
        }
        ++g_launches;
        k_set_spins<<<dim3((n + 255) / 256, GT, e->I), 256, 0, e->stream>>>(e->pwords.p, n, GT, WT, (int)T, nullptr, src,
                                                                            (int)T, e->clamp_ptr(), e->clamp_count());
        CUDA_OK(cudaGetLastError());
        finish_proposals(e, targets, T, false, lqc, lqp, accepted);
        if (!on_device) sync_if(e->stream);  // the caller's host buffer (possibly pinned) is free on return
    });
}

// The refinement sweeps of a proposal round (BASELINE.json configs[1], configs[4]: M Gibbs sweeps of each
// proposal at its target's beta before Eq. 2): the proposal groups [I][GT][n] are swept by the sweep
// kernel with the round's slot streams derive(seed,{kReplica,g,r,q+1}) (e->pfull), draws offset past the
// n + 1 generator draws.  Leaves exact proposal energies in e->pE.  Returns whether it ran.
static bool refine_proposals(tapt_ensemble_s* e, uint32_t T, uint32_t refine) {
    if (!refine) return false;
    const int n = e->n();
    const int WT = std::min<int>((int)T, kW), GT = ((int)T + kW - 1) / kW;
    PTArgs a = e->base_args();
    a.words = e->pwords.p;
    a.G = GT;
    a.W = WT;
    a.B = (int)T;
    a.streams = e->pfull.p;
    a.slot_of = e->pslot.p;
    a.buf_of = nullptr;
    a.E = e->pE.p;
    a.draw_base = (uint64_t)n + 1;
    a.t0 = 0;
    a.n_sweeps = (int)refine;
    a.swap_every = 0;
    a.measure_every = 0;
    a.best = nullptr;
    if (!e->use_k1) {  // K2 tracks energies incrementally: seed them
        CsrArgs g = e->csr_args(false);
        ++g_launches;
        k_energy_csr<<<dim3(GT, e->I), 256, 0, e->stream>>>(e->pwords.p, n, GT, WT, (int)T, g.rowptr, g.col, g.J,
                                                             g.nJ, g.nnz, g.h, e->pE.p);
        CUDA_OK(cudaGetLastError());
    }
    // refinement sweeps of the proposal groups: I x GT CTAs of their own; when they exceed the SMs
    // but fit two 256-thread CTAs per SM, one wave of those beats two of 512-thread CTAs
    // (config 2: 128 x 2 groups)
    int nt = 0;
    if (e->use_k1 && e->k1_threads == 512 && k1_smem_bytes(n, true, e->R) <= (100 - (TAPT_K1_IDXS ? 18 : 0)) * 1024) {
        int dev = 0, nsm = 148;
        CUDA_OK(cudaGetDevice(&dev));
        CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        const long long ctas = (long long)e->I * GT;
        if (ctas > nsm && ctas <= 2ll * nsm) nt = 256;
    }
    e->launch(a, false, nt);
    return true;
}

static void inject_packed(tapt_ensemble_t e, const uint8_t* proposals, int on_device, const uint32_t* targets,
                          uint32_t T, uint32_t refine, uint8_t* accepted) {
    check_ens(e);
    if (e->rx) {
        e->rx->inject_packed(proposals, on_device != 0, targets, T, refine, accepted);
        return;
    }
    prepare_targets(e, targets, T);
    const int n = e->n(), nb = (n + 7) / 8;
    const int WT = std::min<int>((int)T, kW), GT = ((int)T + kW - 1) / kW;
    const uint8_t* src = proposals;
    if (!on_device) {
        e->pbytes.upload(proposals, (size_t)e->I * T * nb, e->stream);
        src = e->pbytes.p;
    }
    ++g_launches;
    k_set_packed<<<dim3((n + 255) / 256, GT, e->I), 256, 0, e->stream>>>(e->pwords.p, n, GT, WT, (int)T, src, (int)T,
                                                                         e->clamp_ptr(), e->clamp_count());
    CUDA_OK(cudaGetLastError());
    if (refine) {  // the round's slot streams for the refinement sweeps
        e->pstreams.alloc((size_t)e->I * T);
        if (e->pfull.n != (size_t)e->I * e->R) {
            e->pfull.alloc((size_t)e->I * e->R);
            e->pfull.zero(e->stream);
        }
        ++g_launches;
        k_derive_round_streams<<<e->I, 64, 0, e->stream>>>(e->seed, e->gid0, e->ptargets.p, (int)T, e->R, e->Q + 1,
                                                           e->pstreams.p, e->pfull.p, nullptr);
        CUDA_OK(cudaGetLastError());
    }
    const bool have_E = refine_proposals(e, T, refine);
    finish_proposals(e, targets, T, have_E, nullptr, nullptr, accepted);
    if (!on_device) sync_if(e->stream);  // the caller's host buffer (possibly pinned) is free on return
}

tapt_status tapt_inject_proposals_packed(tapt_ensemble_t e, const uint8_t* proposals, int on_device,
                                         const uint32_t* targets, uint32_t T, uint8_t* accepted) {
    return guard([&] { inject_packed(e, proposals, on_device, targets, T, 0, accepted); });
}

tapt_status tapt_inject_proposals_packed_refined(tapt_ensemble_t e, const uint8_t* proposals, int on_device,
                                                 const uint32_t* targets, uint32_t T, uint32_t refine,
                                                 uint8_t* accepted) {
    return guard([&] { inject_packed(e, proposals, on_device, targets, T, refine, accepted); });
}


tapt_status tapt_generate_proposals(tapt_ensemble_t e, const uint32_t* targets, uint32_t T, const double* m_bias,
                                    uint32_t refine, uint8_t* accepted) {
    return guard([&] {
        check_ens(e);
        if (e->rx) {
            e->rx->generate(targets, T, m_bias, refine, accepted);
            return;
        }
        prepare_targets(e, targets, T);
        const int n = e->n();
        const int WT = std::min<int>((int)T, kW), GT = ((int)T + kW - 1) / kW;
        // per (instance, target) proposal streams {kReplica, gid, target, round}, derived on the device
        // into [I][T] and slot-indexed [I][R] (the refinement sweeps); per (target, sign) bias thresholds
        std::vector<uint64_t> tup(2 * T);
        e->pstreams.alloc((size_t)e->I * T);
        if (e->pfull.n != (size_t)e->I * e->R) {
            e->pfull.alloc((size_t)e->I * e->R);
            e->pfull.zero(e->stream);
        }
        ++g_launches;
        k_derive_round_streams<<<e->I, 64, 0, e->stream>>>(e->seed, e->gid0, e->ptargets.p, (int)T, e->R, e->Q + 1,
                                                           e->pstreams.p, e->pfull.p, nullptr);
        CUDA_OK(cudaGetLastError());
        for (uint32_t t = 0; t < T; ++t) {
            const double mb = m_bias ? m_bias[t] : 0.0;
            tup[2 * t + 0] = threshold_of((1.0 + -1.0 * mb) / 2.0);
            tup[2 * t + 1] = threshold_of((1.0 + 1.0 * mb) / 2.0);
        }
        e->ptup.upload(tup, e->stream);
        ++g_launches;
        k_gen_proposals<<<dim3((n + 255) / 256, GT, e->I), 256, 0, e->stream>>>(
            e->pwords.p, n, GT, WT, (int)T, e->pstreams.p, e->ptup.p, e->clamp_ptr(), e->clamp_count());
        CUDA_OK(cudaGetLastError());
        const bool have_E = refine_proposals(e, T, refine);
        finish_proposals(e, targets, T, have_E, nullptr, nullptr, accepted);
    });
}

// ------------------------------------------------------------ drop-in sweep

static tapt_real::RealEngine& dropin_real(tapt_model_t m, double beta) {
    if (!m->dropin_real) {
        cudaStream_t st = nullptr;
        CUDA_OK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        m->dropin_stream = st;
        m->dropin_real = std::make_unique<tapt_real::RealEngine>(m->real_graph(), 1, 0, std::vector<double>{beta}, 0,
                                                                 TAPT_ORDER_REFERENCE, st);
    }
    return *m->dropin_real;
}

// gibbs_update (mcmc.cpp:24-28): one heat-bath update of site i with the stream's next draw, on the
// device (K5 with a one-site visit list).  Clamped site -> ClampedSiteError (local_field,
// spin_model.cpp:93), length mismatch -> DimensionError.
tapt_status tapt_gibbs_update(tapt_model_t m, int8_t* s, size_t len, uint32_t site, double beta, uint64_t* rng_state) {
    return guard([&] {
        check_model(m);
        if (len != m->n) throw tapt::DimensionError("configuration length mismatch");
        if (site >= m->n) throw tapt::ConfigError("site index out of range");
        if (m->clamp[site]) throw tapt::ClampedSiteError("spin " + std::to_string(site) + " is clamped");
        if (!(beta >= 0.0)) throw tapt::ConfigError("beta must be >= 0");
        if (!rng_state) throw tapt::ConfigError("null rng state");
        if (tapt_device_count() == 0) throw tapt::CudaError("no CUDA device: the TAPT engine has no CPU fallback");
        std::lock_guard<std::mutex> lock(m->dropin_mu);
        dropin_real(m, beta).dropin_update(s, site, beta, *rng_state, nullptr, 0, 0);
        *rng_state += tapt_dev::kPhi;
    });
}

tapt_status tapt_gibbs_sweep(tapt_model_t m, int8_t* s, size_t len, double beta, uint64_t* rng_state,
                             uint32_t n_sweeps, double* dE) {
    return guard([&] {
        check_model(m);
        if (len != m->n) throw tapt::DimensionError("configuration length mismatch");
        if (!(beta >= 0.0)) throw tapt::ConfigError("beta must be >= 0");
        if (!rng_state) throw tapt::ConfigError("null rng state");
        if (n_sweeps == 0) return;
        if (m->free_sites.empty()) {  // nothing to visit: no draws, dE = 0 (mcmc.cpp:34 loops over free_sites)
            if (dE) std::fill(dE, dE + n_sweeps, 0.0);
            return;
        }
        std::lock_guard<std::mutex> lock(m->dropin_mu);
        if (m->real || (dE && m->free_sites.size() <= 8192)) {
            // K5: the reference's sequential index order in FP64 with every sweep's dE, one launch
            // (real-valued couplings; integer ones decide by their exact tables).  Larger integer
            // graphs keep K4's parallel dependency levels (one launch and one readback per sweep).
            dropin_real(m, beta).dropin_sweeps(s, beta, *rng_state, n_sweeps, dE, nullptr, 0, 0);
            *rng_state += (uint64_t)n_sweeps * (uint64_t)m->free_sites.size() * tapt_dev::kPhi;
            return;
        }
        if (!m->dropin) {
            tapt_ensemble_desc d{};
            d.n_instances = 1;
            d.n_slots = 1;
            d.betas = &beta;
            d.seed = 0;
            d.order = TAPT_ORDER_REFERENCE;
            if (tapt_ensemble_create(m, &d, &m->dropin) != TAPT_OK) throw tapt::CudaError(g_last_error);
        } else if (m->dropin->betas[0] != beta) {
            if (tapt_ensemble_set_betas(m->dropin, &beta, 0) != TAPT_OK) throw tapt::ConfigError(g_last_error);
        }
        tapt_ensemble_t e = m->dropin;
        e->T = 0;  // draws are addressed from the caller's stream state
        e->P = 0;
        const uint64_t st = *rng_state;
        e->streams.upload(&st, 1, e->stream);
        // gibbs_sweep never writes clamped sites and reads whatever they hold (mcmc.cpp:34-37)
        set_spins_impl(e, s, false);
        int64_t e0 = 0;
        tapt_ensemble_get_energies(e, &e0);
        if (dE) {
            for (uint32_t k = 0; k < n_sweeps; ++k) {
                e->run(1, 0, 0, 0);
                int64_t e1 = 0;
                if (tapt_ensemble_get_energies(e, &e1) != TAPT_OK) throw tapt::CudaError(g_last_error);
                dE[k] = (double)(e1 - e0);
                e0 = e1;
            }
        } else {
            e->run(n_sweeps, 0, 0, 0);
        }
        if (tapt_ensemble_get_spins(e, s) != TAPT_OK) throw tapt::CudaError(g_last_error);
        *rng_state = st + (uint64_t)n_sweeps * (uint64_t)m->free_sites.size() * tapt_dev::kPhi;
    });
}

}  // extern "C"

// ============================================================== multi-GPU ===
// Instances are sharded across ranks (one process per GPU); replicas of an instance never span
// GPUs, so the only collectives are the end-of-run observable reductions: per-slot
// sums over every rank's instances, the per-slot energy histograms, and the global best energy --
// ncclAllReduce on the ensemble's stream over NVLink / NVSwitch.  NCCL is loaded at run time
// (dlopen "libnccl.so.2": the copy torch already mapped, else the system one), so the library has no
// link-time NCCL dependency and a missing NCCL is a TAPT_ERR_NCCL at the call.

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("NCCL not available: ") + dlerror();
            return;
        }
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
        api.comm_count = reinterpret_cast<decltype(api.comm_count)>(dlsym(h, "ncclCommCount"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!api.get_unique_id || !api.comm_init_rank || !api.comm_destroy || !api.all_reduce || !api.comm_count ||
            !api.all_gather)
            err = "NCCL library lacks the expected symbols";
    });
    if (!err.empty()) throw tapt::NcclError(err);
    return api;
}

void nccl_ok(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw tapt::NcclError(std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "error"));
}

// per-slot sums over the instances: obs [I][R][5] -> out [R][5]
__global__ void k_obs_slot_sums(const long long* obs, int I, int R, long long* out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= R * 5) return;
    long long v = 0;
    for (int i = 0; i < I; ++i) v += obs[(size_t)i * R * 5 + k];
    out[k] = v;
}
__global__ void k_best_min(const int* best, int I, long long* out) {
    long long m = 0x7FFFFFFFll;
    for (int i = threadIdx.x; i < I; i += blockDim.x) m = min(m, (long long)best[i]);
    for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    if (threadIdx.x == 0) *out = m;
}

}  // namespace

extern "C" {

tapt_status tapt_nccl_unique_id(uint8_t* id, size_t len) {
    return guard([&] {
        if (!id || len < NCCL_UNIQUE_ID_BYTES) throw tapt::ConfigError("unique id buffer must hold 128 bytes");
        ncclUniqueId u;
        nccl_ok(nccl().get_unique_id(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, NCCL_UNIQUE_ID_BYTES);
    });
}

tapt_status tapt_nccl_comm_create(const uint8_t* id, int n_ranks, int rank, void** comm) {
    return guard([&] {
        if (!id || !comm) throw tapt::ConfigError("null unique id / output");
        if (n_ranks < 1 || rank < 0 || rank >= n_ranks) throw tapt::ConfigError("bad rank / world size");
        if (tapt_device_count() == 0) throw tapt::CudaError("no CUDA device");
        ncclUniqueId u;
        std::memcpy(&u, id, NCCL_UNIQUE_ID_BYTES);
        ncclComm_t c = nullptr;
        nccl_ok(nccl().comm_init_rank(&c, n_ranks, u, rank), "ncclCommInitRank");
        *comm = c;
    });
}

tapt_status tapt_nccl_comm_destroy(void* comm) {
    return guard([&] {
        if (comm) nccl_ok(nccl().comm_destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
    });
}

tapt_status tapt_nccl_comm_size(void* comm, int* n_ranks) {
    return guard([&] {
        if (!comm || !n_ranks) throw tapt::ConfigError("null communicator / output");
        nccl_ok(nccl().comm_count(static_cast<ncclComm_t>(comm), n_ranks), "ncclCommCount");
    });
}

tapt_status tapt_allreduce_observables(tapt_ensemble_t e, void* comm, int64_t* obs, uint64_t* hist, int64_t* best) {
    return guard([&] {
        check_ens(e);
        if (!comm) throw tapt::NcclError("null NCCL communicator");
        if (e->rx) throw tapt::ConfigError("observable reductions of real-valued models: use the f64 getters per rank");
        e->poll_sched(true);
        const auto& api = nccl();
        ncclComm_t c = static_cast<ncclComm_t>(comm);
        const int R = e->R;
        DevBuf<long long> o, b;
        if (obs) {
            o.alloc((size_t)R * 5);
            ++g_launches;
            k_obs_slot_sums<<<(R * 5 + 127) / 128, 128, 0, e->stream>>>(e->obs.p, (int)e->I, R, o.p);
            CUDA_OK(cudaGetLastError());
            nccl_ok(api.all_reduce(o.p, o.p, o.n, ncclInt64, ncclSum, c, e->stream), "ncclAllReduce(observables)");
        }
        DevBuf<unsigned long long> h;  // the ensemble keeps its own (rank-local) histogram
        if (hist) {
            if (!e->nbins) throw tapt::ConfigError("no histogram configured");
            h.alloc(e->hist.n);
            nccl_ok(api.all_reduce(e->hist.p, h.p, h.n, ncclUint64, ncclSum, c, e->stream), "ncclAllReduce(histograms)");
        }
        if (best) {
            b.alloc(1);
            ++g_launches;
            k_best_min<<<1, 32, 0, e->stream>>>(e->best.p, (int)e->I, b.p);
            CUDA_OK(cudaGetLastError());
            nccl_ok(api.all_reduce(b.p, b.p, 1, ncclInt64, ncclMin, c, e->stream), "ncclAllReduce(best)");
        }
        if (obs) CUDA_OK(cudaMemcpyAsync(obs, o.p, o.n * sizeof(long long), cudaMemcpyDeviceToHost, e->stream));
        if (hist)
            CUDA_OK(cudaMemcpyAsync(hist, h.p, h.n * sizeof(uint64_t), cudaMemcpyDeviceToHost, e->stream));
        if (best) CUDA_OK(cudaMemcpyAsync(best, b.p, sizeof(long long), cudaMemcpyDeviceToHost, e->stream));
        CUDA_OK(cudaStreamSynchronize(e->stream));
    });
}

}  // extern "C"

extern "C" {

// Per-instance best energies of every rank's shard in global instance order ("per-
// instance results come back by ncclAllGather"): each rank contributes (instance_offset, count) and
// its best energies padded to the largest shard; out[gid] for gid in [0, total).  Shards may be any
// disjoint blocks that cover [0, total).
tapt_status tapt_allgather_best(tapt_ensemble_t e, void* comm, uint64_t total, int64_t* out) {
    return guard([&] {
        check_ens(e);
        if (!comm) throw tapt::NcclError("null NCCL communicator");
        if (!out) throw tapt::ConfigError("null output");
        if (e->rx) throw tapt::ConfigError("best energies of real-valued models: use tapt_get_best_f64 per rank");
        e->poll_sched(true);
        const auto& api = nccl();
        ncclComm_t c = static_cast<ncclComm_t>(comm);
        int world = 0;
        nccl_ok(api.comm_count(c, &world), "ncclCommCount");
        DevBuf<long long> meta, metas;
        meta.alloc(2);
        metas.alloc((size_t)2 * world);
        const long long mine[2] = {(long long)e->gid0, (long long)e->I};
        CUDA_OK(cudaMemcpyAsync(meta.p, mine, sizeof(mine), cudaMemcpyHostToDevice, e->stream));
        nccl_ok(api.all_gather(meta.p, metas.p, 2, ncclInt64, c, e->stream), "ncclAllGather(shards)");
        std::vector<long long> m((size_t)2 * world);
        CUDA_OK(cudaMemcpyAsync(m.data(), metas.p, m.size() * sizeof(long long), cudaMemcpyDeviceToHost, e->stream));
        CUDA_OK(cudaStreamSynchronize(e->stream));
        long long maxc = 0, sum = 0;
        for (int r = 0; r < world; ++r) {
            maxc = std::max(maxc, m[2 * r + 1]);
            sum += m[2 * r + 1];
            if (m[2 * r] < 0 || (uint64_t)(m[2 * r] + m[2 * r + 1]) > total)
                throw tapt::DimensionError("a rank's shard lies outside [0, total)");
        }
        if ((uint64_t)sum != total) throw tapt::DimensionError("the ranks' shards do not cover total instances");
        DevBuf<int> pad;
        DevBuf<int> all;
        pad.alloc((size_t)maxc);
        all.alloc((size_t)maxc * world);
        pad.zero(e->stream);
        CUDA_OK(cudaMemcpyAsync(pad.p, e->best.p, (size_t)e->I * sizeof(int), cudaMemcpyDeviceToDevice, e->stream));
        nccl_ok(api.all_gather(pad.p, all.p, (size_t)maxc, ncclInt32, c, e->stream), "ncclAllGather(best)");
        std::vector<int> h((size_t)maxc * world);
        CUDA_OK(cudaMemcpyAsync(h.data(), all.p, h.size() * sizeof(int), cudaMemcpyDeviceToHost, e->stream));
        CUDA_OK(cudaStreamSynchronize(e->stream));
        for (int r = 0; r < world; ++r)
            for (long long k = 0; k < m[2 * r + 1]; ++k) out[m[2 * r] + k] = h[(size_t)r * maxc + k];
    });
}

}  // extern "C"
