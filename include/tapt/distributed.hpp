// tapt/distributed.hpp -- instance sharding across GPUs for C++ callers (one process per GPU).
//
// The reference parallelises over instances / repetitions with parallel_for and requires results to
// be independent of the worker count (proj/include/tapt/threading.hpp:10-35).  The
// B200 build shards the same way across GPUs: rank g owns a contiguous block of global instance ids
// (Shard), every RNG stream is keyed by the global id, so a sharded run equals the single-GPU run
// instance by instance; replicas never span GPUs, and the only collectives are the end-of-run
// observable reductions (Communicator::allreduce_observables, NCCL over NVLink / NVSwitch).
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <vector>

#include "tapt/spin_model.hpp"
#include "tapt_gpu.h"

namespace tapt {

struct Shard {
    std::uint64_t offset = 0, count = 0;
    // contiguous block of `total` global instance ids for `rank` of `world`
    static Shard of(std::uint64_t total, int world, int rank) {
        if (world < 1 || rank < 0 || rank >= world) throw ConfigError("bad world / rank");
        const std::uint64_t base = total / world, rem = total % world;
        Shard s;
        s.count = base + (std::uint64_t(rank) < rem ? 1 : 0);
        s.offset = std::uint64_t(rank) * base + std::min<std::uint64_t>(rank, rem);
        return s;
    }
};

// One process per GPU: make `device` current for the library on this thread before creating handles.
inline void set_device(int device) { throw_status(tapt_set_device(device)); }

struct ReducedObservables {
    std::vector<std::int64_t> obs;    // [R][5] count, sum E, sum E^2, sum |M|, sum M^2
    std::vector<std::uint64_t> hist;  // [R][nbins] (empty without a histogram)
    std::int64_t best = 0;
};

class Communicator {
  public:
    using UniqueId = std::array<std::uint8_t, 128>;
    static UniqueId unique_id() {  // on rank 0; broadcast the bytes out of band (MPI, a file, torch...)
        UniqueId id{};
        throw_status(tapt_nccl_unique_id(id.data(), id.size()));
        return id;
    }
    Communicator(const UniqueId& id, int n_ranks, int rank) {
        void* c = nullptr;
        throw_status(tapt_nccl_comm_create(id.data(), n_ranks, rank, &c));
        c_ = std::shared_ptr<void>(c, [](void* p) { tapt_nccl_comm_destroy(p); });
    }
    int size() const {
        int n = 0;
        throw_status(tapt_nccl_comm_size(c_.get(), &n));
        return n;
    }
    void* handle() const { return c_.get(); }
    // Sum / min over every rank's instances of an ensemble with R slots (hist needs nbins > 0).
    ReducedObservables allreduce_observables(tapt_ensemble_t e, std::size_t R, std::size_t nbins = 0) const {
        ReducedObservables r;
        r.obs.resize(R * 5);
        r.hist.resize(R * nbins);
        throw_status(tapt_allreduce_observables(e, c_.get(), r.obs.data(), nbins ? r.hist.data() : nullptr, &r.best));
        return r;
    }

    // Per-instance best energies of every rank, in global instance order.
    std::vector<std::int64_t> allgather_best(tapt_ensemble_t e, std::uint64_t total) const {
        std::vector<std::int64_t> out(total);
        throw_status(tapt_allgather_best(e, c_.get(), total, out.data()));
        return out;
    }

  private:
    std::shared_ptr<void> c_;
};

}  // namespace tapt
