// Sequence-sharded decode for C++ hosts (no counterpart in the reference: SURVEY §8(e)).  One
// process per GPU; rank r holds [global | its middle shard | local] of a GLOBAL cache of
// `global_total` rows (shard boundaries: reattn_shard_range).  The library owns the NCCL
// communicator and issues both all-gathers of a step itself (reattn_shard_step), so the whole
// host path is this header over the C-ABI:
//
//   std::array<uint8_t, REATTN_COMM_ID_BYTES> id = reattn::ShardedDecoder::new_comm_id(); // rank 0
//   ... ship `id` to every rank (the launcher's store, MPI_Bcast, a file) ...
//   reattn::ShardedDecoder dec(local_cache, rope, n_head, cfg, global_total, world, rank, id);
//   dec.capture();                                     // optional: the step as one CUDA graph
//   DenseMatrix out = dec.step(q);                     // every rank: the full output
#pragma once

#include <array>
#include <cstdint>
#include <memory>

#include "reattn/dense_matrix.hpp"
#include "reattn/kv_cache.hpp"
#include "reattn/rope.hpp"
#include "reattn/runtime.hpp"
#include "reattn/selection.hpp"

namespace reattn {

class ShardedDecoder {
public:
    using CommId = std::array<std::uint8_t, REATTN_COMM_ID_BYTES>;

    static CommId new_comm_id() {
        CommId id{};
        gpu::check(reattn_comm_unique_id(id.data()));
        return id;
    }
    static std::pair<std::size_t, std::size_t> shard_range(std::size_t middle_len, std::size_t span_m,
                                                           int world, int rank) {
        std::uint64_t b = 0, n = 0;
        gpu::check(reattn_shard_range(middle_len, span_m, world, rank, &b, &n));
        return {b, n};
    }

    // collective over the `world` ranks
    ShardedDecoder(const SegmentedKvCache& local_cache, const RotaryTable& rope, std::size_t n_head,
                   const SelectionConfig& cfg, std::size_t global_total, int world, int rank,
                   const CommId& id)
        : n_head_(n_head), d_(local_cache.d_head()) {
        reattn_comm* c = nullptr;
        gpu::check(reattn_comm_create(gpu::context(), world, rank, id.data(), &c));
        comm_.reset(c);
        const reattn_selection_config sc = cfg.to_c();
        reattn_shard_plan* p = nullptr;
        gpu::check(reattn_shard_plan_create(gpu::context(), local_cache.device(), rope.device(),
                                            n_head, &sc, global_total, world, rank, &p));
        plan_.reset(p);
    }

    // the whole step (scan, NCCL all-gather, select, attend, NCCL all-gather, combine) as one
    // CUDA graph replayed by step(); collective
    void capture() { gpu::check(reattn_shard_capture(plan_.get(), comm_.get())); }

    // one decode step for q (1 x n_head*d, pre-rotation); collective; every rank gets the output
    DenseMatrix step(const DenseMatrix& q) {
        if (q.rows != 1 || q.cols != n_head_ * d_)
            throw std::invalid_argument("attend_step: query width != n_head * d_head");
        DenseMatrix out(1, n_head_ * d_);
        gpu::check(reattn_shard_run_host(plan_.get(), comm_.get(), q.values.data(), out.values.data()));
        return out;
    }

    reattn_step_stats stats() {
        reattn_step_stats st{};
        gpu::check(reattn_shard_stats(plan_.get(), &st, nullptr, nullptr));
        return st;
    }

private:
    struct PlanDel {
        void operator()(reattn_shard_plan* p) const { reattn_shard_plan_destroy(p); }
    };
    struct CommDel {
        void operator()(reattn_comm* c) const { reattn_comm_destroy(c); }
    };
    std::size_t n_head_, d_;
    std::unique_ptr<reattn_comm, CommDel> comm_;  // destroyed after the plan
    std::unique_ptr<reattn_shard_plan, PlanDel> plan_;
};

}  // namespace reattn
