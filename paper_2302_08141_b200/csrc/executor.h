// executor.h — runtime, mesh and partitioned-program structures behind the C-ABI.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <functional>
#include <string>
#include <vector>

#include "common.h"
#include "kernels.h"

using Dims = std::vector<int64_t>;
using Specs = std::vector<rh_spec>;  // one per mesh axis

struct rh_runtime {
  int world = 1;
  bool dist = false;          // one process per GPU (torchrun)
  int first_rank = 0;         // global rank of local rank 0
  std::vector<int> rank_dev;  // local rank -> index into devs
  std::vector<int> devs;      // distinct CUDA device ids
  std::vector<cudaStream_t> streams;  // one per distinct device
  ncclComm_t world_comm = nullptr;    // dist only
  // Mesh-axis communicators (ncclCommSplit of world_comm), created once per (dims, axis) and
  // shared by every mesh with those dims: communicators are costly (NVLS/P2P resources).
  std::vector<std::pair<std::vector<int>, std::vector<ncclComm_t>>> axis_comms;
  int n_local() const { return static_cast<int>(rank_dev.size()); }
  cudaStream_t stream_of(int li) const { return streams[rank_dev[li]]; }
  int device_of(int li) const { return devs[rank_dev[li]]; }
};

struct rh_mesh {
  rh_runtime* rt = nullptr;
  std::vector<int> dims;
  std::vector<ncclComm_t> axis_comm;  // dist only: this process's communicator per axis
  std::vector<int> Coords(int rank) const;
  // Global ranks of `rank`'s group along `axis`, ordered by their coordinate on that axis.
  std::vector<int> Group(int axis, int rank) const;
};

namespace rh {

struct Tensor {
  int op = -1;
  Specs specs;
  Dims gdims;   // global shape
  Dims ldims;   // composed local shape
  int dtype = RH_F32;
  size_t bytes = 0;   // local bytes per rank
  size_t offset = 0;  // arena offset (identical on every rank: the arena is symmetric)
  int alias = -1;      // reshape pass-through: shares the storage of this tensor
  bool storage = true; // owns arena storage (false: alias or bufferless chain member)
  bool recycled = false;  // storage is reused by later tensors within a run (arena planner)
  int stage = -1;         // pipeline programs: the stage whose ranks hold it (-1: every rank)
  int64_t elems() const {
    int64_t n = 1;
    for (auto x : ldims) n *= x;
    return n;
  }
};

struct Step {
  enum Kind { kKernel = 0, kTransition = 1, kSync = 2 };
  int kind = kKernel;
  std::string name;
  int stage = -1;            // pipeline programs: ranks of this stage run it (-1 every rank,
                             // -2 a cross-stage transfer: its closure knows sender / receiver)
  int axis = -1;             // transitions: mesh axis (group) that must be synchronised
  bool p2p = false;          // transition reads peer buffers (needs pre/post group sync)
  bool post_sync = true;     // p2p only: false when a later p2p step on the same axis (same
                             // iteration) already orders the peers' next writes after our reads
  int sync_slot = -1;        // dist p2p: flag row of the barrier fused into the pull kernel
  double alg_bytes = 0, alg_flops = 0, wire_bytes = 0;
  int launches = 0;          // per rank per run
  double ms = 0;             // from the last profile
  std::vector<int> reads, writes;  // tensors (for the arena planner's liveness)
  bool async = false;  // dist p2p transition on the side stream, overlapping the compute
  int post_mode = 0;   // p2p post-barrier: 0 planned (elided when a later barrier orders it),
                       // 1 always (push: peers wrote this rank's destination), 2 never (the
                       // push phase of a two-phase transition: its unpack step's barrier orders it)
  bool no_async = false;  // must stay on the main stream (a two-phase transition's steps)
  int join = -1;       // async: main-stream step that first needs the result (-1: end of run)
  int async_id = -1;   // index into the program's fork/done events
  // Enqueue this step for local rank `li` on stream `s`; returns the launches issued.
  std::function<int(int li, cudaStream_t s)> run;
  // Optional one-time setup after the arena is allocated (device tables that hold arena
  // pointers, e.g. a grouped GEMM's TMA maps) and its teardown at program destruction.
  std::function<void(int li)> init, fini;
  // Peer-memory transitions (p2p, not NCCL): one pull per single-axis transition; several
  // independent transitions of one axis merged into this step run as one grouped launch.
  std::vector<std::function<PullArgs(int li)>> pulls;
  // Fine-grained layouts (LaunchFine): launch with the step's fused barrier and grid cap.
  std::function<int(int li, cudaStream_t s, const PeerSync& sync, int max_blocks)> fine;
};

// Output specs (one per mesh axis) of op i's local computation from its demanded input specs.
Specs NaturalSpecsOf(const rh_op* ops, int n_ops, int i, const std::vector<int>& mesh);

}  // namespace rh

struct rh_program {
  rh_mesh* mesh = nullptr;
  uint32_t flags = 0;
  int n_axes = 0;
  std::vector<rh_op> ops;
  std::vector<std::vector<int>> inputs;
  std::vector<std::vector<Specs>> in_specs;  // [op][slot] -> per axis
  std::vector<Specs> out_specs;
  std::vector<int> outputs;
  std::vector<int> order;

  std::vector<rh::Tensor> tensors;
  std::vector<int> out_tensor;  // op -> tensor index (-1: fused into a successor's kernel)
  std::vector<int> mat_tensor;  // op -> materialized Replicated tensor (outputs)
  std::vector<std::vector<int>> in_tensor;  // [op][slot] -> tensor the op's kernel consumed
  // Extra layouts requested by the caller (rh_reshard): (op, specs) -> tensor index.
  std::vector<std::pair<int, Specs>> requests;
  std::vector<int> request_tensors;
  std::vector<rh::Step> steps;

  // memory
  size_t arena_bytes = 0;
  size_t pool_bytes = 0;  // liveness-planned part of the arena (recycled intermediates)
  size_t flags_off = 0, counter_off = 0;
  size_t err_off = 0;  // bounded cross-GPU waits: first timed-out (me, member) pair (PeerSync)
  size_t sync_off = 0, epoch_off = 0;  // fused-barrier flag rows [slots][world] + run counter
  size_t e2e_sync_off = 0, e2e_epoch_off = 0;  // rh_program_run_host input gather: flag row + counter
  int n_sync_slots = 0;
  std::vector<char*> base;       // per local rank
  std::vector<char*> peer_base;  // per global rank (dist: IPC-mapped; local: = base)
  bool ipc_opened = false;
  std::vector<void*> owned;      // device allocations to free (per distinct device)
  std::vector<std::pair<size_t, std::vector<char>>> uploads;  // constant data (arena offset, bytes)
  size_t gemm_scratch_bytes = 0, gemm_scratch_off = 0;  // 3xTF32 / split-K / stream-K scratch (shared)
  size_t gemm_flags_off = 0;                             // stream-K flags (kGemmSkFlagBytes, zeroed)
  void* graph = nullptr;  // cudaGraphExec_t of one captured run (single-stream runtimes)
  // overlap (dist): side stream for async transitions + its own barrier state
  int n_async = 0;
  size_t side_flags_off = 0, side_counter_off = 0;
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t> fork_ev, done_ev;
  std::vector<std::vector<int>> joins_at;  // main step -> async ids to wait for before it
  bool warmed = false;    // one eager run precedes capture
  // rh_program_step_host staging for sharded inputs: [local rank] -> device buffer (grown, reused)
  std::vector<void*> in_stage;
  std::vector<size_t> in_stage_bytes;

  char* Ptr(const rh::Tensor& t, int global_rank) const { return peer_base[global_rank] + t.offset; }
  int LocalIndex(int global_rank) const;
  // pipeline programs (rh_program_load_pipeline)
  int pipeline_axis = -1;
  int n_stages = 1;
  std::vector<std::pair<int, int>> apply;  // {gradient op, parameter op}
  float lr = 0.f;
  int StageOf(int global_rank) const {
    return pipeline_axis < 0 ? -1 : mesh->Coords(global_rank)[pipeline_axis];
  }
};
