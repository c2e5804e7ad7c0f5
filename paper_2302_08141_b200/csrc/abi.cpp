// abi.cpp — the extern "C" entry points of include/rhino_exec.h: runtime / mesh creation,
// program load (lowering + symmetric arena + CUDA-IPC peer mapping), execution, timing and
// host I/O.  No C++ exception crosses this boundary.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <tuple>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "executor.h"

namespace rh {
void LowerProgram(rh_program* p);
}

using rh::Fail;

namespace rh {
namespace {
thread_local bool g_pdl = false;
}
void SetPdl(bool on) { g_pdl = on; }
bool PdlEnabled() { return g_pdl; }
}  // namespace rh

namespace {

thread_local std::string g_err;

#define RH_NCCL(x)                                                                        \
  do {                                                                                    \
    ncclResult_t r_ = (x);                                                                \
    if (r_ != ncclSuccess)                                                                \
      ::rh::Fail(std::string("NCCL: ") + ncclGetErrorString(r_) + " (" #x ")", RH_ERR_NCCL); \
  } while (0)

template <typename F>
int Guard(F&& f) {
  try {
    f();
    return RH_OK;
  } catch (const rh::Error& e) {
    g_err = e.what();
    return e.status;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RH_ERR_INVALID;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev != prev) RH_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int64_t Prod(const Dims& d) {
  int64_t n = 1;
  for (auto x : d) n *= x;
  return n;
}

rh::ComposedMap MakeComposed(const rh_program* p, const rh::Tensor& t, int global_rank) {
  rh::ComposedMap m{};
  m.nd = static_cast<int>(t.gdims.size());
  for (int k = 0; k < m.nd; ++k) {
    m.gdims[k] = t.gdims[k];
    m.ldims[k] = t.ldims[k];
  }
  const std::vector<int> c = p->mesh->Coords(global_rank);
  for (int a = 0; a < p->n_axes; ++a) {
    if (t.specs[a].kind != RH_SHARD) continue;
    auto& x = m.ax[m.nshard++];
    x.dim = t.specs[a].dim;
    x.d = p->mesh->dims[a];
    x.stride = t.specs[a].stride;
    x.coord = c[a];
  }
  return m;
}

bool SameStream(const rh_runtime* rt) { return rt->streams.size() == 1; }

// Cross-rank ordering around a transition that reads peer buffers.
// `side`: the barrier of an async transition, on the side stream with its own flag/counter
// state (the main and side streams' barriers interleave differently on every rank, but each
// stream's sequence is the same on all ranks).
void GroupSync(rh_program* p, int axis, bool side = false) {
  rh_runtime* rt = p->mesh->rt;
  if (rt->dist) {
    if (rt->world == 1) return;
    const int g = rt->first_rank;
    const std::vector<int> members = p->mesh->Group(axis, g);
    const size_t flags_off = side ? p->side_flags_off : p->flags_off;
    const size_t counter_off = side ? p->side_counter_off : p->counter_off;
    rh::BarrierArgs b{};
    b.d = static_cast<int>(members.size());
    for (int k = 0; k < b.d; ++k) {
      b.members[k] = members[k];
      b.peer_flags[k] = reinterpret_cast<uint32_t*>(p->peer_base[members[k]] + flags_off);
    }
    b.my_flags = reinterpret_cast<uint32_t*>(p->base[0] + flags_off);
    b.counter = reinterpret_cast<uint32_t*>(p->base[0] + counter_off);
    b.me = g;
    b.err = reinterpret_cast<uint32_t*>(p->base[0] + p->err_off);
    b.timeout_ns = rh::SyncTimeoutNs();
    rh::LaunchBarrier(b, side ? p->side : rt->streams[0]);
    return;
  }
  if (SameStream(rt)) return;  // emulated ranks on one GPU share one in-order stream
  // Several GPUs in one process: join every stream (events).
  std::vector<cudaEvent_t> ev(rt->streams.size());
  for (size_t i = 0; i < rt->streams.size(); ++i) {
    DeviceGuard dg(rt->devs[i]);
    RH_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    RH_CUDA(cudaEventRecord(ev[i], rt->streams[i]));
  }
  for (size_t i = 0; i < rt->streams.size(); ++i) {
    DeviceGuard dg(rt->devs[i]);
    for (size_t j = 0; j < ev.size(); ++j)
      if (i != j) RH_CUDA(cudaStreamWaitEvent(rt->streams[i], ev[j], 0));
  }
  for (auto e : ev) cudaEventDestroy(e);
}

// Dist mode: a device-side barrier over the whole world on rank 0's stream, enqueued right
// before a timed region so every rank's timeline starts together (host launch skew between
// processes would otherwise be charged to the first transition's fused barrier).
void WorldSync(rh_program* p) {
  rh_runtime* rt = p->mesh->rt;
  if (!rt->dist || rt->world == 1) return;
  rh::BarrierArgs b{};
  b.d = rt->world;
  for (int k = 0; k < b.d; ++k) {
    b.members[k] = k;
    b.peer_flags[k] = reinterpret_cast<uint32_t*>(p->peer_base[k] + p->flags_off);
  }
  b.my_flags = reinterpret_cast<uint32_t*>(p->base[0] + p->flags_off);
  b.counter = reinterpret_cast<uint32_t*>(p->base[0] + p->counter_off);
  b.me = rt->first_rank;
  b.err = reinterpret_cast<uint32_t*>(p->base[0] + p->err_off);
  b.timeout_ns = rh::SyncTimeoutNs();
  rh::LaunchBarrier(b, rt->streams[0]);
}

// One run of the schedule.  `prof` (optional): n_steps + 1 boundary events recorded on local
// rank 0's stream before every step and after the last, then 2 per async step (begin / end on
// the side stream).
int64_t RunOnce(rh_program* p, std::vector<cudaEvent_t>* prof) {
  rh_runtime* rt = p->mesh->rt;
  int64_t launches = 0;
  const bool multi_dev = rt->devs.size() > 1;
  cudaStream_t main = rt->streams[0];
  if (p->n_sync_slots) {  // new run epoch for the barriers fused into the pull kernels
    rh::LaunchEpochTick(reinterpret_cast<uint32_t*>(p->base[0] + p->epoch_off), main);
    ++launches;
  }
  const size_t n = p->steps.size();
  bool prev_kernel = false;  // the previous main-stream step was a compute kernel step
  for (size_t si = 0; si < n; ++si) {
    rh::Step& st = p->steps[si];
    if (prof) RH_CUDA(cudaEventRecordWithFlags((*prof)[si], main, cudaEventRecordExternal));
    for (int k : p->joins_at[si]) RH_CUDA(cudaStreamWaitEvent(main, p->done_ev[k], 0));
    if (st.async) {  // fork onto the side stream (dist: one local rank)
      const int k = st.async_id;
      RH_CUDA(cudaEventRecord(p->fork_ev[k], main));
      RH_CUDA(cudaStreamWaitEvent(p->side, p->fork_ev[k], 0));
      if (prof) RH_CUDA(cudaEventRecordWithFlags((*prof)[n + 1 + 2 * k], p->side, cudaEventRecordExternal));
      GroupSync(p, st.axis, /*side=*/true);
      if (st.stage < 0 || p->StageOf(rt->first_rank) == st.stage) launches += st.run(0, p->side);
      GroupSync(p, st.axis, /*side=*/true);
      launches += 2;
      if (prof) RH_CUDA(cudaEventRecordWithFlags((*prof)[n + 2 + 2 * k], p->side, cudaEventRecordExternal));
      RH_CUDA(cudaEventRecord(p->done_ev[k], p->side));
      continue;
    }
    if (st.p2p && st.sync_slot < 0) GroupSync(p, st.axis);
    // PDL (launch.cuh) after a compute kernel only: for the next compute kernel, and (opt-in,
    // RH_PDL_PULL=1) for a peer-memory pull, whose CTAs then become resident while the producer
    // drains and publish their arrival at the fused barrier as soon as griddepcontrol.wait
    // returns (measured: no change at N=2/4, profiles/r2/README).  Never after a transition (a
    // kernel must not wait on a grid whose CTAs spin on peers), a cross-stream join or a
    // profiling event.
    static const bool pdl_pull = [] {
      const char* e = std::getenv("RH_PDL_PULL");
      return e && e[0] == '1';
    }();
    const bool pdl = !(p->flags & RH_FLAG_NO_PDL) && !prof && prev_kernel && p->joins_at[si].empty() &&
                     (st.kind == rh::Step::kKernel ||
                      (pdl_pull && st.kind == rh::Step::kTransition && !st.pulls.empty() && !st.fine));
    rh::SetPdl(pdl);
    try {
      for (int li = 0; li < rt->n_local(); ++li) {
        if (st.stage >= 0 && p->StageOf(rt->first_rank + li) != st.stage) continue;  // another stage's step
        if (multi_dev) RH_CUDA(cudaSetDevice(rt->device_of(li)));
        launches += st.run(li, rt->stream_of(li));
      }
    } catch (...) {
      rh::SetPdl(false);
      throw;
    }
    rh::SetPdl(false);
    prev_kernel = st.kind == rh::Step::kKernel;
    if (st.p2p && st.post_sync) GroupSync(p, st.axis);
  }
  for (const auto& st : p->steps)  // join what no later step waited for
    if (st.async && st.join < 0) RH_CUDA(cudaStreamWaitEvent(main, p->done_ev[st.async_id], 0));
  if (prof) RH_CUDA(cudaEventRecordWithFlags((*prof)[n], main, cudaEventRecordExternal));
  if (multi_dev) RH_CUDA(cudaSetDevice(rt->devs[0]));
  return launches;
}

// CUDA graphs: one stream per process (dist mode, or every emulated rank on one GPU).  The
// static schedule is captured once and replayed, removing per-kernel launch latency (the GPT
// block at N>=4 and the MLP configs are launch-bound otherwise).
bool UseGraph(const rh_program* p) {
  return p->mesh->rt->streams.size() == 1 && !(p->flags & RH_FLAG_NO_GRAPH);
}

// Capture `iters` back-to-back runs; `ev` (optional) = iters x (n_steps + 1) boundary events
// recorded as external event nodes.
cudaGraphExec_t CaptureRuns(rh_program* p, int iters, std::vector<std::vector<cudaEvent_t>>* ev) {
  cudaStream_t s = p->mesh->rt->streams[0];
  RH_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  try {
    for (int it = 0; it < iters; ++it) RunOnce(p, ev ? &(*ev)[it] : nullptr);
  } catch (...) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(s, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  cudaGraph_t g = nullptr;
  RH_CUDA(cudaStreamEndCapture(s, &g));
  cudaGraphExec_t e = nullptr;
  const cudaError_t r = cudaGraphInstantiate(&e, g, 0);
  cudaGraphDestroy(g);
  RH_CUDA(r);
  return e;
}

// One run: replay the captured schedule (captured lazily after an eager first run, which also
// performs one-time setup such as kernel attributes and TMA descriptors).
void RunStep(rh_program* p) {
  if (!UseGraph(p)) {
    RunOnce(p, nullptr);
    return;
  }
  if (!p->graph) {
    if (!p->warmed) {
      RunOnce(p, nullptr);
      p->warmed = true;
      return;
    }
    p->graph = CaptureRuns(p, 1, nullptr);
  }
  RH_CUDA(cudaGraphLaunch(static_cast<cudaGraphExec_t>(p->graph), p->mesh->rt->streams[0]));
}

void SyncAll(rh_runtime* rt) {
  for (size_t i = 0; i < rt->streams.size(); ++i) {
    DeviceGuard dg(rt->devs[i]);
    RH_CUDA(cudaStreamSynchronize(rt->streams[i]));
  }
}

// After a run (dist mode): a cross-GPU wait that gave up (PeerSync.err) fails the call.
void CheckSync(rh_program* p) {
  rh_runtime* rt = p->mesh->rt;
  if (!rt->dist || rt->world == 1 || p->base.empty()) return;
  uint32_t e = 0;
  DeviceGuard dg(rt->devs[0]);
  if (p->side) RH_CUDA(cudaStreamSynchronize(p->side));
  RH_CUDA(cudaMemcpy(&e, p->base[0] + p->err_off, 4, cudaMemcpyDeviceToHost));
  if (!e) return;
  const uint32_t zero = 0;
  RH_CUDA(cudaMemcpy(p->base[0] + p->err_off, &zero, 4, cudaMemcpyHostToDevice));
  Fail("cross-GPU barrier timed out: rank " + std::to_string((e >> 8) & 0xff) + " waited more than " +
           std::to_string(rh::SyncTimeoutNs() / 1000000) + " ms for rank " + std::to_string(e & 0xff) +
           " (RH_SYNC_TIMEOUT_MS); the run's results are invalid",
       RH_ERR_TIMEOUT);
}

// Host-side barrier over the world communicator (dist) — used around setup only.
void HostBarrier(rh_runtime* rt) {
  if (!rt->dist || rt->world == 1) return;
  float* buf = nullptr;
  RH_CUDA(cudaMalloc(&buf, 4));
  RH_NCCL(ncclAllReduce(buf, buf, 1, ncclFloat32, ncclSum, rt->world_comm, rt->streams[0]));
  RH_CUDA(cudaStreamSynchronize(rt->streams[0]));
  cudaFree(buf);
}

void Allocate(rh_program* p) {
  rh_runtime* rt = p->mesh->rt;
  const size_t bytes = std::max<size_t>(p->arena_bytes, 256);
  p->base.assign(rt->n_local(), nullptr);
  for (int li = 0; li < rt->n_local(); ++li) {
    DeviceGuard dg(rt->device_of(li));
    void* ptr = nullptr;
    RH_CUDA(cudaMalloc(&ptr, bytes));
    // zero on the rank's own (non-blocking) stream so later work is ordered after it
    RH_CUDA(cudaMemsetAsync(ptr, 0, bytes, rt->stream_of(li)));
    for (const auto& up : p->uploads)  // constant tables (e.g. the bf16 tanh-run tables)
      RH_CUDA(cudaMemcpyAsync(static_cast<char*>(ptr) + up.first, up.second.data(), up.second.size(),
                              cudaMemcpyHostToDevice, rt->stream_of(li)));
    RH_CUDA(cudaStreamSynchronize(rt->stream_of(li)));
    p->base[li] = static_cast<char*>(ptr);
    p->owned.push_back(ptr);
  }
  p->peer_base.assign(rt->world, nullptr);
  if (!rt->dist) {
    for (int li = 0; li < rt->n_local(); ++li) p->peer_base[rt->first_rank + li] = p->base[li];
    return;
  }
  p->peer_base[rt->first_rank] = p->base[0];
  if (rt->world == 1) return;
  // Exchange CUDA IPC handles of the symmetric arenas over the world communicator.
  cudaIpcMemHandle_t mine;
  RH_CUDA(cudaIpcGetMemHandle(&mine, p->base[0]));
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  char* dev = nullptr;
  RH_CUDA(cudaMalloc(&dev, hb * (rt->world + 1)));
  RH_CUDA(cudaMemcpy(dev + hb * rt->world, &mine, hb, cudaMemcpyHostToDevice));
  RH_NCCL(ncclAllGather(dev + hb * rt->world, dev, hb, ncclChar, rt->world_comm, rt->streams[0]));
  RH_CUDA(cudaStreamSynchronize(rt->streams[0]));
  std::vector<cudaIpcMemHandle_t> all(rt->world);
  RH_CUDA(cudaMemcpy(all.data(), dev, hb * rt->world, cudaMemcpyDeviceToHost));
  cudaFree(dev);
  for (int r = 0; r < rt->world; ++r) {
    if (r == rt->first_rank) continue;
    void* ptr = nullptr;
    RH_CUDA(cudaIpcOpenMemHandle(&ptr, all[r], cudaIpcMemLazyEnablePeerAccess));
    p->peer_base[r] = static_cast<char*>(ptr);
  }
  p->ipc_opened = true;
  if (p->n_async) {  // side stream + fork/done events of the async transitions
    DeviceGuard dg(rt->devs[0]);
    RH_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
    p->fork_ev.assign(p->n_async, nullptr);
    p->done_ev.assign(p->n_async, nullptr);
    for (int k = 0; k < p->n_async; ++k) {
      RH_CUDA(cudaEventCreateWithFlags(&p->fork_ev[k], cudaEventDisableTiming));
      RH_CUDA(cudaEventCreateWithFlags(&p->done_ev[k], cudaEventDisableTiming));
    }
  }
  HostBarrier(rt);  // every arena zeroed (flags included) before any barrier kernel runs
}

void DestroyProgram(rh_program* p) {
  if (!p) return;
  rh_runtime* rt = p->mesh->rt;
  try {
    SyncAll(rt);
  } catch (...) {
  }
  if (p->ipc_opened) {
    try {
      HostBarrier(rt);  // peers must be done reading this arena before it is unmapped/freed
    } catch (...) {
    }
    for (int r = 0; r < rt->world; ++r)
      if (r != rt->first_rank && p->peer_base[r]) cudaIpcCloseMemHandle(p->peer_base[r]);
  }
  if (p->graph) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(p->graph));
  for (auto& st : p->steps)
    if (st.fini)
      for (int li = 0; li < rt->n_local() && li < static_cast<int>(p->base.size()); ++li)
        if (p->base[li]) st.fini(li);
  for (auto e : p->fork_ev) cudaEventDestroy(e);
  for (auto e : p->done_ev) cudaEventDestroy(e);
  if (p->side) cudaStreamDestroy(p->side);
  for (int li = 0; li < rt->n_local() && li < static_cast<int>(p->owned.size()); ++li) {
    DeviceGuard dg(rt->device_of(li));
    cudaFree(p->owned[li]);
    if (li < static_cast<int>(p->in_stage.size()) && p->in_stage[li]) cudaFree(p->in_stage[li]);
  }
  delete p;
}

// Host full tensor -> every local rank's buffer of tensor t (H2D staging + slice kernel).
void WriteFull(rh_program* p, const rh::Tensor& t, const void* src, size_t bytes,
               std::vector<void*>* stage_cache) {
  rh_runtime* rt = p->mesh->rt;
  for (int li = 0; li < rt->n_local(); ++li) {
    DeviceGuard dg(rt->device_of(li));
    cudaStream_t s = rt->stream_of(li);
    const int g = rt->first_rank + li;
    bool all_rep = true;
    for (auto& sp : t.specs) all_rep = all_rep && sp.kind == RH_REPLICATED;
    if (all_rep) {
      RH_CUDA(cudaMemcpyAsync(p->base[li] + t.offset, src, bytes, cudaMemcpyHostToDevice, s));
      continue;
    }
    void* stage = nullptr;
    if (stage_cache && static_cast<int>(stage_cache->size()) > li && (*stage_cache)[li]) {
      stage = (*stage_cache)[li];
    } else {
      RH_CUDA(cudaMallocAsync(&stage, bytes, s));
    }
    RH_CUDA(cudaMemcpyAsync(stage, src, bytes, cudaMemcpyHostToDevice, s));
    bool partial_zero = false;
    const std::vector<int> c = p->mesh->Coords(g);
    for (int a = 0; a < p->n_axes; ++a)
      if (t.specs[a].kind == RH_PARTIAL && c[a] != 0) partial_zero = true;
    if (partial_zero) {
      rh::LaunchZero(p->base[li] + t.offset, t.bytes, s);
    } else {
      rh::LaunchSliceComposed(p->base[li] + t.offset, stage, MakeComposed(p, t, g), t.elems(),
                              t.dtype, s);
    }
    if (!(stage_cache && static_cast<int>(stage_cache->size()) > li && (*stage_cache)[li]))
      RH_CUDA(cudaFreeAsync(stage, s));
  }
}

uint16_t F2Bf(float x);
float Bf2F(uint16_t x);

// Global value of tensor t from every rank's local buffer (all ranks must be local): Replicated
// axes read coordinate 0, Partial axes are summed in rank order in fp32 and rounded once.
void AssembleFull(rh_program* p, const rh::Tensor& t, void* dst) {
  rh_runtime* rt = p->mesh->rt;
  if (rt->n_local() != rt->world) Fail("assembling a non-output tensor needs every rank local");
  const int eb = rh::ElemBytes(t.dtype);
  const int64_t n = Prod(t.gdims);
  std::vector<float> full(n, 0.0f);
  std::vector<char> loc(t.bytes);
  for (int r = 0; r < rt->world; ++r) {
    const std::vector<int> c = p->mesh->Coords(r);
    bool skip = false, first = true;
    for (int a = 0; a < p->n_axes; ++a) {
      if (a == p->pipeline_axis) {  // the tensor lives on the ranks of its stage only
        if (c[a] != t.stage) skip = true;
        continue;
      }
      if (t.specs[a].kind == RH_REPLICATED && c[a] != 0) skip = true;
      if (t.specs[a].kind == RH_PARTIAL && c[a] != 0) first = false;
    }
    if (skip) continue;
    {
      DeviceGuard dg(rt->device_of(r));
      RH_CUDA(cudaMemcpy(loc.data(), p->base[r] + t.offset, t.bytes, cudaMemcpyDeviceToHost));
    }
    const rh::ComposedMap m = MakeComposed(p, t, r);
    for (int64_t l = 0; l < t.elems(); ++l) {
      const int64_t f = rh::ComposedLocalToGlobal(m, l);
      float v;
      if (eb == 4) {
        std::memcpy(&v, &loc[l * 4], 4);
      } else {
        uint16_t h;
        std::memcpy(&h, &loc[l * 2], 2);
        v = Bf2F(h);
      }
      full[f] = first ? v : full[f] + v;
    }
  }
  if (eb == 4) {
    std::memcpy(dst, full.data(), static_cast<size_t>(n) * 4);
  } else {
    uint16_t* o = static_cast<uint16_t*>(dst);
    for (int64_t i = 0; i < n; ++i) o[i] = F2Bf(full[i]);
  }
}

uint16_t F2Bf(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return static_cast<uint16_t>((u | 0x400000u) >> 16);
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}
float Bf2F(uint16_t x) {
  uint32_t u = static_cast<uint32_t>(x) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

}  // namespace

extern "C" {

const char* rh_last_error(void) { return g_err.c_str(); }
const char* rh_version(void) { return "rhino-b200 0.1 (sm_100a)"; }

int rh_get_unique_id(uint8_t uid[RH_UID_BYTES]) {
  return Guard([&] {
    static_assert(sizeof(ncclUniqueId) == RH_UID_BYTES, "uid size");
    ncclUniqueId id;
    RH_NCCL(ncclGetUniqueId(&id));
    std::memcpy(uid, &id, RH_UID_BYTES);
  });
}

int rh_runtime_create(int n_ranks, const int* cuda_ids, rh_runtime** out) {
  return Guard([&] {
    if (n_ranks < 1) Fail("rh_runtime_create: n_ranks must be >= 1");
    auto rt = std::make_unique<rh_runtime>();
    rt->world = n_ranks;
    rt->dist = false;
    for (int i = 0; i < n_ranks; ++i) {
      auto it = std::find(rt->devs.begin(), rt->devs.end(), cuda_ids[i]);
      if (it == rt->devs.end()) {
        rt->devs.push_back(cuda_ids[i]);
        rt->rank_dev.push_back(static_cast<int>(rt->devs.size()) - 1);
      } else {
        rt->rank_dev.push_back(static_cast<int>(it - rt->devs.begin()));
      }
    }
    for (int dev : rt->devs) {
      DeviceGuard dg(dev);
      cudaStream_t s;
      RH_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      rt->streams.push_back(s);
      for (int other : rt->devs) {
        if (other == dev) continue;
        int ok = 0;
        RH_CUDA(cudaDeviceCanAccessPeer(&ok, dev, other));
        if (!ok) Fail("rh_runtime_create: no peer access between devices");
        cudaError_t e = cudaDeviceEnablePeerAccess(other, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) RH_CUDA(e);
        cudaGetLastError();
      }
    }
    RH_CUDA(cudaSetDevice(rt->devs[0]));
    *out = rt.release();
  });
}

int rh_runtime_create_dist(int world, int rank, int cuda_id, const uint8_t uid[RH_UID_BYTES],
                           rh_runtime** out) {
  return Guard([&] {
    if (world < 1 || rank < 0 || rank >= world) Fail("rh_runtime_create_dist: bad world/rank");
    auto rt = std::make_unique<rh_runtime>();
    rt->world = world;
    rt->dist = true;
    rt->first_rank = rank;
    rt->devs = {cuda_id};
    rt->rank_dev = {0};
    RH_CUDA(cudaSetDevice(cuda_id));
    cudaStream_t s;
    RH_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    rt->streams = {s};
    ncclUniqueId id;
    std::memcpy(&id, uid, RH_UID_BYTES);
    RH_NCCL(ncclCommInitRank(&rt->world_comm, world, id, rank));
    *out = rt.release();
  });
}

int rh_runtime_world(const rh_runtime* rt, int* world, int* first_local_rank, int* n_local) {
  return Guard([&] {
    *world = rt->world;
    *first_local_rank = rt->first_rank;
    *n_local = rt->n_local();
  });
}

void rh_runtime_destroy(rh_runtime* rt) {
  if (!rt) return;
  for (size_t i = 0; i < rt->streams.size(); ++i) {
    cudaSetDevice(rt->devs[i]);
    cudaStreamSynchronize(rt->streams[i]);
    cudaStreamDestroy(rt->streams[i]);
  }
  for (auto& e : rt->axis_comms)
    for (auto c : e.second)
      if (c) ncclCommDestroy(c);
  if (rt->world_comm) ncclCommDestroy(rt->world_comm);
  delete rt;
}

int rh_mesh_create(rh_runtime* rt, int n_axes, const int* dims, rh_mesh** out) {
  return Guard([&] {
    if (n_axes < 1 || n_axes > RH_MAX_AXES) Fail("rh_mesh_create: 1..4 axes");
    auto m = std::make_unique<rh_mesh>();
    m->rt = rt;
    m->dims.assign(dims, dims + n_axes);
    int64_t prod = 1;
    for (int d : m->dims) {
      if (d < 1 || d > rh::kMaxGroup) Fail("rh_mesh_create: axis size must be 1..8");
      prod *= d;
    }
    if (prod != rt->world) Fail("rh_mesh_create: prod(dims) != world size");
    if (rt->dist) {
      for (const auto& e : rt->axis_comms)
        if (e.first == m->dims) m->axis_comm = e.second;
      if (m->axis_comm.empty()) {
        const std::vector<int> c = m->Coords(rt->first_rank);
        for (int a = 0; a < n_axes; ++a) {
          int color = 0;
          for (int b = 0; b < n_axes; ++b)
            if (b != a) color = color * m->dims[b] + c[b];
          ncclComm_t comm = nullptr;
          RH_NCCL(ncclCommSplit(rt->world_comm, color, c[a], &comm, nullptr));
          m->axis_comm.push_back(comm);
        }
        rt->axis_comms.emplace_back(m->dims, m->axis_comm);
      }
    }
    *out = m.release();
  });
}

void rh_mesh_destroy(rh_mesh* mesh) {
  delete mesh;  // axis communicators belong to the runtime (shared across meshes)
}

}  // extern "C"

namespace {
struct PipelineArgs {
  int axis = -1;
  std::vector<std::pair<int, int>> apply;
  float lr = 0.f;
};

int LoadProgram(rh_mesh* mesh, const rh_op* ops, int n_ops, const int* outputs, int n_out,
                uint32_t flags, const std::vector<std::pair<int, Specs>>& requests,
                rh_program** out, const PipelineArgs& pp = PipelineArgs{}) {
  rh_program* raw = nullptr;
  int rc = Guard([&] {
    auto p = std::make_unique<rh_program>();
    p->requests = requests;
    p->mesh = mesh;
    p->flags = flags;
    p->n_axes = static_cast<int>(mesh->dims.size());
    if (pp.axis >= 0) {
      if (pp.axis >= p->n_axes) Fail("pipeline axis out of range");
      p->pipeline_axis = pp.axis;
      p->n_stages = mesh->dims[pp.axis];
      p->apply = pp.apply;
      p->lr = pp.lr;
      for (const auto& ap : pp.apply)
        if (ap.first < 0 || ap.first >= n_ops || ap.second < 0 || ap.second >= n_ops) Fail("apply: bad op index");
    }
    p->ops.assign(ops, ops + n_ops);
    p->inputs.resize(n_ops);
    p->in_specs.resize(n_ops);
    p->out_specs.resize(n_ops);
    for (int i = 0; i < n_ops; ++i) {
      const rh_op& op = ops[i];
      if (op.rank < 1 || op.rank > RH_MAX_RANK) Fail("op " + std::to_string(i) + ": bad rank");
      if (op.dtype != RH_F32 && op.dtype != RH_BF16) Fail("op " + std::to_string(i) + ": bad dtype");
      p->inputs[i].assign(op.inputs, op.inputs + op.n_in);
      for (int s : p->inputs[i])
        if (s < 0 || s >= n_ops) Fail("op " + std::to_string(i) + ": bad input index");
      p->out_specs[i].assign(op.out_spec, op.out_spec + p->n_axes);
      p->in_specs[i].assign(op.n_in, Specs(p->n_axes));
      for (int a = 0; a < p->n_axes; ++a)
        for (int s = 0; s < op.n_in; ++s) p->in_specs[i][s][a] = op.in_specs[a * op.n_in + s];
      p->ops[i].inputs = nullptr;
      p->ops[i].in_specs = nullptr;
    }
    p->outputs.assign(outputs, outputs + n_out);
    // Kahn order with index tie-break (ops are pure: any topological order gives the same
    // values; the reference's own order is TopoOrderIndices, proj/src/ir.cpp:381-412).
    std::vector<int> indeg(n_ops, 0);
    std::vector<std::vector<int>> cons(n_ops);
    for (int i = 0; i < n_ops; ++i)
      for (int s : p->inputs[i]) {
        ++indeg[i];
        cons[s].push_back(i);
      }
    std::vector<int> q;
    for (int i = 0; i < n_ops; ++i)
      if (!indeg[i]) q.push_back(i);
    for (size_t h = 0; h < q.size(); ++h)
      for (int c : cons[q[h]])
        if (--indeg[c] == 0) q.push_back(c);
    if (static_cast<int>(q.size()) != n_ops) Fail("program has a cycle");
    p->order = q;
    rh::LowerProgram(p.get());
    Allocate(p.get());
    for (auto& st : p->steps)  // one-time device tables (arena pointers are final now)
      if (st.init)
        for (int li = 0; li < p->mesh->rt->n_local(); ++li) {
          DeviceGuard dg(p->mesh->rt->device_of(li));
          st.init(li);
        }
    raw = p.release();
  });
  if (rc == RH_OK) *out = raw;
  return rc;
}
}  // namespace

extern "C" {

int rh_op_natural_specs(const rh_op* ops, int n_ops, int op, int n_axes, const int* mesh_dims, rh_spec* out) {
  return Guard([&] {
    if (n_axes < 1 || n_axes > RH_MAX_AXES) Fail("bad mesh");
    const std::vector<int> mesh(mesh_dims, mesh_dims + n_axes);
    const Specs nat = rh::NaturalSpecsOf(ops, n_ops, op, mesh);
    for (int a = 0; a < n_axes; ++a) out[a] = nat[a];
  });
}

int rh_program_load(rh_mesh* mesh, const rh_op* ops, int n_ops, const int* outputs, int n_out,
                    uint32_t flags, rh_program** out) {
  return LoadProgram(mesh, ops, n_ops, outputs, n_out, flags, {}, out);
}

int rh_program_load_pipeline(rh_mesh* mesh, int pipeline_axis, const rh_op* ops, int n_ops, const int* outputs,
                             int n_out, const int* apply, int n_apply, float lr, uint32_t flags,
                             rh_program** out) {
  PipelineArgs pp;
  pp.axis = pipeline_axis;
  pp.lr = lr;
  for (int k = 0; k < n_apply; ++k) pp.apply.emplace_back(apply[2 * k], apply[2 * k + 1]);
  if (pipeline_axis < 0) {
    g_err = "rh_program_load_pipeline: pipeline_axis must be a mesh axis";
    return RH_ERR_INVALID;
  }
  return LoadProgram(mesh, ops, n_ops, outputs, n_out, flags, {}, out, pp);
}

void rh_program_destroy(rh_program* prog) { DestroyProgram(prog); }

int rh_program_init_synthetic(rh_program* p, uint64_t seed) {
  return Guard([&] {
    rh_runtime* rt = p->mesh->rt;
    for (size_t i = 0; i < p->ops.size(); ++i) {
      const rh_op& op = p->ops[i];
      if (op.kind != RH_OP_PARAMETER && op.kind != RH_OP_INPUT) continue;
      const rh::Tensor& t = p->tensors[p->out_tensor[i]];
      const float scale = op.kind == RH_OP_PARAMETER
                              ? static_cast<float>(std::sqrt(3.0 / static_cast<double>(op.dims[0])))
                              : 1.0f;
      for (int li = 0; li < rt->n_local(); ++li) {
        DeviceGuard dg(rt->device_of(li));
        const int g = rt->first_rank + li;
        bool zero = false;
        const std::vector<int> c = p->mesh->Coords(g);
        for (int a = 0; a < p->n_axes; ++a)
          if (t.specs[a].kind == RH_PARTIAL && c[a] != 0) zero = true;
        if (zero) {
          rh::LaunchZero(p->base[li] + t.offset, t.bytes, rt->stream_of(li));
        } else {
          rh::LaunchSynthetic(p->base[li] + t.offset, MakeComposed(p, t, g), t.elems(), seed,
                              static_cast<uint32_t>(i), scale, t.dtype, rt->stream_of(li));
        }
      }
    }
    SyncAll(rt);
  });
}

int rh_program_write_full(rh_program* p, int op, const void* src, size_t bytes) {
  return Guard([&] {
    if (op < 0 || op >= static_cast<int>(p->ops.size())) Fail("bad op index");
    if (p->ops[op].kind != RH_OP_PARAMETER && p->ops[op].kind != RH_OP_INPUT)
      Fail("rh_program_write_full: op is not a source");
    const rh::Tensor& t = p->tensors[p->out_tensor[op]];
    if (bytes != static_cast<size_t>(Prod(t.gdims)) * rh::ElemBytes(t.dtype)) Fail("size mismatch");
    WriteFull(p, t, src, bytes, nullptr);
    SyncAll(p->mesh->rt);
  });
}

int rh_program_run(rh_program* p, int iters, double* ms_per_iter) {
  return Guard([&] {
    rh_runtime* rt = p->mesh->rt;
    // graph capture / instantiation is host work: do it before the timed region (the eager
    // first run it needs is one extra, identical run of the program)
    if (UseGraph(p) && !p->graph && iters > 0) {
      if (!p->warmed) RunStep(p);
      p->graph = CaptureRuns(p, 1, nullptr);
    }
    SyncAll(rt);
    WorldSync(p);
    std::vector<cudaEvent_t> ev0(rt->streams.size()), ev1(rt->streams.size());
    for (size_t i = 0; i < rt->streams.size(); ++i) {
      DeviceGuard dg(rt->devs[i]);
      RH_CUDA(cudaEventCreate(&ev0[i]));
      RH_CUDA(cudaEventCreate(&ev1[i]));
      RH_CUDA(cudaEventRecord(ev0[i], rt->streams[i]));
    }
    for (int it = 0; it < iters; ++it) RunStep(p);
    float worst = 0;
    for (size_t i = 0; i < rt->streams.size(); ++i) {
      DeviceGuard dg(rt->devs[i]);
      RH_CUDA(cudaEventRecord(ev1[i], rt->streams[i]));
      RH_CUDA(cudaEventSynchronize(ev1[i]));
      float ms = 0;
      RH_CUDA(cudaEventElapsedTime(&ms, ev0[i], ev1[i]));
      worst = std::max(worst, ms);
      cudaEventDestroy(ev0[i]);
      cudaEventDestroy(ev1[i]);
    }
    CheckSync(p);
    if (ms_per_iter) *ms_per_iter = iters > 0 ? worst / iters : 0.0;
  });
}

int rh_program_profile(rh_program* p, int iters, double* ms_per_iter) {
  return Guard([&] {
    rh_runtime* rt = p->mesh->rt;
    SyncAll(rt);
    DeviceGuard dg(rt->devs[0]);
    const size_t n = p->steps.size();
    // Boundary events for every (iteration, step); no host sync inside the timed region.
    std::vector<std::vector<cudaEvent_t>> ev(std::max(iters, 0), std::vector<cudaEvent_t>(n + 1 + 2 * p->n_async));
    for (auto& row : ev)
      for (auto& e : row) RH_CUDA(cudaEventCreate(&e));
    if (UseGraph(p) && iters > 0) {
      // the whole timed region is one graph: K runs back to back with external event nodes
      cudaGraphExec_t g = CaptureRuns(p, iters, &ev);
      WorldSync(p);
      RH_CUDA(cudaGraphLaunch(g, rt->streams[0]));
      SyncAll(rt);
      cudaGraphExecDestroy(g);
    } else {
      for (int it = 0; it < iters; ++it) RunOnce(p, &ev[it]);
    }
    SyncAll(rt);
    CheckSync(p);
    std::vector<double> acc(n, 0.0);
    for (int it = 0; it < iters; ++it)
      for (size_t i = 0; i < n; ++i) {
        float ms = 0;
        const rh::Step& st = p->steps[i];
        if (st.async) {  // side-stream duration (fork to done, including its barriers)
          const size_t k = static_cast<size_t>(st.async_id);
          RH_CUDA(cudaEventElapsedTime(&ms, ev[it][n + 1 + 2 * k], ev[it][n + 2 + 2 * k]));
        } else {
          RH_CUDA(cudaEventElapsedTime(&ms, ev[it][i], ev[it][i + 1]));
        }
        acc[i] += ms;
      }
    float total = 0;
    if (iters > 0) RH_CUDA(cudaEventElapsedTime(&total, ev[0][0], ev[iters - 1][n]));
    for (size_t i = 0; i < n; ++i) p->steps[i].ms = iters > 0 ? acc[i] / iters : 0.0;
    for (auto& row : ev)
      for (auto& e : row) cudaEventDestroy(e);
    if (ms_per_iter) *ms_per_iter = iters > 0 ? total / iters : 0.0;
  });
}

// Every rank's copy of a symmetric device buffer, mapped here (CUDA IPC handles all-gathered
// over the world communicator); entry `first_rank` is `mine` itself.
std::vector<char*> ExchangeIpc(rh_runtime* rt, char* mine) {
  cudaIpcMemHandle_t h;
  RH_CUDA(cudaIpcGetMemHandle(&h, mine));
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  char* dev = nullptr;
  RH_CUDA(cudaMalloc(&dev, hb * (rt->world + 1)));
  RH_CUDA(cudaMemcpy(dev + hb * rt->world, &h, hb, cudaMemcpyHostToDevice));
  RH_NCCL(ncclAllGather(dev + hb * rt->world, dev, hb, ncclChar, rt->world_comm, rt->streams[0]));
  RH_CUDA(cudaStreamSynchronize(rt->streams[0]));
  std::vector<cudaIpcMemHandle_t> all(rt->world);
  RH_CUDA(cudaMemcpy(all.data(), dev, hb * rt->world, cudaMemcpyDeviceToHost));
  cudaFree(dev);
  std::vector<char*> out(rt->world, nullptr);
  for (int r = 0; r < rt->world; ++r) {
    if (r == rt->first_rank) {
      out[r] = mine;
      continue;
    }
    void* ptr = nullptr;
    RH_CUDA(cudaIpcOpenMemHandle(&ptr, all[r], cudaIpcMemLazyEnablePeerAccess));
    out[r] = static_cast<char*>(ptr);
  }
  return out;
}

// Host read of output k: a materialized (replicated) output in a multi-process run is read as
// this process's 1/world contiguous slice (the processes' slices together are the full tensor;
// every rank copying the whole replicated tensor would multiply the PCIe traffic by world).
std::pair<size_t, size_t> OutSlice(const rh_program* p, int op, const rh::Tensor& t) {
  const rh_runtime* rt = p->mesh->rt;
  if (rt->dist && rt->world > 1 && p->mat_tensor[op] >= 0 && t.bytes % (static_cast<size_t>(rt->world) * 16) == 0) {
    const size_t part = t.bytes / rt->world;
    return {part * rt->first_rank, part};
  }
  return {0, t.bytes};
}

// A fully replicated input in a multi-process run: each process copies only its 1/world
// contiguous slice over PCIe and the slices are all-gathered over NVLink (every process copying
// the whole tensor multiplies the host->device traffic by world: at N=4 the 16 MiB C3 input per
// process and step made e2e PCIe-bound, 0.60 ms against a 0.31 ms run).  The gather runs on its
// own stream between the H2D and the step that consumes it, so it overlaps the previous step's
// run (round 1 had it, with host-ordered world barriers, on the compute stream: slower).
// Returns the slice bytes, 0 when the input is copied whole.  RH_E2E_SCATTER=0 disables.
size_t ScatterPart(const rh_program* p, const rh::Tensor& t) {
  const rh_runtime* rt = p->mesh->rt;
  if (!rt->dist || rt->world <= 1 || rt->world > rh::kMaxGroup || !p->e2e_epoch_off) return 0;
  const char* env = std::getenv("RH_E2E_SCATTER");
  if (env && env[0] == '0') return 0;
  for (int a = 0; a < p->n_axes; ++a)
    if (t.specs[a].kind != RH_REPLICATED) return 0;
  if (t.bytes % (static_cast<size_t>(rt->world) * 16) != 0) return 0;
  return t.bytes / rt->world;
}

// Pipelined end-to-end steps through host buffers (one local rank per process): step i's H2D
// (copy-in stream, into a double-buffered device stage) overlaps step i-1's run and step i-2's
// D2H (copy-out stream); the compute stream moves stage -> arena input (D2D copy, or the slice
// kernel for a sharded input) before the run and arena output -> output stage after it.  Every
// step still copies its inputs in and its outputs out; only the copies of neighbouring steps
// overlap, as in a serving / training loop that prefetches the next batch.
int rh_program_run_host(rh_program* p, int iters, int n_in, const int* in_ops, const void* const* in_ptrs,
                        int n_outs, void* const* out_ptrs, double* ms_per_iter) {
  return Guard([&] {
    rh_runtime* rt = p->mesh->rt;
    if (rt->n_local() != 1) Fail("rh_program_run_host: needs one local rank per process");
    if (iters <= 0) Fail("rh_program_run_host: iters must be positive");
    if (n_outs > static_cast<int>(p->outputs.size())) Fail("too many output buffers");
    DeviceGuard dg(rt->devs[0]);
    cudaStream_t cs = rt->streams[0];
    const int g = rt->first_rank;
    struct In {
      const rh::Tensor* t;
      size_t bytes;
      void* stage[2];
      size_t part;  // > 0: scattered (this process copies bytes [part*g, part*(g+1)) over PCIe)
      std::vector<char*> peer_stage[2];  // scattered: every rank's stage[b] (IPC-mapped)
    };
    struct Out {
      const rh::Tensor* t;
      size_t off, bytes;  // OutSlice
      void* stage[2];
    };
    std::vector<In> ins(n_in);
    std::vector<Out> outs(n_outs);
    bool any_part = false;
    for (int k = 0; k < n_in; ++k) {
      const rh::Tensor& t = p->tensors[p->out_tensor[in_ops[k]]];
      ins[k].t = &t;
      ins[k].bytes = static_cast<size_t>(Prod(t.gdims)) * rh::ElemBytes(t.dtype);
      ins[k].part = ScatterPart(p, t);
      any_part = any_part || ins[k].part;
      for (int b = 0; b < 2; ++b) RH_CUDA(cudaMalloc(&ins[k].stage[b], ins[k].bytes));
    }
    // scattered inputs: map every rank's stage buffers (CUDA IPC over the world communicator)
    std::vector<char*> opened;
    for (auto& x : ins) {
      if (!x.part) continue;
      for (int b = 0; b < 2; ++b) {
        x.peer_stage[b] = ExchangeIpc(rt, static_cast<char*>(x.stage[b]));
        for (int q = 0; q < rt->world; ++q)
          if (q != g) opened.push_back(x.peer_stage[b][q]);
      }
    }
    rh::PeerSync gsync{};
    if (any_part) {
      gsync.d = rt->world;
      gsync.me = g;
      for (int q = 0; q < rt->world; ++q) {
        gsync.members[q] = q;
        gsync.peer_slot[q] = reinterpret_cast<uint32_t*>(p->peer_base[q] + p->e2e_sync_off);
      }
      gsync.my_slot = reinterpret_cast<uint32_t*>(p->base[0] + p->e2e_sync_off);
      gsync.epoch = reinterpret_cast<const uint32_t*>(p->base[0] + p->e2e_epoch_off);
      gsync.err = reinterpret_cast<uint32_t*>(p->base[0] + p->err_off);
      gsync.timeout_ns = rh::SyncTimeoutNs();
    }
    for (int k = 0; k < n_outs; ++k) {
      const int op = p->outputs[k];
      const int ti = p->mat_tensor[op] >= 0 ? p->mat_tensor[op] : p->out_tensor[op];
      if (ti < 0) Fail("output has no buffer");
      outs[k].t = &p->tensors[ti];
      std::tie(outs[k].off, outs[k].bytes) = OutSlice(p, op, *outs[k].t);
      for (int b = 0; b < 2; ++b) RH_CUDA(cudaMalloc(&outs[k].stage[b], outs[k].bytes));
    }
    cudaStream_t sin = nullptr, sout = nullptr, sg = nullptr;
    RH_CUDA(cudaStreamCreateWithFlags(&sin, cudaStreamNonBlocking));
    RH_CUDA(cudaStreamCreateWithFlags(&sout, cudaStreamNonBlocking));
    RH_CUDA(cudaStreamCreateWithFlags(&sg, cudaStreamNonBlocking));
    cudaEvent_t in_ready[2], in_free[2], out_ready[2], out_free[2], h2d_done[2], gathered[2], e0, e1;
    for (int b = 0; b < 2; ++b) {
      RH_CUDA(cudaEventCreateWithFlags(&h2d_done[b], cudaEventDisableTiming));
      RH_CUDA(cudaEventCreateWithFlags(&gathered[b], cudaEventDisableTiming));
      RH_CUDA(cudaEventCreateWithFlags(&in_ready[b], cudaEventDisableTiming));
      RH_CUDA(cudaEventCreateWithFlags(&in_free[b], cudaEventDisableTiming));
      RH_CUDA(cudaEventCreateWithFlags(&out_ready[b], cudaEventDisableTiming));
      RH_CUDA(cudaEventCreateWithFlags(&out_free[b], cudaEventDisableTiming));
    }
    RH_CUDA(cudaEventCreate(&e0));
    RH_CUDA(cudaEventCreate(&e1));
    auto cleanup = [&] {
      cudaStreamSynchronize(sin);
      cudaStreamSynchronize(sg);
      cudaStreamSynchronize(sout);
      cudaStreamSynchronize(cs);
      if (!opened.empty()) {
        try {
          HostBarrier(rt);  // no peer still reads this rank's stage buffers
        } catch (...) {
        }
        for (char* q : opened) cudaIpcCloseMemHandle(q);
      }
      for (auto& x : ins)
        for (void* q : x.stage) cudaFree(q);
      for (auto& x : outs)
        for (void* q : x.stage) cudaFree(q);
      for (int b = 0; b < 2; ++b) {
        cudaEventDestroy(h2d_done[b]);
        cudaEventDestroy(gathered[b]);
        cudaEventDestroy(in_ready[b]);
        cudaEventDestroy(in_free[b]);
        cudaEventDestroy(out_ready[b]);
        cudaEventDestroy(out_free[b]);
      }
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      cudaStreamDestroy(sin);
      cudaStreamDestroy(sout);
      cudaStreamDestroy(sg);
    };
    try {
      if (UseGraph(p) && !p->graph) {  // capture outside the timed region
        if (!p->warmed) RunStep(p);
        RunStep(p);
      }
      SyncAll(rt);
      WorldSync(p);
      RH_CUDA(cudaEventRecord(e0, cs));
      RH_CUDA(cudaStreamWaitEvent(sin, e0, 0));
      RH_CUDA(cudaStreamWaitEvent(sg, e0, 0));
      for (int it = 0; it < iters; ++it) {
        const int b = it & 1;
        RH_CUDA(cudaStreamWaitEvent(sin, in_free[b], 0));
        // scattered inputs: stage[b] is rewritten only after this rank's previous gather, whose
        // barrier every peer passed after finishing the gather that read stage[b] two steps ago
        if (any_part && it > 0) RH_CUDA(cudaStreamWaitEvent(sin, gathered[b ^ 1], 0));
        for (auto& x : ins) {
          const size_t off = x.part * static_cast<size_t>(g), n = x.part ? x.part : x.bytes;
          RH_CUDA(cudaMemcpyAsync(static_cast<char*>(x.stage[b]) + off,
                                  static_cast<const char*>(in_ptrs[&x - ins.data()]) + off, n,
                                  cudaMemcpyHostToDevice, sin));
        }
        RH_CUDA(cudaEventRecord(in_ready[b], sin));
        if (any_part) {  // gather stream: world barrier fused into the pull of the peers' pieces
          RH_CUDA(cudaStreamWaitEvent(sg, in_ready[b], 0));
          rh::LaunchEpochTick(reinterpret_cast<uint32_t*>(p->base[0] + p->e2e_epoch_off), sg);
          for (auto& x : ins)
            if (x.part) rh::LaunchGatherSlices(x.peer_stage[b].data(), rt->world, g, x.part, gsync, sg);
          RH_CUDA(cudaEventRecord(gathered[b], sg));
          RH_CUDA(cudaStreamWaitEvent(cs, gathered[b], 0));
        } else {
          RH_CUDA(cudaStreamWaitEvent(cs, in_ready[b], 0));
        }
        for (auto& x : ins) {
          const rh::Tensor& t = *x.t;
          bool all_rep = true, partial_zero = false;
          const std::vector<int> c = p->mesh->Coords(g);
          for (int a = 0; a < p->n_axes; ++a) {
            all_rep = all_rep && t.specs[a].kind == RH_REPLICATED;
            if (t.specs[a].kind == RH_PARTIAL && c[a] != 0) partial_zero = true;
          }
          if (all_rep) {  // (a scattered input's stage is whole again after its gather)
            RH_CUDA(cudaMemcpyAsync(p->base[0] + t.offset, x.stage[b], x.bytes, cudaMemcpyDeviceToDevice, cs));
          } else if (partial_zero) {
            rh::LaunchZero(p->base[0] + t.offset, t.bytes, cs);
          } else {
            rh::LaunchSliceComposed(p->base[0] + t.offset, x.stage[b], MakeComposed(p, t, g), t.elems(), t.dtype, cs);
          }
        }
        RH_CUDA(cudaEventRecord(in_free[b], cs));
        RunStep(p);
        RH_CUDA(cudaStreamWaitEvent(cs, out_free[b], 0));
        for (auto& x : outs)
          RH_CUDA(cudaMemcpyAsync(x.stage[b], p->base[0] + x.t->offset + x.off, x.bytes, cudaMemcpyDeviceToDevice, cs));
        RH_CUDA(cudaEventRecord(out_ready[b], cs));
        RH_CUDA(cudaStreamWaitEvent(sout, out_ready[b], 0));
        for (auto& x : outs)
          RH_CUDA(cudaMemcpyAsync(static_cast<char*>(out_ptrs[&x - outs.data()]) + x.off, x.stage[b], x.bytes,
                                  cudaMemcpyDeviceToHost, sout));
        RH_CUDA(cudaEventRecord(out_free[b], sout));
      }
      RH_CUDA(cudaStreamWaitEvent(cs, out_free[(iters - 1) & 1], 0));
      RH_CUDA(cudaEventRecord(e1, cs));
      RH_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      RH_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      if (ms_per_iter) *ms_per_iter = ms / iters;
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
    CheckSync(p);
  });
}

int rh_program_step_host(rh_program* p, int n_in, const int* in_ops, const void* const* in_ptrs,
                         int n_outs, void* const* out_ptrs, double* ms) {
  return Guard([&] {
    rh_runtime* rt = p->mesh->rt;
    SyncAll(rt);
    DeviceGuard dg(rt->devs[0]);
    cudaEvent_t e0, e1;
    RH_CUDA(cudaEventCreate(&e0));
    RH_CUDA(cudaEventCreate(&e1));
    WorldSync(p);
    RH_CUDA(cudaEventRecord(e0, rt->streams[0]));
    auto h0 = std::chrono::steady_clock::now();
    // persistent staging (one buffer per local rank, grown to the largest input): no per-step
    // cudaMallocAsync / cudaFreeAsync inside the timed region
    size_t need = 0;
    for (int k = 0; k < n_in; ++k) {
      const rh::Tensor& t = p->tensors[p->out_tensor[in_ops[k]]];
      need = std::max(need, static_cast<size_t>(Prod(t.gdims)) * rh::ElemBytes(t.dtype));
    }
    p->in_stage.resize(rt->n_local(), nullptr);
    p->in_stage_bytes.resize(rt->n_local(), 0);
    for (int li = 0; li < rt->n_local(); ++li)
      if (p->in_stage_bytes[li] < need) {
        DeviceGuard dgl(rt->device_of(li));
        if (p->in_stage[li]) RH_CUDA(cudaFree(p->in_stage[li]));
        RH_CUDA(cudaMalloc(&p->in_stage[li], need));
        p->in_stage_bytes[li] = need;
      }
    for (int k = 0; k < n_in; ++k) {
      const int op = in_ops[k];
      const rh::Tensor& t = p->tensors[p->out_tensor[op]];
      WriteFull(p, t, in_ptrs[k], static_cast<size_t>(Prod(t.gdims)) * rh::ElemBytes(t.dtype), &p->in_stage);
    }
    RunStep(p);
    if (n_outs > static_cast<int>(p->outputs.size())) Fail("too many output buffers");
    for (int k = 0; k < n_outs; ++k) {
      const int op = p->outputs[k];
      // materialized: the full tensor; otherwise this process's first local rank's shard
      const int ti = p->mat_tensor[op] >= 0 ? p->mat_tensor[op] : p->out_tensor[op];
      if (ti < 0) Fail("output has no buffer");
      const rh::Tensor& t = p->tensors[ti];
      const auto sl = OutSlice(p, op, t);
      RH_CUDA(cudaMemcpyAsync(static_cast<char*>(out_ptrs[k]) + sl.first, p->base[0] + t.offset + sl.first,
                              sl.second, cudaMemcpyDeviceToHost, rt->streams[0]));
    }
    RH_CUDA(cudaEventRecord(e1, rt->streams[0]));
    SyncAll(rt);
    RH_CUDA(cudaEventSynchronize(e1));
    float dev_ms = 0;
    RH_CUDA(cudaEventElapsedTime(&dev_ms, e0, e1));
    const double host_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CheckSync(p);
    if (ms) *ms = std::max<double>(dev_ms, host_ms);
  });
}

int rh_program_memory(const rh_program* p, size_t* arena_bytes, size_t* pool_bytes) {
  return Guard([&] {
    if (arena_bytes) *arena_bytes = p->arena_bytes;
    if (pool_bytes) *pool_bytes = p->pool_bytes;
  });
}

namespace {
void RequireLive(const rh::Tensor& t) {
  if (t.recycled)
    Fail("intermediate buffer is reused by the arena planner after its last use; load the program "
         "with RH_FLAG_KEEP_ALL to read intermediates");
}
}  // namespace

int rh_program_local_bytes(const rh_program* p, int op, int rank, size_t* bytes) {
  return Guard([&] {
    (void)rank;
    if (op < 0 || op >= static_cast<int>(p->ops.size())) Fail("bad op index");
    if (p->out_tensor[op] < 0) Fail("op was fused into its consumer's kernel (use RH_FLAG_NO_FUSION)");
    *bytes = p->tensors[p->out_tensor[op]].bytes;
  });
}

int rh_program_read_local(rh_program* p, int op, int rank, void* dst, size_t bytes) {
  return Guard([&] {
    if (op < 0 || op >= static_cast<int>(p->ops.size())) Fail("bad op index");
    if (p->out_tensor[op] < 0) Fail("op was fused into its consumer's kernel (use RH_FLAG_NO_FUSION)");
    const rh::Tensor& t = p->tensors[p->out_tensor[op]];
    if (bytes != t.bytes) Fail("rh_program_read_local: size mismatch");
    RequireLive(t);
    const int li = p->LocalIndex(rank);
    if (t.stage >= 0 && p->StageOf(rank) != t.stage)
      Fail("op is held by pipeline stage " + std::to_string(t.stage) + ", not by rank " + std::to_string(rank));
    SyncAll(p->mesh->rt);
    DeviceGuard dg(p->mesh->rt->device_of(li));
    RH_CUDA(cudaMemcpy(dst, p->base[li] + t.offset, bytes, cudaMemcpyDeviceToHost));
  });
}

int rh_program_read_full(rh_program* p, int op, void* dst, size_t bytes) {
  return Guard([&] {
    if (op < 0 || op >= static_cast<int>(p->ops.size())) Fail("bad op index");
    rh_runtime* rt = p->mesh->rt;
    SyncAll(rt);
    const int dtype = p->ops[op].dtype;
    const int eb = rh::ElemBytes(dtype);
    Dims g(p->ops[op].dims, p->ops[op].dims + p->ops[op].rank);
    const int64_t n = Prod(g);
    if (bytes != static_cast<size_t>(n) * eb) Fail("rh_program_read_full: size mismatch");
    if (p->mat_tensor[op] >= 0) {
      const rh::Tensor& t = p->tensors[p->mat_tensor[op]];
      int li = 0;  // a local rank that holds it (pipeline programs: of the output's stage)
      if (t.stage >= 0) {
        li = -1;
        for (int k = 0; k < rt->n_local() && li < 0; ++k)
          if (p->StageOf(rt->first_rank + k) == t.stage) li = k;
        if (li < 0) Fail("output is held by pipeline stage " + std::to_string(t.stage) + ", not by this process");
      }
      DeviceGuard dg(rt->device_of(li));
      RH_CUDA(cudaMemcpy(dst, p->base[li] + t.offset, bytes, cudaMemcpyDeviceToHost));
      return;
    }
    if (p->out_tensor[op] < 0) Fail("op was fused into its consumer's kernel (use RH_FLAG_NO_FUSION)");
    RequireLive(p->tensors[p->out_tensor[op]]);
    AssembleFull(p, p->tensors[p->out_tensor[op]], dst);
  });
}

int rh_program_read_input_full(rh_program* p, int op, int slot, void* dst, size_t bytes) {
  return Guard([&] {
    if (op < 0 || op >= static_cast<int>(p->ops.size())) Fail("bad op index");
    if (slot < 0 || slot >= static_cast<int>(p->in_tensor[op].size()) || p->in_tensor[op][slot] < 0)
      Fail("rh_program_read_input_full: op has no recorded input (source, fused or reshape-free)");
    SyncAll(p->mesh->rt);
    const rh::Tensor& t = p->tensors[p->in_tensor[op][slot]];
    if (bytes != static_cast<size_t>(Prod(t.gdims)) * rh::ElemBytes(t.dtype)) Fail("size mismatch");
    RequireLive(t);
    AssembleFull(p, t, dst);
  });
}

int rh_program_num_steps(const rh_program* p, int* n) {
  return Guard([&] { *n = static_cast<int>(p->steps.size()); });
}

int rh_program_step_info(const rh_program* p, int i, rh_step_info* out) {
  return Guard([&] {
    if (i < 0 || i >= static_cast<int>(p->steps.size())) Fail("bad step index");
    const rh::Step& s = p->steps[i];
    std::memset(out, 0, sizeof(*out));
    std::strncpy(out->name, s.name.c_str(), sizeof(out->name) - 1);
    out->kind = s.kind;
    out->launches = s.launches;
    out->alg_bytes = s.alg_bytes;
    out->alg_flops = s.alg_flops;
    out->wire_bytes = s.wire_bytes;
    out->ms = s.ms;
  });
}

int rh_program_launch_count(const rh_program* p, int64_t* launches) {
  return Guard([&] {
    int64_t n = 0;
    for (const auto& s : p->steps) n += static_cast<int64_t>(s.launches) * p->mesh->rt->n_local();
    for (const auto& s : p->steps)
      if (s.p2p && p->mesh->rt->dist && p->mesh->rt->world > 1)
        n += (s.sync_slot < 0 || s.async ? 1 : 0) + (s.post_sync ? 1 : 0);  // separate barrier kernels
    if (p->n_sync_slots) n += 1;                                 // epoch tick
    *launches = n;
  });
}

int rh_reshard(rh_mesh* mesh, int axis, rh_spec from, rh_spec to, int ndim, const int64_t* dims,
               int dtype, void* const* src, void* const* dst, uint32_t flags, int iters, double* ms) {
  return Guard([&] {
    if (axis < 0 || axis >= static_cast<int>(mesh->dims.size())) Fail("rh_reshard: bad axis");
    if (from.kind == RH_PARTIAL && to.kind == RH_PARTIAL) Fail("rh_reshard: identity");
    const int na = static_cast<int>(mesh->dims.size());
    // Program: x = input (spec `from` on `axis`, Replicated elsewhere) plus a request for x in
    // `to`: the schedule is exactly the transition.
    std::vector<rh_spec> xs(na, rh_spec{RH_REPLICATED, -1, 0}), ys = xs;
    xs[axis] = from;
    ys[axis] = to;
    rh_op op0;
    std::memset(&op0, 0, sizeof(op0));
    op0.kind = RH_OP_INPUT;
    op0.dtype = dtype;
    op0.rank = ndim;
    for (int i = 0; i < ndim; ++i) op0.dims[i] = dims[i];
    for (int a = 0; a < na; ++a) op0.out_spec[a] = xs[a];
    int outs[1] = {0};
    rh_program* p = nullptr;
    int rc = LoadProgram(mesh, &op0, 1, outs, 1, flags | RH_FLAG_NO_MATERIALIZE, {{0, ys}}, &p);
    if (rc != RH_OK) throw rh::Error(rc, g_err);
    std::unique_ptr<rh_program, void (*)(rh_program*)> guard(p, DestroyProgram);
    rh_runtime* rt = mesh->rt;
    const rh::Tensor& x = p->tensors[p->out_tensor[0]];
    const int ti = p->request_tensors.at(0);
    if (p->steps.empty()) Fail("rh_reshard: no transition was scheduled");
    const rh::Tensor& y = p->tensors[ti];
    for (int li = 0; li < rt->n_local(); ++li) {
      DeviceGuard dg(rt->device_of(li));
      RH_CUDA(cudaMemcpy(p->base[li] + x.offset, src[li], x.bytes, cudaMemcpyDeviceToDevice));
    }
    HostBarrier(rt);
    RunStep(p);  // warm-up (eager), then capture + first replay: both outside the timed runs
    RunStep(p);
    SyncAll(rt);
    HostBarrier(rt);
    double t = 0;
    rc = rh_program_run(p, std::max(iters, 1), &t);
    if (rc != RH_OK) throw rh::Error(rc, g_err);
    for (int li = 0; li < rt->n_local(); ++li) {
      DeviceGuard dg(rt->device_of(li));
      RH_CUDA(cudaMemcpy(dst[li], p->base[li] + y.offset, y.bytes, cudaMemcpyDeviceToDevice));
    }
    if (ms) *ms = t;
  });
}

}  // extern "C"
