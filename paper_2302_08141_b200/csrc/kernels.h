// kernels.h — launchers of the sm_100a kernels (one translation unit per family).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.h"
#include "ew_defs.h"

namespace rh {

constexpr int kMaxGroup = 8;  // ranks per mesh-axis group (one B200 box)

// Programmatic dependent launch for the next compute-kernel launches of this host thread
// (launch.cuh; set per step by the executor's run loop).
void SetPdl(bool on);
bool PdlEnabled();

// Unsigned 32-bit division by an invariant (Granlund & Montgomery 1994, Fig. 4.1): exact for
// every 32-bit dividend.  Used for the block-cyclic index maps inside the resharding kernels.
struct FastDiv {
  uint32_t d, mul, s1, s2;
};
FastDiv MakeFastDiv(uint32_t d);
__host__ __device__ inline uint32_t Div(const FastDiv& f, uint32_t n) {
#ifdef __CUDA_ARCH__
  uint32_t t = __umulhi(f.mul, n);
#else
  uint32_t t = static_cast<uint32_t>((static_cast<uint64_t>(f.mul) * n) >> 32);
#endif
  return (t + ((n - t) >> f.s1)) >> f.s2;
}

// ------------------------------------ resharding (K9-K14) ------------------------------------
// One rank's side of a single-axis transition in the pull form: the rank fills its destination
// buffer (layout `to`, group coordinate `coord`) by reading the d group members' source buffers
// (layout `from`) directly — device-local, peer (NVLink P2P / CUDA IPC) or, for the NCCL
// baseline, sub-buffers of a staging buffer.  Partial sources are summed in rank order
// 0..d-1 in fp32 (bf16 rounded once), matching the oracle bit for bit.
// Fused pre-transition group barrier (one process per GPU): every CTA of the pull kernel
// first publishes this run's epoch into each member's flag slot for this transition (idempotent
// 4-byte peer stores, so no CTA depends on another CTA of its own grid being resident), then
// waits until every member's epoch has arrived in its own slot.  Replaces a separate barrier
// kernel launch per transition.
struct PeerSync {
  uint32_t* peer_slot[kMaxGroup];  // member k's flag row for this transition (mapped): [world]
  uint32_t* my_slot;               // this rank's flag row for this transition
  const uint32_t* epoch;           // this rank's run counter (device)
  int members[kMaxGroup];
  int d;                           // 0: no fused barrier
  int me;
  // Bounded wait: a peer that has not arrived within timeout_ns (globaltimer) records
  // SyncErrorCode(me, member) in *err and the kernel proceeds; the host turns it into
  // RH_ERR_TIMEOUT after the run instead of hanging the GPU.
  uint32_t* err;
  uint64_t timeout_ns;
};
// Host: RH_SYNC_TIMEOUT_MS (default 60000) in ns; error word encoding / decoding.
uint64_t SyncTimeoutNs();
__host__ __device__ inline uint32_t SyncErrorCode(int me, int member) {
  return 0x80000000u | (static_cast<uint32_t>(me & 0xff) << 8) | static_cast<uint32_t>(member & 0xff);
}

struct PullArgs {
  void* dst;
  const void* src[kMaxGroup];
  AxisView to, from;
  int coord;
  int64_t n_dst;  // destination elements
  int dtype;
  PeerSync sync;  // sync.d == 0 unless fused
  int max_blocks = 0;  // grid cap (0: default).  Spinning pull grids never fill the GPU (at most
                       // 6 of 8 CTA slots per SM), so a pull on the side stream can always be
                       // scheduled next to a main-stream pull that waits for a peer.
};
// Increments the device run counter (start of every run with fused barriers).
void LaunchEpochTick(uint32_t* epoch, cudaStream_t s);
// Returns the number of kernel launches (0 or 1).
int LaunchPull(const PullArgs& a, cudaStream_t s);
// Fine-grained block-cyclic layouts (runs shorter than a sector): register-permute kernels that
// keep every global access a 16-byte vector (k_reshard.cu, FineDeinterleaveKernel /
// FineInterleaveKernel).  kind 0 = de-interleave (push: the running rank c splits n contiguous
// local elements into d targets, unit m -> member m % d); kind 1 = interleave (pull: d streams
// into n contiguous elements).  The strided side's element offset of super-vector s is s * n/(d*
// n_sv) when `lin`, else f0/d with i0 = s*sv, f0 = ((i0/run)*d + c)*run + i0%run.
struct FineArgs {
  int kind;
  int d;
  int unit_bytes;  // 2, 4, 8, 16 or 32
  int eb;
  const void* in[kMaxGroup];
  void* out[kMaxGroup];
  int64_t n;       // elements on the contiguous side
  int lin;
  int64_t run;
  int c;
  int only = -1;   // de-interleave: write only member `only` (a local slice)
  PeerSync sync;
  int max_blocks = 0;
};
bool FineSupported(int d, int unit_bytes, int eb, int64_t n_contig);
int LaunchFine(const FineArgs& a, cudaStream_t s);
// Push all-gather (S -> R into a persistent destination): a.src[k] = member k's replicated
// destination, a.dst = this rank's local shard (roles reversed against a pull).
bool PushGatherSupported(const PullArgs& a);
int LaunchPushGather(const PullArgs& a, cudaStream_t s);
// Grouped transitions: n independent pulls of one mesh axis as ONE launch behind ONE fused
// barrier (`sync` of LaunchPullMulti; the PullArgs' own sync is ignored).  PreparePullMulti
// writes the segment table (PullMultiTableBytes) once and returns false when the pulls cannot
// share a launch (zero-fill, staged fine-grained sources, mixed source kinds or dtypes).
size_t PullMultiTableBytes(int n);
bool PreparePullMulti(const PullArgs* a, int n, int max_blocks, void* table);
void ReleasePullMulti(const void* table);
int LaunchPullMulti(const void* table, const PeerSync& sync, cudaStream_t s);

// dst_local[l] = full[ComposedLocalToGlobal(m, l)]  (R -> any composed spec slice)
void LaunchSliceComposed(void* dst, const void* full, const ComposedMap& m, int64_t n, int dtype,
                         cudaStream_t s);
// Synthetic init of one rank's local buffer (Philox4x32-10 by global flat index).
void LaunchSynthetic(void* dst, const ComposedMap& m, int64_t n, uint64_t seed, uint32_t op_index,
                     float scale, int dtype, cudaStream_t s);

// ----------------------------------------- local ops -----------------------------------------
constexpr int kMaxChain = 64;
struct ChainArgs {
  int32_t n_fn;
  int32_t fns[kMaxChain];
  int32_t n_tab;
  uint64_t tab_off[kMaxTanhRuns];        // arena offsets (host side)
  const uint16_t* tab[kMaxTanhRuns];     // device pointers, patched per rank at launch
};
// Host: T^k table (kTanhRunEntries values) of the correctly rounded bf16 tanh.
void TanhRunTable(int k, uint16_t* out);
// Elementwise unary chain (one fused pass).  softmax is not elementwise and has its own kernel.
void LaunchUnaryChain(void* out, const void* in, int64_t n, const ChainArgs& c, int dtype,
                      cudaStream_t s);
void LaunchSoftmaxRows(void* out, const void* in, int64_t rows, int64_t cols, int dtype,
                       cudaStream_t s);
// Elementwise chain program (one kernel for a chain of add / mul / unary ops that crosses
// multi-use values: the forward tanh chains whose outputs the backward keeps, the backward's
// dy * (1 - y^2) accumulations).  An accumulator walks the chain; every instruction is
// warp-uniform, so the interpreter costs one switch per 8 elements:
//   LOAD k          acc = in[k]
//   UNARY fn        acc = fn(acc)        (fn >= kFnTanhRun: T^k table lookup, bf16)
//   ADD src/MUL src acc = acc op src     (src: input k, kEwSrcKeep, kEwSrcAcc)
//   KEEP            keep = acc
//   STORE j         out[j] = acc
//   TBWD k          keep = acc; acc = keep + -((acc * in[k]) * in[k])  — the backward of tanh
//                   (peephole of KEEP, MUL k, MUL k, UNARY neg, ADD keep; same roundings)
// Every op result is rounded to the program dtype, as in the one-op-per-kernel path.
inline int32_t EwIns(int op, int arg) { return op | (arg << 8); }
void TanhLadderTable(const int* powers, int n, uint16_t* out);
void LaunchEwProg(const EwArgs& a, int dtype, cudaStream_t s);
// Kernel family a program runs in (LaunchEwProg's choice; the JIT compiles the same family).
enum EwKind { kEwKindF32 = 0, kEwKindBf16 = 1, kEwKindRematHalf = 2, kEwKindRematFull = 3, kEwKindLadder = 4,
              kEwKindLadderRemat = 5 };
int EwKindOf(const EwArgs& a, int dtype);
// Per-program kernels (ew_jit.cpp): EwJitRegister returns the EwArgs::jit value for a program
// (0 when RH_EW_JIT=0); EwJitBuild compiles every registered, not yet compiled program with
// NVRTC (one call per executor build); EwJitLaunch launches a's compiled kernel and returns
// false when there is none (compile failure: the interpreter kernel runs instead).
int32_t EwJitRegister(const EwArgs& a, int dtype);
void EwJitBuild();
bool EwJitLaunch(const EwArgs& a, int blocks, size_t smem, cudaStream_t s);
// out = a (+|*) b, then an optional unary chain (epilogue fusion).
void LaunchBinary(void* out, const void* a, const void* b, int64_t n, bool mul, const ChainArgs& c,
                  int dtype, cudaStream_t s);
void LaunchReduceSum(void* out, const void* in, int64_t outer, int64_t e, int64_t inner, int dtype,
                     cudaStream_t s);
void LaunchTranspose(void* out, const void* in, int nd, const int64_t* in_dims, const int* perm,
                     int dtype, cudaStream_t s);
void LaunchBroadcast(void* out, const void* in, int64_t n_out, int64_t n_in, int dtype,
                     cudaStream_t s);
// Concat of every piece in one launch (16-byte units): row16/off16/orow16 in 16-byte units.
// Returns false when a row, offset or pointer is not 16-byte aligned (use the per-piece form).
constexpr int kMaxConcat = 64;
struct ConcatArgs {
  void* out;
  const void* in[kMaxConcat];
  int64_t row16[kMaxConcat], off16[kMaxConcat];
  int64_t outer, orow16;
  int n;
};
bool LaunchConcat(const ConcatArgs& a, cudaStream_t s);
// Concat: copies `in` ([outer, row] contiguous) into out at column offset `off` of rows `orow`.
void LaunchConcatPiece(void* out, const void* in, int64_t outer, int64_t row, int64_t orow,
                       int64_t off, int dtype, cudaStream_t s);
void LaunchZero(void* dst, size_t bytes, cudaStream_t s);
// ApplyGradients (taskgraph.cpp:161-165): w -= lr * g elementwise, in place (fp32 arithmetic,
// bf16 rounded once).
void LaunchSgd(void* w, const void* g, int64_t n, float lr, int dtype, cudaStream_t s);
// A fused-barrier rendezvous on its own (one CTA): the sending side of a cross-stage transfer.
void LaunchPeerSync(const PeerSync& sync, cudaStream_t s);
// End-to-end input gather (rh_program_run_host): every member q of the world holds its piece
// [q*part, (q+1)*part) of a replicated input in its stage buffer src[q] (mapped); behind the
// fused barrier `sync` (every member's H2D of this step landed) this rank pulls the peers'
// pieces into the same offsets of dst = src[me].  part % 16 == 0.
void LaunchGatherSlices(char* const* src, int world, int me, size_t part, const PeerSync& sync, cudaStream_t s);

// ------------------------------------------ GEMM (K1) ----------------------------------------
// C[m,n] = op(A)[m,k] . op(B)[k,n]; A stored [m,k] (ta=0) or [k,m] (ta=1), B stored [k,n]
// (tb=0) or [n,k] (tb=1); fp32 accumulation; C row-major in `dtype`; optional unary chain
// applied in the epilogue.
// The output all-gather of a row-sharded GEMM output, fused into the GEMM's epilogue (executor
// TryPushMaterialize): every output row r of this rank's C also goes to dst[k] + (row_off + r)
// * n for each of the n group members k (this rank included), behind a barrier fused into the
// kernel (block 0 arrives at the start: this rank's copy is free; every epilogue warp waits for
// all members before its first push).  n = 0: none.
struct GemmPush {
  int n;
  void* dst[kMaxGroup];  // member k's replicated copy: [rows_full, GemmArgs::n] row-major
  int64_t row_off, rows_full;
  PeerSync sync;
  // scatter_dim >= 0 (the reduce-scatter of a Partial output, executor TryPushReduceScatter):
  // output box (row, col) goes only to its owner k = (scatter_dim ? col : row) / part, into
  // dst[k] = this rank's slot of k's staging, [m, part] (dim 1) or [part, n] (dim 0).
  int scatter_dim = -1;
  int64_t part = 0;
};
struct GemmArgs {
  void* c;
  const void* a;
  const void* b;
  int64_t m, n, k;
  bool ta, tb;
  int dtype;
  ChainArgs epi;
  // fp32 tensor-core path (3xTF32): device scratch for the hi/lo splits of A and B
  // (GemmTf32x3ScratchBytes bytes, reused by every GEMM of a program: they run in stream order).
  void* scratch = nullptr;
  // bf16 stream-K (CTA-pair kernel): kGemmSkFlagBytes of zeroed flags, owned by the caller and
  // left zeroed by every launch; the partial accumulators live in `scratch`.  nullptr: no
  // stream-K.
  uint32_t* sk_flags = nullptr;
  // Fused residual add (bf16): C = round(GEMM [+ chain]) + resid, resid [m, n] row-major like C
  // (the add op after the GEMM, executor PlanFusion), every kernel and the split-K reduce
  // included.  nullptr: none.
  const void* resid = nullptr;
  GemmPush push{};
};
// A push epilogue is available when the GEMM runs without split-K / stream-K (one kernel writes
// the final values).
bool GemmTcPushSupported(const GemmArgs& g, bool single_pass = false);
constexpr size_t kGemmSkFlagBytes = 4096;
size_t GemmTf32x3ScratchBytes(const GemmArgs& g);
// Scratch the tensor-core path wants for this GEMM (3xTF32 splits, or bf16 split-K partials).
size_t GemmTcScratchBytes(const GemmArgs& g);
// CUDA-core kernel (any shape/layout); the test reference for the tensor-core path.  With
// g.scratch (>= GemmSimtScratchBytes) small-M shapes run split-K.  Returns the launches issued.
int LaunchGemmSimt(const GemmArgs& g, cudaStream_t s);
size_t GemmSimtScratchBytes(const GemmArgs& g);
// tcgen05 / TMEM / TMA kernel.  Returns false when the shape/layout is not supported by it.
bool GemmTcSupported(const GemmArgs& g);
void LaunchGemmTc(const GemmArgs& g, cudaStream_t s);
// Launches LaunchGemmTc issues: 3xTF32 3 (two splits + GEMM), bf16 split-K 2 (+ reduce), else 1.
int GemmTcLaunches(const GemmArgs& g);
const char* GemmTcSchedule(const GemmArgs& g);  // " [split-k]" or ""
// Grouped tcgen05 GEMM: n_prob independent problems of g's shape (m, n, k, ta, tb, dtype, epi)
// in ONE persistent launch (the per-head q/k/v, score and context GEMMs of an attention block),
// laid side by side along a virtual N; a tile spans problems when they all read the same A.
// PrepareGemmTcGroup writes the device table (GemmTcGroupTableBytes: per-problem TMA maps and
// output pointers) once; LaunchGemmTcGroup replays it.
bool GemmTcGroupSupported(const GemmArgs& g, int n_prob, bool shared_a);
size_t GemmTcGroupTableBytes(int n_prob);
const char* GemmTcGroupSchedule(const GemmArgs& g, int n_prob, bool shared_a);
void PrepareGemmTcGroup(const GemmArgs& g, int n_prob, const void* const* a, const void* const* b,
                        void* const* c, void* table);
void ReleaseGemmTcGroup(const void* table);
void LaunchGemmTcGroup(const GemmArgs& g, const void* table, cudaStream_t s);

// Fused attention-head chain (the 32-head block): per head h, O_h = chain(round(Q_h K_h^T)) V_h
// with Q_h [sq, 128], K_h / V_h [sk, 128], O_h [sq, 128] bf16 row-major and `epi` the score
// GEMM's epilogue chain; the sq x sk scores stay on chip.  PrepareAttnChain writes the per-head
// TMA maps (AttnChainTableBytes) once.
bool AttnChainSupported(int n_heads, int64_t sq, int64_t sk, int64_t d);
size_t AttnChainTableBytes(int n_heads);
void PrepareAttnChain(int n_heads, int64_t sq, int64_t sk, const void* const* q, const void* const* k,
                      const void* const* v, void* const* o, void* table);
void LaunchAttnChain(int n_heads, int64_t sq, int64_t sk, const ChainArgs& epi, const void* table, cudaStream_t s);

// --------------------------------------- cross-GPU sync --------------------------------------
// Group barrier over CUDA-IPC-mapped flag arrays (one process per GPU only: every member runs on
// its own GPU, so the spin never waits on a kernel of the same GPU).
struct BarrierArgs {
  uint32_t* peer_flags[kMaxGroup];  // member k's flag array (mapped)
  uint32_t* my_flags;               // this rank's flag array
  uint32_t* counter;                // this rank's barrier sequence counter (device)
  int members[kMaxGroup];           // global ranks of the group
  int d;
  int me;                           // my global rank
  uint32_t* err;                    // bounded wait (PeerSync)
  uint64_t timeout_ns;
};
void LaunchBarrier(const BarrierArgs& b, cudaStream_t s);

}  // namespace rh
