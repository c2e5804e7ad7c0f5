// k_reshard.cu — resharding transitions (K9 slice, K10 all-gather, K11 reduce-scatter,
// K12 all-reduce, K13 all-to-all, K14 zero-fill), synthetic init (K17) and the cross-GPU
// group barrier.
//
// Every transition of sharding.cpp:104-142 is one "pull" kernel per destination rank: the rank
// walks its destination buffer in order (coalesced 16-byte stores), maps each 16-byte unit to
// its global position and reads it from whichever group member owns it (Shard), from its own
// copy (Replicated) or from all members summed in rank order (Partial).  Sources are device
// pointers that may live on this GPU, on a peer GPU over NVLink, or in an NCCL staging buffer.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "kernels.h"
#include "launch.cuh"

namespace rh {

FastDiv MakeFastDiv(uint32_t d) {
  if (d == 0) Fail("FastDiv: division by zero");
  FastDiv f{};
  f.d = d;
  uint32_t l = 0;
  while ((uint64_t{1} << l) < d) ++l;  // l = ceil(log2 d)
  f.mul = static_cast<uint32_t>(((uint64_t{1} << 32) * ((uint64_t{1} << l) - d)) / d + 1);
  f.s1 = l > 0 ? 1 : 0;
  f.s2 = l > 0 ? l - 1 : 0;
  const uint32_t probes[] = {0u, 1u, d - 1, d, d + 1, 2 * d - 1, 0x7fffffffu, 0xfffffffeu, 0xffffffffu};
  for (uint32_t n : probes) {
    if (Div(f, n) != n / d) Fail("FastDiv self-check failed");
  }
  return f;
}

namespace {

template <int VB>
struct VecT;
template <>
struct VecT<16> {
  using T = uint4;
};
template <>
struct VecT<8> {
  using T = uint2;
};
template <>
struct VecT<4> {
  using T = uint32_t;
};
template <>
struct VecT<2> {
  using T = uint16_t;
};

struct PullDev {
  char* dst;
  const char* src[kMaxGroup];
  int to_shard;
  FastDiv qst;  // destination run length (units)
  int from_kind;
  FastDiv qsf;  // source run length (units)
  FastDiv dd;   // group size
  uint32_t coord;
  uint32_t n;   // destination units
  uint32_t rot; // traversal start (units): coord * n / d, so that at any moment the d ranks of a
                // group read from d different sources instead of all hammering the same peer
  PeerSync sync;
  uint32_t blk0, nblk;  // grouped launches (PullMultiKernel): this segment's block range
  int32_t d_sum;        // Partial sources: members summed
};

__device__ __forceinline__ uint32_t Rotate(uint32_t i, uint32_t rot, uint32_t n) {
  const uint32_t j = i + rot;
  return j >= n ? j - n : j;
}

__device__ __forceinline__ void StRelaxedSys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t LdRelaxedSys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Fused pre-transition barrier (see PeerSync): arrive (every CTA, idempotent), then wait.
__device__ __forceinline__ uint32_t LdAcquireSysU32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t GlobalTimerNs() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin until *f reaches `want` (wrapping compare), at most timeout_ns: on timeout record the
// (me, member) pair in *err (first one wins) and give up — the run then fails loudly on the
// host (RH_ERR_TIMEOUT) instead of hanging the GPU.
__device__ __forceinline__ void WaitFlag(const uint32_t* f, uint32_t want, uint32_t* err, uint64_t timeout_ns,
                                         int me, int member, bool sleep) {
  if (static_cast<int32_t>(LdAcquireSysU32(f) - want) >= 0) return;
  const uint64_t t0 = GlobalTimerNs();
  uint32_t n = 0;
  while (static_cast<int32_t>(LdAcquireSysU32(f) - want) < 0) {
    if (sleep) __nanosleep(64);
    if ((++n & 1023) == 0 && timeout_ns && GlobalTimerNs() - t0 > timeout_ns) {
      if (err) atomicCAS(err, 0u, SyncErrorCode(me, member));
      return;
    }
  }
}

// Block 0 publishes the arrival (it is dispatched first; every other CTA only polls its own,
// local flag row, so no CTA waits on a CTA of its own grid that might not be resident).
__device__ __forceinline__ void ArriveAndWait(const PeerSync& s) {
  PdlWait();  // launched with PDL after a compute kernel: its writes are complete and visible
  if (s.d == 0) return;
  const int t = threadIdx.x;
  if (t < s.d) {
    const uint32_t e = *reinterpret_cast<const volatile uint32_t*>(s.epoch);
    if (blockIdx.x == 0) {
      __threadfence_system();  // this rank's producer writes precede the signal
      StRelaxedSys(s.peer_slot[t] + s.me, e);
    }
    WaitFlag(s.my_slot + s.members[t], e, s.err, s.timeout_ns, s.me, s.members[t], false);
  }
  __syncthreads();
}

__global__ void EpochTickKernel(uint32_t* epoch) { *epoch += 1; }

__global__ void PeerSyncKernel(PeerSync s) { ArriveAndWait(s); }

struct GatherArgs {
  char* src[kMaxGroup];
  int world, me;
  uint64_t part16;  // 16-byte chunks per piece
  PeerSync sync;
};

// Peer q's piece comes from peer (me + 1 + k) % world for k = 0..world-2: at any moment the
// ranks read from different peers.
__global__ void __launch_bounds__(256) GatherSlicesKernel(const __grid_constant__ GatherArgs a) {
  ArriveAndWait(a.sync);
  const uint64_t total = a.part16 * static_cast<uint64_t>(a.world - 1);
  uint4* dst = reinterpret_cast<uint4*>(a.src[a.me]);
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i / a.part16);
    const uint64_t j = i - static_cast<uint64_t>(k) * a.part16;
    const int q = (a.me + 1 + k) % a.world;
    const uint64_t o = static_cast<uint64_t>(q) * a.part16 + j;
    dst[o] = reinterpret_cast<const uint4*>(a.src[q])[o];
  }
}

__device__ __forceinline__ uint32_t DstToGlobal(const PullDev& a, uint32_t i) {
  if (!a.to_shard) return i;
  const uint32_t p = Div(a.qst, i);
  const uint32_t u = i - p * a.qst.d;
  return (p * a.dd.d + a.coord) * a.qst.d + u;
}

// Shard / Replicated sources: a pure copy of VB-byte units.  `bid` / `nb`: this block's index
// among the blocks working on this transition (the whole grid, or a grouped launch's segment).
template <int VB, bool kFromShard>
__device__ __forceinline__ void PullCopyBody(const PullDev& a, uint32_t bid, uint32_t nb) {
  using V = typename VecT<VB>::T;
  constexpr int U = 4;
  const uint32_t stride = nb * blockDim.x;
  uint32_t i = bid * blockDim.x + threadIdx.x;
  for (; i < a.n; i += U * stride) {
    V v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const uint32_t ii = Rotate(i + j * stride, a.rot, a.n);
      if (i + j * stride < a.n) {
        const uint32_t f = DstToGlobal(a, ii);
        if (kFromShard) {
          const uint32_t q = Div(a.qsf, f);
          const uint32_t u = f - q * a.qsf.d;
          const uint32_t pp = Div(a.dd, q);
          const uint32_t r = q - pp * a.dd.d;
          v[j] = reinterpret_cast<const V*>(a.src[r])[pp * a.qsf.d + u];
        } else {
          v[j] = reinterpret_cast<const V*>(a.src[a.coord])[f];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (i + j * stride < a.n) reinterpret_cast<V*>(a.dst)[Rotate(i + j * stride, a.rot, a.n)] = v[j];
    }
  }
}

template <int VB, bool kFromShard>
__global__ void __launch_bounds__(256) PullCopyKernel(PullDev a) {
  ArriveAndWait(a.sync);
  PullCopyBody<VB, kFromShard>(a, blockIdx.x, gridDim.x);
}

template <typename T>
__device__ __forceinline__ float ToF(T x);
template <>
__device__ __forceinline__ float ToF<float>(float x) {
  return x;
}
template <>
__device__ __forceinline__ float ToF<__nv_bfloat16>(__nv_bfloat16 x) {
  return __bfloat162float(x);
}
template <typename T>
__device__ __forceinline__ T FromF(float x);
template <>
__device__ __forceinline__ float FromF<float>(float x) {
  return x;
}
template <>
__device__ __forceinline__ __nv_bfloat16 FromF<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// Partial sources: sum of the d members' values at the same global position, rank order.
template <typename T, int VB>
__device__ __forceinline__ void PullSumBody(const PullDev& a, int d, uint32_t bid, uint32_t nb) {
  using V = typename VecT<VB>::T;
  constexpr int E = VB / sizeof(T);
  const uint32_t stride = nb * blockDim.x;
  for (uint32_t i0 = bid * blockDim.x + threadIdx.x; i0 < a.n; i0 += stride) {
    const uint32_t i = Rotate(i0, a.rot, a.n);
    const uint32_t f = DstToGlobal(a, i);
    float acc[E];
    for (int k = 0; k < d; ++k) {
      V v = reinterpret_cast<const V*>(a.src[k])[f];
      const T* t = reinterpret_cast<const T*>(&v);
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] = k == 0 ? ToF<T>(t[e]) : __fadd_rn(acc[e], ToF<T>(t[e]));
    }
    V o;
    T* t = reinterpret_cast<T*>(&o);
#pragma unroll
    for (int e = 0; e < E; ++e) t[e] = FromF<T>(acc[e]);
    reinterpret_cast<V*>(a.dst)[i] = o;
  }
}

template <typename T, int VB>
__global__ void __launch_bounds__(256) PullSumKernel(PullDev a, int d) {
  ArriveAndWait(a.sync);
  PullSumBody<T, VB>(a, d, blockIdx.x, gridDim.x);
}

// Grouped transitions: independent single-axis transitions of one mesh axis (the per-head K / V
// all-gathers of an attention block) as ONE launch behind ONE fused barrier.  Segment k owns
// blocks [blk0, blk0 + nblk); the segment table lives in device memory (written at load).
// kKind: 0 Shard-source copy, 1 Replicated-source copy, 2 Partial-source sum.
template <int VB, int kKind, typename T>
__global__ void __launch_bounds__(256) PullMultiKernel(const PullDev* __restrict__ seg, int n, PeerSync sync) {
  ArriveAndWait(sync);
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seg[mid].blk0 <= blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const PullDev& a = seg[lo];
  if constexpr (kKind == 2) {
    PullSumBody<T, VB>(a, a.d_sum, blockIdx.x - a.blk0, a.nblk);
  } else {
    PullCopyBody<VB, kKind == 0>(a, blockIdx.x - a.blk0, a.nblk);
  }
}

// Fine-grained (strided) sources: Shard(dim, s) with runs shorter than 16 bytes interleave the
// d members element by element, so a per-element pull would issue 2-4-byte gathers.  Instead a
// block takes L consecutive destination elements whose global range [f0, f0+L) is aligned to a
// full round-robin cycle Lr = Qs_from * d: each member then owns ONE contiguous L/d slice of it
// (local offset (f0/Lr)*Qs_from).  The block copies the d slices into shared memory with 16-byte
// loads (local HBM or NVLink peer), then writes the L destination elements with 16-byte stores,
// re-interleaving through shared memory.
struct StagedDev {
  char* dst;
  const char* src[kMaxGroup];
  int to_shard;
  FastDiv qst;  // destination run (elements)
  FastDiv qsf;  // source run (elements)
  FastDiv dd;
  uint32_t coord;
  uint32_t L;       // elements per chunk
  uint32_t per;     // L / d
  uint32_t chunks;  // destination chunks
  uint32_t cpb;     // chunks per block iteration
  PeerSync sync;
};

// A block iteration handles `cpb` consecutive chunks (cpb x L ~ 4096 elements), so short chunks
// (L = 32..64 elements for stride-1 sources) still give every thread 16-byte work.
template <typename T>
__global__ void __launch_bounds__(256) PullStagedKernel(StagedDev a) {
  extern __shared__ __align__(16) unsigned char smem_stage[];
  T* tile = reinterpret_cast<T*>(smem_stage);
  ArriveAndWait(a.sync);
  constexpr int E = 16 / sizeof(T);  // elements per 16-byte vector
  const uint32_t d = a.dd.d;
  const uint32_t Lr = a.qsf.d * d;
  const uint32_t vper = a.per / E, vchunk_in = vper * d, vchunk_out = a.L / E;
  const uint32_t rot = a.coord * (a.chunks / d);
  auto chunk_base = [&](uint32_t chunk, uint32_t* i0) {  // dst offset, each member's local start
    *i0 = chunk * a.L;
    uint32_t f0 = *i0;
    if (a.to_shard) {
      const uint32_t p = Div(a.qst, *i0);
      f0 = (p * d + a.coord) * a.qst.d + (*i0 - p * a.qst.d);
    }
    return (f0 / Lr) * a.qsf.d;
  };
  for (uint32_t g0 = blockIdx.x * a.cpb; g0 < a.chunks; g0 += gridDim.x * a.cpb) {
    const uint32_t ng = min(a.cpb, a.chunks - g0);
    for (uint32_t v = threadIdx.x; v < ng * vchunk_in; v += blockDim.x) {
      const uint32_t cg = v / vchunk_in, rem = v - cg * vchunk_in;
      const uint32_t k = rem / vper, j = rem - k * vper;
      uint32_t i0;
      const uint32_t base = chunk_base(Rotate(g0 + cg, rot, a.chunks), &i0);
      reinterpret_cast<uint4*>(tile + cg * a.L)[k * vper + j] =
          reinterpret_cast<const uint4*>(a.src[k] + size_t(base) * sizeof(T))[j];
    }
    __syncthreads();
    for (uint32_t v = threadIdx.x; v < ng * vchunk_out; v += blockDim.x) {
      const uint32_t cg = v / vchunk_out, vv = v - cg * vchunk_out;
      const uint32_t chunk = Rotate(g0 + cg, rot, a.chunks);
      const T* t = tile + cg * a.L;
      T out[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t i = vv * E + e;        // offset in the chunk == offset from f0
        const uint32_t q = Div(a.qsf, i);     // run index
        const uint32_t qd = Div(a.dd, q);
        const uint32_t r = q - qd * d;        // owner
        out[e] = t[r * a.per + qd * a.qsf.d + (i - q * a.qsf.d)];
      }
      reinterpret_cast<uint4*>(a.dst + size_t(chunk) * a.L * sizeof(T))[vv] = *reinterpret_cast<uint4*>(out);
    }
    __syncthreads();
  }
}

// Returns true when the staged kernel was launched.
bool TryLaunchStaged(const PullArgs& a, cudaStream_t s) {
  if (a.from.kind != RH_SHARD) return false;
  const int eb = ElemBytes(a.dtype);
  const int64_t qsf = a.from.Qs, d = a.from.d;
  if (qsf * eb >= 16) return false;  // runs already vectorize in the plain pull kernel
  const int64_t Lr = qsf * d;
  const int64_t run = a.to.kind == RH_SHARD ? a.to.Qs : a.n_dst;
  if (a.to.kind == RH_SHARD && a.to.Qs % Lr != 0) return false;
  const int64_t E = 16 / eb;
  int64_t L = 0;
  for (int64_t m = 1; Lr * m <= 8192; m *= 2) {
    const int64_t cand = Lr * m;
    if (run % cand == 0 && (cand / d) % E == 0) L = cand;
  }
  if (L == 0) return false;
  for (int k = 0; k < d; ++k)
    if (reinterpret_cast<uintptr_t>(a.src[k]) % 16) return false;
  if (reinterpret_cast<uintptr_t>(a.dst) % 16) return false;
  const int64_t total = a.to.kind == RH_SHARD ? a.n_dst * a.to.d : a.n_dst;
  if (total >= (int64_t{1} << 32)) return false;
  StagedDev sd{};
  sd.dst = static_cast<char*>(a.dst);
  for (int k = 0; k < kMaxGroup; ++k) sd.src[k] = static_cast<const char*>(a.src[k]);
  sd.to_shard = a.to.kind == RH_SHARD;
  sd.qst = MakeFastDiv(sd.to_shard ? static_cast<uint32_t>(a.to.Qs) : 1u);
  sd.qsf = MakeFastDiv(static_cast<uint32_t>(qsf));
  sd.dd = MakeFastDiv(static_cast<uint32_t>(d));
  sd.coord = static_cast<uint32_t>(a.coord);
  sd.sync = a.sync;
  sd.L = static_cast<uint32_t>(L);
  sd.per = static_cast<uint32_t>(L / d);
  sd.chunks = static_cast<uint32_t>(a.n_dst / L);
  sd.cpb = static_cast<uint32_t>(std::max<int64_t>(1, 4096 / L));
  const int64_t groups = (sd.chunks + sd.cpb - 1) / sd.cpb;
  const int blocks = static_cast<int>(std::min<int64_t>(groups, a.max_blocks > 0 ? a.max_blocks : SmCount() * 6));
  const size_t smem = static_cast<size_t>(sd.cpb) * L * eb;
  if (eb == 2) PullStagedKernel<uint16_t><<<blocks, 256, smem, s>>>(sd);
  else PullStagedKernel<uint32_t><<<blocks, 256, smem, s>>>(sd);
  RH_CUDA(cudaGetLastError());
  return true;
}

int Gcd(int64_t a, int64_t b) {
  while (b) {
    int64_t t = a % b;
    a = b;
    b = t;
  }
  return static_cast<int>(std::min<int64_t>(a, 1 << 30));
}

template <int VB>
void LaunchPullVB(const PullArgs& a, PullDev& dv, cudaStream_t s) {
  const uint32_t n = dv.n;
  const int cap = a.max_blocks > 0 ? a.max_blocks : SmCount() * 6;
  int blocks = static_cast<int>(std::min<int64_t>((n + 1023) / 1024, cap));
  blocks = std::max(blocks, 1);
  if (a.from.kind == RH_PARTIAL) {
    const int sb = static_cast<int>(std::min<int64_t>((n + 255) / 256, cap));
    if (a.dtype == RH_BF16) {
      if constexpr (VB >= 2) LaunchPdl(PullSumKernel<__nv_bfloat16, VB>, sb, 256, 0, s, dv, a.from.d);
    } else {
      if constexpr (VB >= 4) LaunchPdl(PullSumKernel<float, VB>, sb, 256, 0, s, dv, a.from.d);
    }
  } else if (a.from.kind == RH_SHARD) {
    LaunchPdl(PullCopyKernel<VB, true>, blocks, 256, 0, s, dv);
  } else {
    LaunchPdl(PullCopyKernel<VB, false>, blocks, 256, 0, s, dv);
  }
  RH_CUDA(cudaGetLastError());
}

// ------------------------ fine-grained layouts: unit (de)interleave ------------------------
// Block-cyclic layouts whose runs are shorter than a sector (Shard(1,1) of a [N,4096] tensor:
// 2-byte runs) make a plain pull read or write 2..16-byte pieces across NVLink.  Instead:
//   De-interleave (push, run by source rank c): a thread reads D*W contiguous bytes of its local
//     buffer (W = max(16, UB) bytes per member; UB = the pattern's unit), unit m of them belongs
//     to member m % D at position m / D, and writes W contiguous bytes to each member's target
//     (the member's destination directly, or its staging stream for this source).
//   Interleave (pull, run by destination rank c): a thread reads W contiguous bytes from each
//     member's stream, unit m of its output comes from member m % D, and writes D*W contiguous
//     bytes.
// The unit permutation runs in registers (compile-time D and UB: register moves / PRMT), every
// global access is a 16-byte vector and every warp access 512 contiguous bytes per stream.
// Offsets (elements) of super-vector s on the strided side: lin ? s*Wel
//   : f0 / D with i0 = s*D*Wel, f0 = ((i0 / R)*D + c)*R + i0 % R   (R: that side's run length).
struct FineDev {
  const char* in[kMaxGroup];
  char* out[kMaxGroup];
  uint32_t n_sv;   // super-vectors
  uint32_t sv;     // elements per super-vector (D * Wel)
  FastDiv run;     // R (elements), non-linear offsets only
  uint32_t c;      // coordinate of the running rank
  uint32_t eb;     // element bytes
  int lin;
  int only;        // de-interleave: write member `only` only (local slice), -1: every member
  PeerSync sync;
};

__device__ __forceinline__ uint64_t FineOffset(const FineDev& a, uint32_t s, uint32_t d) {
  const uint32_t wel = a.sv / d;
  if (a.lin) return static_cast<uint64_t>(s) * wel;
  const uint64_t i0 = static_cast<uint64_t>(s) * a.sv;
  const uint32_t q = Div(a.run, static_cast<uint32_t>(i0));  // i0 < 2^32 (host-checked)
  const uint64_t f0 = (static_cast<uint64_t>(q) * d + a.c) * a.run.d + (i0 - static_cast<uint64_t>(q) * a.run.d);
  return f0 / d;
}

// 16-bit unit x of a word array (compile-time x after unrolling)
template <int N>
__device__ __forceinline__ uint32_t Half2(const uint32_t (&w)[N], int lo, int hi) {
  // halfword lo -> bits 0..15, halfword hi -> bits 16..31
  const uint32_t sel = ((lo & 1) ? 0x32u : 0x10u) | (((hi & 1) ? 0x76u : 0x54u) << 8);
  return __byte_perm(w[lo >> 1], w[hi >> 1], sel);
}

template <int D, int UB>
__global__ void __launch_bounds__(256) FineDeinterleaveKernel(FineDev a) {
  constexpr int W = UB < 16 ? 16 : UB;  // bytes per member per super-vector
  constexpr int NV = W / 16;            // uint4 per member
  ArriveAndWait(a.sync);
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < a.n_sv; s += gridDim.x * blockDim.x) {
    const uint4* src = reinterpret_cast<const uint4*>(a.in[0]) + static_cast<size_t>(s) * D * NV;
    uint32_t w[4 * D * NV];
#pragma unroll
    for (int j = 0; j < D * NV; ++j) {
      const uint4 v = src[j];
      w[4 * j] = v.x;
      w[4 * j + 1] = v.y;
      w[4 * j + 2] = v.z;
      w[4 * j + 3] = v.w;
    }
    const uint64_t off = FineOffset(a, s, D) * a.eb;
#pragma unroll
    for (int r = 0; r < D; ++r) {
      if (a.only >= 0 && a.only != r) continue;
      uint32_t o[4 * NV];
      if constexpr (UB >= 16) {  // unit = NV uint4, unit m -> member m
#pragma unroll
        for (int q = 0; q < 4 * NV; ++q) o[q] = w[r * 4 * NV + q];
      } else if constexpr (UB == 8) {  // 2 units of 2 words per member
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          o[2 * e] = w[2 * (e * D + r)];
          o[2 * e + 1] = w[2 * (e * D + r) + 1];
        }
      } else if constexpr (UB == 4) {
#pragma unroll
        for (int e = 0; e < 4; ++e) o[e] = w[e * D + r];
      } else {  // UB == 2: 8 halfwords per member
#pragma unroll
        for (int q = 0; q < 4; ++q) o[q] = Half2(w, (2 * q) * D + r, (2 * q + 1) * D + r);
      }
      uint4* dst = reinterpret_cast<uint4*>(a.out[r] + off);
#pragma unroll
      for (int q = 0; q < NV; ++q) dst[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
    }
  }
}

template <int D, int UB>
__global__ void __launch_bounds__(256) FineInterleaveKernel(FineDev a) {
  constexpr int W = UB < 16 ? 16 : UB;
  constexpr int NV = W / 16;
  ArriveAndWait(a.sync);
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < a.n_sv; s += gridDim.x * blockDim.x) {
    const uint64_t off = FineOffset(a, s, D) * a.eb;
    uint32_t w[4 * D * NV];  // member-major: member r's W bytes at w[r*4*NV ..]
#pragma unroll
    for (int r = 0; r < D; ++r) {
      const uint4* src = reinterpret_cast<const uint4*>(a.in[r] + off);
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const uint4 v = src[q];
        w[r * 4 * NV + 4 * q] = v.x;
        w[r * 4 * NV + 4 * q + 1] = v.y;
        w[r * 4 * NV + 4 * q + 2] = v.z;
        w[r * 4 * NV + 4 * q + 3] = v.w;
      }
    }
    uint32_t o[4 * D * NV];
    if constexpr (UB >= 16) {  // unit m <- member m
#pragma unroll
      for (int q = 0; q < 4 * D * NV; ++q) o[q] = w[q];
    } else if constexpr (UB == 8) {  // output unit m (2 words) <- member m % D, its unit m / D
#pragma unroll
      for (int m = 0; m < 2 * D; ++m) {
        o[2 * m] = w[(m % D) * 4 + 2 * (m / D)];
        o[2 * m + 1] = w[(m % D) * 4 + 2 * (m / D) + 1];
      }
    } else if constexpr (UB == 4) {
#pragma unroll
      for (int m = 0; m < 4 * D; ++m) o[m] = w[(m % D) * 4 + m / D];
    } else {  // UB == 2: output halfword x <- member x % D, its halfword x / D
#pragma unroll
      for (int q = 0; q < 4 * D; ++q) {
        const int x0 = 2 * q, x1 = 2 * q + 1;
        o[q] = Half2(w, (x0 % D) * 8 + x0 / D, (x1 % D) * 8 + x1 / D);
      }
    }
    uint4* dst = reinterpret_cast<uint4*>(a.out[0]) + static_cast<size_t>(s) * D * NV;
#pragma unroll
    for (int j = 0; j < D * NV; ++j) dst[j] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
  }
}

// Units of 16 / 32 bytes need no permutation inside a vector: one thread per 16-byte chunk, the
// contiguous side walked in order by consecutive lanes (fully coalesced) and every member given
// 512/D contiguous bytes per warp instruction (the super-vector form stores 32-byte units with a
// 32-byte lane stride: half-sector writes, which cost 2x across NVLink).
template <int D, int NV>
__global__ void __launch_bounds__(256) FineChunkKernel(FineDev a, int kind) {
  ArriveAndWait(a.sync);
  const uint32_t total = a.n_sv * NV * D;  // 16-byte chunks on the contiguous side
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    // chunk g = (q*D + r)*NV + j: super-vector q, member r, chunk j of its unit.  Consecutive
    // lanes walk the contiguous side in order and give each member 512/D contiguous bytes per
    // warp instruction.
    if (kind == 0) {  // de-interleave: input chunk g -> member r's chunk q*NV + j
      const uint32_t q = g / (D * NV), rem = g - q * (D * NV), r = rem / NV, j = rem % NV;
      if (a.only >= 0 && a.only != static_cast<int>(r)) continue;
      const uint64_t off = FineOffset(a, q, D) * a.eb + j * 16;
      *reinterpret_cast<uint4*>(a.out[r] + off) = reinterpret_cast<const uint4*>(a.in[0])[g];
    } else {  // interleave: output chunk g <- member (g/NV)%D, its chunk ((g/NV)/D)*NV + g%NV
      const uint32_t m = g / NV, r = m % D, p = (m / D) * NV + g % NV;
      const uint64_t off = FineOffset(a, p / NV, D) * a.eb + (p % NV) * 16;
      reinterpret_cast<uint4*>(a.out[0])[g] = *reinterpret_cast<const uint4*>(a.in[r] + off);
    }
  }
}

template <int D>
bool LaunchFineD(const FineArgs& a, const FineDev& dv, int blocks, int cap, cudaStream_t s) {
  auto chunk_blocks = [&](int nv) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((int64_t{dv.n_sv} * nv * D + 255) / 256, cap)));
  };
#define RH_FINE(UBV)                                                                      \
  case UBV:                                                                               \
    if (a.kind == 0) FineDeinterleaveKernel<D, UBV><<<blocks, 256, 0, s>>>(dv);          \
    else FineInterleaveKernel<D, UBV><<<blocks, 256, 0, s>>>(dv);                        \
    return true;
  switch (a.unit_bytes) {
    RH_FINE(2)
    RH_FINE(4)
    RH_FINE(8)
    case 16:
      FineChunkKernel<D, 1><<<chunk_blocks(1), 256, 0, s>>>(dv, a.kind);
      return true;
    case 32:
      FineChunkKernel<D, 2><<<chunk_blocks(2), 256, 0, s>>>(dv, a.kind);
      return true;
    default:
      return false;
  }
#undef RH_FINE
}

}  // namespace

bool FineSupported(int d, int unit_bytes, int eb, int64_t n_contig) {
  if (d != 2 && d != 4 && d != 8) return false;
  if (unit_bytes != 2 && unit_bytes != 4 && unit_bytes != 8 && unit_bytes != 16 && unit_bytes != 32) return false;
  if (unit_bytes < eb) return false;
  const int64_t sv = static_cast<int64_t>(d) * std::max(16, unit_bytes) / eb;
  return n_contig > 0 && n_contig % sv == 0 && n_contig < (int64_t{1} << 32);
}

int LaunchFine(const FineArgs& a, cudaStream_t s) {
  if (!FineSupported(a.d, a.unit_bytes, a.eb, a.n)) Fail("fine-grained reshard: unsupported pattern");
  FineDev dv{};
  for (int k = 0; k < kMaxGroup; ++k) {
    dv.in[k] = static_cast<const char*>(a.in[k]);
    dv.out[k] = static_cast<char*>(a.out[k]);
  }
  dv.sv = static_cast<uint32_t>(static_cast<int64_t>(a.d) * std::max(16, a.unit_bytes) / a.eb);
  dv.n_sv = static_cast<uint32_t>(a.n / dv.sv);
  dv.run = MakeFastDiv(static_cast<uint32_t>(a.lin ? 1 : a.run));
  dv.c = static_cast<uint32_t>(a.c);
  dv.eb = static_cast<uint32_t>(a.eb);
  dv.lin = a.lin;
  dv.only = a.only;
  dv.sync = a.sync;
  const int cap = a.max_blocks > 0 ? a.max_blocks : SmCount() * 6;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((dv.n_sv + 255) / 256, cap)));
  bool ok = false;
  switch (a.d) {
    case 2: ok = LaunchFineD<2>(a, dv, blocks, cap, s); break;
    case 4: ok = LaunchFineD<4>(a, dv, blocks, cap, s); break;
    default: ok = LaunchFineD<8>(a, dv, blocks, cap, s); break;
  }
  if (!ok) Fail("fine-grained reshard: unsupported unit");
  RH_CUDA(cudaGetLastError());
  return 1;
}

namespace {

// Push all-gather (S -> R into a persistent destination, the output materialization): the
// source rank writes each of its 16-byte local units to its global position in every member's
// replicated destination — posted NVLink writes instead of round-trip reads.  Unit l of the
// local buffer: run q = l / Qs, offset u: global (q*d + c)*Qs + u.
struct PushDev {
  const uint4* src;
  uint4* dst[kMaxGroup];
  FastDiv qs;  // source run (16-byte units)
  uint32_t d, c, n;
  PeerSync sync;
};

__global__ void __launch_bounds__(256) PushGatherKernel(PushDev a) {
  ArriveAndWait(a.sync);
  for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < a.n; l += gridDim.x * blockDim.x) {
    const uint32_t q = Div(a.qs, l);
    const uint64_t f = (static_cast<uint64_t>(q) * a.d + a.c) * a.qs.d + (l - q * a.qs.d);
    const uint4 v = a.src[l];
    for (uint32_t k = 0; k < a.d; ++k) {
      const uint32_t r = (a.c + k) % a.d;  // rotated: the d ranks start on d different peers
      a.dst[r][f] = v;
    }
  }
}

}  // namespace

bool PushGatherSupported(const PullArgs& a) {
  const int eb = ElemBytes(a.dtype);
  if (a.from.kind != RH_SHARD || a.to.kind != RH_REPLICATED) return false;
  if ((a.from.Qs * eb) % 16) return false;
  const int64_t n16 = a.n_dst * eb / 16;
  if (n16 >= (int64_t{1} << 32)) return false;
  for (int k = 0; k < a.from.d; ++k)
    if (reinterpret_cast<uintptr_t>(a.src[k]) % 16) return false;
  return reinterpret_cast<uintptr_t>(a.dst) % 16 == 0;
}

// a.src[k]: member k's DESTINATION (replicated) buffer; a.dst: this rank's SOURCE shard (the
// roles of a pull, reversed); a.n_dst: elements of the replicated destination.
int LaunchPushGather(const PullArgs& a, cudaStream_t s) {
  if (!PushGatherSupported(a)) Fail("push all-gather: unsupported layout");
  const int eb = ElemBytes(a.dtype);
  PushDev dv{};
  dv.src = static_cast<const uint4*>(a.dst);
  for (int k = 0; k < a.from.d; ++k) dv.dst[k] = static_cast<uint4*>(const_cast<void*>(a.src[k]));
  dv.qs = MakeFastDiv(static_cast<uint32_t>(a.from.Qs * eb / 16));
  dv.d = static_cast<uint32_t>(a.from.d);
  dv.c = static_cast<uint32_t>(a.coord);
  dv.n = static_cast<uint32_t>(a.n_dst / a.from.d * eb / 16);
  dv.sync = a.sync;
  const int cap = a.max_blocks > 0 ? a.max_blocks : SmCount() * 6;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((dv.n + 255) / 256, cap)));
  PushGatherKernel<<<blocks, 256, 0, s>>>(dv);
  RH_CUDA(cudaGetLastError());
  return 1;
}

namespace {

// Vector width of a plain pull: the largest power-of-two unit (<= 16 B) that divides every
// contiguous run and every buffer alignment.
int PullVB(const PullArgs& a) {
  const int eb = ElemBytes(a.dtype);
  int64_t g = a.n_dst;
  if (a.to.kind == RH_SHARD) g = Gcd(g, a.to.Qs);
  if (a.from.kind == RH_SHARD) g = Gcd(g, a.from.Qs);
  int vb = 16;
  auto aligned = [&](const void* p) { return (reinterpret_cast<uintptr_t>(p) % vb) == 0; };
  while (vb > eb) {
    bool ok = (g * eb) % vb == 0 && aligned(a.dst);
    const int nsrc = a.from.kind == RH_REPLICATED ? 0 : a.from.d;
    for (int k = 0; k < nsrc; ++k) ok = ok && aligned(a.src[k]);
    if (a.from.kind == RH_REPLICATED) ok = ok && aligned(a.src[a.coord]);
    if (ok) break;
    vb /= 2;
  }
  return vb;
}

PullDev MakePullDev(const PullArgs& a, int vb) {
  const int eb = ElemBytes(a.dtype);
  const int64_t units_per = vb / eb;
  PullDev dv{};
  dv.dst = static_cast<char*>(a.dst);
  for (int k = 0; k < kMaxGroup; ++k) dv.src[k] = static_cast<const char*>(a.src[k]);
  const int64_t total = a.to.kind == RH_SHARD ? a.n_dst * a.to.d : a.n_dst;
  if (total / units_per >= (int64_t{1} << 32)) Fail("reshard: tensor too large for 32-bit unit indices");
  dv.n = static_cast<uint32_t>(a.n_dst / units_per);
  dv.to_shard = a.to.kind == RH_SHARD;
  dv.qst = MakeFastDiv(dv.to_shard ? static_cast<uint32_t>(a.to.Qs / units_per) : 1u);
  dv.from_kind = a.from.kind;
  dv.qsf = MakeFastDiv(a.from.kind == RH_SHARD ? static_cast<uint32_t>(a.from.Qs / units_per) : 1u);
  const int d = a.to.kind == RH_SHARD ? a.to.d : a.from.d;
  dv.dd = MakeFastDiv(static_cast<uint32_t>(std::max(d, 1)));
  dv.coord = static_cast<uint32_t>(a.coord);
  dv.rot = static_cast<uint32_t>((static_cast<uint64_t>(dv.n) / std::max(d, 1)) * a.coord % std::max<uint32_t>(dv.n, 1));
  dv.sync = a.sync;
  dv.d_sum = a.from.d;
  return dv;
}

}  // namespace

int LaunchPull(const PullArgs& a, cudaStream_t s) {
  const int eb = ElemBytes(a.dtype);
  if (a.n_dst == 0) return 0;
  if (a.to.kind == RH_PARTIAL && a.coord != 0) {  // zero-fill (sharding.cpp:132-135)
    if (a.sync.d) Fail("internal: fused barrier on a zero-fill transition");
    RH_CUDA(cudaMemsetAsync(a.dst, 0, a.n_dst * eb, s));
    return 1;
  }
  if (TryLaunchStaged(a, s)) return 1;
  const int vb = PullVB(a);
  PullDev dv = MakePullDev(a, vb);
  switch (vb) {
    case 16: LaunchPullVB<16>(a, dv, s); break;
    case 8: LaunchPullVB<8>(a, dv, s); break;
    case 4: LaunchPullVB<4>(a, dv, s); break;
    default: LaunchPullVB<2>(a, dv, s); break;
  }
  return 1;
}

// Grouped transitions (one launch, one fused barrier).  Eligible when every segment is a plain
// pull (no zero-fill, no staged fine-grained source) of the same source kind and dtype; the
// common vector width is the smallest segment's.
namespace {
struct MultiHost {
  int vb, kind, dtype, blocks, n;
};
std::mutex g_multi_mu;
std::map<const void*, MultiHost> g_multi;
}  // namespace

size_t PullMultiTableBytes(int n) { return static_cast<size_t>(n) * sizeof(PullDev); }

bool PreparePullMulti(const PullArgs* a, int n, int max_blocks, void* table) {
  if (n < 2) return false;
  int vb = 16;
  for (int k = 0; k < n; ++k) {
    if (a[k].n_dst == 0 || a[k].to.kind == RH_PARTIAL || a[k].from.kind != a[0].from.kind ||
        a[k].dtype != a[0].dtype)
      return false;
    if (a[k].from.kind == RH_SHARD && a[k].from.Qs * ElemBytes(a[k].dtype) < 16) return false;  // staged
    vb = std::min(vb, PullVB(a[k]));
  }
  if (a[0].from.kind == RH_PARTIAL && vb < (a[0].dtype == RH_BF16 ? 2 : 4)) return false;
  std::vector<PullDev> seg(n);
  double units = 0;
  for (int k = 0; k < n; ++k) {
    seg[k] = MakePullDev(a[k], vb);
    units += seg[k].n;
  }
  const int cap = max_blocks > 0 ? max_blocks : SmCount() * 6;
  const double per_blk = a[0].from.kind == RH_PARTIAL ? 256.0 : 1024.0;
  const double scale = std::min(1.0, cap / std::max(1.0, units / per_blk));
  uint32_t b0 = 0;
  for (int k = 0; k < n; ++k) {
    const uint32_t want = static_cast<uint32_t>(std::ceil(seg[k].n / per_blk * scale));
    seg[k].blk0 = b0;
    seg[k].nblk = std::max<uint32_t>(1, want);
    b0 += seg[k].nblk;
  }
  RH_CUDA(cudaMemcpy(table, seg.data(), seg.size() * sizeof(PullDev), cudaMemcpyHostToDevice));
  std::lock_guard<std::mutex> lk(g_multi_mu);
  g_multi[table] = MultiHost{vb, a[0].from.kind, a[0].dtype, static_cast<int>(b0), n};
  return true;
}

void ReleasePullMulti(const void* table) {
  std::lock_guard<std::mutex> lk(g_multi_mu);
  g_multi.erase(table);
}

int LaunchPullMulti(const void* table, const PeerSync& sync, cudaStream_t s) {
  MultiHost h;
  {
    std::lock_guard<std::mutex> lk(g_multi_mu);
    auto it = g_multi.find(table);
    if (it == g_multi.end()) Fail("grouped transition: table not prepared", RH_ERR_STATE);
    h = it->second;
  }
  const PullDev* seg = static_cast<const PullDev*>(table);
  const bool bf = h.dtype == RH_BF16;
#define RH_MULTI(VB)                                                                                   \
  if (h.kind == RH_SHARD) LaunchPdl(PullMultiKernel<VB, 0, float>, h.blocks, 256, 0, s, seg, h.n, sync);       \
  else if (h.kind == RH_REPLICATED) LaunchPdl(PullMultiKernel<VB, 1, float>, h.blocks, 256, 0, s, seg, h.n, sync); \
  else if (bf) LaunchPdl(PullMultiKernel<VB, 2, __nv_bfloat16>, h.blocks, 256, 0, s, seg, h.n, sync);         \
  else if (VB >= 4) LaunchPdl(PullMultiKernel<(VB >= 4 ? VB : 4), 2, float>, h.blocks, 256, 0, s, seg, h.n, sync);
  switch (h.vb) {
    case 16: RH_MULTI(16) break;
    case 8: RH_MULTI(8) break;
    case 4: RH_MULTI(4) break;
    default: RH_MULTI(2) break;
  }
#undef RH_MULTI
  RH_CUDA(cudaGetLastError());
  return 1;
}

// ----------------------------------------------------------------------------------------------

namespace {

template <typename T>
__global__ void SliceComposedKernel(T* dst, const T* full, ComposedMap m, int64_t n) {
  for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < n;
       l += int64_t(gridDim.x) * blockDim.x)
    dst[l] = full[ComposedLocalToGlobal(m, l)];
}

__device__ __forceinline__ void Philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

template <typename T>
__global__ void SyntheticKernel(T* dst, ComposedMap m, int64_t n, uint64_t seed, uint32_t op_index,
                                float scale) {
  for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < n;
       l += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t f = static_cast<uint64_t>(ComposedLocalToGlobal(m, l));
    const uint64_t blk = f >> 2;
    uint32_t c[4] = {static_cast<uint32_t>(blk), static_cast<uint32_t>(blk >> 32),
                     static_cast<uint32_t>(seed >> 32), 0u};
    Philox(c, static_cast<uint32_t>(seed), op_index);
    const uint32_t w = c[f & 3];
    const float v = static_cast<float>(static_cast<int32_t>(w >> 8) - 8388608) * (1.0f / 8388608.0f);
    const float x = __fmul_rn(v, scale);
    if constexpr (sizeof(T) == 4) {
      dst[l] = x;
    } else {
      dst[l] = __float2bfloat16_rn(x);
    }
  }
}

__device__ __forceinline__ void StReleaseSys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t LdAcquireSys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void BarrierKernel(BarrierArgs b) {
  __shared__ uint32_t seq;
  if (threadIdx.x == 0) {
    seq = *b.counter + 1;
    *b.counter = seq;
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t < b.d) {
    __threadfence_system();
    StReleaseSys(b.peer_flags[t] + b.me, seq);
    WaitFlag(b.my_flags + b.members[t], seq, b.err, b.timeout_ns, b.me, b.members[t], true);
  }
  __syncthreads();
}

int Blocks(int64_t n) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, SmCount() * 16))); }

}  // namespace

void LaunchSliceComposed(void* dst, const void* full, const ComposedMap& m, int64_t n, int dtype,
                         cudaStream_t s) {
  if (n == 0) return;
  if (dtype == RH_BF16) {
    SliceComposedKernel<<<Blocks(n), 256, 0, s>>>(static_cast<uint16_t*>(dst),
                                                 static_cast<const uint16_t*>(full), m, n);
  } else {
    SliceComposedKernel<<<Blocks(n), 256, 0, s>>>(static_cast<uint32_t*>(dst),
                                                 static_cast<const uint32_t*>(full), m, n);
  }
  RH_CUDA(cudaGetLastError());
}

void LaunchSynthetic(void* dst, const ComposedMap& m, int64_t n, uint64_t seed, uint32_t op_index,
                     float scale, int dtype, cudaStream_t s) {
  if (n == 0) return;
  if (dtype == RH_BF16) {
    SyntheticKernel<<<Blocks(n), 256, 0, s>>>(static_cast<__nv_bfloat16*>(dst), m, n, seed,
                                             op_index, scale);
  } else {
    SyntheticKernel<<<Blocks(n), 256, 0, s>>>(static_cast<float*>(dst), m, n, seed, op_index, scale);
  }
  RH_CUDA(cudaGetLastError());
}

uint64_t SyncTimeoutNs() {
  static const uint64_t ns = [] {
    const char* e = std::getenv("RH_SYNC_TIMEOUT_MS");
    const double ms = e && *e ? std::atof(e) : 60000.0;
    return static_cast<uint64_t>(std::max(0.0, ms) * 1e6);
  }();
  return ns;
}

void LaunchBarrier(const BarrierArgs& b, cudaStream_t s) {
  BarrierKernel<<<1, 32, 0, s>>>(b);
  RH_CUDA(cudaGetLastError());
}

void LaunchGatherSlices(char* const* src, int world, int me, size_t part, const PeerSync& sync, cudaStream_t s) {
  if (world > kMaxGroup || part % 16) Fail("gather slices: unsupported world / piece size");
  GatherArgs a{};
  for (int q = 0; q < world; ++q) a.src[q] = src[q];
  a.world = world;
  a.me = me;
  a.part16 = part / 16;
  a.sync = sync;
  const uint64_t total = a.part16 * static_cast<uint64_t>(world - 1);
  static const int cap = [] {  // grid cap (A/B knob; profiles/r2/e2e_scatter_ab.txt: 148 best)
    const char* e = getenv("RH_E2E_GATHER_BLOCKS");
    return e && *e ? std::max(1, atoi(e)) : SmCount();
  }();
  const int blocks = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, cap)));
  GatherSlicesKernel<<<blocks, 256, 0, s>>>(a);
  RH_CUDA(cudaGetLastError());
}

void LaunchPeerSync(const PeerSync& sync, cudaStream_t s) {
  if (sync.d == 0) return;
  PeerSyncKernel<<<1, 32, 0, s>>>(sync);
  RH_CUDA(cudaGetLastError());
}

void LaunchEpochTick(uint32_t* epoch, cudaStream_t s) {
  EpochTickKernel<<<1, 1, 0, s>>>(epoch);
  RH_CUDA(cudaGetLastError());
}

void LaunchZero(void* dst, size_t bytes, cudaStream_t s) {
  if (bytes) RH_CUDA(cudaMemsetAsync(dst, 0, bytes, s));
}

}  // namespace rh
