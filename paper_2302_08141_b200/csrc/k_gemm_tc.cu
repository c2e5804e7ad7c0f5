// k_gemm_tc.cu — the sharded-GEMM kernel (K1) on Blackwell 5th-gen tensor cores.
//
// bf16 x bf16 -> fp32 accumulate in TMEM -> bf16 (+ fused unary-chain epilogue).
// Persistent, warp-specialised, one CTA per SM:
//   warp 0 (one lane)  TMA producer: A [BM x 64] and B [64 x BN] k-blocks into a 4-stage ring
//                      (cp.async.bulk.tensor, 128-byte swizzle, mbarrier complete_tx);
//   warp 1 (one lane)  MMA issuer: tcgen05.mma.cta_group::1.kind::f16 128 x BN x 16 into one of
//                      two TMEM accumulators, tcgen05.commit frees smem stages / signals the
//                      epilogue;
//   warp 2             TMEM allocator (2 x BN fp32 columns);
//   warps 4-7          epilogue: tcgen05.ld 32x32b.x32 -> registers -> chain -> bf16 -> global,
//                      overlapped with the next tile's MMAs (double-buffered accumulator).
// A is K-major ([M,K] row-major); B is MN-major ([K,N] row-major) or K-major ([N,K], transpose_b).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "kernels.h"
#include "launch.cuh"
#include "unary.cuh"

namespace rh {
namespace {

constexpr int BM = 128, BK = 64;
constexpr int kThreads = 256;

// Residual add of the fused `add` op: the same add.rn.bf16x2 as the chain kernels (ew_core.cuh),
// so the fused result is bit-identical to the separate add kernel's.
__device__ __forceinline__ uint32_t AddBf16x2Epi(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// Output push (GemmPush): the fused barrier's arrival and wait (the same flag protocol as the
// resharding kernels' PeerSync, k_reshard.cu) and the pushed rows.
__device__ __forceinline__ uint32_t PushLdAcquireSys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// kernel-side form of GemmPush: a 32 x 32 box tensor map of every member's replicated copy
// (LaunchGemmTc builds them from the pointers); the epilogue's staged output box is stored
// through each of them right after the local store (bulk NVLink writes to the peers).
struct PushDev {
  int n;
  int row_off;
  int scatter_dim, part;  // scatter_dim >= 0: one owner per box (GemmPush)
  PeerSync sync;
  CUtensorMap map[kMaxGroup];
};
// block 0, threads < d: this rank's destination copy is free (every earlier reader of it is
// done: stream order), signalled into every member's flag row
__device__ __forceinline__ void SyncArrive(const PeerSync& y) {
  if (y.d == 0 || blockIdx.x != 0 || static_cast<int>(threadIdx.x) >= y.d) return;
  const uint32_t e = *reinterpret_cast<const volatile uint32_t*>(y.epoch);
  __threadfence_system();
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(y.peer_slot[threadIdx.x] + y.me), "r"(e) : "memory");
}
__device__ __forceinline__ void PushArrive(const PushDev& p) {
  if (p.n) SyncArrive(p.sync);
}
// one thread: every member arrived (bounded: a missing peer records the error and gives up)
__device__ __forceinline__ void SyncWaitAll(const PeerSync& y) {
  const uint32_t e = *reinterpret_cast<const volatile uint32_t*>(y.epoch);
  for (int t = 0; t < y.d; ++t) {
    const uint32_t* f = y.my_slot + y.members[t];
    if (static_cast<int32_t>(PushLdAcquireSys(f) - e) >= 0) continue;
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (uint32_t n = 1; static_cast<int32_t>(PushLdAcquireSys(f) - e) < 0; ++n) {
      if ((n & 1023) == 0 && y.timeout_ns) {
        uint64_t t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > y.timeout_ns) {
          if (y.err) atomicCAS(y.err, 0u, SyncErrorCode(y.me, y.members[t]));
          break;
        }
      }
    }
  }
}
__device__ __forceinline__ void PushWaitAll(const PushDev& p) { SyncWaitAll(p.sync); }

__device__ __forceinline__ uint32_t SmemU32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void MbarInit(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(SmemU32(bar)), "r"(count));
}
__device__ __forceinline__ void MbarExpectTx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(SmemU32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void MbarArrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(SmemU32(bar)) : "memory");
}
__device__ __forceinline__ void MbarWait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(SmemU32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void TmaLoad2D(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                          int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          SmemU32(dst)),
      "l"(map), "r"(SmemU32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Epilogue output: 32 x 32 bf16 boxes (64-byte rows, 64-byte swizzle) staged in shared memory and
// written by the TMA engine (cp.async.bulk.tensor store): fully coalesced, asynchronous global
// writes instead of one 16-byte store per row per thread (32 rows per store instruction).
__device__ __forceinline__ void TmaStore2D(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(SmemU32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void BulkCommit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void BulkWaitRead() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void BulkWaitAll() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void FenceProxyAsyncSmem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
constexpr int kEpiStageBytes = 4 * 2 * 2048;  // 4 epilogue warps x 2 buffers x (32 x 64 B)

// One 32-row x 32-column bf16 box of the epilogue (lane = row, p = its 16 packed pairs) through
// staging buffer `buf` (of 2, alternating) and a TMA store at (c0, c1).  `cnt` = boxes this warp
// stored before: the buffer's previous store must have been read out before it is rewritten.
struct PushDev;
__device__ __forceinline__ void EpiStoreBox(uint8_t* stage, uint32_t cnt, const uint32_t (&p)[16],
                                            const CUtensorMap* map, int c0, int c1, int lane,
                                            const PushDev* push = nullptr, bool* push_ready = nullptr);

// One 32-row x 32-column bf16 box of the epilogue (lane = row, p = its 16 packed pairs) through
// staging buffer `buf` (of 2, alternating) and a TMA store at (c0, c1) — and, with `push`, the
// same box into every member's replicated copy (rows offset by push->row_off), after the fused
// barrier (first box only).  `cnt` = boxes this warp stored before: the buffer's previous
// stores must have been read out before it is rewritten.
__device__ __forceinline__ void EpiStoreBox(uint8_t* stage, uint32_t cnt, const uint32_t (&p)[16],
                                            const CUtensorMap* map, int c0, int c1, int lane,
                                            const PushDev* push, bool* push_ready) {
  uint8_t* sb = stage + (cnt & 1) * 2048;
  if (lane == 0 && cnt >= 2) BulkWaitRead<1>();
  __syncwarp();
  const int sw = (lane >> 1) & 3;  // 64-byte swizzle: 16-byte chunk ^= address bits [7,9)
#pragma unroll
  for (int q = 0; q < 4; ++q)
    *reinterpret_cast<uint4*>(sb + lane * 64 + ((q ^ sw) << 4)) = make_uint4(p[4 * q], p[4 * q + 1], p[4 * q + 2], p[4 * q + 3]);
  FenceProxyAsyncSmem();
  __syncwarp();
  if (lane == 0) {
    TmaStore2D(map, sb, c0, c1);
    if (push && push->n) {
      if (!*push_ready) {
        PushWaitAll(*push);
        *push_ready = true;
      }
      if (push->scatter_dim == 1) {
        const int k = c0 / push->part;
        TmaStore2D(&push->map[k], sb, c0 - k * push->part, c1);
      } else if (push->scatter_dim == 0) {
        const int k = c1 / push->part;
        TmaStore2D(&push->map[k], sb, c0, c1 - k * push->part);
      } else {
        for (int k = 0; k < push->n; ++k) TmaStore2D(&push->map[k], sb, c0, c1 + push->row_off);
      }
    }
    BulkCommit();
  }
}



__device__ __forceinline__ void FenceBefore() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void FenceAfter() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void MmaF16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void Commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   SmemU32(bar))
               : "memory");
}

// Shared-memory matrix descriptor, 128-byte swizzle (version 1, base offset 0).
__device__ __forceinline__ uint64_t DescSw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

__device__ __forceinline__ void TmemLd32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Split-K finish: sum the fp32 partials in split order, round to bf16, apply the chain.
// Output push of a split-K GEMM: the reduce writes every final 4-element group into each
// member's replicated copy too (dst[k] = the copy + this rank's row offset), behind the barrier.
struct ReducePush {
  int n;
  uint2* dst[kMaxGroup];
  PeerSync sync;
};
__global__ void __launch_bounds__(256) SplitReduceBf16(__nv_bfloat16* __restrict__ C, const float4* __restrict__ ws,
                                                       int64_t n4, int splits, ChainArgs epi,
                                                       const __nv_bfloat16* __restrict__ resid,
                                                       const __grid_constant__ ReducePush rp);

// The packed bf16 ops the lowering lets into a bf16 GEMM epilogue (executor.cpp: relu / neg /
// identity, and tanh runs = one T^k table lookup; LaunchGemmTc rejects anything else).
// Warp-uniform fn loop outside the element loop: small code.  tabs[t] = table of run slot t
// (shared memory in the GEMM kernels, global in the split-K reduce).
template <int P>
__device__ __forceinline__ void EpiPackedBf16(const ChainArgs& epi, uint32_t (&p)[P], const uint16_t* const* tabs) {
  for (int i = 0; i < epi.n_fn; ++i) {
    const int fn = epi.fns[i];
    if (fn >= kFnTanhRun) {
      const uint16_t* tab = tabs[fn - kFnTanhRun];
#pragma unroll
      for (int j = 0; j < P; ++j)
        p[j] = TanhRunLookup(p[j] & 0xffffu, tab) | (TanhRunLookup(p[j] >> 16, tab) << 16);
    } else if (fn == RH_FN_RELU) {
#pragma unroll
      for (int j = 0; j < P; ++j) p[j] = ReluBf16x2(p[j]);
    } else if (fn == RH_FN_NEG) {
#pragma unroll
      for (int j = 0; j < P; ++j) p[j] ^= 0x80008000u;
    }
  }
}

// Epilogue warps (`nthreads` threads, named barrier 1) stage the chain's T^k tables in shared
// memory.
__device__ __forceinline__ void StageEpiTables(const ChainArgs& epi, uint16_t* tab_s, int t,
                                               const uint16_t* (&tp)[kMaxTanhRuns], int nthreads = 128) {
  for (int i = t; i < epi.n_tab * kTanhRunEntries; i += nthreads)
    tab_s[i] = epi.tab[i / kTanhRunEntries][i % kTanhRunEntries];
#pragma unroll
  for (int k = 0; k < kMaxTanhRuns; ++k) tp[k] = tab_s + k * kTanhRunEntries;
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
constexpr int kEpiTabBytes = 8192;  // >= kMaxTanhRuns * kTanhRunEntries * 2

__global__ void __launch_bounds__(256) SplitReduceBf16(__nv_bfloat16* __restrict__ C, const float4* __restrict__ ws,
                                                       int64_t n4, int splits, ChainArgs epi,
                                                       const __nv_bfloat16* __restrict__ resid,
                                                       const __grid_constant__ ReducePush rp) {
  PdlTrigger();
  PdlWait();
  if (rp.n) {  // block 0 arrives (this rank's copy is free); every block waits for all members
    SyncArrive(rp.sync);
    if (threadIdx.x == 0) SyncWaitAll(rp.sync);
    __syncthreads();
  }
  const uint16_t* tabs[kMaxTanhRuns];
#pragma unroll
  for (int k = 0; k < kMaxTanhRuns; ++k) tabs[k] = epi.tab[k];
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x) {
    float4 v = ws[i];
    for (int z = 1; z < splits; ++z) {
      const float4 w = ws[int64_t(z) * n4 + i];
      v.x = __fadd_rn(v.x, w.x);
      v.y = __fadd_rn(v.y, w.y);
      v.z = __fadd_rn(v.z, w.z);
      v.w = __fadd_rn(v.w, w.w);
    }
    uint32_t p[2] = {PackBf16x2(v.x, v.y), PackBf16x2(v.z, v.w)};
    EpiPackedBf16(epi, p, tabs);
    if (resid) {
      const uint2 r = reinterpret_cast<const uint2*>(resid)[i];
      p[0] = AddBf16x2Epi(p[0], r.x);
      p[1] = AddBf16x2Epi(p[1], r.y);
    }
    reinterpret_cast<uint2*>(C)[i] = make_uint2(p[0], p[1]);
    for (int k = 0; k < rp.n; ++k) rp.dst[k][i] = make_uint2(p[0], p[1]);
  }
}

// Grouped launches (GemmTcGroup): independent problems of equal shape, laid side by side along
// a virtual N = n_prob * seg_n.  Tables live in device memory (written once at program load).
struct GroupDev {
  const CUtensorMap* b;       // [n_prob] B maps
  const CUtensorMap* a;       // [n_prob] A maps, or nullptr: every problem reads the kernel's A
  const CUtensorMap* cm;      // [n_prob] output maps (TMA-store epilogue)
  int seg_n;                  // columns per problem
};

template <int BN, bool kBKMajor, bool kAKMajor, int KB = BK>
struct TcCfg {
  static constexpr int kABytes = BM * KB * 2;
  static constexpr int kBBytes = BN * KB * 2;
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered fp32 accumulator
  static constexpr int kStages = (192 * 1024) / kStage;  // 4 (BN 256, KB 64) / 3 (BN 128, KB 128)
  static constexpr int kSmem = kStages * kStage + 1024 /*barriers*/ + kEpiTabBytes + kEpiStageBytes + 1024 /*align*/;
  static constexpr uint32_t kIdesc = (1u << 4)                     // D = F32
                                     | (1u << 7) | (1u << 10)      // A, B = BF16
                                     | ((kAKMajor ? 0u : 1u) << 15)  // A major
                                     | ((kBKMajor ? 0u : 1u) << 16)  // B major
                                     | (static_cast<uint32_t>(BN >> 3) << 17) |
                                     (static_cast<uint32_t>(BM >> 4) << 24);
};

// A and B each either K-major ([M,K] / [N,K] row-major: one rows x 64 box per 64-wide K chunk)
// or MN-major ([K,M] / [K,N]: 64-wide column chunks of KB rows, the transpose_a /
// non-transposed-B layouts) — the MMA reads both straight from the swizzled tiles, no
// transpose pass.  KB = K elements per pipeline stage: 64, or 128 for the 128-wide tiles (twice
// the MMA work per barrier round trip: their 128 x 128 x 64 k-blocks were issue-latency-bound).
template <int BN, bool kBKMajor, bool kAKMajor, int KB, bool kGroup = false>
__global__ void __launch_bounds__(kThreads, 1)
    GemmTcKernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                 const __grid_constant__ CUtensorMap tma_c, int M, int N, int K, ChainArgs epi, int ksplit,
                 float* __restrict__ ws, GroupDev grp, const __nv_bfloat16* __restrict__ resid,
                 const __grid_constant__ PushDev push) {
  PdlTrigger();
  // Work unit = (m tile, n tile, k split).  ksplit > 1 (few tiles: the sharded GEMMs at N >= 4)
  // writes fp32 partial tiles to ws[split][M][N]; SplitReduceBf16 finishes them.
  using Cfg = TcCfg<BN, kBKMajor, kAKMajor, KB>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::kStages * Cfg::kStage);
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* tfull = empty + Cfg::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int num_m = M / BM, num_n = N / BN, mn = num_m * num_n, tiles = mn * ksplit;
  const int kblocks = K / KB / ksplit;  // per split

  if (warp == 0 && lane == 0) {
    if (!kGroup) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
    }
    for (int s = 0; s < Cfg::kStages; ++s) {
      MbarInit(&full[s], 1);
      MbarInit(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      MbarInit(&tfull[a], 1);
      MbarInit(&tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(SmemU32(tmem_slot)),
                 "r"(Cfg::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  FenceBefore();
  __syncthreads();
  FenceAfter();
  const uint32_t tmem = *tmem_slot;
  PdlWait();  // prologue above overlaps the previous kernel's tail (launch.cuh)
  PushArrive(push);

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer ----------------
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int t = tile % mn, ks = tile / mn;
        const int m_blk = t % num_m, n_blk = t / num_m;
        // operand maps of this tile: grouped launches pick each problem's map (the B column
        // chunk's problem; A per problem unless shared) from the device table
        const CUtensorMap* ma = &tma_a;
        const CUtensorMap* mb[BN / 64];
        int cb[BN / 64];
#pragma unroll
        for (int j = 0; j < BN / 64; ++j) {
          const int col = n_blk * BN + (kBKMajor ? 0 : j * 64);
          mb[j] = &tma_b;
          cb[j] = col;
          if constexpr (kGroup) {
            mb[j] = grp.b + col / grp.seg_n;
            cb[j] = col % grp.seg_n;
          }
        }
        if constexpr (kGroup) {
          if (grp.a) ma = grp.a + (n_blk * BN) / grp.seg_n;
        }
        for (int kb = ks * kblocks; kb < (ks + 1) * kblocks; ++kb) {
          MbarWait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::kStage;
          uint8_t* sb = sa + Cfg::kABytes;
          MbarExpectTx(&full[stage], Cfg::kStage);
          if constexpr (kAKMajor) {
#pragma unroll
            for (int q = 0; q < KB / 64; ++q)
              TmaLoad2D(sa + q * (BM * 128), ma, &full[stage], kb * KB + q * 64, m_blk * BM);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              TmaLoad2D(sa + j * (64 * KB * 2), ma, &full[stage], m_blk * BM + j * 64, kb * KB);
          }
          if constexpr (kBKMajor) {
#pragma unroll
            for (int q = 0; q < KB / 64; ++q)
              TmaLoad2D(sb + q * (BN * 128), mb[0], &full[stage], kb * KB + q * 64, cb[0]);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              TmaLoad2D(sb + j * (64 * KB * 2), mb[j], &full[stage], cb[j], kb * KB);
          }
          if (++stage == Cfg::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer ----------------
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        MbarWait(&tempty[acc], acc_phase ^ 1);
        FenceAfter();
        const uint32_t d_tmem = tmem + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          MbarWait(&full[stage], phase);
          FenceAfter();
          const uint32_t sa = SmemU32(smem + stage * Cfg::kStage);
          const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
          for (int k = 0; k < KB / 16; ++k) {
            const uint64_t ad = kAKMajor ? DescSw128(sa + (k / 4) * (BM * 128) + (k % 4) * 32, 16, 1024)
                                         : DescSw128(sa + k * 16 * 128, 64 * KB * 2, 1024);
            const uint64_t bd = kBKMajor ? DescSw128(sb + (k / 4) * (BN * 128) + (k % 4) * 32, 16, 1024)
                                         : DescSw128(sb + k * 16 * 128, 64 * KB * 2, 1024);
            MmaF16(d_tmem, ad, bd, Cfg::kIdesc, (kb | k) != 0);
          }
          Commit(&empty[stage]);
          if (++stage == Cfg::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        Commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue ----------------
    const int ew = warp - 4;  // TMEM lanes [32*ew, 32*ew+32)
    const uint16_t* tp[kMaxTanhRuns];
    StageEpiTables(epi, reinterpret_cast<uint16_t*>(smem + Cfg::kStages * Cfg::kStage + 1024), threadIdx.x - 128, tp);
    uint8_t* stage_c = smem + Cfg::kStages * Cfg::kStage + 1024 + kEpiTabBytes + ew * 4096;
    uint32_t boxes = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    bool push_ready = false;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      const int t = tile % mn, ks = tile / mn;
      const int m_blk = t % num_m, n_blk = t / num_m;
      MbarWait(&tfull[acc], acc_phase);
      FenceAfter();
      const int row = m_blk * BM + ew * 32 + lane;
      float* wrow = ws ? ws + (static_cast<int64_t>(ks) * M + row) * N + n_blk * BN : nullptr;
      // residual (fused add): 64 bytes of the thread's row per 32-column chunk, loaded one chunk
      // ahead so the loads overlap the previous chunk's TMEM load, chain and store
      const uint4* rrow = resid && !wrow ? reinterpret_cast<const uint4*>(resid + static_cast<int64_t>(row) * N + n_blk * BN)
                                         : nullptr;
      uint4 rn[4];
      if (rrow) {
#pragma unroll
        for (int q = 0; q < 4; ++q) rn[q] = rrow[q];
      }
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint4 rv[4];
        if (rrow) {
#pragma unroll
          for (int q = 0; q < 4; ++q) rv[q] = rn[q];
          if (c + 1 < BN / 32) {
#pragma unroll
            for (int q = 0; q < 4; ++q) rn[q] = rrow[(c + 1) * 4 + q];
          }
        }
        uint32_t r[32];
        TmemLd32(tmem + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN + c * 32, r);
        if (wrow) {  // split-K partial (fp32, unrounded)
          float4* dst = reinterpret_cast<float4*>(wrow + c * 32);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            dst[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                 __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
          continue;
        }
        // fp32 -> bf16 pairs (one cvt.rn.bf16x2 each), then the exact packed ops: the epilogue
        // stays a few hundred instructions (a generic per-element chain inlined 32x made the
        // kernel ~10k instructions and its first tile instruction-fetch-bound)
        uint32_t p[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) p[j] = PackBf16x2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
        EpiPackedBf16(epi, p, tp);
        if (rrow) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            p[4 * q] = AddBf16x2Epi(p[4 * q], rv[q].x);
            p[4 * q + 1] = AddBf16x2Epi(p[4 * q + 1], rv[q].y);
            p[4 * q + 2] = AddBf16x2Epi(p[4 * q + 2], rv[q].z);
            p[4 * q + 3] = AddBf16x2Epi(p[4 * q + 3], rv[q].w);
          }
        }
        int col = n_blk * BN + c * 32;
        const CUtensorMap* cmap = &tma_c;
        if constexpr (kGroup) {  // this 32-column chunk's problem and column within it
          cmap = grp.cm + col / grp.seg_n;
          col %= grp.seg_n;
        }
        EpiStoreBox(stage_c, boxes++, p, cmap, col, m_blk * BM + ew * 32, lane, &push, &push_ready);
      }
      FenceBefore();
      __syncwarp();
      if (lane == 0) MbarArrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) BulkWaitAll();  // staged outputs written before the CTA retires
  }
  FenceBefore();
  __syncthreads();
  FenceAfter();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::kTmemCols));
  }
}

// ------------------------- bf16 GEMM on a CTA pair (tcgen05 cta_group::2) -------------------------
// Two CTAs of a cluster (the two SMs of a TPC) compute one 256 x BN tile: each CTA stages its
// own 128 rows of A and HALF of the BN columns of B, and the leader's single thread issues
// tcgen05.mma.cta_group::2 (M = 256), which reads A from each CTA and B from both; each CTA's
// TMEM receives its 128 rows.  Per SM and k-block the shared-memory operand traffic drops from
// (128 + BN) x 64 to (128 + BN/2) x 64 elements for the same 128 x BN x 64 MMA work, which is what
// lets 128-wide pair tiles (the small sharded GEMMs at N >= 4) run near the MMA rate.
//   both CTAs, warp 0: TMA of own A half / B half into own smem; completion is counted on the
//                      LEADER's full barrier (cp.async.bulk.tensor .cta_group::2);
//   leader, warp 1:    MMA issuer; tcgen05.commit .multicast::cluster frees the stage in both
//                      CTAs and signals both epilogues;
//   both, warps 4-7:   epilogue of own TMEM rows; release the accumulator on the leader's
//                      tempty barrier (8 arrivals: 4 warps x 2 CTAs).
__device__ __forceinline__ uint32_t ClusterRank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t MapaShared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void ClusterSync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void MbarWaitCluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(SmemU32(bar)),
      "r"(parity)
      : "memory");
}
// Release at CTA scope (the PTX default): the epilogue's TMEM reads are ordered by
// tcgen05.wait::ld + fence::before_thread_sync.  A .release.cluster arrive compiles to
// MEMBAR.GPU, which waits for the warp's 16 KB of epilogue stores to drain on every tile (the
// K = 128 score GEMMs of the 32-head block spent most of their time there).
__device__ __forceinline__ void MbarArriveRemote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void TmaLoad2D2Sm(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                             int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          SmemU32(dst)),
      "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void MmaF16Pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void CommitPair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          SmemU32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

// Work units of one CTA pair.  Tile stepping: output tiles pair, pair + n_pairs, .. (tile index
// includes the split-K index), all k-blocks of each.  Stream-K: the tiles' mn * kbt k-block
// iterations are cut into n_pairs contiguous ranges, so every pair runs the same number of
// k-blocks whatever the wave quantization; a range starts and ends inside tiles.  A unit
// [k0, k1) of a tile with k0 > 0 (at most one per pair: its first) is a contributor: fp32
// partial accumulator to the pair's workspace slot, then a flag; the unit with k0 == 0 of a
// split tile (the pair's last) finishes it: waits for the later pairs that contribute to the
// tile (their first units, so no wait cycle), adds their partials in pair order, and runs the
// epilogue.  All pairs are co-resident (grid <= cudaOccupancyMaxActiveClusters).
struct PairWork {
  int64_t g, end;  // stream-K: [g, end) of the mn * kbt iterations
  int next, step, tiles, kbt;
  bool sk;
};
__device__ __forceinline__ int64_t SkStart(int pair, int n_pairs, int64_t total) { return total * pair / n_pairs; }
__device__ __forceinline__ PairWork PairWorkOf(int pair, int n_pairs, int tiles, int kbt, bool sk) {
  PairWork w;
  w.sk = sk;
  w.kbt = kbt;
  w.next = pair;
  w.step = n_pairs;
  w.tiles = tiles;
  const int64_t total = static_cast<int64_t>(tiles) * kbt;
  w.g = SkStart(pair, n_pairs, total);
  w.end = SkStart(pair + 1, n_pairs, total);
  return w;
}
__device__ __forceinline__ bool NextPairWork(PairWork& w, int& tile, int& k0, int& k1) {
  if (w.sk) {
    if (w.g >= w.end) return false;
    tile = static_cast<int>(w.g / w.kbt);
    k0 = static_cast<int>(w.g - static_cast<int64_t>(tile) * w.kbt);
    k1 = static_cast<int>(min(static_cast<int64_t>(w.kbt), k0 + (w.end - w.g)));
    w.g += k1 - k0;
    return true;
  }
  if (w.next >= w.tiles) return false;
  tile = w.next;
  w.next += w.step;
  k0 = 0;
  k1 = w.kbt;
  return true;
}
__device__ __forceinline__ uint32_t LdAcquireGpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Bounded wait for a stream-K contributor (a schedule bug must not hang the GPU).
__device__ __forceinline__ void SkWaitFlag(const uint32_t* f) {
  if (LdAcquireGpu(f)) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (uint32_t n = 1;; ++n) {
    if (LdAcquireGpu(f)) return;
    if ((n & 1023) == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 5000000000ull) __trap();
    }
  }
}

// kEpi = epilogue warps: 4, or 8 for short-K GEMMs whose epilogue is the critical path (the
// 32-head block's K = 128 score GEMMs, each output through a T^14 lookup): two warps per TMEM
// lane quarter, alternate 32-column chunks; one pipeline stage less pays for their staging.
template <int BN, bool kBKMajor, bool kAKMajor, int kEpi = 4>
struct Tc2Cfg {
  static constexpr int kABytes = BM * BK * 2;        // own 128 rows
  static constexpr int kBBytes = (BN / 2) * BK * 2;  // own half of the columns
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kStages = ((kEpi == 4 ? 192 : kEpi == 8 ? 160 : 128) * 1024) / kStage;
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kSmem = kStages * kStage + 1024 + kEpiTabBytes + kEpi * 4096 + 1024;
  static constexpr uint32_t kIdesc = (1u << 4)                     // D = F32
                                     | (1u << 7) | (1u << 10)      // A, B = BF16
                                     | ((kAKMajor ? 0u : 1u) << 15) | ((kBKMajor ? 0u : 1u) << 16) |
                                     (static_cast<uint32_t>(BN >> 3) << 17) |
                                     (static_cast<uint32_t>((2 * BM) >> 4) << 24);  // M = 256
};

template <int BN, bool kBKMajor, bool kAKMajor, bool kGroup = false, int kEpi = 4>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128 + 32 * kEpi, 1)
    GemmTcPairKernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                     const __grid_constant__ CUtensorMap tma_c, int M, int N, int K, ChainArgs epi, int ksplit,
                     float* __restrict__ ws, GroupDev grp, uint32_t* __restrict__ sk_flags,
                     const __nv_bfloat16* __restrict__ resid, const __grid_constant__ PushDev push) {
  PdlTrigger();
  using Cfg = Tc2Cfg<BN, kBKMajor, kAKMajor, kEpi>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::kStages * Cfg::kStage);
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* tfull = empty + Cfg::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = ClusterRank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int num_m = M / (2 * BM), num_n = N / BN, mn = num_m * num_n, tiles = mn * ksplit;
  const int kblocks = K / BK / ksplit;
  const bool sk = sk_flags != nullptr;  // stream-K (ksplit == 1; ws = the pairs' partial slots)

  if (warp == 0 && lane == 0) {
    if (!kGroup) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_a) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tma_b) : "memory");
    }
    for (int st = 0; st < Cfg::kStages; ++st) {
      MbarInit(&full[st], 1);
      MbarInit(&empty[st], 1);
    }
    for (int a = 0; a < 2; ++a) {
      MbarInit(&tfull[a], 1);
      MbarInit(&tempty[a], 2 * kEpi);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(SmemU32(tmem_slot)),
                 "r"(Cfg::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  FenceBefore();
  ClusterSync();  // barrier inits and TMEM allocation visible to both CTAs of the pair
  FenceAfter();
  const uint32_t tmem = *tmem_slot;
  PdlWait();
  PushArrive(push);

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs) ----------------
      int stage = 0;
      uint32_t phase = 0;
      PairWork w = PairWorkOf(pair, n_pairs, tiles, kblocks, sk);
      int tile, k0, k1;
      while (NextPairWork(w, tile, k0, k1)) {
        const int t = tile % mn, ks = tile / mn;
        const int m_blk = t % num_m, n_blk = t / num_m;
        const int m0 = m_blk * 2 * BM + static_cast<int>(rank) * BM;
        const int n0 = n_blk * BN + static_cast<int>(rank) * (BN / 2);
        const CUtensorMap* ma = &tma_a;
        const CUtensorMap* mb[BN / 128];
        int cb[BN / 128];
#pragma unroll
        for (int j = 0; j < BN / 128; ++j) {
          const int col = n0 + (kBKMajor ? 0 : j * 64);
          mb[j] = &tma_b;
          cb[j] = col;
          if constexpr (kGroup) {
            mb[j] = grp.b + col / grp.seg_n;
            cb[j] = col % grp.seg_n;
          }
        }
        if constexpr (kGroup) {
          if (grp.a) ma = grp.a + (n_blk * BN) / grp.seg_n;
        }
        for (int kb = ks * kblocks + k0; kb < ks * kblocks + k1; ++kb) {
          MbarWait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::kStage;
          uint8_t* sb = sa + Cfg::kABytes;
          const uint32_t fb = MapaShared(SmemU32(&full[stage]), 0);
          if (leader) MbarExpectTx(&full[stage], 2 * Cfg::kStage);
          if constexpr (kAKMajor) {
            TmaLoad2D2Sm(sa, ma, fb, kb * BK, m0);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) TmaLoad2D2Sm(sa + j * (64 * BK * 2), ma, fb, m0 + j * 64, kb * BK);
          }
          if constexpr (kBKMajor) {
            TmaLoad2D2Sm(sb, mb[0], fb, kb * BK, cb[0]);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 128; ++j) TmaLoad2D2Sm(sb + j * (64 * BK * 2), mb[j], fb, cb[j], kb * BK);
          }
          if (++stage == Cfg::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---------------- MMA issuer (leader) ----------------
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      PairWork w = PairWorkOf(pair, n_pairs, tiles, kblocks, sk);
      int tile, k0, k1;
      while (NextPairWork(w, tile, k0, k1)) {
        MbarWaitCluster(&tempty[acc], acc_phase ^ 1);
        FenceAfter();
        const uint32_t d_tmem = tmem + acc * BN;
        for (int kb = 0; kb < k1 - k0; ++kb) {
          MbarWait(&full[stage], phase);
          FenceAfter();
          const uint32_t sa = SmemU32(smem + stage * Cfg::kStage);
          const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = kAKMajor ? DescSw128(sa + k * 32, 16, 1024)
                                         : DescSw128(sa + k * 16 * 128, 64 * BK * 2, 1024);
            const uint64_t bd = kBKMajor ? DescSw128(sb + k * 32, 16, 1024)
                                         : DescSw128(sb + k * 16 * 128, 64 * BK * 2, 1024);
            MmaF16Pair(d_tmem, ad, bd, Cfg::kIdesc, (kb | k) != 0);
          }
          CommitPair(&empty[stage]);
          if (++stage == Cfg::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        CommitPair(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue (both CTAs) ----------------
    const int ew = warp - 4, quarter = ew % 4, half = ew / 4;  // TMEM lanes of warp w: 32 * (w % 4)
    const uint16_t* tp[kMaxTanhRuns];
    StageEpiTables(epi, reinterpret_cast<uint16_t*>(smem + Cfg::kStages * Cfg::kStage + 1024), threadIdx.x - 128, tp,
                   32 * kEpi);
    const uint32_t tempty_leader[2] = {MapaShared(SmemU32(&tempty[0]), 0), MapaShared(SmemU32(&tempty[1]), 0)};
    uint8_t* stage_c = smem + Cfg::kStages * Cfg::kStage + 1024 + kEpiTabBytes + ew * 4096;
    uint32_t boxes = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    PairWork w = PairWorkOf(pair, n_pairs, tiles, kblocks, sk);
    const int64_t sk_total = static_cast<int64_t>(tiles) * kblocks;
    bool push_ready = false;
    constexpr int kSlot = BM * BN;  // floats per CTA slot: [BN/32 chunks][128 rows][32]
    int tile, k0, k1;
    while (NextPairWork(w, tile, k0, k1)) {
      const int t = tile % mn, ks = tile / mn;
      const int m_blk = t % num_m, n_blk = t / num_m;
      const bool contrib = sk && k0 > 0, finish = sk && k0 == 0 && k1 < kblocks;
      // contributors of a finished tile: the next pairs whose ranges start inside it
      int cp_end = pair + 1;
      if (finish) {
        const int64_t tile_end = static_cast<int64_t>(tile + 1) * kblocks;
        while (cp_end < n_pairs && SkStart(cp_end, n_pairs, sk_total) < tile_end) ++cp_end;
        if (lane == 0)
          for (int cp = pair + 1; cp < cp_end; ++cp) SkWaitFlag(sk_flags + 2 * cp + rank);
        __syncwarp();
      }
      MbarWait(&tfull[acc], acc_phase);
      FenceAfter();
      const int row0 = m_blk * 2 * BM + static_cast<int>(rank) * BM + quarter * 32;
      const int row = row0 + lane;
      float* wrow = ws && !sk ? ws + (static_cast<int64_t>(ks) * M + row) * N + n_blk * BN : nullptr;
      // residual (fused add): 64 bytes of the thread's row per 32-column chunk, loaded one chunk
      // ahead so the loads overlap the previous chunk's TMEM load, chain and store
      const bool radd = resid && !wrow && !contrib;
      const uint4* rrow = radd ? reinterpret_cast<const uint4*>(resid + static_cast<int64_t>(row) * N + n_blk * BN)
                               : nullptr;
      uint4 rn[4];
      if (radd) {
#pragma unroll
        for (int q = 0; q < 4; ++q) rn[q] = rrow[half * 4 + q];
      }
#pragma unroll 1
      for (int c = half; c < BN / 32; c += kEpi / 4) {
        uint4 rv[4];
        if (radd) {
#pragma unroll
          for (int q = 0; q < 4; ++q) rv[q] = rn[q];
          if (c + kEpi / 4 < BN / 32) {
#pragma unroll
            for (int q = 0; q < 4; ++q) rn[q] = rrow[(c + kEpi / 4) * 4 + q];
          }
        }
        uint32_t r[32];
        TmemLd32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN + c * 32, r);
        const int64_t so = (static_cast<int64_t>(c) * BM + quarter * 32 + lane) * 32;
        if (contrib) {
          float4* dst = reinterpret_cast<float4*>(ws + static_cast<int64_t>(2 * pair + rank) * kSlot + so);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            dst[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                 __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
          continue;
        }
        if (finish) {
          for (int cp = pair + 1; cp < cp_end; ++cp) {
            const float4* src = reinterpret_cast<const float4*>(ws + static_cast<int64_t>(2 * cp + rank) * kSlot + so);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 v = src[q];
              r[4 * q] = __float_as_uint(__uint_as_float(r[4 * q]) + v.x);
              r[4 * q + 1] = __float_as_uint(__uint_as_float(r[4 * q + 1]) + v.y);
              r[4 * q + 2] = __float_as_uint(__uint_as_float(r[4 * q + 2]) + v.z);
              r[4 * q + 3] = __float_as_uint(__uint_as_float(r[4 * q + 3]) + v.w);
            }
          }
        }
        if (wrow) {
          float4* dst = reinterpret_cast<float4*>(wrow + c * 32);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            dst[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                 __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
          continue;
        }
        uint32_t p[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) p[j] = PackBf16x2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
        EpiPackedBf16(epi, p, tp);
        if (radd) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            p[4 * q] = AddBf16x2Epi(p[4 * q], rv[q].x);
            p[4 * q + 1] = AddBf16x2Epi(p[4 * q + 1], rv[q].y);
            p[4 * q + 2] = AddBf16x2Epi(p[4 * q + 2], rv[q].z);
            p[4 * q + 3] = AddBf16x2Epi(p[4 * q + 3], rv[q].w);
          }
        }
        int col = n_blk * BN + c * 32;
        const CUtensorMap* cmap = &tma_c;
        if constexpr (kGroup) {
          cmap = grp.cm + col / grp.seg_n;
          col %= grp.seg_n;
        }
        EpiStoreBox(stage_c, boxes++, p, cmap, col, row0, lane, &push, &push_ready);
      }
      FenceBefore();
      __syncwarp();
      if (lane == 0) MbarArriveRemote(tempty_leader[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
      if (contrib || finish) {
        if (contrib) __threadfence();  // this thread's partials, before the flag (below)
        asm volatile("bar.sync 1, %0;" ::"r"(32 * kEpi) : "memory");  // the epilogue warps
        if (threadIdx.x == 128) {
          if (contrib) {
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(sk_flags + 2 * pair + rank), "r"(1u) : "memory");
          } else {  // consumed: re-arm the contributors' flags for the next stream-K GEMM
            for (int cp = pair + 1; cp < cp_end; ++cp) sk_flags[2 * cp + rank] = 0;
          }
        }
      }
    }
    if (lane == 0) BulkWaitAll();
  }
  FenceBefore();
  __syncthreads();
  ClusterSync();  // the peer's last remote arrivals / MMAs done before TMEM is released
  FenceAfter();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::kTmemCols));
  }
}

// ------------------------------- fp32 GEMM: 3xTF32 on tcgen05 -------------------------------
// fp32 programs need fp32-level accuracy (parity 1e-5), which one TF32 pass (10-bit mantissa)
// cannot give.  Each operand is split exactly into hi = x with the low 13 mantissa bits cleared
// (exactly representable in TF32, so hardware truncation or rounding leaves it unchanged) and
// lo = x - hi (exact in fp32); D += A_hi B_hi + A_hi B_lo + A_lo B_hi with kind::tf32 MMAs,
// fp32 accumulation in TMEM (the dropped A_lo B_lo term is < 2^-22 relative).

__global__ void __launch_bounds__(256) SplitTf32Kernel(const float4* __restrict__ x, float4* __restrict__ hi,
                                                       float4* __restrict__ lo, int64_t n4) {
  PdlTrigger();
  PdlWait();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 v = x[i];
    float4 h, l;
    h.x = __uint_as_float(__float_as_uint(v.x) & 0xffffe000u);
    h.y = __uint_as_float(__float_as_uint(v.y) & 0xffffe000u);
    h.z = __uint_as_float(__float_as_uint(v.z) & 0xffffe000u);
    h.w = __uint_as_float(__float_as_uint(v.w) & 0xffffe000u);
    l.x = __fsub_rn(v.x, h.x);
    l.y = __fsub_rn(v.y, h.y);
    l.z = __fsub_rn(v.z, h.z);
    l.w = __fsub_rn(v.w, h.w);
    hi[i] = h;
    lo[i] = l;
  }
}

// B stored [K,N] (MN-major): split AND transpose to [N,K] in the same pass (32x33 smem tile),
// so the MMA always reads K-major TF32 operands.
__global__ void __launch_bounds__(256) SplitTransposeTf32Kernel(const float* __restrict__ b, float* __restrict__ hi_t,
                                                                float* __restrict__ lo_t, int64_t K, int64_t N) {
  PdlTrigger();
  PdlWait();
  __shared__ float tile[32][33];
  const int64_t k0 = int64_t(blockIdx.y) * 32, n0 = int64_t(blockIdx.x) * 32;
  for (int j = threadIdx.y; j < 32; j += 8) tile[j][threadIdx.x] = b[(k0 + j) * N + n0 + threadIdx.x];
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const float v = tile[threadIdx.x][j];
    const float h = __uint_as_float(__float_as_uint(v) & 0xffffe000u);
    hi_t[(n0 + j) * K + k0 + threadIdx.x] = h;
    lo_t[(n0 + j) * K + k0 + threadIdx.x] = __fsub_rn(v, h);
  }
}

constexpr int BK32 = 32;   // fp32 elements per k-block (128 bytes: one swizzle row)
constexpr int STAGES32 = 3;
constexpr int kChunkKb = 8;  // k-blocks (8 x 32 = K 256) per TMEM accumulation chunk

template <int BN, bool kBKMajor>
struct Tf32Cfg {
  static constexpr int kA = BM * BK32 * 4;           // 16 KB
  static constexpr int kB = BN * BK32 * 4;           // 16 KB at BN=128
  static constexpr int kStage = 2 * kA + 2 * kB;     // hi + lo of A and B
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kSmem = STAGES32 * kStage + 1024 + 1024;
  static constexpr uint32_t kIdesc = (1u << 4)                     // D = F32
                                     | (2u << 7) | (2u << 10)      // A, B = TF32
                                     | (0u << 15) | ((kBKMajor ? 0u : 1u) << 16) |
                                     (static_cast<uint32_t>(BN >> 3) << 17) |
                                     (static_cast<uint32_t>(BM >> 4) << 24);
};

__device__ __forceinline__ void MmaTf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// maps: 0 A_hi, 1 A_lo, 2 B_hi, 3 B_lo
template <int BN, bool kBKMajor>
__global__ void __launch_bounds__(kThreads, 1)
    GemmTf32x3Kernel(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
                     const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo,
                     float* __restrict__ C, int M, int N, int K, ChainArgs epi) {
  PdlTrigger();
  using Cfg = Tf32Cfg<BN, kBKMajor>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES32 * Cfg::kStage);
  uint64_t* empty = full + STAGES32;
  uint64_t* tfull = empty + STAGES32;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int num_m = M / BM, num_n = N / BN, tiles = num_m * num_n, kblocks = K / BK32;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES32; ++s) {
      MbarInit(&full[s], 1);
      MbarInit(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      MbarInit(&tfull[a], 1);
      MbarInit(&tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(SmemU32(tmem_slot)),
                 "r"(Cfg::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  FenceBefore();
  __syncthreads();
  FenceAfter();
  const uint32_t tmem = *tmem_slot;
  PdlWait();  // prologue above overlaps the previous kernel's tail (launch.cuh)

  if (warp == 0) {
    if (lane == 0) {  // TMA producer: A_hi, A_lo, B_hi, B_lo per stage
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int m_blk = tile % num_m, n_blk = tile / num_m;
        for (int kb = 0; kb < kblocks; ++kb) {
          MbarWait(&empty[stage], phase ^ 1);
          uint8_t* s_ahi = smem + stage * Cfg::kStage;
          uint8_t* s_alo = s_ahi + Cfg::kA;
          uint8_t* s_bhi = s_alo + Cfg::kA;
          uint8_t* s_blo = s_bhi + Cfg::kB;
          MbarExpectTx(&full[stage], Cfg::kStage);
          TmaLoad2D(s_ahi, &ta_hi, &full[stage], kb * BK32, m_blk * BM);
          TmaLoad2D(s_alo, &ta_lo, &full[stage], kb * BK32, m_blk * BM);
          if constexpr (kBKMajor) {
            TmaLoad2D(s_bhi, &tb_hi, &full[stage], kb * BK32, n_blk * BN);
            TmaLoad2D(s_blo, &tb_lo, &full[stage], kb * BK32, n_blk * BN);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 32; ++j) {
              TmaLoad2D(s_bhi + j * (32 * BK32 * 4), &tb_hi, &full[stage], n_blk * BN + j * 32, kb * BK32);
              TmaLoad2D(s_blo + j * (32 * BK32 * 4), &tb_lo, &full[stage], n_blk * BN + j * 32, kb * BK32);
            }
          }
          if (++stage == STAGES32) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer: 3 TF32 products per k-substep
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      // The TMEM accumulator adds each MMA's partial sums with truncation (measured: error
      // growing linearly in K, 3.7e-5 at K=4096).  So TMEM accumulates only a K-chunk of
      // kChunkKb k-blocks; the epilogue warps add the chunks in fp32 registers with
      // round-to-nearest (error ~(chunk/8) * 2^-24 + RN noise: ~1e-6).
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        for (int kb0 = 0; kb0 < kblocks; kb0 += kChunkKb) {
          MbarWait(&tempty[acc], acc_phase ^ 1);
          FenceAfter();
          const uint32_t d_tmem = tmem + acc * BN;
          const int kb1 = min(kb0 + kChunkKb, kblocks);
          for (int kb = kb0; kb < kb1; ++kb) {
            MbarWait(&full[stage], phase);
            FenceAfter();
            const uint32_t ahi = SmemU32(smem + stage * Cfg::kStage);
            const uint32_t alo = ahi + Cfg::kA;
            const uint32_t bhi = alo + Cfg::kA;
            const uint32_t blo = bhi + Cfg::kB;
#pragma unroll
            for (int k = 0; k < BK32 / 8; ++k) {  // UMMA_K = 8 for tf32 (32 bytes)
              const uint64_t dahi = DescSw128(ahi + k * 32, 16, 1024);
              const uint64_t dalo = DescSw128(alo + k * 32, 16, 1024);
              const uint64_t dbhi = DescSw128(bhi + k * 32, 16, 1024);
              const uint64_t dblo = DescSw128(blo + k * 32, 16, 1024);
              MmaTf32(d_tmem, dalo, dbhi, Cfg::kIdesc, (kb != kb0) || k != 0);  // small terms first
              MmaTf32(d_tmem, dahi, dblo, Cfg::kIdesc, 1);
              MmaTf32(d_tmem, dahi, dbhi, Cfg::kIdesc, 1);
            }
            Commit(&empty[stage]);
            if (++stage == STAGES32) {
              stage = 0;
              phase ^= 1;
            }
          }
          Commit(&tfull[acc]);
          if (++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4) {  // epilogue: RN accumulation of the chunks, fp32 out (+ chain)
    const int ew = warp - 4;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      const int m_blk = tile % num_m, n_blk = tile / num_m;
      float sum[BN];
#pragma unroll
      for (int j = 0; j < BN; ++j) sum[j] = 0.0f;
      for (int kb0 = 0; kb0 < kblocks; kb0 += kChunkKb) {
        MbarWait(&tfull[acc], acc_phase);
        FenceAfter();
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          TmemLd32(tmem + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN + c * 32, r);
#pragma unroll
          for (int j = 0; j < 32; ++j) sum[c * 32 + j] = __fadd_rn(sum[c * 32 + j], __uint_as_float(r[j]));
        }
        FenceBefore();
        __syncwarp();
        if (lane == 0) MbarArrive(&tempty[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      const int row = m_blk * BM + ew * 32 + lane;
      float* crow = C + static_cast<int64_t>(row) * N + n_blk * BN;
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        float* v = sum + c * 32;
        if (epi.n_fn) {
          float t[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) t[j] = v[j];
          ApplyChainVecF32<32>(epi.fns, epi.n_fn, t);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = t[j];
        }
        float4* dst = reinterpret_cast<float4*>(crow + c * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
    }
  }
  FenceBefore();
  __syncthreads();
  FenceAfter();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::kTmemCols));
  }
}

// ------------------------------------------- host ------------------------------------------

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn GetEncode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  if (!fn) Fail("cuTensorMapEncodeTiled unavailable", RH_ERR_CUDA);
  return fn;
}

// 2-D tensor map (bf16 or fp32): inner dim `d0` (contiguous), outer `d1` with row pitch `pitch`
// elements, 128-byte swizzle.
CUtensorMap MakeMap(const void* base, uint64_t d0, uint64_t d1, uint64_t pitch, uint32_t box0,
                    uint32_t box1, bool f32 = false,
                    CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  cuuint64_t dims[2] = {d0, d1};
  cuuint64_t strides[1] = {pitch * (f32 ? 4 : 2)};
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = GetEncode()(&m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                           2, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) Fail("cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")", RH_ERR_CUDA);
  return m;
}

struct Maps {
  CUtensorMap a, b, c;  // c: output, 32 x 32 boxes, 64-byte swizzle (TMA-store epilogue)
};

// Tensor maps depend only on (pointer, shape); arena pointers are static, so cache them.
// bn = B rows per CTA tile (K-major box), kb = K rows per stage (MN-major box).
const Maps& GetMaps(const GemmArgs& g, int bn, int kb = BK) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, const void*, const void*, int64_t, int64_t, int64_t, bool, bool, int, int>, Maps> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(g.a, g.b, g.c, g.m, g.n, g.k, g.ta, g.tb, bn, kb);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  Maps m;
  if (g.ta) {
    m.a = MakeMap(g.a, g.m, g.k, g.m, 64, kb);  // A stored [K,M]: MN-major, 64-wide chunks
  } else {
    m.a = MakeMap(g.a, g.k, g.m, g.k, BK, BM);  // A stored [M,K]: K-major, one 64-wide K chunk
  }
  if (g.tb) {
    m.b = MakeMap(g.b, g.k, g.n, g.k, BK, bn);  // B stored [N,K]: K-major
  } else {
    m.b = MakeMap(g.b, g.n, g.k, g.n, 64, kb);  // B stored [K,N]: MN-major, 64-wide chunks
  }
  m.c = MakeMap(g.c, g.n, g.m, g.n, 32, 32, false, CU_TENSOR_MAP_SWIZZLE_64B);
  return cache.emplace(key, m).first->second;
}

int NumSms() { return SmCount(); }

// Experiment knobs (profiles/gemm_shapes.py A/B runs): RH_GEMM_BN forces the tile width,
// RH_GEMM_MAX_SPLIT caps split-K.  Unset in production.
int EnvInt(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// Tile width: BN = 256 halves the A-operand shared-memory traffic per flop, so it is used
// whenever it yields >= 96 tiles; else BN = 128 (twice the tiles); split-K only when even
// 128-wide tiles cannot fill the SMs.  Measured (profiles/gemm_shapes.py, B200): 2048x1024
// output, K = 4096: BN=256 + split-K 2 28.3 us, BN=128 21.0 us; 2048x2048 output, K = 1024:
// 24.3 vs 12.3 us; the fp32 partials' round trip costs more than the idle SMs it fills.
int PickBN(const GemmArgs& g) {
  if (g.dtype == RH_F32) return g.n % 128 == 0 ? 128 : 0;
  static const int force = EnvInt("RH_GEMM_BN", 0);
  if (force && g.n % force == 0) return force;
  const int64_t mt = g.m / BM;
  if (g.n % 256 == 0 && mt * (g.n / 256) >= 96) return 256;
  if (g.n % 128 == 0) return 128;
  return 0;
}

// bf16 split-K factor: when the output tiles cannot fill the SMs (< 96 tiles), split K so that
// work units reach ~1-2 waves while every split keeps >= 8 k-blocks (K >= 512).
int KSplit(const GemmArgs& g, int bn) {
  if (g.dtype != RH_BF16) return 1;
  static const int max_split = EnvInt("RH_GEMM_MAX_SPLIT", 8);
  const int64_t tiles = (g.m / BM) * (g.n / bn), kb = g.k / BK;
  if (tiles >= 96) return 1;
  int best = 1;
  for (int ks = 2; ks <= max_split; ks *= 2) {
    if (kb % ks || kb / ks < 8 || tiles * (ks / 2) > SmCount()) break;
    best = ks;
  }
  return best;
}

// CTA-pair kernel: bf16 with M a multiple of 256 (RH_GEMM_PAIR=0 disables it, for A/B).
bool UsePair(const GemmArgs& g) {
  static const int on = EnvInt("RH_GEMM_PAIR", 1);
  return on && g.dtype == RH_BF16 && g.m % (2 * BM) == 0;
}

int KSplitPair(const GemmArgs& g, int bn) {
  static const int max_split = EnvInt("RH_GEMM_MAX_SPLIT", 8);
  const int64_t ctas = 2 * (g.m / (2 * BM)) * (g.n / bn), kb = g.k / BK;
  if (ctas >= 96) return 1;
  int best = 1;
  for (int ks = 2; ks <= max_split; ks *= 2) {
    if (kb % ks || kb / ks < 8 || ctas * (ks / 2) > SmCount()) break;
    best = ks;
  }
  return best;
}

// Kernel-side push arguments: a 32 x 32 box (64-byte swizzle) tensor map of every member's
// replicated copy; nothing when g.push.n == 0 or when the schedule cannot push (split-K).
PushDev MakePushDev(const GemmArgs& g, bool allowed) {
  PushDev d{};
  if (!g.push.n || !allowed) return d;  // (split-K: the reduce pushes, MakeReducePush)
  static std::mutex mu;
  static std::map<std::tuple<const void*, int64_t, int64_t>, CUtensorMap> cache;
  std::lock_guard<std::mutex> lk(mu);
  d.n = g.push.n;
  d.row_off = static_cast<int>(g.push.row_off);
  d.scatter_dim = g.push.scatter_dim;
  d.part = static_cast<int>(g.push.part);
  d.sync = g.push.sync;
  // destination [rows, cols]: the replicated copy, or the owner's slot of its staging
  const int64_t cols = g.push.scatter_dim == 1 ? g.push.part : g.n;
  const int64_t rows = g.push.scatter_dim == 0 ? g.push.part : g.push.scatter_dim == 1 ? g.m : g.push.rows_full;
  for (int k = 0; k < g.push.n; ++k) {
    const auto key = std::make_tuple(static_cast<const void*>(g.push.dst[k]), rows, cols);
    auto it = cache.find(key);
    if (it == cache.end())
      it = cache.emplace(key, MakeMap(g.push.dst[k], cols, rows, cols, 32, 32, false, CU_TENSOR_MAP_SWIZZLE_64B)).first;
    d.map[k] = it->second;
  }
  return d;
}

ReducePush MakeReducePush(const GemmArgs& g) {
  ReducePush r{};
  if (!g.push.n) return r;
  if (g.push.scatter_dim >= 0) Fail("internal: scatter push from a split-K reduce");
  r.n = g.push.n;
  r.sync = g.push.sync;
  for (int k = 0; k < g.push.n; ++k)
    r.dst[k] = reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(g.push.dst[k]) + g.push.row_off * g.n);
  return r;
}

// Stream-K for the CTA-pair kernel (opt-in: RH_GEMM_STREAMK=1): when whole pair tiles leave
// >= 8% of the pairs idle in the last wave (e.g. 128 tiles on 74 pairs: 1.73 waves run as 2),
// and every pair still gets >= 16 k-blocks.  Needs the caller's flags and scratch
// (StreamKScratchBytes).  Measured slower than the tile-stepping schedule on every C3/C5 shape
// (profiles/r2/streamk_ab.txt): without the fixup the k-balanced main loop is 10-16% faster
// (2048^3: 14.4 -> 13.2 us class), but the finisher's partial reads run in the 4-warp
// epilogue's serial chunk loop (128 KB per CTA and contributor, L2-latency-bound: +8 us) and the
// contributors' writes +5 us; long-K shapes also lose the L2 reuse of the lock-step k order
// (2048x16384x4096: 183 -> 272 us).
int StreamKPairs() { return NumSms() / 2; }
bool UseStreamK(const GemmArgs& g) {
  static const int on = EnvInt("RH_GEMM_STREAMK", 0);
  if (!on || !g.sk_flags || !UsePair(g) || g.n % 256) return false;
  const int64_t tiles = (g.m / (2 * BM)) * (g.n / 256), kb = g.k / BK, pairs = StreamKPairs();
  const int64_t waves = (tiles + pairs - 1) / pairs;
  if (tiles * 100 >= waves * pairs * 92) return false;
  return tiles * kb >= pairs * 16;
}
size_t StreamKScratchBytes() { return static_cast<size_t>(2 * StreamKPairs()) * BM * 256 * 4; }

// Pairs of the CTA-pair kernel that can be resident at once (stream-K requires co-residency:
// a finishing pair waits for later pairs' partials).  Cached per device.
template <int BN, bool kBK, bool kAK, bool kG, int kEpi>
int MaxPairs() {
  static int cache[64] = {};
  int dev = 0;
  RH_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && cache[dev]) return cache[dev];
  using Cfg = Tc2Cfg<BN, kBK, kAK, kEpi>;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * StreamKPairs());
  cfg.blockDim = dim3(128 + 32 * kEpi);
  cfg.dynamicSmemBytes = Cfg::kSmem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  RH_CUDA(cudaOccupancyMaxActiveClusters(&n, GemmTcPairKernel<BN, kBK, kAK, kG, kEpi>, &cfg));
  n = std::max(1, std::min(n, StreamKPairs()));
  if (dev < 64) cache[dev] = n;
  return n;
}

// A grouped launch (GemmTcGroup): problem 0's maps as the kernel-param maps (the shared A),
// the device table, and the problem count.
struct GroupLaunch {
  Maps m0;
  GroupDev dev;
  int n_prob;
};

template <int BN, bool kBK, bool kAK, int KB, bool kG = false>
void LaunchKB(const GemmArgs& g, cudaStream_t s, const GroupLaunch* gl = nullptr) {
  using Cfg = TcCfg<BN, kBK, kAK, KB>;
  int dev = 0;
  RH_CUDA(cudaGetDevice(&dev));
  static bool attr[64] = {};  // per device (local multi-GPU runtimes)
  if (dev < 64 && !attr[dev]) {
    RH_CUDA(cudaFuncSetAttribute(GemmTcKernel<BN, kBK, kAK, KB, kG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cfg::kSmem));
    attr[dev] = true;
  }
  const Maps& mp = kG ? gl->m0 : GetMaps(g, BN, KB);
  const int64_t n = kG ? g.n * gl->n_prob : g.n;
  const int ks = g.scratch && !kG ? KSplit(g, BN) : 1;
  const int tiles = static_cast<int>((g.m / BM) * (n / BN)) * ks;
  const int grid = std::min(tiles, NumSms());
  float* ws = ks > 1 ? static_cast<float*>(g.scratch) : nullptr;
  LaunchPdl(GemmTcKernel<BN, kBK, kAK, KB, kG>, grid, kThreads, Cfg::kSmem, s,
      mp.a, mp.b, mp.c, static_cast<int>(g.m), static_cast<int>(n),
      static_cast<int>(g.k), g.epi, ks, ws, kG ? gl->dev : GroupDev{},
      kG ? nullptr : static_cast<const __nv_bfloat16*>(g.resid), MakePushDev(g, ks == 1 && !kG));
  RH_CUDA(cudaGetLastError());
  if (ws) {
    const int64_t n4 = g.m * g.n / 4;
    const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n4 + 255) / 256, SmCount() * 8)));
    LaunchPdl(SplitReduceBf16, blocks, 256, 0, s, static_cast<__nv_bfloat16*>(g.c), reinterpret_cast<const float4*>(ws),
              n4, ks, g.epi, static_cast<const __nv_bfloat16*>(g.resid), MakeReducePush(g));
    RH_CUDA(cudaGetLastError());
  }
}

// KB = 128 K elements per stage for 128-wide tiles when every split holds whole 128-chunks.
template <int BN, bool kBK, bool kAK, bool kG = false>
void Launch(const GemmArgs& g, cudaStream_t s, const GroupLaunch* gl = nullptr) {
  const int ks = g.scratch && !kG ? KSplit(g, BN) : 1;
  if (BN == 128 && g.k % (128 * ks) == 0) LaunchKB<BN, kBK, kAK, 128, kG>(g, s, gl);
  else LaunchKB<BN, kBK, kAK, 64, kG>(g, s, gl);
}

// Pair-tile (256 x BN) launch: clusters of 2 CTAs, one pair per TPC, persistent over the tiles.
template <int BN, bool kBK, bool kAK, bool kG = false, int kEpi = 4>
void LaunchPair(const GemmArgs& g, cudaStream_t s, const GroupLaunch* gl = nullptr) {
  using Cfg = Tc2Cfg<BN, kBK, kAK, kEpi>;
  int dev = 0;
  RH_CUDA(cudaGetDevice(&dev));
  static bool attr[64] = {};
  if (dev < 64 && !attr[dev]) {
    RH_CUDA(cudaFuncSetAttribute(GemmTcPairKernel<BN, kBK, kAK, kG, kEpi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cfg::kSmem));
    attr[dev] = true;
  }
  const Maps& mp = kG ? gl->m0 : GetMaps(g, BN / 2);  // B box: half of the pair's columns per CTA
  const int64_t n = kG ? g.n * gl->n_prob : g.n;
  const bool sk = !kG && UseStreamK(g);
  if (sk && !g.scratch) Fail("internal: stream-K GEMM without scratch (GemmTcScratchBytes)");
  const int ks = g.scratch && !kG && !sk ? KSplitPair(g, BN) : 1;
  const int tiles = static_cast<int>((g.m / (2 * BM)) * (n / BN)) * ks;
  int pairs = std::min(tiles, NumSms() / 2);
  if (sk) {
    static const int force = EnvInt("RH_GEMM_SK_PAIRS", 0);
    pairs = std::min<int64_t>(int64_t{tiles} * (g.k / BK), force ? force : MaxPairs<BN, kBK, kAK, kG, kEpi>());
    static const int dbg = EnvInt("RH_GEMM_SK_DEBUG", 0);
    if (dbg) fprintf(stderr, "[stream-k] m %lld n %lld k %lld tiles %d pairs %d (max %d)\n", (long long)g.m,
                     (long long)g.n, (long long)g.k, tiles, pairs, MaxPairs<BN, kBK, kAK, kG, kEpi>());
  }
  float* ws = ks > 1 || sk ? static_cast<float*>(g.scratch) : nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(128 + 32 * kEpi);
  cfg.dynamicSmemBytes = Cfg::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = PdlEnabled() ? 2 : 1;
  RH_CUDA(cudaLaunchKernelEx(&cfg, GemmTcPairKernel<BN, kBK, kAK, kG, kEpi>, mp.a, mp.b, mp.c,
                             static_cast<int>(g.m), static_cast<int>(n), static_cast<int>(g.k), g.epi, ks, ws,
                             kG ? gl->dev : GroupDev{}, sk ? g.sk_flags : nullptr,
                             kG ? nullptr : static_cast<const __nv_bfloat16*>(g.resid),
                             MakePushDev(g, ks == 1 && !sk && !kG)));
  if (ws && !sk) {
    const int64_t n4 = g.m * g.n / 4;
    const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n4 + 255) / 256, SmCount() * 8)));
    LaunchPdl(SplitReduceBf16, blocks, 256, 0, s, static_cast<__nv_bfloat16*>(g.c), reinterpret_cast<const float4*>(ws),
              n4, ks, g.epi, static_cast<const __nv_bfloat16*>(g.resid), MakeReducePush(g));
    RH_CUDA(cudaGetLastError());
  }
}

struct Maps4 {
  CUtensorMap a_hi, a_lo, b_hi, b_lo;
};

template <bool kBK>
void LaunchTf32x3(const GemmArgs& g, cudaStream_t s) {
  constexpr int BN = 128;
  using Cfg = Tf32Cfg<BN, true>;
  int dev = 0;
  RH_CUDA(cudaGetDevice(&dev));
  static bool attr[64] = {};
  if (dev < 64 && !attr[dev]) {
    RH_CUDA(cudaFuncSetAttribute(GemmTf32x3Kernel<BN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cfg::kSmem));
    attr[dev] = true;
  }
  const int64_t na = g.m * g.k, nb = g.k * g.n;
  float* a_hi = static_cast<float*>(g.scratch);
  float* a_lo = a_hi + na;
  float* b_hi = a_lo + na;
  float* b_lo = b_hi + nb;
  const int threads = 256;
  auto blocks = [](int64_t n4) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n4 + 255) / 256, SmCount() * 8))); };
  if (!g.ta) {
    LaunchPdl(SplitTf32Kernel, blocks(na / 4), threads, 0, s, static_cast<const float4*>(g.a), reinterpret_cast<float4*>(a_hi),
                                                       reinterpret_cast<float4*>(a_lo), na / 4);
  } else {  // [K,M] -> hi/lo of [M,K]
    LaunchPdl(SplitTransposeTf32Kernel, dim3(static_cast<unsigned>(g.m / 32), static_cast<unsigned>(g.k / 32)),
                               dim3(32, 8), 0, s, static_cast<const float*>(g.a), a_hi, a_lo, g.k, g.m);
  }
  if (kBK) {
    LaunchPdl(SplitTf32Kernel, blocks(nb / 4), threads, 0, s, static_cast<const float4*>(g.b),
                                                       reinterpret_cast<float4*>(b_hi),
                                                       reinterpret_cast<float4*>(b_lo), nb / 4);
  } else {  // [K,N] -> hi/lo of [N,K]
    LaunchPdl(SplitTransposeTf32Kernel, dim3(static_cast<unsigned>(g.n / 32), static_cast<unsigned>(g.k / 32)),
                               dim3(32, 8), 0, s, static_cast<const float*>(g.b), b_hi, b_lo, g.k, g.n);
  }
  RH_CUDA(cudaGetLastError());
  static std::mutex mu;
  static std::map<std::tuple<const void*, int64_t, int64_t, int64_t, bool>, Maps4> cache;
  Maps4 mp;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(g.scratch, g.m, g.n, g.k, g.tb);
    auto it = cache.find(key);
    if (it == cache.end()) {
      Maps4 m4;
      m4.a_hi = MakeMap(a_hi, g.k, g.m, g.k, BK32, BM, true);
      m4.a_lo = MakeMap(a_lo, g.k, g.m, g.k, BK32, BM, true);
      // the split buffers of B are always [N,K] (K-major)
      m4.b_hi = MakeMap(b_hi, g.k, g.n, g.k, BK32, BN, true);
      m4.b_lo = MakeMap(b_lo, g.k, g.n, g.k, BK32, BN, true);
      it = cache.emplace(key, m4).first;
    }
    mp = it->second;
  }
  const int tiles = static_cast<int>((g.m / BM) * (g.n / BN));
  const int grid = std::min(tiles, NumSms());
  LaunchPdl(GemmTf32x3Kernel<BN, true>, grid, kThreads, Cfg::kSmem, s, 
      mp.a_hi, mp.a_lo, mp.b_hi, mp.b_lo, static_cast<float*>(g.c), static_cast<int>(g.m),
      static_cast<int>(g.n), static_cast<int>(g.k), g.epi);
  RH_CUDA(cudaGetLastError());
}


// ------------------------- fused score -> chain -> context (attention heads) -------------------------
// One kernel for a head's S = Q K^T (K = 128), the elementwise chain on S (bf16 rounding, then
// the score GEMM's epilogue chain: T^14 for the fixture's unlabeled tanh chain), and
// O = chain(S) V — the score and context groups of the 32-head block without the 2048 x 2048
// score tensor ever leaving the SM.  One CTA per (head, 128-row block of Q):
//   warp 0: TMA producer (Q once; K_j and V_j per 128-key block, 2 stages),
//   warp 1: MMA issuer (S_j into one of 2 TMEM buffers, O += P_j V_j into a third),
//   warps 4-7: S_j -> bf16 -> chain -> P_j in shared memory (128-byte swizzled K-major, the
//   A operand of the next MMA), then O -> bf16 -> TMA-store epilogue.
// P_j is exactly the score group's output (same rounding, same chain code) and O accumulates the
// same K = 16 MMA steps in key order as the context group's 128 x 128 tiles.
constexpr int kAttnD = 128, kAttnBlk = 128;
constexpr int kAttnChunk = kAttnBlk * 128;                     // one 64-wide K chunk of a 128-row tile
constexpr int kAttnQ = 2 * kAttnChunk;                         // Q_i: [128 rows x 128 K]
constexpr int kAttnKV = 4 * kAttnChunk;                        // K_j + V_j per stage
constexpr int kAttnP = 2 * kAttnChunk;                         // P_j: [128 rows x 128 keys]
constexpr int kAttnEpi = 16;  // epilogue warps: 4 per TMEM lane quarter, one 32-column chunk each per block
constexpr int kAttnThreads = 128 + 32 * kAttnEpi;
// (the output staging of the final epilogue reuses the P buffer: the last MMA has read it)
constexpr int kAttnSmem = kAttnQ + 2 * kAttnKV + kAttnP + 1024 + kEpiTabBytes + 1024;
constexpr uint32_t kAttnIdescS = TcCfg<128, true, true, 128>::kIdesc;   // B = K_j, K-major
constexpr uint32_t kAttnIdescO = TcCfg<128, false, true, 128>::kIdesc;  // B = V_j, MN-major

__global__ void __launch_bounds__(kAttnThreads, 1)
    AttnChainKernel(const CUtensorMap* __restrict__ maps, int q_blocks, int k_blocks, ChainArgs epi) {
  PdlTrigger();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;
  uint8_t* skv = sq + kAttnQ;
  uint8_t* sp = skv + 2 * kAttnKV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sp + kAttnP);
  // K_j and V_j have their own stages: K_j is free once S_j is computed, V_j only after O += P_j V_j,
  // so K can be fetched two blocks ahead of its use (one shared stage serialized the TMA latency)
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2]
  uint64_t* s_empty = bars + 11; // [2]
  uint64_t* p_full = bars + 13;
  uint64_t* p_empty = bars + 14;
  uint64_t* o_full = bars + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
  uint8_t* tab_area = reinterpret_cast<uint8_t*>(bars) + 1024;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int head = blockIdx.x / q_blocks, qi = blockIdx.x % q_blocks;
  const CUtensorMap* mq = maps + 4 * head;
  const CUtensorMap* mk = mq + 1;
  const CUtensorMap* mv = mq + 2;
  const CUtensorMap* mo = mq + 3;

  if (warp == 0 && lane == 0) {
    MbarInit(q_full, 1);
    for (int b = 0; b < 2; ++b) {
      MbarInit(&k_full[b], 1);
      MbarInit(&k_empty[b], 1);
      MbarInit(&v_full[b], 1);
      MbarInit(&v_empty[b], 1);
      MbarInit(&s_full[b], 1);
      MbarInit(&s_empty[b], kAttnEpi);
    }
    MbarInit(p_full, kAttnEpi);
    MbarInit(p_empty, 1);
    MbarInit(o_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(SmemU32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  FenceBefore();
  __syncthreads();
  FenceAfter();
  const uint32_t tmem = *tmem_slot;  // S_0 at column 0, S_1 at 128, O at 256
  PdlWait();

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer ----------------
      MbarExpectTx(q_full, kAttnQ);
      for (int c = 0; c < 2; ++c) TmaLoad2D(sq + c * kAttnChunk, mq, q_full, c * 64, qi * kAttnBlk);
      auto load_k = [&](int j) {
        const int st = j & 1;
        MbarWait(&k_empty[st], ((j >> 1) & 1) ^ 1);
        uint8_t* sk = skv + st * kAttnKV;
        MbarExpectTx(&k_full[st], 2 * kAttnChunk);
        for (int c = 0; c < 2; ++c) TmaLoad2D(sk + c * kAttnChunk, mk, &k_full[st], c * 64, j * kAttnBlk);
      };
      auto load_v = [&](int j) {
        const int st = j & 1;
        MbarWait(&v_empty[st], ((j >> 1) & 1) ^ 1);
        uint8_t* sv = skv + st * kAttnKV + 2 * kAttnChunk;
        MbarExpectTx(&v_full[st], 2 * kAttnChunk);
        for (int c = 0; c < 2; ++c) TmaLoad2D(sv + c * kAttnChunk, mv, &v_full[st], c * 64, j * kAttnBlk);
      };
      // K runs one block ahead of V: K0 K1 V0 K2 V1 ... (a V wait never delays the next K)
      for (int j = 0; j <= k_blocks; ++j) {
        if (j < k_blocks) load_k(j);
        if (j > 0) load_v(j - 1);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer ----------------
      MbarWait(q_full, 0);
      const uint32_t aq = SmemU32(sq);
      auto issue_s = [&](int j) {
        const int st = j & 1;
        MbarWait(&k_full[st], (j >> 1) & 1);
        MbarWait(&s_empty[st], ((j >> 1) & 1) ^ 1);
        FenceAfter();
        const uint32_t ak = SmemU32(skv + st * kAttnKV);
#pragma unroll
        for (int k = 0; k < kAttnD / 16; ++k)
          MmaF16(tmem + st * kAttnBlk, DescSw128(aq + (k / 4) * kAttnChunk + (k % 4) * 32, 16, 1024),
                 DescSw128(ak + (k / 4) * kAttnChunk + (k % 4) * 32, 16, 1024), kAttnIdescS, k != 0);
        Commit(&s_full[st]);
        Commit(&k_empty[st]);
      };
      issue_s(0);
      const uint32_t ap = SmemU32(sp);
      for (int j = 0; j < k_blocks; ++j) {
        if (j + 1 < k_blocks) issue_s(j + 1);
        MbarWait(p_full, j & 1);
        MbarWait(&v_full[j & 1], (j >> 1) & 1);
        FenceAfter();
        const uint32_t av = SmemU32(skv + (j & 1) * kAttnKV + 2 * kAttnChunk);
#pragma unroll
        for (int k = 0; k < kAttnBlk / 16; ++k)
          MmaF16(tmem + 2 * kAttnBlk, DescSw128(ap + (k / 4) * kAttnChunk + (k % 4) * 32, 16, 1024),
                 DescSw128(av + k * 16 * 128, 64 * kAttnBlk * 2, 1024), kAttnIdescO, (j | k) != 0);
        Commit(p_empty);
        Commit(&v_empty[j & 1]);
      }
      Commit(o_full);
    }
  } else if (warp >= 4) {  // ---------------- chain + output epilogue ----------------
    // warp ew: TMEM lane quarter ew % 4 (rows [32*q, 32*q + 32)), 32-column chunks ew / 4 + 2i
    const int ew = warp - 4, quarter = ew % 4, half = ew / 4;
    const uint16_t* tp[kMaxTanhRuns];
    StageEpiTables(epi, reinterpret_cast<uint16_t*>(tab_area), threadIdx.x - 128, tp, 32 * kAttnEpi);
    const int r = quarter * 32 + lane;  // row of the 128-row tile
    constexpr int kCh = kAttnBlk / 32 / (kAttnEpi / 4);  // 32-column chunks per warp and block
    for (int j = 0; j < k_blocks; ++j) {
      const int st = j & 1;
      MbarWait(&s_full[st], (j >> 1) & 1);
      FenceAfter();
      // S_j -> bf16 -> chain into registers first: this overlaps the previous O MMA, and the S
      // buffer goes back to the MMA warp before P is written
      uint32_t pk[kCh][16];
#pragma unroll
      for (int ci = 0; ci < kCh; ++ci) {
        const int c = half + ci * (kAttnEpi / 4);
        uint32_t v[32];
        TmemLd32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + st * kAttnBlk + c * 32, v);
#pragma unroll
        for (int t = 0; t < 16; ++t) pk[ci][t] = PackBf16x2(__uint_as_float(v[2 * t]), __uint_as_float(v[2 * t + 1]));
        EpiPackedBf16(epi, pk[ci], tp);
      }
      FenceBefore();
      __syncwarp();
      if (lane == 0) MbarArrive(&s_empty[st]);
      if (j > 0) MbarWait(p_empty, (j - 1) & 1);  // the previous O MMA has read P
#pragma unroll
      for (int ci = 0; ci < kCh; ++ci) {
        const int c = half + ci * (kAttnEpi / 4);
        // keys c*32 .. c*32+31 of row r: 64-key chunk c/2, 16-byte units (c%2)*4 + t, 128-byte swizzle
        uint8_t* row = sp + (c >> 1) * kAttnChunk + r * 128;
#pragma unroll
        for (int t = 0; t < 4; ++t)
          *reinterpret_cast<uint4*>(row + ((((c & 1) * 4 + t) ^ (r & 7)) << 4)) =
              make_uint4(pk[ci][4 * t], pk[ci][4 * t + 1], pk[ci][4 * t + 2], pk[ci][4 * t + 3]);
      }
      FenceProxyAsyncSmem();  // generic-proxy P stores -> the MMA's async-proxy reads
      __syncwarp();
      if (lane == 0) MbarArrive(p_full);
    }
    MbarWait(o_full, 0);  // every MMA done: P is free for the output staging
    FenceAfter();
    // one or two 2 KB boxes per warp: kAttnEpi warps x that fit in the 32 KB P buffer
    constexpr int kBoxes = kAttnD / 32 / (kAttnEpi / 4);
    static_assert(kAttnEpi * (kBoxes > 1 ? 4096 : 2048) <= kAttnP, "output staging exceeds the P buffer");
    uint8_t* stage_c = sp + ew * (kBoxes > 1 ? 4096 : 2048);
    uint32_t boxes = 0;
#pragma unroll 1
    for (int c = half; c < kAttnD / 32; c += kAttnEpi / 4) {
      uint32_t v[32];
      TmemLd32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + 2 * kAttnBlk + c * 32, v);
      uint32_t p[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) p[t] = PackBf16x2(__uint_as_float(v[2 * t]), __uint_as_float(v[2 * t + 1]));
      EpiStoreBox(stage_c, boxes++, p, mo, c * 32, qi * kAttnBlk + quarter * 32, lane);
    }
    if (lane == 0) BulkWaitAll();
  }
  FenceBefore();
  __syncthreads();
  FenceAfter();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}
}  // namespace

size_t GemmTf32x3ScratchBytes(const GemmArgs& g) {
  return static_cast<size_t>(2 * (g.m * g.k + g.k * g.n)) * 4;
}

namespace {
struct Sched {
  bool pair;
  int bn, ks;
  bool sk = false;  // stream-K (pair kernel)
};
// Measured (profiles/gemm_shapes.py, B200, bf16): the CTA-pair kernel with 256 x 256 pair
// tiles wins once they fill a wave (2048x4096 output, K 4096: 46.8 vs 49.4 us; K 16384: 174 vs
// 200 us) and, with split-K, for long-K GEMMs with few tiles (512x4096 output, K 16384: 61 vs
// 77 us); below a wave, and with 256 x 128 pair tiles, the single-CTA kernel is faster (2048^3:
// 14.7 vs 15.6 us; 512x4096 output, K 4096: 19.3 vs 23.4 us).
Sched ScheduleOf(const GemmArgs& g) {
  if (UseStreamK(g)) return {true, 256, 1, true};
  if (UsePair(g) && g.n % 256 == 0) {
    static const int force = EnvInt("RH_GEMM_BN", 0);
    const int64_t ctas = (g.m / BM) * (g.n / 256);
    if (force == 256 || ctas >= SmCount()) return {true, 256, 1};
    if (force == 128 && EnvInt("RH_GEMM_PAIR128", 0)) return {true, 128, 1};
    if (ctas < 96 && g.k / BK >= 128) return {true, 256, KSplitPair(g, 256)};
  }
  const int bn = PickBN(g);
  return {false, bn, bn ? KSplit(g, bn) : 1};
}
}  // namespace

size_t GemmTcScratchBytes(const GemmArgs& g) {
  if (g.dtype == RH_F32) return GemmTf32x3ScratchBytes(g);
  const Sched sc = ScheduleOf(g);
  if (sc.sk) return StreamKScratchBytes();
  return sc.ks > 1 ? static_cast<size_t>(sc.ks) * g.m * g.n * 4 : 0;
}

bool GemmTcSupported(const GemmArgs& g) {
  if (g.dtype == RH_F32) {
    if (g.m % BM || g.n % 128 || g.k % BK32 || g.k == 0 || !g.scratch) return false;
  } else if (g.dtype == RH_BF16) {
    if (g.m % BM || g.k % BK || g.k == 0) return false;
  } else {
    return false;
  }
  if (g.m > (int64_t{1} << 30) || g.n > (int64_t{1} << 30) || g.k > (int64_t{1} << 30)) return false;
  if (g.dtype == RH_F32 ? PickBN(g) == 0 : ScheduleOf(g).bn == 0) return false;
  const uintptr_t a = reinterpret_cast<uintptr_t>(g.a), b = reinterpret_cast<uintptr_t>(g.b);
  if ((a | b) % 16) return false;
  return true;
}

const char* GemmTcSchedule(const GemmArgs& g) {
  if (g.dtype == RH_F32) return "";
  const Sched sc = ScheduleOf(g);
  if (sc.sk) return " [pair, stream-k]";
  if (sc.pair) return sc.ks > 1 ? " [pair, split-k]" : " [pair]";
  return sc.ks > 1 ? " [split-k]" : "";
}

bool GemmTcPushSupported(const GemmArgs& g, bool single_pass) {
  if (g.dtype != RH_BF16 || !GemmTcSupported(g)) return false;
  const Sched sc = ScheduleOf(g);
  if (sc.sk) return false;
  return !single_pass || sc.ks == 1;  // single pass: the epilogue pushes; split-K: the reduce
}

int GemmTcLaunches(const GemmArgs& g) {
  if (g.dtype == RH_F32) return 3;
  return ScheduleOf(g).ks > 1 ? 2 : 1;
}

// ------------------------------- grouped GEMM (horizontal fusion) -------------------------------
namespace {
// 8 epilogue warps when the main loop is a handful of k-blocks (K <= 256): the epilogue is the
// critical path there.  RH_GEMM_EPI8=0 disables (A/B).
bool UseEpi8(const GemmArgs& g) {
  static const int on = EnvInt("RH_GEMM_EPI8", 1);
  return on && g.k <= 256;
}
// Problems side by side along a virtual N = n_prob * g.n.  A tile may span problems only when
// they share A; B column chunks (64 wide, MN-major) or boxes (K-major: bn or bn/2 rows) must not
// straddle two problems; no split-K (the partials' reduce would need the same scatter).
Sched GroupScheduleOf(const GemmArgs& g, int n_prob, bool shared_a) {
  GemmArgs v = g;
  v.n = g.n * n_prob;
  auto ok = [&](int bn, bool pair) {
    const int64_t half = pair ? bn / 2 : bn;
    if (v.n % bn || g.n % 64) return false;
    if (!shared_a && g.n % bn) return false;
    if (g.tb && g.n % half) return false;
    return true;
  };
  static const int force = EnvInt("RH_GEMM_BN", 0);
  if (UsePair(v) && ok(256, true)) {
    const int64_t ctas = (v.m / BM) * (v.n / 256);
    if (ctas >= SmCount() || force == 256) return {true, 256, 1};
  }
  if (force != 128 && (v.m / BM) * (v.n / 256) >= 96 && ok(256, false)) return {false, 256, 1};
  if (ok(128, false)) return {false, 128, 1};
  return {false, 0, 1};
}

struct GroupHost {
  GroupLaunch gl;
  Sched sc;
};
std::mutex g_group_mu;
std::map<const void*, GroupHost> g_groups;  // device table -> launch parameters
}  // namespace

bool GemmTcGroupSupported(const GemmArgs& g, int n_prob, bool shared_a) {
  if (g.dtype != RH_BF16 || n_prob < 2 || !GemmTcSupported(g)) return false;
  if (g.n * n_prob > (int64_t{1} << 30)) return false;
  return GroupScheduleOf(g, n_prob, shared_a).bn != 0;
}

size_t GemmTcGroupTableBytes(int n_prob) {
  return static_cast<size_t>(n_prob) * 3 * sizeof(CUtensorMap);
}

const char* GemmTcGroupSchedule(const GemmArgs& g, int n_prob, bool shared_a) {
  const Sched sc = GroupScheduleOf(g, n_prob, shared_a);
  if (sc.pair) return " [pair]";
  return sc.bn == 256 ? " [256]" : " [128]";
}

void PrepareGemmTcGroup(const GemmArgs& g, int n_prob, const void* const* a, const void* const* b,
                        void* const* c, void* table) {
  const bool shared_a = std::all_of(a, a + n_prob, [&](const void* x) { return x == a[0]; });
  if (!GemmTcGroupSupported(g, n_prob, shared_a)) Fail("tcgen05 grouped GEMM: unsupported shape/layout", RH_ERR_UNSUPPORTED);
  GroupHost h{};
  h.sc = GroupScheduleOf(g, n_prob, shared_a);
  const int box_n = h.sc.pair ? h.sc.bn / 2 : h.sc.bn;
  const int kb = !h.sc.pair && h.sc.bn == 128 && g.k % 128 == 0 ? 128 : 64;
  std::vector<char> host(GemmTcGroupTableBytes(n_prob));
  CUtensorMap* bm = reinterpret_cast<CUtensorMap*>(host.data());
  CUtensorMap* am = bm + n_prob;
  CUtensorMap* cm = am + n_prob;
  for (int p = 0; p < n_prob; ++p) {
    GemmArgs gp = g;
    gp.a = a[p];
    gp.b = b[p];
    gp.c = c[p];
    const Maps& mp = GetMaps(gp, box_n, kb);
    if (p == 0) h.gl.m0 = mp;
    bm[p] = mp.b;
    am[p] = mp.a;
    cm[p] = mp.c;
    if (reinterpret_cast<uintptr_t>(c[p]) % 16) Fail("tcgen05 grouped GEMM: unaligned output");
  }
  RH_CUDA(cudaMemcpy(table, host.data(), host.size(), cudaMemcpyHostToDevice));
  const CUtensorMap* tb = static_cast<const CUtensorMap*>(table);
  h.gl.dev.b = tb;
  h.gl.dev.a = shared_a ? nullptr : tb + n_prob;
  h.gl.dev.cm = tb + 2 * n_prob;
  h.gl.dev.seg_n = static_cast<int>(g.n);
  h.gl.n_prob = n_prob;
  std::lock_guard<std::mutex> lk(g_group_mu);
  g_groups[table] = h;
}

void ReleaseGemmTcGroup(const void* table) {
  std::lock_guard<std::mutex> lk(g_group_mu);
  g_groups.erase(table);
}

void LaunchGemmTcGroup(const GemmArgs& g, const void* table, cudaStream_t s) {
  GroupHost h;
  {
    std::lock_guard<std::mutex> lk(g_group_mu);
    auto it = g_groups.find(table);
    if (it == g_groups.end()) Fail("tcgen05 grouped GEMM: table not prepared", RH_ERR_STATE);
    h = it->second;
  }
  for (int i = 0; i < g.epi.n_fn; ++i) {
    const int fn = g.epi.fns[i];
    if (fn != RH_FN_RELU && fn != RH_FN_NEG && fn != RH_FN_IDENTITY && !(fn >= kFnTanhRun && fn - kFnTanhRun < g.epi.n_tab))
      Fail("tcgen05 bf16 GEMM epilogue takes only relu / neg / identity / tanh runs", RH_ERR_UNSUPPORTED);
  }
  const GroupLaunch* gl = &h.gl;
  const int v = (h.sc.bn == 256 ? 4 : 0) | (g.tb ? 2 : 0) | (g.ta ? 0 : 1);
  if (h.sc.pair) {
    if (UseEpi8(g)) {
      static const int w = EnvInt("RH_GEMM_EPI_WARPS", 12);
      if (w == 12) {
        switch (v) {
          case 4: LaunchPair<256, false, false, true, 12>(g, s, gl); break;
          case 5: LaunchPair<256, false, true, true, 12>(g, s, gl); break;
          case 6: LaunchPair<256, true, false, true, 12>(g, s, gl); break;
          case 7: LaunchPair<256, true, true, true, 12>(g, s, gl); break;
          default: Fail("internal: grouped pair schedule");
        }
        return;
      }
      switch (v) {
        case 4: LaunchPair<256, false, false, true, 8>(g, s, gl); break;
        case 5: LaunchPair<256, false, true, true, 8>(g, s, gl); break;
        case 6: LaunchPair<256, true, false, true, 8>(g, s, gl); break;
        case 7: LaunchPair<256, true, true, true, 8>(g, s, gl); break;
        default: Fail("internal: grouped pair schedule");
      }
      return;
    }
    switch (v) {
      case 4: LaunchPair<256, false, false, true>(g, s, gl); break;
      case 5: LaunchPair<256, false, true, true>(g, s, gl); break;
      case 6: LaunchPair<256, true, false, true>(g, s, gl); break;
      case 7: LaunchPair<256, true, true, true>(g, s, gl); break;
      default: Fail("internal: grouped pair schedule");
    }
    return;
  }
  switch (v) {
    case 0: Launch<128, false, false, true>(g, s, gl); break;
    case 1: Launch<128, false, true, true>(g, s, gl); break;
    case 2: Launch<128, true, false, true>(g, s, gl); break;
    case 3: Launch<128, true, true, true>(g, s, gl); break;
    case 4: Launch<256, false, false, true>(g, s, gl); break;
    case 5: Launch<256, false, true, true>(g, s, gl); break;
    case 6: Launch<256, true, false, true>(g, s, gl); break;
    default: Launch<256, true, true, true>(g, s, gl); break;
  }
}

void LaunchGemmTc(const GemmArgs& g, cudaStream_t s) {
  if (!GemmTcSupported(g)) Fail("tcgen05 GEMM: unsupported shape/layout", RH_ERR_UNSUPPORTED);
  if (g.dtype == RH_F32) {
    if (g.tb) LaunchTf32x3<true>(g, s);
    else LaunchTf32x3<false>(g, s);
    return;
  }
  for (int i = 0; i < g.epi.n_fn; ++i) {
    const int fn = g.epi.fns[i];
    if (fn != RH_FN_RELU && fn != RH_FN_NEG && fn != RH_FN_IDENTITY && !(fn >= kFnTanhRun && fn - kFnTanhRun < g.epi.n_tab))
      Fail("tcgen05 bf16 GEMM epilogue takes only relu / neg / identity / tanh runs", RH_ERR_UNSUPPORTED);
  }
  const Sched sc = ScheduleOf(g);
  const int v = (sc.bn == 256 ? 4 : 0) | (g.tb ? 2 : 0) | (g.ta ? 0 : 1);
  if (sc.pair) {
    switch (v) {
      case 0: LaunchPair<128, false, false>(g, s); break;
      case 1: LaunchPair<128, false, true>(g, s); break;
      case 2: LaunchPair<128, true, false>(g, s); break;
      case 3: LaunchPair<128, true, true>(g, s); break;
      case 4: LaunchPair<256, false, false>(g, s); break;
      case 5: LaunchPair<256, false, true>(g, s); break;
      case 6: LaunchPair<256, true, false>(g, s); break;
      default: LaunchPair<256, true, true>(g, s); break;
    }
    return;
  }
  switch (v) {
    case 0: Launch<128, false, false>(g, s); break;
    case 1: Launch<128, false, true>(g, s); break;
    case 2: Launch<128, true, false>(g, s); break;
    case 3: Launch<128, true, true>(g, s); break;
    case 4: Launch<256, false, false>(g, s); break;
    case 5: Launch<256, false, true>(g, s); break;
    case 6: Launch<256, true, false>(g, s); break;
    default: Launch<256, true, true>(g, s); break;
  }
}


// ------------------------- fused score -> chain -> context: host side -------------------------
bool AttnChainSupported(int n_heads, int64_t sq, int64_t sk, int64_t d) {
  return n_heads > 0 && d == kAttnD && sq > 0 && sk > 0 && sq % kAttnBlk == 0 && sk % kAttnBlk == 0 &&
         static_cast<int64_t>(n_heads) * (sq / kAttnBlk) < (int64_t{1} << 31) && sk / kAttnBlk < (1 << 30);
}
size_t AttnChainTableBytes(int n_heads) { return static_cast<size_t>(n_heads) * 4 * sizeof(CUtensorMap); }

void PrepareAttnChain(int n_heads, int64_t sq, int64_t sk, const void* const* q, const void* const* k,
                      const void* const* v, void* const* o, void* table) {
  std::vector<CUtensorMap> m(static_cast<size_t>(n_heads) * 4);
  for (int h = 0; h < n_heads; ++h) {
    for (const void* ptr : {q[h], k[h], v[h], static_cast<const void*>(o[h])})
      if (reinterpret_cast<uintptr_t>(ptr) % 16) Fail("attention chain: unaligned operand");
    m[4 * h + 0] = MakeMap(q[h], kAttnD, sq, kAttnD, 64, kAttnBlk);  // Q [sq, 128]: K-major A
    m[4 * h + 1] = MakeMap(k[h], kAttnD, sk, kAttnD, 64, kAttnBlk);  // K [sk, 128]: K-major B
    m[4 * h + 2] = MakeMap(v[h], kAttnD, sk, kAttnD, 64, kAttnBlk);  // V [sk, 128]: MN-major B
    m[4 * h + 3] = MakeMap(o[h], kAttnD, sq, kAttnD, 32, 32, false, CU_TENSOR_MAP_SWIZZLE_64B);
  }
  RH_CUDA(cudaMemcpy(table, m.data(), m.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
}

void LaunchAttnChain(int n_heads, int64_t sq, int64_t sk, const ChainArgs& epi, const void* table, cudaStream_t s) {
  for (int i = 0; i < epi.n_fn; ++i) {
    const int fn = epi.fns[i];
    if (fn != RH_FN_RELU && fn != RH_FN_NEG && fn != RH_FN_IDENTITY && !(fn >= kFnTanhRun && fn - kFnTanhRun < epi.n_tab))
      Fail("attention chain: the score chain takes only relu / neg / identity / tanh runs", RH_ERR_UNSUPPORTED);
  }
  int dev = 0;
  RH_CUDA(cudaGetDevice(&dev));
  static bool attr[64] = {};
  if (dev < 64 && !attr[dev]) {
    RH_CUDA(cudaFuncSetAttribute(AttnChainKernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnSmem));
    attr[dev] = true;
  }
  const int qb = static_cast<int>(sq / kAttnBlk), kb = static_cast<int>(sk / kAttnBlk);
  LaunchPdl(AttnChainKernel, n_heads * qb, kAttnThreads, kAttnSmem, s, static_cast<const CUtensorMap*>(table), qb, kb, epi);
  RH_CUDA(cudaGetLastError());
}
}  // namespace rh
