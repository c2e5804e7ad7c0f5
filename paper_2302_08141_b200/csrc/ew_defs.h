// ew_defs.h — elementwise chain program format shared by the host (executor, launchers), the
// nvcc-built kernels and the kernels specialized at run time with NVRTC (ew_jit.cpp): plain
// constants and structs only, so the file compiles under both.
#pragma once

#ifndef __CUDACC_RTC__
#include <stdint.h>
#include <vector_types.h>
#endif

namespace rh {

// bf16 only: a run of k consecutive tanh ops is one lookup in the table of T^k, T = the
// correctly rounded bf16 tanh (bf16 has 2^16 inputs; T^k composes the per-op-rounded
// semantics exactly).  fns[i] = kFnTanhRun + j selects table j.
constexpr int kFnTanhRun = 100;
constexpr int kMaxTanhRuns = 4;
constexpr int kTanhRunEntries = 897;  // 896 table binades [2^-5, 4) + the |x| >= 4 constant
constexpr int kMaxEwIn = 8, kMaxEwOut = 16, kMaxEwCode = 192;
enum EwOpcode : int32_t { kEwLoad = 0, kEwUnary = 1, kEwAdd = 2, kEwMul = 3, kEwKeep = 4, kEwStore = 5,
                          kEwTanhBwd = 6, kEwTanhBwdLad = 7 };
// kEwTanhBwdLad (rematerializing programs): a run of TBWD on ladder columns hi, hi-1, ..,
// hi-cnt+1 (arg = hi | cnt << 4), unrolled over compile-time columns.
constexpr int kEwSrcKeep = 30, kEwSrcAcc = 31;
struct EwArgs {
  int32_t n_code, n_in;
  int32_t code[kMaxEwCode];
  const void* in[kMaxEwIn];
  void* out[kMaxEwOut];
  int32_t n_tab;
  uint64_t tab_off[kMaxTanhRuns];     // arena offsets (host side)
  const uint16_t* tab[kMaxTanhRuns];  // device pointers, patched per rank at launch
  int64_t n;
  // tanh ladder (bf16): code[lad_pc..] is only tanh runs and stores.  Store s of the suffix
  // holds T^{c_s}(x0) with x0 = acc at lad_pc, so the vector path reads all lad_n outputs of an
  // element from one 32-byte row of the ladder table (TanhLadderTable) instead of walking the
  // chain one lookup per op.  lad_n = 0: no ladder.
  int32_t lad_pc, lad_n;
  int32_t lad_out[kMaxEwOut];
  uint64_t lad_off;  // arena offset (host side)
  const uint4* lad;  // device pointer, patched per rank at launch
  // rematerialized operands (bf16): operand kEwSrcVirt + s = T^{powers[s]}(in[vlad_in]), read
  // from column s of a ladder table (the forward tanh values the backward would otherwise load;
  // the table composes the per-op rounding, so the value is bit-identical).  vlad_n = 0: none.
  int32_t vlad_in, vlad_n;
  uint64_t vlad_off;  // arena offset (host side)
  const uint4* vlad;  // device pointer, patched per rank at launch
  // specialized kernel (ew_jit.cpp): 1 + its id in the JIT registry; 0 runs the interpreter
  int32_t jit;
};
constexpr int kEwSrcVirt = 32;
// Ladder rows: kTanhRunEntries rows x kLadderWidth u16; row r, column s = T^{powers[s]} of the
// row's representative |x| (the TanhRunTable indexing).
constexpr int kLadderWidth = 16;

}  // namespace rh
