// ew_jit.cpp — per-program elementwise chain kernels, compiled with NVRTC at program load.
//
// The interpreter kernels (k_elementwise.cu) decode every instruction of a chain program per
// 8-element vector: on the 24-layer backward chains the decode (instruction fetch, dispatch
// branches, operand-select switches) is most of the issued instructions (ncu: IMAD / ISETP /
// BRA / MOV / LDC ahead of the bf16 math).  Here each distinct program becomes its own kernel:
// the same body (ew_core.cuh EwProgBody / EwLadderBody) with the instruction sequence written
// out as EwStep calls on literal constants, which the compiler folds into straight-line code.
// EwStep is the one definition of an instruction's semantics for both paths, so results are
// bit-identical to the interpreter's.
//
// Programs are registered while the executor lowers (EwJitRegister: deduplicated by kernel
// family, input count and instruction sequence) and compiled together at the end of the build
// (EwJitBuild: one NVRTC unit per batch of programs, batches in parallel threads, loaded as a
// context-independent cudaLibrary so one handle serves every local device).  RH_EW_JIT=0 keeps
// the interpreter; a failed compile prints NVRTC's log once and falls back to it.
#include <nvrtc.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "kernels.h"

#include "ew_jit_src.inc"  // kEwJitParts (build.py: the device headers as string literals)

namespace rh {
namespace {

struct JitEntry {
  std::string key;
  int kind = 0;
  int n_in = 0;
  std::vector<int32_t> code;  // the instructions the kernel inlines
  bool tried = false;
  cudaKernel_t k = nullptr;
  unsigned attr_devs = 0;  // devices whose max dynamic shared memory attribute is set
};

std::mutex g_mu;
std::deque<JitEntry> g_entries;
std::unordered_map<std::string, int> g_by_key;
std::vector<cudaLibrary_t> g_libs;

bool JitEnabled() {
  static const bool on = [] {
    const char* e = getenv("RH_EW_JIT");
    return !(e && e[0] == '0');
  }();
  return on;
}

std::string KernelName(int id) { return "rh_ew_" + std::to_string(id); }

// One kernel: EwProgBody / EwLadderBody with the instruction sequence inlined.
std::string KernelSource(const JitEntry& e, int id) {
  const bool bf = e.kind != kEwKindF32;
  const bool remat = e.kind == kEwKindRematHalf || e.kind == kEwKindRematFull || e.kind == kEwKindLadderRemat;
  const bool half = e.kind == kEwKindRematHalf;
  const bool ladder = e.kind == kEwKindLadder || e.kind == kEwKindLadderRemat;
  // resident blocks per SM the register budget is sized for (the interpreter's, except the
  // plain programs: straight-line code fits 64 registers)
  const int min_blocks = half ? 4 : e.kind == kEwKindRematFull ? 1 : ladder ? (remat ? 1 : 2) : 4;
  const int nin = std::max(1, e.n_in);
  const std::string tp = std::string(bf ? "true" : "false") + ", " + (remat ? "true" : "false") + ", " +
                         (half ? "true" : "false") + ", " + std::to_string(nin);
  std::string s;
  s += "extern \"C\" __global__ void __launch_bounds__(256, " + std::to_string(min_blocks) + ") " + KernelName(id) +
       "(const __grid_constant__ rh::EwArgs a) {\n";
  s += "  struct P {\n    __device__ __forceinline__ void operator()(const rh::EwArgs& a, int64_t i, "
       "const uint16_t* t, rh::EwVec<" + std::to_string(nin) + ">& v) const {\n";
  for (int32_t ins : e.code)
    s += "      rh::EwStep<" + tp + ">(a, i, t, v, " + std::to_string(ins & 0xff) + ", " + std::to_string(ins >> 8) +
         ");\n";
  s += "    }\n  };\n";
  if (ladder)
    s += "  rh::EwLadderBody<" + std::string(remat ? "true" : "false") + ", " + std::to_string(nin) + ", true>(a, P{});\n";
  else
    s += "  rh::EwProgBody<" + tp + ", true>(a, P{});\n";
  s += "}\n";
  return s;
}

std::string Prelude() {
  // RH_EW_PAIR=0: one vector per thread-iteration (A/B of EwProgBody's two-vector loop)
  const char* pair = getenv("RH_EW_PAIR");
  std::string s = std::string("#define RH_EW_PAIR_VECTORS ") + (pair && pair[0] == '0' ? "0" : "1") + "\n" +
      "#include <cuda_bf16.h>\n#include <cuda/std/cstdint>\n"
      "using cuda::std::int8_t; using cuda::std::uint8_t; using cuda::std::int16_t; using cuda::std::uint16_t;\n"
      "using cuda::std::int32_t; using cuda::std::uint32_t; using cuda::std::int64_t; using cuda::std::uint64_t;\n";
  for (const char* part : kEwJitParts) s += part;
  return s;
}

const char* CudaInclude() {
  static std::string inc = [] {
    const char* home = getenv("CUDA_HOME");
    return std::string("-I") + (home && *home ? home : "/usr/local/cuda") + "/include";
  }();
  return inc.c_str();
}

// Compiles entries [ids] as one NVRTC unit; returns the cubin (empty on failure, log printed).
std::vector<char> Compile(const std::vector<int>& ids, const std::vector<std::string>& bodies) {
  std::string src = Prelude();
  for (const auto& b : bodies) src += b;
  nvrtcProgram prog = nullptr;
  if (nvrtcCreateProgram(&prog, src.c_str(), "rh_ew_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) return {};
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", CudaInclude()};
  const nvrtcResult r = nvrtcCompileProgram(prog, 4, opts);
  std::vector<char> cubin;
  if (r == NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetCUBINSize(prog, &n);
    cubin.resize(n);
    nvrtcGetCUBIN(prog, cubin.data());
  } else {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, log.data());
    static std::once_flag once;
    std::call_once(once, [&] {
      fprintf(stderr, "[rhino] elementwise JIT: NVRTC failed (%s) for %zu programs; using the interpreter\n%s\n",
              nvrtcGetErrorString(r), ids.size(), log.c_str());
    });
  }
  nvrtcDestroyProgram(&prog);
  return cubin;
}

}  // namespace

int32_t EwJitRegister(const EwArgs& a, int dtype) {
  if (!JitEnabled()) return 0;
  JitEntry e;
  e.kind = EwKindOf(a, dtype);
  e.n_in = a.n_in;
  const bool ladder = e.kind == kEwKindLadder || e.kind == kEwKindLadderRemat;
  e.code.assign(a.code, a.code + (ladder ? a.lad_pc : a.n_code));
  e.key = std::to_string(e.kind) + ":" + std::to_string(e.n_in) + ":";
  for (int32_t c : e.code) e.key += std::to_string(c) + ",";
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_by_key.find(e.key);
  if (it != g_by_key.end()) return it->second + 1;
  const int id = static_cast<int>(g_entries.size());
  g_by_key[e.key] = id;
  g_entries.push_back(std::move(e));
  return id + 1;
}

void EwJitBuild() {
  std::lock_guard<std::mutex> lk(g_mu);
  std::vector<int> todo;
  for (size_t i = 0; i < g_entries.size(); ++i)
    if (!g_entries[i].tried) todo.push_back(static_cast<int>(i));
  if (todo.empty()) return;
  // batches of <= 8 programs compiled in parallel (the NVRTC front end parses cuda_bf16.h once
  // per unit; code generation is per kernel)
  const size_t per = 8;
  const size_t nb = (todo.size() + per - 1) / per;
  std::vector<std::vector<int>> ids(nb);
  std::vector<std::vector<std::string>> bodies(nb);
  for (size_t j = 0; j < todo.size(); ++j) {
    ids[j / per].push_back(todo[j]);
    bodies[j / per].push_back(KernelSource(g_entries[todo[j]], todo[j]));
  }
  std::vector<std::vector<char>> cubins(nb);
  std::vector<std::thread> th;
  for (size_t b = 0; b < nb; ++b) th.emplace_back([&, b] { cubins[b] = Compile(ids[b], bodies[b]); });
  for (auto& t : th) t.join();
  for (size_t b = 0; b < nb; ++b) {
    for (int id : ids[b]) g_entries[id].tried = true;
    if (cubins[b].empty()) continue;
    cudaLibrary_t lib = nullptr;
    RH_CUDA(cudaLibraryLoadData(&lib, cubins[b].data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    g_libs.push_back(lib);
    for (int id : ids[b]) RH_CUDA(cudaLibraryGetKernel(&g_entries[id].k, lib, KernelName(id).c_str()));
  }
}

bool EwJitLaunch(const EwArgs& a, int blocks, size_t smem, cudaStream_t s) {
  cudaKernel_t k = nullptr;
  int dev = 0;
  RH_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (a.jit <= 0 || a.jit > static_cast<int>(g_entries.size())) return false;
    JitEntry& e = g_entries[a.jit - 1];
    if (!e.k) return false;
    k = e.k;
    if (smem > 48 * 1024 && dev < 32 && !(e.attr_devs & (1u << dev))) {
      RH_CUDA(cudaKernelSetAttributeForDevice(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              static_cast<int>(smem), dev));
      e.attr_devs |= 1u << dev;
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(blocks));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  if (PdlEnabled()) {
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  void* args[] = {const_cast<EwArgs*>(&a)};
  RH_CUDA(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(k), args));
  return true;
}

}  // namespace rh

// Test hook (not part of include/rhino_exec.h): NVRTC-compiles one program of every kernel
// family from the embedded headers — no GPU needed — so the CPU suite catches a header the
// run-time compiler rejects.  Returns the cubin size, 0 on a compile failure (log printed).
extern "C" long long rh_test_ew_jit_compile() {
  using namespace rh;
  auto I = [](int op, int arg) { return op | (arg << 8); };
  std::vector<JitEntry> es(6);
  es[0].kind = kEwKindRematHalf;
  es[0].n_in = 2;
  es[0].code = {I(kEwLoad, 0), I(kEwTanhBwdLad, 6 | (7 << 4)), I(kEwStore, 0)};
  es[1].kind = kEwKindBf16;
  es[1].n_in = 2;
  es[1].code = {I(kEwLoad, 0), I(kEwUnary, kFnTanhRun), I(kEwStore, 0), I(kEwUnary, kFnTanhRun + 1), I(kEwKeep, 0),
                I(kEwAdd, 1), I(kEwStore, 1), I(kEwUnary, RH_FN_GELU)};
  es[2].kind = kEwKindF32;
  es[2].n_in = 2;
  es[2].code = {I(kEwLoad, 0), I(kEwUnary, RH_FN_TANH), I(kEwTanhBwd, 1), I(kEwStore, 0), I(kEwMul, kEwSrcKeep)};
  es[3].kind = kEwKindLadder;
  es[3].n_in = 1;
  es[3].code = {I(kEwLoad, 0), I(kEwUnary, kFnTanhRun)};
  es[4].kind = kEwKindRematFull;
  es[4].n_in = 3;
  es[4].code = {I(kEwLoad, 0), I(kEwTanhBwd, kEwSrcVirt + 1), I(kEwTanhBwdLad, 12 | (3 << 4)), I(kEwAdd, 1),
                I(kEwMul, kEwSrcVirt + 8), I(kEwStore, 0)};
  es[5].kind = kEwKindLadderRemat;
  es[5].n_in = 2;
  es[5].code = {I(kEwLoad, 1), I(kEwMul, kEwSrcVirt)};
  std::vector<int> ids;
  std::vector<std::string> bodies;
  for (int i = 0; i < static_cast<int>(es.size()); ++i) {
    ids.push_back(i);
    bodies.push_back(KernelSource(es[i], i));
  }
  return static_cast<long long>(Compile(ids, bodies).size());
}
