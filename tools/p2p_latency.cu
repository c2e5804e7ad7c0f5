// p2p_latency.cu — NVLink peer-memory physics on 2 GPUs (one process, peer access): the costs
// the transition kernels are built from.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   (1) flag ping-pong round trip: st.release.sys / ld.acquire.sys, and relaxed + fence variants
//   (2) peer-read copy kernel (pull) of S bytes, 1 .. 64 MiB: duration via events
//   (3) local copy kernel of the same sizes; empty-kernel graph replay gap
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) { asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) { uint32_t v; asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) { asm volatile("st.relaxed.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) { uint32_t v; asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }

// me writes peer_flag (on the peer GPU), waits on my_flag (local, written by the peer)
__global__ void PingPong(uint32_t* my_flag, uint32_t* peer_flag, int iters, int first, int mode, unsigned long long* out) {
  unsigned long long t0 = clock64();
  for (int i = 1; i <= iters; ++i) {
    if (first) {
      if (mode == 0) st_release(peer_flag, i); else { __threadfence_system(); st_relaxed(peer_flag, i); }
      while ((mode == 0 ? ld_acquire(my_flag) : ld_relaxed(my_flag)) < (uint32_t)i) {}
    } else {
      while ((mode == 0 ? ld_acquire(my_flag) : ld_relaxed(my_flag)) < (uint32_t)i) {}
      if (mode == 0) st_release(peer_flag, i); else { __threadfence_system(); st_relaxed(peer_flag, i); }
    }
  }
  *out = clock64() - t0;
}

__global__ void Copy(uint4* dst, const uint4* src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) dst[i] = src[i];
}
__global__ void Empty() {}
__global__ void FenceSys(int n) { for (int i = 0; i < n; ++i) __threadfence_system(); }

int main() {
  int nd = 0;
  CK(cudaGetDeviceCount(&nd));
  if (nd < 2) { printf("need 2 GPUs\n"); return 1; }
  CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0));
  uint32_t* f[2];
  unsigned long long* o[2];
  for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaMalloc(&f[d], 256)); CK(cudaMalloc(&o[d], 8)); }
  int clk = 0; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  for (int mode = 0; mode < 2; ++mode) {
    for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaMemset(f[d], 0, 256)); CK(cudaDeviceSynchronize()); }
    const int iters = 2000;
    CK(cudaSetDevice(1)); PingPong<<<1, 1>>>(f[1], f[0], iters, 0, mode, o[1]);
    CK(cudaSetDevice(0)); PingPong<<<1, 1>>>(f[0], f[1], iters, 1, mode, o[0]);
    for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
    unsigned long long cyc = 0; CK(cudaSetDevice(0)); CK(cudaMemcpy(&cyc, o[0], 8, cudaMemcpyDeviceToHost));
    printf("pingpong mode=%s round trip %.2f us (clock %d kHz)\n", mode == 0 ? "release/acquire" : "fence+relaxed", cyc / (double)iters / (clk * 1e-3), clk);
  }
  CK(cudaSetDevice(0));
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  // fence cost
  FenceSys<<<1, 32, 0, s>>>(1); CK(cudaStreamSynchronize(s));
  CK(cudaEventRecord(e0, s)); FenceSys<<<1, 32, 0, s>>>(1000); CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
  float ms = 0; CK(cudaEventElapsedTime(&ms, e0, e1)); printf("__threadfence_system: %.3f us each\n", ms * 1e3 / 1000);
  // empty-kernel graph gap
  cudaGraph_t g; cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < 100; ++i) Empty<<<148, 256, 0, s>>>();
  CK(cudaStreamEndCapture(s, &g)); CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, s)); CK(cudaStreamSynchronize(s));
  CK(cudaEventRecord(e0, s)); for (int r = 0; r < 10; ++r) CK(cudaGraphLaunch(ge, s)); CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
  CK(cudaEventElapsedTime(&ms, e0, e1)); printf("graph empty kernel (148x256): %.2f us each\n", ms * 1e3 / 1000);
  // copies
  size_t maxb = 64ull << 20;
  void *loc, *loc2, *peer;
  CK(cudaMalloc(&loc, maxb)); CK(cudaMalloc(&loc2, maxb));
  CK(cudaSetDevice(1)); CK(cudaMalloc(&peer, maxb)); CK(cudaMemset(peer, 1, maxb)); CK(cudaDeviceSynchronize()); CK(cudaSetDevice(0));
  for (size_t b = 1 << 20; b <= maxb; b *= 4) {
    for (int grid : {148, 148 * 4, 148 * 8}) {
      int64_t n = b / 16;
      for (int pass = 0; pass < 2; ++pass) {
        const void* src = pass == 0 ? peer : loc2;
        Copy<<<grid, 256, 0, s>>>((uint4*)loc, (const uint4*)src, n);
        CK(cudaStreamSynchronize(s));
        CK(cudaEventRecord(e0, s));
        for (int r = 0; r < 20; ++r) Copy<<<grid, 256, 0, s>>>((uint4*)loc, (const uint4*)src, n);
        CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double us = ms * 1e3 / 20;
        printf("%s copy %6zu KiB grid %4d: %8.2f us  %7.1f GB/s\n", pass == 0 ? "peer " : "local", b >> 10, grid, us, b / (us * 1e-6) / 1e9);
      }
    }
  }
  return 0;
}
