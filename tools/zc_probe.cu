// PCIe throughput of SM-driven copies (a kernel loading from / storing to
// pinned host memory through its UVA address) against the copy engines
// (cudaMemcpyAsync), for copies cut into parts like the host pipeline's
// per-column copies.  Diagnostic only.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o zc_probe tools/zc_probe.cu && ./zc_probe
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>

struct Seg { const char* src; char* dst; long long bytes; };

// one launch moves a list of segments; each CTA takes 16-byte vectors with a
// grid-stride loop over the concatenated segments, 4 loads in flight per thread
__global__ void __launch_bounds__(512) k_copy_segs(const Seg* segs, int nseg, long long total_vec) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i < total_vec; i += 4 * stride) {
    uint4 v[4];
    long long idx[4];
    int sg[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      idx[u] = i + u * stride;
      sg[u] = -1;
      if (idx[u] < total_vec) {
        long long off = idx[u];
        int s = 0;
        while (s < nseg && off >= segs[s].bytes / 16) { off -= segs[s].bytes / 16; ++s; }
        sg[u] = s;
        idx[u] = off;
        v[u] = __ldcs(reinterpret_cast<const uint4*>(segs[s].src) + off);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (sg[u] >= 0) __stcs(reinterpret_cast<uint4*>(segs[sg[u]].dst) + idx[u], v[u]);
  }
}

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

int main() {
  const long long n = 1ll << 28;
  char *h1, *h2, *d1, *d2;
  CK(cudaHostAlloc(&h1, n, cudaHostAllocDefault));
  CK(cudaHostAlloc(&h2, n, cudaHostAllocDefault));
  CK(cudaMalloc(&d1, n));
  CK(cudaMalloc(&d2, n));
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  Seg *dsegA, *dsegB;
  CK(cudaMalloc(&dsegA, sizeof(Seg) * 1024));
  CK(cudaMalloc(&dsegB, sizeof(Seg) * 1024));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int grids[] = {16, 32, 64, 148};
  long long parts[] = {16ll << 20, 2ll << 20, 512ll << 10};
  for (long long part : parts) {
    // segments of `part` bytes; a launch moves 8 of them (one chunk's columns)
    const int per_launch = 8;
    const int nseg = (int)(n / part);
    std::vector<Seg> a(nseg), b(nseg);
    for (int s = 0; s < nseg; ++s) {
      a[s] = {h1 + s * part, d1 + s * part, part};
      b[s] = {d2 + s * part, h2 + s * part, part};
    }
    CK(cudaMemcpy(dsegA, a.data(), sizeof(Seg) * nseg, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dsegB, b.data(), sizeof(Seg) * nseg, cudaMemcpyHostToDevice));
    auto dma = [&](bool h2d, bool d2h) {
      for (int s = 0; s < nseg; ++s) {
        if (h2d) cudaMemcpyAsync(d1 + s * part, h1 + s * part, part, cudaMemcpyHostToDevice, s1);
        if (d2h) cudaMemcpyAsync(h2 + s * part, d2 + s * part, part, cudaMemcpyDeviceToHost, s2);
      }
    };
    auto kern = [&](bool h2d, bool d2h, int grid) {
      for (int s = 0; s < nseg; s += per_launch) {
        int k = nseg - s < per_launch ? nseg - s : per_launch;
        long long tv = k * part / 16;
        if (h2d) k_copy_segs<<<grid, 512, 0, s1>>>(dsegA + s, k, tv);
        if (d2h) k_copy_segs<<<grid, 512, 0, s2>>>(dsegB + s, k, tv);
      }
    };
    auto timeit = [&](auto f) {
      f();
      cudaDeviceSynchronize();
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        cudaDeviceSynchronize();
        cudaEventRecord(e0, 0);
        f();
        cudaStreamSynchronize(s1);
        cudaStreamSynchronize(s2);
        cudaEventRecord(e1, 0);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      return n / (best * 1e-3) / 1e9;
    };
    printf("part %6lld KB  DMA: H2D %5.1f  D2H %5.1f  both %5.1f GB/s each\n", part >> 10,
           timeit([&] { dma(true, false); }), timeit([&] { dma(false, true); }),
           timeit([&] { dma(true, true); }));
    for (int g : grids)
      printf("part %6lld KB  kernel grid %3d: H2D %5.1f  D2H %5.1f  both %5.1f GB/s each;  kernel H2D + DMA D2H %5.1f\n",
             part >> 10, g, timeit([&] { kern(true, false, g); }), timeit([&] { kern(false, true, g); }),
             timeit([&] { kern(true, true, g); }), timeit([&] { kern(true, false, g); dma(false, true); }));
  }
  // correctness of the copy kernel
  for (long long i = 0; i < 1024; ++i) h1[i] = (char)(i * 7);
  std::vector<Seg> a1 = {{h1, d1, 1024}};
  cudaMemcpy(dsegA, a1.data(), sizeof(Seg), cudaMemcpyHostToDevice);
  k_copy_segs<<<4, 512>>>(dsegA, 1, 64);
  std::vector<char> back(1024);
  cudaMemcpy(back.data(), d1, 1024, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 1024; ++i) bad += back[i] != (char)(i * 7);
  printf("copy kernel check: %d bad bytes\n", bad);
  return 0;
}
