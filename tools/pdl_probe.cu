// When do the CTAs of a programmatic-dependent grid B start on SMs freed by
// early-exiting CTAs of the primary grid A?  A: 144 CTAs x 200 KB smem, CTAs
// with blockIdx.x % 2 == 0 exit after ~10 us, the others after ~30 us
// (spinning on the global timer); every CTA triggers launch_dependents
// first.  B: 144 CTAs x 200 KB smem; stamps its start.  nvcc -arch=sm_100a.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }

__global__ void kA(unsigned long long *rec, int mode) {
  extern __shared__ char s[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  unsigned long long t0 = gt();
  unsigned long long dur = (blockIdx.x % 2 == 0) ? 10000 : 30000;
  if (mode == 1) dur = (blockIdx.x < 8) ? 30000 : 10000;   // only 8 long CTAs
  while (gt() - t0 < dur) { s[threadIdx.x] += 1; }
  if (threadIdx.x == 0) { rec[2 * blockIdx.x] = t0; rec[2 * blockIdx.x + 1] = gt() | ((unsigned long long)smid() << 56); }
}
__global__ void kB(unsigned long long *rec) {
  extern __shared__ char s[];
  if (threadIdx.x == 0) { rec[2 * blockIdx.x] = gt(); rec[2 * blockIdx.x + 1] = smid(); }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  s[threadIdx.x] = 0;
}

int main() {
  const int smem = 200 * 1024, N = 144;
  cudaFuncSetAttribute(kA, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(kB, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long *ra, *rb;
  cudaMalloc(&ra, 16 * N); cudaMalloc(&rb, 16 * N);
  cudaStream_t st; cudaStreamCreate(&st);
  for (int mode = 0; mode < 4; ++mode)
  for (int rep = 0; rep < 3; ++rep) {
    auto launch = [&]() {
      kA<<<N, 256, smem, st>>>(ra, mode & 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = N; cfg.blockDim = 256; cfg.dynamicSmemBytes = smem; cfg.stream = st;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, kB, rb);
    };
    if (mode < 2) {
      launch();
    } else {   // modes 2, 3: the same pair captured in a CUDA graph and replayed
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      launch();
      cudaStreamEndCapture(st, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, st);
    }
    cudaStreamSynchronize(st);
    std::vector<unsigned long long> a(2 * N), b(2 * N);
    cudaMemcpy(a.data(), ra, 16 * N, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), rb, 16 * N, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, aend = 0;
    for (int i = 0; i < N; ++i) { t0 = std::min(t0, a[2 * i]); aend = std::max(aend, a[2 * i + 1] & ((1ull << 56) - 1)); }
    aend = 0;
    std::vector<double> bs;
    for (int i = 0; i < N; ++i) bs.push_back((b[2 * i] - t0) / 1e3);
    std::sort(bs.begin(), bs.end());
    printf("mode %d rep %d: A end %.1f us; B start: min %.1f p10 %.1f med %.1f p90 %.1f max %.1f\n", mode, rep,
           (aend - t0) / 1e3, bs[0], bs[N / 10], bs[N / 2], bs[9 * N / 10], bs[N - 1]);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
