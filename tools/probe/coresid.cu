// Co-residency probe: can a 202 KB-smem, cluster-2, 192-thread persistent kernel
// (the fused GEMM's footprint) run next to small spinning kernels?
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
__device__ unsigned long long g_t[4096];
__device__ volatile int g_go;
__global__ void spinner(unsigned long long ns, int wait_flag) {
  unsigned long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (threadIdx.x == 0) {
    while (true) {
      unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (wait_flag ? g_go != 0 : (t - t0 > ns)) break;
      if (t - t0 > 3000000000ull) { printf("spinner timeout\n"); break; }
      __nanosleep(200);
    }
  }
  __syncthreads();
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1) big(int n) {
  extern __shared__ char sm[];
  sm[threadIdx.x] = 1;
  unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0) g_t[blockIdx.x] = t;
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd((int*)&g_t[4000], 1) == n - 1) g_go = 1;
}
int main(int argc, char** argv) {
  int dyn_spin = argc > 1 ? atoi(argv[1]) : 0;
  int carve = argc > 2 ? atoi(argv[2]) : -1;
  int wait_flag = argc > 3 ? atoi(argv[3]) : 1;
  int ctas = argc > 4 ? atoi(argv[4]) : 32;
  int bigsmem = 202 * 1024;
  cudaFuncSetAttribute(big, cudaFuncAttributeMaxDynamicSharedMemorySize, bigsmem);
  if (carve >= 0) cudaFuncSetAttribute(spinner, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
  if (dyn_spin > 48 * 1024) cudaFuncSetAttribute(spinner, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_spin);
  cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  int zero = 0; cudaMemcpyToSymbol(g_go, &zero, 4);
  spinner<<<ctas, 256, dyn_spin, s1>>>(200000000ull, wait_flag);
  big<<<148, 192, bigsmem, s2>>>(148);
  cudaError_t e = cudaDeviceSynchronize();
  int go; cudaMemcpyFromSymbol(&go, g_go, 4);
  printf("dyn_spin=%d carve=%d ctas=%d wait_flag=%d: %s, big finished while spinner waited: %s\n", dyn_spin, carve, ctas, wait_flag,
         cudaGetErrorString(e), go ? "yes" : "no");
  return 0;
}
