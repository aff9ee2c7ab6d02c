// Co-residency probe 2: the fused GEMM's launch pattern -- spinner forked from the
// GEMM stream by an event, GEMM launched with cudaLaunchKernelEx (cluster 2,
// programmatic stream serialization attribute = 0) and calling griddepcontrol.wait.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
__device__ unsigned int g_flag;
__device__ unsigned long long g_seen;
__global__ void spinner() {
  if (threadIdx.x == 0) {
    unsigned long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      unsigned int v; asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(&g_flag) : "memory");
      unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (v) { if (blockIdx.x == 0) g_seen = t - t0; break; }
      if (t - t0 > 2000000000ull) { if (blockIdx.x == 0) g_seen = 0; break; }
      __nanosleep(256);
    }
  }
  __syncthreads();
}
__global__ void __launch_bounds__(192, 1) big(int use_gdc) {
  extern __shared__ char sm[];
  if (use_gdc) asm volatile("griddepcontrol.wait;" ::: "memory");
  sm[threadIdx.x] = 1;
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(&g_flag), "r"(1u) : "memory");
}
int main(int argc, char** argv) {
  int use_gdc = atoi(argv[1]), use_ex = atoi(argv[2]), fork = atoi(argv[3]), torch_like = argc > 4 ? atoi(argv[4]) : 0;
  int bigsmem = 202 * 1024;
  cudaFuncSetAttribute(big, cudaFuncAttributeMaxDynamicSharedMemorySize, bigsmem);
  cudaStream_t st, side; cudaEvent_t ev;
  if (torch_like) cudaStreamCreate(&st); else cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  unsigned int z = 0; cudaMemcpyToSymbol(g_flag, &z, 4);
  if (fork) { cudaEventRecord(ev, st); cudaStreamWaitEvent(side, ev, 0); }
  spinner<<<12, 256, 0, side>>>();
  if (use_ex) {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(16); cfg.blockDim = dim3(192); cfg.dynamicSmemBytes = bigsmem; cfg.stream = st;
    cudaLaunchAttribute at[2]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[1].val.programmaticStreamSerializationAllowed = 0;
    cfg.attrs = at; cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, big, use_gdc); if (e) printf("launch: %s\n", cudaGetErrorString(e));
  } else big<<<16, 192, bigsmem, st>>>(use_gdc);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long seen; cudaMemcpyFromSymbol(&seen, g_seen, 8);
  printf("gdc=%d ex=%d fork=%d torch_like=%d: %s; spinner saw the flag after %llu ns (0 = never)\n", use_gdc, use_ex, fork, torch_like, cudaGetErrorString(e), seen);
  return 0;
}
