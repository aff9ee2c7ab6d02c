#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s -> %d %s\n", #x, (int)r, s); return 1; } } while (0)
__global__ void k(unsigned int* mc, float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    float v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc + i) : "memory");
    out[i] = v;
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" :: "l"(mc + i), "f"(v * 2.0f) : "memory");
  }
}
int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  int mcs = -1; CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  printf("MULTICAST_SUPPORTED=%d\n", mcs);
  int ndev; cudaGetDeviceCount(&ndev); printf("devices=%d\n", ndev);
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  if (!mcs) return 0;
  CUmulticastObjectProp prop = {};
  prop.numDevices = 1; prop.handleTypes = CU_MEM_HANDLE_TYPE_NONE; prop.size = 2 << 20;
  const char* ht = getenv("HT"); if (ht) prop.handleTypes = (unsigned long long)atoi(ht);
  const char* nd = getenv("ND"); if (nd) prop.numDevices = atoi(nd);
  size_t gran = 0; CK(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  printf("gran=%zu\n", gran);
  prop.size = (prop.size + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle mch; CK(cuMulticastCreate(&mch, &prop));
  CK(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {}; ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = 0;
  ap.requestedHandleTypes = (CUmemAllocationHandleType)prop.handleTypes;
  CUmemGenericAllocationHandle ph; CK(cuMemCreate(&ph, prop.size, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, ph, 0, prop.size, 0));
  CUdeviceptr uc, mc;
  CK(cuMemAddressReserve(&uc, prop.size, gran, 0, 0)); CK(cuMemMap(uc, prop.size, 0, ph, 0));
  CUmemAccessDesc acc = {}; acc.location = ap.location; acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, prop.size, &acc, 1));
  CK(cuMemAddressReserve(&mc, prop.size, gran, 0, 0)); CK(cuMemMap(mc, prop.size, 0, mch, 0));
  CK(cuMemSetAccess(mc, prop.size, &acc, 1));
  int n = 1024; float h[1024]; for (int i = 0; i < n; ++i) h[i] = i;
  cudaMemcpy((void*)uc, h, n * 4, cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, n * 4);
  k<<<4, 256>>>((unsigned int*)mc, out, n);
  cudaError_t e = cudaDeviceSynchronize(); printf("kernel: %s\n", cudaGetErrorString(e));
  float o[1024], u[1024]; cudaMemcpy(o, out, n * 4, cudaMemcpyDeviceToHost); cudaMemcpy(u, (void*)uc, n * 4, cudaMemcpyDeviceToHost);
  printf("o[5]=%f u[5]=%f o[1000]=%f u[1000]=%f\n", o[5], u[5], o[1000], u[1000]);
  return 0;
}
