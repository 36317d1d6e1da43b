// Probe: CUDA multicast (NVLS) objects on this box -- attributes, a 1-device
// multicast object bound to a buffer, multimem.st and multimem.ld_reduce
// through the multicast address.  Build: nvcc -arch=sm_100a mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); \
  printf("FAIL %s: %s\n", #x, s); return 1; } } while (0)

__global__ void st_kernel(float* mc, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    float v = (float)i * 0.5f;
    asm volatile("multimem.st.global.f32 [%0], %1;" :: "l"(mc + i), "f"(v) : "memory");
  }
}
__global__ void ldred_kernel(const float* mc, float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    float v;
    asm volatile("multimem.ld_reduce.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc + i) : "memory");
    out[i] = v;
  }
}

int main() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  int mcs = -1, fab = -1, vmm = -1;
  cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, dev);
  printf("multicast_supported=%d fabric_handles=%d vmm=%d\n", mcs, fab, vmm);
  cudaFree(0);
  if (mcs != 1) return 0;
  const size_t n = 1 << 20, bytes = n * sizeof(float);
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  size_t gran = 0;
  CUmemGenericAllocationHandle mch;
  const CUmemAllocationHandleType types[3] = {(CUmemAllocationHandleType)0, CU_MEM_HANDLE_TYPE_FABRIC,
                                              CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR};
  int ok = 0;
  for (int k = 0; k < 3 && !ok; ++k) {
    mp.handleTypes = types[k];
    if (cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS) { printf("gran fail type %d\n", (int)types[k]); continue; }
    mp.size = ((bytes + gran - 1) / gran) * gran;
    CUresult r = cuMulticastCreate(&mch, &mp);
    const char* es; cuGetErrorString(r, &es);
    printf("handle type %d: granularity %zu create: %s\n", (int)types[k], gran, es);
    ok = (r == CUDA_SUCCESS);
  }
  if (!ok) return 1;
  CK(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  size_t ugran = 0;
  CK(cuMemGetAllocationGranularity(&ugran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  size_t usize = ((mp.size + ugran - 1) / ugran) * ugran;
  CUmemGenericAllocationHandle uh;
  CK(cuMemCreate(&uh, usize, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, uh, 0, usize, 0));
  CUdeviceptr uva, mcva;
  CK(cuMemAddressReserve(&uva, usize, 0, 0, 0));
  CK(cuMemMap(uva, usize, 0, uh, 0));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = 0;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uva, usize, &acc, 1));
  CK(cuMemAddressReserve(&mcva, mp.size, 0, 0, 0));
  CK(cuMemMap(mcva, mp.size, 0, mch, 0));
  CK(cuMemSetAccess(mcva, mp.size, &acc, 1));
  st_kernel<<<(n + 255) / 256, 256>>>((float*)mcva, (int)n);
  float* out;
  cudaMalloc(&out, bytes);
  ldred_kernel<<<(n + 255) / 256, 256>>>((const float*)mcva, out, (int)n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernels: %s\n", cudaGetErrorString(e));
  float h[4], u[4];
  cudaMemcpy(h, out + 1000, sizeof(h), cudaMemcpyDeviceToHost);
  cudaMemcpy(u, (void*)(uva + 1000 * 4), sizeof(u), cudaMemcpyDeviceToHost);
  printf("ld_reduce[1000..] = %g %g %g %g ; unicast view = %g %g %g %g (expect 500 500.5 501 501.5)\n",
         h[0], h[1], h[2], h[3], u[0], u[1], u[2], u[3]);
  return 0;
}
