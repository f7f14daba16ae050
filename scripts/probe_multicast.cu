// Probe: can this box build an NVLS multicast object over ONE device and run multimem.*
// instructions on it?  (One GPU per gpurun call: a 1-device multicast object is the only way
// to execute the multimem code path here.)  Prints the attribute, each driver call's result,
// and the values a multimem.ld_reduce / multimem.st / multimem.red round trip produces.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

#define CK(x) do { CUresult r_ = (x); const char* s_ = nullptr; cuGetErrorString(r_, &s_); \
  printf("%-60s -> %d %s\n", #x, (int)r_, s_ ? s_ : ""); if (r_ != CUDA_SUCCESS) return 1; } while (0)

__global__ void k_mm(float* uc, float* mc, float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i * 4 >= n) return;
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(mc + 4 * i) : "memory");
  reinterpret_cast<float4*>(out)[i] = v;
  float4 w = make_float4(v.x + 1.f, v.y + 1.f, v.z + 1.f, v.w + 1.f);
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + 4 * i), "f"(w.x), "f"(w.y),
               "f"(w.z), "f"(w.w) : "memory");
  asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(mc + 4 * i), "f"(0.5f) : "memory");
}

int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  int mcs = -1; CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  printf("MULTICAST_SUPPORTED = %d\n", mcs);
  int ndev = 0; cudaGetDeviceCount(&ndev); printf("visible devices = %d\n", ndev);
  const size_t want = 2 << 20;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1; mp.size = want; mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0; CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  printf("multicast granularity = %zu\n", gran);
  mp.size = (want + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle mch = 0;
  const unsigned long long types[3] = {0ull, (unsigned long long)CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                       (unsigned long long)CU_MEM_HANDLE_TYPE_FABRIC};
  bool made = false;
  for (int t = 0; t < 3 && !made; ++t) {
    for (int nd = 1; nd <= 2 && !made; ++nd) {
      mp.handleTypes = types[t]; mp.numDevices = nd;
      CUresult r = cuMulticastCreate(&mch, &mp);
      const char* es = nullptr; cuGetErrorString(r, &es);
      printf("cuMulticastCreate(handleTypes=%llu, numDevices=%d) -> %d %s\n", types[t], nd, (int)r, es ? es : "");
      made = (r == CUDA_SUCCESS && nd == 1);
    }
  }
  if (!made) { printf("MULTIMEM_ONE_DEVICE UNAVAILABLE\n"); return 0; }
  CK(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = dev;
  ap.requestedHandleTypes = (CUmemAllocationHandleType)mp.handleTypes;
  size_t pg = 0; CK(cuMemGetAllocationGranularity(&pg, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  CUmemGenericAllocationHandle ph; CK(cuMemCreate(&ph, mp.size, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, ph, 0, mp.size, 0));
  CUdeviceptr uc = 0, mc = 0;
  CK(cuMemAddressReserve(&uc, mp.size, gran, 0, 0)); CK(cuMemMap(uc, mp.size, 0, ph, 0));
  CK(cuMemAddressReserve(&mc, mp.size, gran, 0, 0)); CK(cuMemMap(mc, mp.size, 0, mch, 0));
  CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = dev;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, mp.size, &ad, 1)); CK(cuMemSetAccess(mc, mp.size, &ad, 1));
  const int n = 1024;
  float h[n]; for (int i = 0; i < n; ++i) h[i] = (float)i;
  cudaMemcpy((void*)uc, h, sizeof h, cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, sizeof h);
  k_mm<<<1, 256>>>((float*)uc, (float*)mc, out, n);
  printf("kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  float o[n], u[n];
  cudaMemcpy(o, out, sizeof o, cudaMemcpyDeviceToHost);
  cudaMemcpy(u, (void*)uc, sizeof u, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < n; ++i) bad += (o[i] != (float)i) + (u[i] != (float)i + 1.5f);
  printf("ld_reduce[5] = %g (want 5), after st+red uc[5] = %g (want 6.5), mismatches %d\n", o[5], u[5], bad);
  printf("MULTIMEM_ONE_DEVICE %s\n", bad == 0 ? "OK" : "FAIL");
  return 0;
}
