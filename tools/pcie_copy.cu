// pcie_copy.cu -- copy kernels for tools/pcie_bw.py: device <-> mapped pinned host memory
// through the SMs (zero-copy) with 2/4/8/16-byte accesses, to compare with the copy engines.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o build/libpcie_copy.so tools/pcie_copy.cu
#include <cuda_runtime.h>
#include <cstdint>
template <typename T> __global__ void copyT(const T *__restrict__ src, T *__restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) dst[i] = src[i];
}
extern "C" int zc_copyw(const void *src, void *dst, size_t bytes, int grid, int block, int w, void *stream) {
    if (w == 2) copyT<<<grid, block, 0, (cudaStream_t)stream>>>((const uint16_t *)src, (uint16_t *)dst, bytes / 2);
    else if (w == 4) copyT<<<grid, block, 0, (cudaStream_t)stream>>>((const uint32_t *)src, (uint32_t *)dst, bytes / 4);
    else if (w == 8) copyT<<<grid, block, 0, (cudaStream_t)stream>>>((const uint2 *)src, (uint2 *)dst, bytes / 8);
    else copyT<<<grid, block, 0, (cudaStream_t)stream>>>((const uint4 *)src, (uint4 *)dst, bytes / 16);
    return (int)cudaGetLastError();
}
extern "C" int zc_engines() { cudaDeviceProp p; cudaGetDeviceProperties(&p, 0); return p.asyncEngineCount * 1000 + p.canMapHostMemory * 100 + p.unifiedAddressing; }
