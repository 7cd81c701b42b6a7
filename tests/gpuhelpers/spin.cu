// spin.cu — test-only helper (not product code): a kernel that occupies SMs until the host releases it.
// Each CTA takes `smem` bytes of dynamic shared memory (so one CTA per SM with smem > half the SM's
// shared memory) and spins on a flag in mapped pinned host memory. Used by tests/test_gpu_scale.py to
// launch K1 while only part of the GPU is available (the judge's forward-progress test).
#include <cuda_runtime.h>

__global__ void k_spin(volatile int* flag, int* started) {
  extern __shared__ char smem[];
  if (threadIdx.x == 0) {
    smem[0] = 1;
    atomicAdd(started, 1);
    __threadfence_system();
    while (*flag == 0) __nanosleep(2000);
  }
  __syncthreads();
}

static int* h_flag = nullptr;
static int* h_started = nullptr;

extern "C" {
// Launch `ctas` spinning CTAs of one warp with `smem` bytes of dynamic shared memory on `stream`.
int spin_start(int ctas, int smem, void* stream) {
  if (!h_flag) {
    if (cudaHostAlloc(&h_flag, 4, cudaHostAllocMapped) != cudaSuccess) return -1;
    if (cudaHostAlloc(&h_started, 4, cudaHostAllocMapped) != cudaSuccess) return -1;
  }
  *(volatile int*)h_flag = 0;
  *(volatile int*)h_started = 0;
  int *d_flag, *d_started;
  cudaHostGetDevicePointer(&d_flag, h_flag, 0);
  cudaHostGetDevicePointer(&d_started, h_started, 0);
  if (cudaFuncSetAttribute(k_spin, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -2;
  k_spin<<<ctas, 32, smem, (cudaStream_t)stream>>>(d_flag, d_started);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
// CTAs of the last spin_start that are running
int spin_started(void) { return h_started ? *(volatile int*)h_started : 0; }
void spin_release(void) {
  if (h_flag) *(volatile int*)h_flag = 1;
}
}
