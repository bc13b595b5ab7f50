// Dependent-load latency: shared memory reached through a generic pointer (LD) vs an
// explicit shared-space load (LDS).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
__global__ void chase(int* out, int hops, int* gp_in, int mode) {
  __shared__ int a[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) a[i] = (i * 97 + 13) & 4095;
  __syncthreads();
  // opaque generic pointer into shared memory: round-trip it through global memory
  if (threadIdx.x == 0) reinterpret_cast<int**>(gp_in)[0] = a;
  __syncthreads();
  int* gp = reinterpret_cast<int* volatile*>(gp_in)[0];
  int s = threadIdx.x;
  long long t0 = clock64();
  if (mode == 0) {
    for (int h = 0; h < hops; ++h) s = gp[s];
  } else {
    for (int h = 0; h < hops; ++h) s = a[s];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (int)((t1 - t0) / hops); out[1] = s; }
}
int main() {
  int* d; cudaMalloc(&d, 8);
  int* pbuf; cudaMalloc(&pbuf, 16);
  int h[2];
  for (int mode = 0; mode < 2; ++mode) {
    chase<<<1, 32>>>(d, 4096, pbuf, mode);
    chase<<<1, 32>>>(d, 4096, pbuf, mode);
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("%s: %d cycles per dependent load\n", mode == 0 ? "generic LD -> smem" : "LDS", h[0]);
  }
  return 0;
}
