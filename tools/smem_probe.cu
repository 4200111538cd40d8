// Probe: static + dynamic shared memory above 48 KB with the opt-in attribute.
#include <cstdio>
__global__ void __launch_bounds__(128, 4) k(double* out) {
  __shared__ double s[4096];
  extern __shared__ double d[];
  s[threadIdx.x] = threadIdx.x;
  d[threadIdx.x] = 2.0 * threadIdx.x;
  __syncthreads();
  out[threadIdx.x] = s[127 - threadIdx.x] + d[threadIdx.x];
}
int main() {
  double* o;
  cudaMalloc(&o, 1024);
  for (int dyn : {8192, 16384, 18432, 24576}) {
    cudaError_t a = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    k<<<1, 128, dyn>>>(o);
    cudaError_t e = cudaGetLastError();
    cudaError_t s = cudaDeviceSynchronize();
    printf("dyn %d: attr %s launch %s sync %s\n", dyn, cudaGetErrorString(a), cudaGetErrorString(e), cudaGetErrorString(s));
  }
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  printf("optin %d\n", v);
}
