// Streaming ceilings on B200: copy / read / triad with 8 B and 16 B accesses.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void copy8(const double* __restrict__ a, double* __restrict__ b, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void copy16(const double2* __restrict__ a, double2* __restrict__ b, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void add3_8(const double* __restrict__ a, const double* __restrict__ c, double* __restrict__ b, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i] + c[i];
}
__global__ void add3_16(const double2* __restrict__ a, const double2* __restrict__ c, double2* __restrict__ b, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    double2 x = a[i], y = c[i]; b[i] = make_double2(x.x + y.x, x.y + y.y); }
}
template <int U>
__global__ void add3_8u(const double* __restrict__ a, const double* __restrict__ c, double* __restrict__ b, long n) {
  long base = (blockIdx.x * (long)blockDim.x) * U + threadIdx.x;
  double x[U], y[U];
#pragma unroll
  for (int t = 0; t < U; ++t) { long i = base + (long)t * blockDim.x; x[t] = i < n ? a[i] : 0; y[t] = i < n ? c[i] : 0; }
#pragma unroll
  for (int t = 0; t < U; ++t) { long i = base + (long)t * blockDim.x; if (i < n) b[i] = x[t] + y[t]; }
}
__global__ void read8(const double* __restrict__ a, double* out, long n) {
  double s = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) s += a[i];
  if (s == 1.2345) out[0] = s;
}
int main() {
  long n = 1L << 27;  // 1 GiB of doubles
  double *a, *b, *c, *o;
  cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8); cudaMalloc(&c, n * 8); cudaMalloc(&o, 8);
  cudaMemset(a, 0, n * 8); cudaMemset(b, 0, n * 8); cudaMemset(c, 0, n * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](const char* name, auto fn, double bytes) {
    fn(); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) fn();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-22s %8.1f GB/s\n", name, bytes * 10 / (ms * 1e-3) / 1e9);
  };
  int g = sms * 8;
  run("copy8 gridstride", [&] { copy8<<<g, 256>>>(a, b, n); }, 16.0 * n);
  run("copy8 full grid", [&] { copy8<<<(n + 255) / 256, 256>>>(a, b, n); }, 16.0 * n);
  run("copy16 gridstride", [&] { copy16<<<g, 256>>>((double2*)a, (double2*)b, n / 2); }, 16.0 * n);
  run("add3_8 gridstride", [&] { add3_8<<<g, 256>>>(a, c, b, n); }, 24.0 * n);
  run("add3_8 full", [&] { add3_8<<<(n + 255) / 256, 256>>>(a, c, b, n); }, 24.0 * n);
  run("add3_16 gridstride", [&] { add3_16<<<g, 256>>>((double2*)a, (double2*)c, (double2*)b, n / 2); }, 24.0 * n);
  run("add3_8 unroll4", [&] { add3_8u<4><<<(n + 1023) / 1024, 256>>>(a, c, b, n); }, 24.0 * n);
  run("add3_8 unroll8", [&] { add3_8u<8><<<(n + 2047) / 2048, 256>>>(a, c, b, n); }, 24.0 * n);
  run("read8 gridstride", [&] { read8<<<g, 256>>>(a, o, n); }, 8.0 * n);
  return 0;
}
