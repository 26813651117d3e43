// Half-sweep access pattern without the arithmetic, real field layout
// [c][j][k][pitch] (pitch 520 doubles, 1024^2 x 128).  Variants of tile
// order / per-thread batching, to separate DRAM-pattern from compute costs.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NX = 1024, NY = 1024, NZ = 128, OFF = 4, PITCH = 520;
constexpr long long JS = (long long)NZ * PITCH, CS = (long long)(NY + 2) * JS;
__device__ __forceinline__ long long at(int c, int k, int j, int h) {
  return c * CS + (long long)(j + 1) * JS + (long long)k * PITCH + OFF + h;
}
template <int B>
__global__ void __launch_bounds__(256) tilewalk(const double* __restrict__ f, double* __restrict__ u, int c, int ntiles) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5; int o = c ^ 1;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int j = t / 16, h = (t % 16) * 32 + lane, k0 = w * 16;
    double acc[16];
    for (int b = 0; b < 16; b += B) {
      double a[B], bb[B], cc[B], d[B];
#pragma unroll
      for (int e = 0; e < B; ++e) { int k = k0 + b + e;
        a[e] = f[at(c, k, j, h)]; bb[e] = u[at(o, k, j, h)]; cc[e] = u[at(o, k, j - 1, h)]; d[e] = u[at(o, k, j + 1, h)]; }
#pragma unroll
      for (int e = 0; e < B; ++e) acc[b + e] = a[e] + bb[e] + cc[e] + d[e];
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) u[at(c, k0 + e, j, h)] = acc[e];
  }
}
template <int B>
__global__ void __launch_bounds__(256) tilewalk_sync(const double* __restrict__ f, double* __restrict__ u, int c, int ntiles) {
  __shared__ double x[8][32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5; int o = c ^ 1;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int j = t / 16, h = (t % 16) * 32 + lane, k0 = w * 16;
    double acc[16];
    for (int b = 0; b < 16; b += B) {
      double a[B], bb[B], cc[B], d[B];
#pragma unroll
      for (int e = 0; e < B; ++e) { int k = k0 + b + e;
        a[e] = f[at(c, k, j, h)]; bb[e] = u[at(o, k, j, h)]; cc[e] = u[at(o, k, j - 1, h)]; d[e] = u[at(o, k, j + 1, h)]; }
#pragma unroll
      for (int e = 0; e < B; ++e) acc[b + e] = a[e] + bb[e] + cc[e] + d[e];
    }
    x[w][lane] = acc[15];
    __syncthreads();
    double G = 0; for (int s = 0; s < w; ++s) G = G * 0.5 + x[s][lane];
    acc[0] += G;
    __syncthreads();
    x[w][lane] = acc[0];
    __syncthreads();
    double X = 0; for (int s = 7; s > w; --s) X = X * 0.5 + x[s][lane];
#pragma unroll
    for (int e = 0; e < 16; ++e) u[at(c, k0 + e, j, h)] = acc[e] + X;
    __syncthreads();
  }
}
__global__ void slab(const double* __restrict__ f, double* __restrict__ u, int c) {
  int h = blockIdx.x * 32 + (threadIdx.x & 31); int j = blockIdx.z * 8 + (threadIdx.x >> 5); int k = blockIdx.y; int o = c ^ 1;
  u[at(c, k, j, h)] = f[at(c, k, j, h)] + u[at(o, k, j, h)] + u[at(o, k, j - 1, h)] + u[at(o, k, j + 1, h)];
}
__global__ void __launch_bounds__(256) tileread(const double* __restrict__ f, const double* __restrict__ u, double* out, int c, int ntiles) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5; int o = c ^ 1; double s = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int j = t / 16, h = (t % 16) * 32 + lane, k0 = w * 16;
    for (int b = 0; b < 16; b += 4) {
      double a[4], bb[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) { int k = k0 + b + e; a[e] = f[at(c, k, j, h)]; bb[e] = u[at(o, k, j, h)]; }
#pragma unroll
      for (int e = 0; e < 4; ++e) s += a[e] * bb[e];
    }
  }
  if (s == 1.2345) out[0] = s;
}
int main() {
  size_t n = 2 * CS;
  double *f, *u, *o; cudaMalloc(&f, n * 8); cudaMalloc(&u, n * 8); cudaMalloc(&o, 8);
  cudaMemset(f, 0, n * 8); cudaMemset(u, 0, n * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double alg = 12.0 * NX * NY * NZ;
  auto run = [&](const char* name, auto fn, double bytes) {
    fn(); cudaDeviceSynchronize(); cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) fn();
    cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %8.1f us  %7.1f GB/s\n", name, ms * 100, bytes * 10 / (ms * 1e-3) / 1e9);
  };
  int ntiles = 16 * NY;
  for (int g : {296, 444, 592, 1184}) {
    char nm[64]; snprintf(nm, 64, "tilewalk B4 grid %d", g);
    run(nm, [&] { tilewalk<4><<<g, 256>>>(f, u, 0, ntiles); }, alg);
  }
  run("tilewalk_sync B4 grid 296", [&] { tilewalk_sync<4><<<296, 256>>>(f, u, 0, ntiles); }, alg);
  run("tilewalk_sync B4 grid 444", [&] { tilewalk_sync<4><<<444, 256>>>(f, u, 0, ntiles); }, alg);
  run("tilewalk B8 grid 296", [&] { tilewalk<8><<<296, 256>>>(f, u, 0, ntiles); }, alg);
  run("tilewalk B2 grid 592", [&] { tilewalk<2><<<592, 256>>>(f, u, 0, ntiles); }, alg);
  run("slab (h,k,j) 1/thread", [&] { slab<<<dim3(16, NZ, NY / 8), 256>>>(f, u, 0); }, alg);
  run("tileread f+u_o (2/3)", [&] { tileread<<<592, 256>>>(f, u, o, 0, ntiles); }, 8.0 * NX * NY * NZ);
  return 0;
}
