// Microbenchmark: dependent-chain latency of FP64 FMA / sqrt / div / rsqrt
// and of shuffles, smem round trips and __syncthreads on this GPU (clock64).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double seed, int iters) {
  double x = seed + threadIdx.x * 1e-9, y = 1.0000001, z = 0.9999999;
  __shared__ double sm[64];
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, y, z);
  t1 = clock64();
  cyc[0] = (t1 - t0) / iters;
  // sqrt chain
  double s = x + 2.0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) s = sqrt(s) + 1.0;
  t1 = clock64();
  cyc[1] = (t1 - t0) / iters;
  // div chain
  double d = s;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) d = 3.0 / (d + 1.0);
  t1 = clock64();
  cyc[2] = (t1 - t0) / iters;
  // rsqrt chain
  double r = d + 1.0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) r = rsqrt(r) + 1.0;
  t1 = clock64();
  cyc[3] = (t1 - t0) / iters;
  // shuffle chain (double)
  double q = r;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) q = __shfl_sync(0xffffffffu, q, (threadIdx.x + 1) & 31) + 1.0;
  t1 = clock64();
  cyc[4] = (t1 - t0) / iters;
  // smem store -> load round trip
  double m = q;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    sm[threadIdx.x] = m;
    __syncwarp();
    m = sm[(threadIdx.x + 1) & 31] + 1.0;
  }
  t1 = clock64();
  cyc[5] = (t1 - t0) / iters;
  // __syncthreads (block of blockDim threads)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  t1 = clock64();
  cyc[6] = (t1 - t0) / iters;
  // DADD chain
  double a = m;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) a = a + z;
  t1 = clock64();
  cyc[7] = (t1 - t0) / iters;
  out[threadIdx.x] = x + s + d + r + q + m + a;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  const char* names[] = {"dfma", "sqrt+add", "div+add", "rsqrt+add", "shfl.f64+add", "sts/lds+add", "syncthreads",
                         "dadd"};
  for (int threads : {32, 256, 1024}) {
    lat<<<1, threads>>>(out, cyc, 1.0, 1000);
    lat<<<1, threads>>>(out, cyc, 1.0, 1000);
    cudaDeviceSynchronize();
    printf("threads=%d:", threads);
    for (int i = 0; i < 8; ++i) printf(" %s=%lld", names[i], cyc[i]);
    printf("\n");
  }
  return 0;
}
