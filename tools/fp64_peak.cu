// fp64 ceiling probe on B200: DMMA (mma.sync f64 shapes) vs DFMA, register-only.
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void dmma_loop(double *out, int iters) {
  double a[8], b[4], c[8][4];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-9 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - i * 1e-9;
  for (int t = 0; t < 8; ++t)
    for (int i = 0; i < 4; ++i) c[t][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {  // 8 independent accumulators per warp
      if (SHAPE == 4)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      else if (SHAPE == 8)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
  for (int t = 0; t < 8; ++t)
    for (int i = 0; i < 4; ++i) s += c[t][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_loop(double *out, int iters) {
  double x[16];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
  const double m = 0.999999, a = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], m, a);
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
double run(F f, int blocks, int threads, double flops) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return flops / (ms * 1e-3) / 1e12;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  cudaMalloc(&out, 1 << 26);
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    int blocks = sms * 4, threads = 32 * warps;
    double n = (double)blocks * warps * iters * 8;
    printf("warps/blk %2d  m16n8k4 %.2f TF  m16n8k8 %.2f TF  m16n8k16 %.2f TF\n", warps,
           run([&] { dmma_loop<4><<<blocks, threads>>>(out, iters); }, blocks, threads, n * 2 * 16 * 8 * 4),
           run([&] { dmma_loop<8><<<blocks, threads>>>(out, iters); }, blocks, threads, n * 2 * 16 * 8 * 8),
           run([&] { dmma_loop<16><<<blocks, threads>>>(out, iters / 2); }, blocks, threads, n / 2 * 2 * 16 * 8 * 16));
  }
  int blocks = sms * 8, threads = 256;
  printf("dfma %.2f TF\n", run([&] { dfma_loop<<<blocks, threads>>>(out, iters); }, blocks, threads,
                                 (double)blocks * threads * iters * 16 * 2));
  return 0;
}
