// Per-SM throughput of ex2.approx.ftz.f32 (MUFU) and fma.rn.f32x2 (FFMA2) on sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/sfu_rate scripts/sfu_rate.cu && scripts/sfu_rate
// One CTA per SM, W warps, 8 independent chains per thread; prints results per SM per clock.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k_rate(int iters, float* out, long long* cyc) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = 0.001f * (threadIdx.x + j);
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
      } else {
        unsigned long long p;
        asm volatile("mov.b64 %0, {%1, %2};" : "=l"(p) : "f"(a[j]), "f"(a[(j + 1) & 7]));
        asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(p));
        float x, y;
        asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(p));
        a[j] = x + 0.f * y;
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  const int iters = 4096;
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  for (int op = 0; op < 2; ++op) {
    for (int warps = 2; warps <= 32; warps *= 2) {
      const int th = 32 * warps;
      for (int rep = 0; rep < 2; ++rep) {
        if (op == 0) k_rate<0><<<148, th>>>(iters, out, cyc);
        else k_rate<1><<<148, th>>>(iters, out, cyc);
      }
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
      const double ops = (double)iters * 8 * th;  // thread-level ops per SM
      printf("%s warps %2d: %.2f thread-ops per SM per clock\n", op == 0 ? "ex2.approx " : "fma.f32x2  ", warps,
             ops / (double)c);
    }
  }
  return 0;
}
