// Micro-benchmark: FP64 add / mul / div issue rates on the B200 (sm_100a).
// Used once to fill the FP64 roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, double a, double b, int iters) {
  double x0 = a + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) { x0 = __dadd_rn(x0, b); x1 = __dadd_rn(x1, b); x2 = __dadd_rn(x2, b); x3 = __dadd_rn(x3, b);
                   x4 = __dadd_rn(x4, b); x5 = __dadd_rn(x5, b); x6 = __dadd_rn(x6, b); x7 = __dadd_rn(x7, b); }
    if (OP == 1) { x0 = __dmul_rn(x0, b); x1 = __dmul_rn(x1, b); x2 = __dmul_rn(x2, b); x3 = __dmul_rn(x3, b);
                   x4 = __dmul_rn(x4, b); x5 = __dmul_rn(x5, b); x6 = __dmul_rn(x6, b); x7 = __dmul_rn(x7, b); }
    if (OP == 2) { x0 = __fma_rn(x0, b, a); x1 = __fma_rn(x1, b, a); x2 = __fma_rn(x2, b, a); x3 = __fma_rn(x3, b, a);
                   x4 = __fma_rn(x4, b, a); x5 = __fma_rn(x5, b, a); x6 = __fma_rn(x6, b, a); x7 = __fma_rn(x7, b, a); }
    if (OP == 3) { x0 = __ddiv_rn(b, x0); x1 = __ddiv_rn(b, x1); x2 = __ddiv_rn(b, x2); x3 = __ddiv_rn(b, x3);
                   x4 = __ddiv_rn(b, x4); x5 = __ddiv_rn(b, x5); x6 = __ddiv_rn(b, x6); x7 = __ddiv_rn(b, x7); }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
template <int OP> void run(const char* name, double* out, int iters) {
  cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
  int blocks = 148 * 8, threads = 256;
  k<OP><<<blocks, threads>>>(out, 1.0000001, 0.9999999, 16);
  cudaEventRecord(s);
  k<OP><<<blocks, threads>>>(out, 1.0000001, 0.9999999, iters);
  cudaEventRecord(e); cudaEventSynchronize(e);
  float ms; cudaEventElapsedTime(&ms, s, e);
  double ops = double(blocks) * threads * iters * 8;
  printf("%s: %.3f ms  %.3f Gop/s (lane-ops)\n", name, ms, ops / ms / 1e6);
}
int main() {
  double* out; cudaMalloc(&out, 148 * 8 * 256 * sizeof(double));
  run<0>("dadd", out, 4096); run<1>("dmul", out, 4096); run<2>("dfma", out, 4096); run<3>("ddiv", out, 512);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock kHz %d\n", clk);
  return 0;
}
