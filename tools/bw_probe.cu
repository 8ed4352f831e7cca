// Practical HBM roofline for the evaluate kernel's traffic pattern: per
// candidate read one 8-byte word, write one reason byte and one f64 (17 B),
// with no compute. Compares against a plain 16 B/thread copy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bw_probe tools/bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void rw17(const uint4* __restrict__ in, uint32_t* __restrict__ reason, uint4* __restrict__ raw, int64_t n4) {
  // thread handles 4 candidates: 32 B in, 4 B + 32 B out
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 a = in[2 * i], b = in[2 * i + 1];
    uint32_t r = (a.x ^ b.y) & 0x01010101u;  // keep the loads live
    reason[i] = r;
    raw[2 * i] = make_uint4(r & 0, 0, 0, 0);
    raw[2 * i + 1] = make_uint4(0, 0, 0, 0);
  }
}
// same, raw stores warp-contiguous (lane-strided 16 B)
__global__ void rw17c(const uint4* __restrict__ in, uint32_t* __restrict__ reason, uint4* __restrict__ raw, int64_t n4) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w0 = i - lane;  // warp's first thread index
    uint4 a = in[2 * w0 + lane], b = in[2 * w0 + 32 + lane];
    uint32_t r = (a.x ^ b.y) & 0x01010101u;
    reason[i] = r;
    raw[2 * w0 + lane] = make_uint4(r & 0, 0, 0, 0);
    raw[2 * w0 + 32 + lane] = make_uint4(0, 0, 0, 0);
  }
}
__global__ void copy16(const uint4* __restrict__ in, uint4* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) out[i] = in[i];
}
__global__ void read8(const uint4* __restrict__ in, uint32_t* __restrict__ sink, int64_t n) {
  uint32_t acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) acc ^= in[i].x;
  if (acc == 0x12345678u) sink[0] = acc;
}
__global__ void write9(uint32_t* __restrict__ reason, uint4* __restrict__ raw, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    reason[i] = 0;
    raw[2 * i] = make_uint4(0, 0, 0, 0);
    raw[2 * i + 1] = make_uint4(0, 0, 0, 0);
  }
}

int main() {
  const int64_t n = 1ll << 27;  // candidates
  uint4 *in, *raw, *out;
  uint32_t* reason;
  cudaMalloc(&in, n * 8);
  cudaMalloc(&raw, n * 8);
  cudaMalloc(&reason, n);
  cudaMalloc(&out, n * 8);
  cudaMemset(in, 1, n * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 148;
  auto run = [&](const char* name, double bytes, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    float best = 1e9, sum = 0;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
      sum += ms;
    }
    printf("%-34s best %.3f ms  %.0f GB/s   mean %.0f GB/s\n", name, best, bytes / best / 1e6, bytes / (sum / 10) / 1e6);
  };
  for (int bpsm : {4, 8, 16}) {
    const int grid = sms * bpsm, thr = 256;
    char nm[64];
    snprintf(nm, 64, "rw17 (8 in, 9 out) grid %d", grid);
    run(nm, 17.0 * n, [&] { rw17<<<grid, thr>>>(in, reason, raw, n / 4); });
    snprintf(nm, 64, "rw17c coalesced grid %d", grid);
    run(nm, 17.0 * n, [&] { rw17c<<<grid, thr>>>(in, reason, raw, n / 4); });
    snprintf(nm, 64, "copy16 (1 GB -> 1 GB) grid %d", grid);
    run(nm, 16.0 * n, [&] { copy16<<<grid, thr>>>(in, out, n / 2); });
    snprintf(nm, 64, "read8 grid %d", grid);
    run(nm, 8.0 * n, [&] { read8<<<grid, thr>>>(in, reason, n / 2); });
    snprintf(nm, 64, "write9 grid %d", grid);
    run(nm, 9.0 * n, [&] { write9<<<grid, thr>>>(reason, raw, n / 4); });
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
