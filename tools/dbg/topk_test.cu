// Debug: standalone launch of the select-kernel top-k with RegList (k<=32).
#include <cstdio>
#include <vector>
#include "../../paper_2509_00217_b200/csrc/ls_select.cu"
using namespace ls;
int main(int argc, char** argv) {
  const int n = 4096, k = argc > 1 ? atoi(argv[1]) : 3;
  std::vector<uint8_t> reason(n), planes(16 * n);
  std::vector<double> thr(n);
  for (int i = 0; i < n; ++i) { reason[i] = (i % 7 == 0) ? 0 : 2; thr[i] = (i * 37 % 101); for (int h = 0; h < 16; ++h) planes[h * n + i] = (i >> h) & 1; }
  uint8_t *dr, *dp; double* dt; ls_elite_rec* out; int* cnt; void* scratch;
  cudaMalloc(&dr, n); cudaMalloc(&dp, 16 * n); cudaMalloc(&dt, 8 * n); cudaMalloc(&out, 64 * 32); cudaMalloc(&cnt, 4);
  cudaMalloc(&scratch, topk_scratch_bytes(n, k, 148));
  cudaMemcpy(dr, reason.data(), n, cudaMemcpyHostToDevice); cudaMemcpy(dp, planes.data(), 16 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dt, thr.data(), 8 * n, cudaMemcpyHostToDevice);
  TopkMeta tm; tm.A = 16; for (int h = 0; h < LS_MAX_HEADS; ++h) tm.code_stride[h] = h < 16 ? (1ll << (15 - h)) : 0;
  cudaError_t e = launch_topk(tm, dp, n, dr, dt, dt, n, k, 0, out, cnt, scratch, 148, 0);
  printf("launch: %s\n", cudaGetErrorString(e));
  e = cudaDeviceSynchronize();
  printf("sync: %s\n", cudaGetErrorString(e));
  int c = 0; ls_elite_rec h[64]; cudaMemcpy(&c, cnt, 4, cudaMemcpyDeviceToHost); cudaMemcpy(h, out, 64 * 32, cudaMemcpyDeviceToHost);
  printf("count %d first %g idx %ld\n", c, h[0].key, (long)h[0].index);
  return 0;
}
