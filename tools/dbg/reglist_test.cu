// Debug: exercise RegList insert/offer on one warp.
#include <cstdio>
#include "../../paper_2509_00217_b200/csrc/ls_topk.cuh"
using namespace ls;
__global__ void k1(ls_elite_rec* out, int* cnt, int k, int stage) {
  RegList l;
  l.init();
  const int lane = threadIdx.x & 31;
  if (stage >= 1) {
    for (int it = 0; it < 4; ++it) {
      Rec r{double((lane * 7 + it * 13) % 50), 0.0, lane + 32 * it, (uint64_t)((lane * 7 + it * 13) % 50)};
      l.offer(true, r, k);
    }
  }
  if (stage >= 2) l.emit(out, cnt);
}
int main() {
  ls_elite_rec* out; int* cnt;
  cudaMalloc(&out, 64 * sizeof(ls_elite_rec)); cudaMalloc(&cnt, 4);
  for (int stage = 0; stage < 3; ++stage) {
    k1<<<1, 32>>>(out, cnt, 3, stage);
    cudaError_t e = cudaDeviceSynchronize();
    printf("stage %d: %s\n", stage, cudaGetErrorString(e));
    if (e) return 1;
  }
  ls_elite_rec h[3]; int c;
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost); cudaMemcpy(&c, cnt, 4, cudaMemcpyDeviceToHost);
  printf("count %d: %g %g %g\n", c, h[0].key, h[1].key, h[2].key);
  return 0;
}
