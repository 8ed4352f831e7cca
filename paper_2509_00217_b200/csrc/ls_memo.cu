// ls_memo.cu — the layer-sum memo table of a workload.
//
// The layer plan's two Python sums (simulator.py:224-236: the compute and the
// collective time of one transformer layer) depend only on (tp, ep, batch)
// and the axes of qkv, attn_core (DIM1 or not), attn_out, ffn1, ffn2 and the
// shared-expert pair: 7·7·11 x 1458 = 785,862 combinations for the default
// 12-op domains. build_memo evaluates every combination once, with the same
// device code the per-candidate walk uses (layer_sums) and the workload's sum()
// semantics, into a double2 table (12.6 MB, L2-resident); full_path then reads
// one 16-byte entry instead of ~18 table gathers and compensated adds. The
// values are the walk's own results, so verdicts stay bit-identical.
#include <cuda_runtime.h>

#include "ls_evaluate.cuh"
#include "ls_kernels.h"

namespace ls {

namespace {

template <bool NEU>
__global__ void build_memo_kernel(const uint64_t* __restrict__ tab, const TabLayout L, const EvalMeta M, int64_t n,
                                  double2* __restrict__ memo) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = k;
    int ax_s1 = 0, ax_s2 = 0;
    if (L.has_shared) {
      ax_s2 = (int)(r % 3);
      r /= 3;
      ax_s1 = (int)(r % 3);
      r /= 3;
    }
    const int ax_f2 = (int)(r % 3);
    r /= 3;
    const int ax_f1 = (int)(r % 3);
    r /= 3;
    const int ax_out = (int)(r % 3);
    r /= 3;
    const int a2 = (int)(r % 2);
    r /= 2;
    const int ax_qkv = (int)(r % 3);
    r /= 3;
    const int b = (int)(r % L.nb);
    r /= L.nb;
    const int e = (int)(r % L.ne);
    const int t = (int)(r / L.ne);
    const bool tp_gt1 = (int64_t)gword(tab, L.tpv + t) > 1, ep_gt1 = (int64_t)gword(tab, L.epv + e) > 1;
    double lc, lm;
    layer_sums<NEU, true, false, double>(tab, nullptr, L, t, e, b, tp_gt1, ep_gt1, ax_qkv, a2, ax_out, ax_f1, ax_f2,
                                         ax_s1, ax_s2, lc, lm);
    memo[k] = make_double2(lc, lm);
  }
}

}  // namespace

int64_t memo_entries(const TabLayout& L) {
  return (int64_t)L.nt * L.ne * L.nb * 3 * 2 * 3 * 3 * 3 * (L.has_shared ? 9 : 1);
}

cudaError_t build_memo(bool neumaier, const uint64_t* tab, const TabLayout& L, const EvalMeta& M, double2* memo,
                       cudaStream_t s) {
  const int64_t n = memo_entries(L);
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (neumaier) build_memo_kernel<true><<<(unsigned)blocks, 256, 0, s>>>(tab, L, M, n, memo);
  else build_memo_kernel<false><<<(unsigned)blocks, 256, 0, s>>>(tab, L, M, n, memo);
  return cudaGetLastError();
}

}  // namespace ls
