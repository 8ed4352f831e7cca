// ls_evaluate.cu — the batched strategy-evaluation kernels.
//
// Data path (per CTA, persistent over a grid-stride range of candidates):
//   1. one elected thread bulk-copies (TMA, cp.async.bulk) the workload's
//      table buffer from HBM into shared memory, tracked by an mbarrier;
//   2. each thread owns 4 consecutive candidates and reads them with one
//      32-bit load per head plane (a warp reads 128 contiguous bytes per
//      plane: fully coalesced), decodes, scores (ls_evaluate.cuh) and
//      writes the verdict planes with 32-bit (reason) and 16-byte (float64
//      fields) stores.
// A generic one-candidate-per-thread kernel covers vectors longer than 16
// heads, unaligned planes and ragged strides.
#include <cuda_runtime.h>

#include "ls_evaluate.cuh"
#include "ls_kernels.h"

namespace ls {

namespace {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Stage `words` 8-byte words from global memory into shared memory with
// 1-D bulk async copies (TMA engine) completing on one mbarrier.
__device__ void stage_tables(uint64_t* dst, const uint64_t* __restrict__ src, int words) {
  __shared__ __align__(8) uint64_t bar;
  const uint32_t bar_a = smem_addr(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t bytes = static_cast<uint32_t>(words) * 8u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a), "r"(bytes) : "memory");
    const uint32_t chunk = 16384;
    for (uint32_t off = 0; off < bytes; off += chunk) {
      const uint32_t sz = bytes - off < chunk ? bytes - off : chunk;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_addr(reinterpret_cast<const char*>(dst) + off)),
          "l"(reinterpret_cast<const char*>(src) + off), "r"(sz), "r"(bar_a)
          : "memory");
    }
  }
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar_a)
        : "memory");
  }
}

__device__ __forceinline__ void store_verdict(const EvalArgs& a, int64_t i, const Verdict& v) {
  a.reason[i] = static_cast<uint8_t>(v.reason);
  if (a.thr) a.thr[i] = v.thr;
  if (a.tpot) a.tpot[i] = v.tpot;
  if (a.mem) a.mem[i] = v.mem;
  if (a.comp) a.comp[i] = v.comp;
  if (a.comm) a.comm[i] = v.comm;
  if (a.pipe) a.pipe[i] = v.pipe;
}

__device__ __forceinline__ void store2(double* base, int64_t i, double x, double y) {
  if (base) *reinterpret_cast<double2*>(base + i) = make_double2(x, y);
}

// 4 candidates per thread, A <= 16 heads, planes 4-byte aligned, outputs
// 16-byte aligned.
template <bool NEU, bool SMEM>
__global__ void __launch_bounds__(256) eval_vec4_kernel(const uint64_t* __restrict__ gtab, const TabLayout L,
                                                        const EvalMeta M, const EvalArgs a) {
  extern __shared__ __align__(16) uint64_t s_tab[];
  const uint64_t* T = gtab;
  if (SMEM) {
    stage_tables(s_tab, gtab, L.words);
    T = s_tab;
  }
  const int64_t nquads = (a.n + 3) >> 2;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nquads; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t base = q << 2;
    const bool full = base + 4 <= a.n;
    uint32_t w[16];
#pragma unroll
    for (int h = 0; h < 16; ++h) {
      w[h] = 0;
      if (h < M.A) {
        const uint8_t* src = a.planes + (int64_t)h * a.stride + base;
        if (full) {
          w[h] = __ldcs(reinterpret_cast<const unsigned int*>(src));
        } else {
          for (int j = 0; base + j < a.n; ++j) w[h] |= (uint32_t)src[j] << (8 * j);
        }
      }
    }
    Verdict v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t bad = 0, X = M.pinned_axes;
      int idx[4];
#pragma unroll
      for (int h = 0; h < 16; ++h) {
        if (h < M.A) {
          const uint32_t byte = (w[h] >> (8 * j)) & 0xffu;
          bad |= byte >= M.head_size[h];
          if (h < 4) {
            idx[h] = (int)byte;
          } else {
            const int op = M.head_op[h];
            if (op >= 0) X = (X & ~(3u << (2 * op))) | ((byte & 3u) << (2 * op));
          }
        }
      }
      if (bad) {
        v[j].reason = LS_REASON_DECODE_ERROR;
        v[j].thr = v[j].tpot = v[j].mem = v[j].comp = v[j].comm = v[j].pipe = 0.0;
      } else {
        score<NEU>(T, L, M, idx[0], idx[1], idx[2], idx[3], X, v[j]);
      }
    }
    if (full) {
      const uint32_t r = v[0].reason | (v[1].reason << 8) | (v[2].reason << 16) | (v[3].reason << 24);
      __stcs(reinterpret_cast<unsigned int*>(a.reason + base), r);
      store2(a.thr, base, v[0].thr, v[1].thr);
      store2(a.thr, base + 2, v[2].thr, v[3].thr);
      store2(a.tpot, base, v[0].tpot, v[1].tpot);
      store2(a.tpot, base + 2, v[2].tpot, v[3].tpot);
      store2(a.mem, base, v[0].mem, v[1].mem);
      store2(a.mem, base + 2, v[2].mem, v[3].mem);
      store2(a.comp, base, v[0].comp, v[1].comp);
      store2(a.comp, base + 2, v[2].comp, v[3].comp);
      store2(a.comm, base, v[0].comm, v[1].comm);
      store2(a.comm, base + 2, v[2].comm, v[3].comm);
      store2(a.pipe, base, v[0].pipe, v[1].pipe);
      store2(a.pipe, base + 2, v[2].pipe, v[3].pipe);
    } else {
      for (int j = 0; j < 4 && base + j < a.n; ++j) store_verdict(a, base + j, v[j]);
    }
  }
}

// One candidate per thread, any A <= LS_MAX_HEADS, any alignment.
template <bool NEU, bool SMEM>
__global__ void __launch_bounds__(256) eval_generic_kernel(const uint64_t* __restrict__ gtab, const TabLayout L,
                                                           const EvalMeta M, const EvalArgs a) {
  extern __shared__ __align__(16) uint64_t s_tab[];
  const uint64_t* T = gtab;
  if (SMEM) {
    stage_tables(s_tab, gtab, L.words);
    T = s_tab;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t bad = 0, X = M.pinned_axes;
    int idx[4] = {0, 0, 0, 0};
    for (int h = 0; h < M.A; ++h) {
      const uint32_t byte = a.planes[(int64_t)h * a.stride + i];
      bad |= byte >= M.head_size[h];
      if (h < 4) {
        idx[h & 3] = (int)byte;
      } else {
        const int op = M.head_op[h];
        if (op >= 0) X = (X & ~(3u << (2 * op))) | ((byte & 3u) << (2 * op));
      }
    }
    Verdict v;
    if (bad) {
      v.reason = LS_REASON_DECODE_ERROR;
      v.thr = v.tpot = v.mem = v.comp = v.comm = v.pipe = 0.0;
    } else {
      score<NEU>(T, L, M, idx[0], idx[1], idx[2], idx[3], X, v);
    }
    store_verdict(a, i, v);
  }
}

template <bool NEU, bool SMEM>
cudaError_t launch_eval(const LaunchPlan& lp, const uint64_t* tab, const TabLayout& L, const EvalMeta& M,
                        const EvalArgs& a, cudaStream_t s) {
  const size_t smem = SMEM ? (size_t)L.words * 8 : 0;
  if (lp.vec4) {
    auto k = eval_vec4_kernel<NEU, SMEM>;
    const int64_t nquads = (a.n + 3) >> 2;
    int64_t blocks = (nquads + 255) / 256;
    if (blocks > lp.max_blocks) blocks = lp.max_blocks;
    k<<<(unsigned)blocks, 256, smem, s>>>(tab, L, M, a);
  } else {
    auto k = eval_generic_kernel<NEU, SMEM>;
    int64_t blocks = (a.n + 255) / 256;
    if (blocks > lp.max_blocks) blocks = lp.max_blocks;
    k<<<(unsigned)blocks, 256, smem, s>>>(tab, L, M, a);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_evaluate(const LaunchPlan& lp, bool neumaier, bool smem_tables, const uint64_t* tab,
                            const TabLayout& L, const EvalMeta& M, const EvalArgs& a, cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  if (neumaier) {
    return smem_tables ? launch_eval<true, true>(lp, tab, L, M, a, s) : launch_eval<true, false>(lp, tab, L, M, a, s);
  }
  return smem_tables ? launch_eval<false, true>(lp, tab, L, M, a, s) : launch_eval<false, false>(lp, tab, L, M, a, s);
}

cudaError_t prepare_eval_kernels(size_t smem) {
  const int b = (int)smem;
  cudaFuncSetAttribute(eval_vec4_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(eval_vec4_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(eval_generic_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(eval_generic_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  return cudaGetLastError();
}

int occupancy_blocks_per_sm(bool vec4, bool smem_tables, size_t smem) {
  int nb = 0;
  if (vec4)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &nb, smem_tables ? eval_vec4_kernel<true, true> : eval_vec4_kernel<true, false>, 256, smem);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &nb, smem_tables ? eval_generic_kernel<true, true> : eval_generic_kernel<true, false>, 256, smem);
  return nb;
}

}  // namespace ls
