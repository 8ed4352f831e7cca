// ls_evaluate.cu — the batched strategy-evaluation kernels.
//
// eval_tma_kernel (the hot path; 16-byte aligned SoA planes, A <= 16):
//   persistent CTAs walk 1024-candidate tiles. Per CTA:
//   * one thread bulk-copies (TMA, cp.async.bulk + mbarrier) the workload's
//     gate tables into shared memory, then keeps a 3-stage ring of candidate
//     tiles in flight (A plane slices of 1 KB per tile), so HBM latency is
//     hidden by the copy engine instead of by registers;
//   * pass A: each thread pulls its 4 candidates (one 32-bit shared load per
//     head plane), decodes them and runs the integer/bitmask gates and the
//     memory model (gate()); the ~98% of candidates a uniform batch gates out
//     are finished here with coalesced 32-bit / 128-bit stores;
//   * survivors (fit in memory) are compacted into a shared-memory queue with
//     warp-aggregated atomics; when half full, all 256 threads drain it
//     through the fp64 cost model (full_path()) — dense warps, no divergence
//     between cheap and expensive candidates.
// eval_generic_kernel covers everything else (any alignment, A <= 64), one
// candidate per thread.
#include <cuda_runtime.h>

#include "ls_evaluate.cuh"
#include "ls_kernels.h"

namespace ls {

namespace {

constexpr int kThreads = 256;
constexpr int kTile = 4 * kThreads;  // candidates per tile
constexpr int kStages = 3;
constexpr int kQueue = 2048;  // survivor queue entries per CTA

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

// 1-D bulk async copy global -> shared (TMA engine), completing on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Decode byte j of the packed plane words: head range check + domain
// indices + 2-bit axis word in canonical op order.
__device__ __forceinline__ bool decode_quad(const uint32_t* w, int j, const EvalMeta& M, Decoded& c) {
  uint32_t bad = 0, X = M.pinned_axes;
  const int sh = 8 * j;
  const uint32_t b0 = (w[0] >> sh) & 0xffu, b1 = (w[1] >> sh) & 0xffu, b2 = (w[2] >> sh) & 0xffu,
                 b3 = (w[3] >> sh) & 0xffu;
  bad |= (b0 >= M.head_size[0]) | (b1 >= M.head_size[1]) | (b2 >= M.head_size[2]) | (b3 >= M.head_size[3]);
#pragma unroll
  for (int h = 4; h < 16; ++h) {
    if (h < M.A) {
      const uint32_t byte = (w[h] >> sh) & 0xffu;
      bad |= byte > 2u;
      const int op = M.head_op[h];
      if (op >= 0) X = (X & ~(3u << (2 * op))) | ((byte & 3u) << (2 * op));
    }
  }
  c.t = (int)b0;
  c.e = (int)b1;
  c.p = (int)b2;
  c.b = (int)b3;
  c.X = X;
  return !bad;
}

__device__ __forceinline__ uint64_t pack_key(int64_t idx, const Decoded& c) {
  return (uint64_t)idx | ((uint64_t)c.t << 40) | ((uint64_t)c.e << 46) | ((uint64_t)c.p << 52) |
         ((uint64_t)c.b << 58);
}

__device__ __forceinline__ void unpack_key(uint64_t k, uint32_t X, int64_t& idx, Decoded& c) {
  idx = (int64_t)(k & ((1ull << 40) - 1));
  c.t = (int)((k >> 40) & 63);
  c.e = (int)((k >> 46) & 63);
  c.p = (int)((k >> 52) & 63);
  c.b = (int)((k >> 58) & 63);
  c.X = X;
}

__device__ __forceinline__ void st2(double* base, int64_t i, double x, double y) {
  *reinterpret_cast<double2*>(base + i) = make_double2(x, y);
}

template <bool NEU, bool FULL>
__device__ __forceinline__ void write_full(const EvalArgs& a, int64_t idx, const Verdict& v) {
  a.reason[idx] = (uint8_t)v.reason;
  if (a.thr) a.thr[idx] = v.thr;
  if (FULL) {
    if (a.tpot) a.tpot[idx] = v.tpot;
    if (a.comp) a.comp[idx] = v.comp;
    if (a.comm) a.comm[idx] = v.comm;
    if (a.pipe) a.pipe[idx] = v.pipe;
  }
}

template <bool NEU, bool FULL, bool SMEM_GATE>
__global__ void __launch_bounds__(kThreads, 2)
    eval_tma_kernel(const uint64_t* __restrict__ gtab, const TabLayout L, const EvalMeta M, const EvalArgs a,
                    const int64_t ntiles) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full_bar[kStages];
  __shared__ __align__(8) uint64_t gate_bar;
  __shared__ int qcount;
  const int A = M.A;
  const uint32_t stage_bytes = (uint32_t)A * kTile;
  uint8_t* ring = smem;
  uint64_t* G = reinterpret_cast<uint64_t*>(smem + kStages * stage_bytes);
  uint64_t* qkey = SMEM_GATE ? G + L.gate_words : G;
  uint32_t* qx = reinterpret_cast<uint32_t*>(qkey + kQueue);
  const uint64_t* Gt = SMEM_GATE ? G : gtab;
  const int tid = threadIdx.x, lane = tid & 31;

  auto issue_tile = [&](int stage, int64_t tile) {
    uint64_t* bar = &full_bar[stage];
    mbar_expect_tx(bar, stage_bytes);
    const uint8_t* src = a.planes + tile * kTile;
    uint8_t* dst = ring + stage * stage_bytes;
    for (int h = 0; h < A; ++h) bulk_g2s(dst + h * kTile, src + (int64_t)h * a.stride, kTile, bar);
  };

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full_bar[s], 1);
    mbar_init(&gate_bar, 1);
    qcount = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async();
  }
  __syncthreads();
  if (tid == 0) {
    if (SMEM_GATE) {
      mbar_expect_tx(&gate_bar, (uint32_t)L.gate_words * 8u);
      bulk_g2s(G, gtab, (uint32_t)L.gate_words * 8u, &gate_bar);
    }
    for (int s = 0; s < kStages; ++s) {
      const int64_t tile = blockIdx.x + (int64_t)s * gridDim.x;
      if (tile < ntiles) issue_tile(s, tile);
    }
  }
  if (SMEM_GATE) mbar_wait(&gate_bar, 0);

  // Drain the survivor queue through the fp64 path (all threads).
  auto drain = [&]() {
    const int qc = qcount;
    for (int q = tid; q < qc; q += kThreads) {
      int64_t idx;
      Decoded c;
      unpack_key(qkey[q], qx[q], idx, c);
      Verdict v;
      full_path<NEU>(gtab, L, M, c, v);
      write_full<NEU, FULL>(a, idx, v);
    }
    __syncthreads();
    if (tid == 0) qcount = 0;
    __syncthreads();
  };

  // Pass A over 4 consecutive candidates starting at `base` (count valid).
  auto pass_a = [&](const uint32_t* w, int64_t base, int count) {
    uint32_t r4 = 0;
    double m[4];
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
      Decoded c;
      const bool ok = decode_quad(w, j, M, c);
      double mem = 0.0;
      uint32_t reason = LS_REASON_DECODE_ERROR;
      if (ok) reason = gate(Gt, L, M, c, mem);
      const bool surv = j < count && ok && reason == LS_REASON_NONE;
      const unsigned mask = __ballot_sync(0xffffffffu, surv);
      if (mask) {
        const int leader = __ffs(mask) - 1;
        int qb = 0;
        if (lane == leader) qb = atomicAdd(&qcount, __popc(mask));
        qb = __shfl_sync(0xffffffffu, qb, leader);
        if (surv) {
          const int pos = qb + __popc(mask & ((1u << lane) - 1u));
          qkey[pos] = pack_key(base + j, c);
          qx[pos] = c.X;
        }
      }
      r4 |= reason << (8 * j);
      m[j] = mem;
    }
    if (count == 4) {
      *reinterpret_cast<uint32_t*>(a.reason + base) = r4;
      if (a.thr) {
        st2(a.thr, base, 0.0, 0.0);
        st2(a.thr, base + 2, 0.0, 0.0);
      }
      if (FULL) {
        if (a.mem) {
          st2(a.mem, base, m[0], m[1]);
          st2(a.mem, base + 2, m[2], m[3]);
        }
        double* zf[4] = {a.tpot, a.comp, a.comm, a.pipe};
#pragma unroll
        for (int f = 0; f < 4; ++f)
          if (zf[f]) {
            st2(zf[f], base, 0.0, 0.0);
            st2(zf[f], base + 2, 0.0, 0.0);
          }
      }
    } else {
      for (int j = 0; j < count; ++j) {
        a.reason[base + j] = (uint8_t)(r4 >> (8 * j));
        if (a.thr) a.thr[base + j] = 0.0;
        if (FULL) {
          if (a.mem) a.mem[base + j] = m[j];
          if (a.tpot) a.tpot[base + j] = 0.0;
          if (a.comp) a.comp[base + j] = 0.0;
          if (a.comm) a.comm[base + j] = 0.0;
          if (a.pipe) a.pipe[base + j] = 0.0;
        }
      }
    }
  };

  int i = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
    const int s = i % kStages;
    mbar_wait(&full_bar[s], (uint32_t)((i / kStages) & 1));
    uint32_t w[16];
    const uint8_t* st = ring + s * stage_bytes + 4 * tid;
#pragma unroll
    for (int h = 0; h < 16; ++h) w[h] = h < A ? *reinterpret_cast<const uint32_t*>(st + h * kTile) : 0u;
    __syncthreads();  // stage s fully pulled into registers: refill it
    if (tid == 0) {
      const int64_t next = tile + (int64_t)kStages * gridDim.x;
      if (next < ntiles) {
        fence_proxy_async();
        issue_tile(s, next);
      }
    }
    pass_a(w, tile * kTile + 4 * tid, 4);
    __syncthreads();
    if (qcount >= kQueue / 2) drain();
  }
  // ragged tail (< one tile): the CTA that would own the next tile
  const int64_t tail0 = ntiles * kTile;
  if (tail0 < a.n && blockIdx.x == (unsigned)(ntiles % gridDim.x)) {
    const int64_t base = tail0 + 4 * tid;
    int count = 0;
    uint32_t w[16];
    if (base < a.n) {
      count = a.n - base < 4 ? (int)(a.n - base) : 4;
#pragma unroll
      for (int h = 0; h < 16; ++h) {
        w[h] = 0;
        if (h < A)
          for (int j = 0; j < count; ++j) w[h] |= (uint32_t)a.planes[(int64_t)h * a.stride + base + j] << (8 * j);
      }
    } else {
#pragma unroll
      for (int h = 0; h < 16; ++h) w[h] = 0;
    }
    pass_a(w, base, count);
    __syncthreads();
  }
  if (qcount > 0) drain();
}

// One candidate per thread, any alignment, any A <= LS_MAX_HEADS.
template <bool NEU>
__global__ void __launch_bounds__(kThreads) eval_generic_kernel(const uint64_t* __restrict__ gtab, const TabLayout L,
                                                                const EvalMeta M, const EvalArgs a) {
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
    Decoded c;
    c.t = idx[0];
    c.e = idx[1];
    c.p = idx[2];
    c.b = idx[3];
    c.X = X;
    Verdict v;
    v.thr = v.tpot = v.comp = v.comm = v.pipe = 0.0;
    double mem = 0.0;
    v.reason = bad ? LS_REASON_DECODE_ERROR : gate(gtab, L, M, c, mem);
    if (!bad && v.reason == LS_REASON_NONE) full_path<NEU>(gtab, L, M, c, v);
    a.reason[i] = (uint8_t)v.reason;
    if (a.thr) a.thr[i] = v.thr;
    if (a.tpot) a.tpot[i] = v.tpot;
    if (a.mem) a.mem[i] = mem;
    if (a.comp) a.comp[i] = v.comp;
    if (a.comm) a.comm[i] = v.comm;
    if (a.pipe) a.pipe[i] = v.pipe;
  }
}

template <bool NEU, bool FULL, bool SG>
void set_attr(size_t smem) {
  cudaFuncSetAttribute(eval_tma_kernel<NEU, FULL, SG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

}  // namespace

size_t tma_smem_bytes(const TabLayout& L, int A, bool smem_gate) {
  return (size_t)kStages * A * kTile + (smem_gate ? (size_t)L.gate_words * 8 : 0) + (size_t)kQueue * 12;
}

bool tma_eligible(const EvalArgs& a, int A) {
  const bool al16 = ((uintptr_t)a.planes % 16) == 0 && a.stride % 16 == 0;
  bool out_al = ((uintptr_t)a.reason % 4) == 0;
  const double* fs[6] = {a.thr, a.tpot, a.mem, a.comp, a.comm, a.pipe};
  for (const double* f : fs) out_al = out_al && ((uintptr_t)f % 16) == 0;
  return A <= 16 && al16 && out_al && a.n < (int64_t(1) << 40);
}

cudaError_t prepare_eval_kernels(const TabLayout& L, int A, bool smem_gate) {
  const size_t smem = tma_smem_bytes(L, A, smem_gate);
  if (smem_gate) {
    set_attr<true, true, true>(smem);
    set_attr<true, false, true>(smem);
    set_attr<false, true, true>(smem);
    set_attr<false, false, true>(smem);
  } else {
    set_attr<true, true, false>(smem);
    set_attr<true, false, false>(smem);
    set_attr<false, true, false>(smem);
    set_attr<false, false, false>(smem);
  }
  return cudaGetLastError();
}

int tma_blocks_per_sm(const TabLayout& L, int A, bool smem_gate) {
  int nb = 0;
  const size_t smem = tma_smem_bytes(L, A, smem_gate);
  if (smem_gate)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, eval_tma_kernel<true, false, true>, kThreads, smem);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, eval_tma_kernel<true, false, false>, kThreads, smem);
  return nb;
}

int generic_blocks_per_sm() {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, eval_generic_kernel<true>, kThreads, 0);
  return nb;
}

template <bool NEU, bool FULL>
static void launch_tma_t(const LaunchPlan& lp, const uint64_t* tab, const TabLayout& L, const EvalMeta& M,
                         const EvalArgs& a, cudaStream_t s) {
  const int64_t ntiles = a.n / kTile;
  int64_t blocks = ntiles > 0 ? ntiles : 1;
  if (blocks > lp.max_blocks) blocks = lp.max_blocks;
  const size_t smem = tma_smem_bytes(L, M.A, lp.smem_gate);
  if (lp.smem_gate)
    eval_tma_kernel<NEU, FULL, true><<<(unsigned)blocks, kThreads, smem, s>>>(tab, L, M, a, ntiles);
  else
    eval_tma_kernel<NEU, FULL, false><<<(unsigned)blocks, kThreads, smem, s>>>(tab, L, M, a, ntiles);
}

cudaError_t launch_evaluate(const LaunchPlan& lp, bool neumaier, const uint64_t* tab, const TabLayout& L,
                            const EvalMeta& M, const EvalArgs& a, cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  const bool full = a.tpot || a.mem || a.comp || a.comm || a.pipe;
  if (lp.tma) {
    if (neumaier) {
      if (full) launch_tma_t<true, true>(lp, tab, L, M, a, s);
      else launch_tma_t<true, false>(lp, tab, L, M, a, s);
    } else {
      if (full) launch_tma_t<false, true>(lp, tab, L, M, a, s);
      else launch_tma_t<false, false>(lp, tab, L, M, a, s);
    }
  } else {
    int64_t blocks = (a.n + kThreads - 1) / kThreads;
    if (blocks > lp.max_blocks) blocks = lp.max_blocks;
    if (neumaier) eval_generic_kernel<true><<<(unsigned)blocks, kThreads, 0, s>>>(tab, L, M, a);
    else eval_generic_kernel<false><<<(unsigned)blocks, kThreads, 0, s>>>(tab, L, M, a);
  }
  return cudaGetLastError();
}

}  // namespace ls
