// ls_select.cu — device-side reward shaping scan and elite top-k.
//
// Reward scan: SearchEnv.step shapes every valid candidate against the best
// raw seen strictly BEFORE it (env.py:159-164, best updated after at
// :178-179). Over a batch that is an exclusive prefix-max scan, done in
// three passes: per-tile max -> single-CTA scan of tile maxima -> per-tile
// exclusive scan + reward write.
//
// Top-k: EliteBuffer.offer (policy.py:86-102) keeps the best `capacity`
// DISTINCT vectors, older first among equal rewards; build_report(by_raw)
// (ppo.py:441-447) keeps the earliest best raw. Both equal "top-k over
// distinct vectors by (key desc, index asc), each vector ranked by its best
// occurrence" for an empty start. Each warp keeps
// such a list in shared memory (warp-cooperative sorted insert with dedupe by
// mixed-radix vector code), warps merge per CTA, CTAs merge in one final CTA.
// The insert rule (replace a duplicate only by a better occurrence, evict the
// worst when full) keeps the invariant "list = top-k distinct of everything
// seen" for any arrival order, so the same merge serves the cross-GPU
// all-gather of per-rank lists.
#include <cuda_runtime.h>
#include <float.h>

#include "ls_kernels.h"

namespace ls {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanPerThread = 16;
constexpr int kScanTile = kScanThreads * kScanPerThread;

__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void tile_max_kernel(const uint8_t* __restrict__ reason, const double* __restrict__ thr, int64_t n,
                                double* __restrict__ tile_max) {
  __shared__ double red[kScanThreads / 32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  double m = -DBL_MAX;
  for (int j = 0; j < kScanPerThread; ++j) {
    const int64_t i = base + (int64_t)j * kScanThreads + threadIdx.x;
    if (i < n && reason[i] == LS_REASON_NONE) m = fmax(m, thr[i]);
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < kScanThreads / 32 ? red[threadIdx.x] : -DBL_MAX;
    v = warp_max(v);
    if (threadIdx.x == 0) tile_max[blockIdx.x] = v;
  }
}

// Exclusive prefix max over tile maxima, seeded with b0. One CTA.
__global__ void tile_scan_kernel(const double* __restrict__ tile_max, int64_t tiles, double b0,
                                 double* __restrict__ tile_base, double* __restrict__ best_out) {
  __shared__ double warp_tot[32];
  __shared__ double carry;
  if (threadIdx.x == 0) carry = b0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t start = 0; start < tiles; start += blockDim.x) {
    const int64_t i = start + threadIdx.x;
    const double x = i < tiles ? tile_max[i] : -DBL_MAX;
    double incl = x;
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl = fmax(incl, y);
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      double t = lane < nw ? warp_tot[lane] : -DBL_MAX;
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t = fmax(t, y);
      }
      if (lane < nw) warp_tot[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const double before_warp = wid ? warp_tot[wid - 1] : -DBL_MAX;
    double excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = -DBL_MAX;
    const double c = carry;
    if (i < tiles) tile_base[i] = fmax(c, fmax(before_warp, excl));
    __syncthreads();
    if (threadIdx.x == 0) carry = fmax(c, warp_tot[nw - 1]);
    __syncthreads();
  }
  if (threadIdx.x == 0 && best_out) *best_out = carry;
}

__global__ void reward_kernel(const uint8_t* __restrict__ reason, const double* __restrict__ thr, int64_t n,
                              const double* __restrict__ tile_base, double alpha, double beta, double penalty,
                              double* __restrict__ reward) {
  __shared__ double warp_tot[kScanThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanPerThread;
  double raw[kScanPerThread];
  bool ok[kScanPerThread];
  double m = -DBL_MAX;
#pragma unroll
  for (int j = 0; j < kScanPerThread; ++j) {
    const int64_t i = base + j;
    ok[j] = i < n && reason[i] == LS_REASON_NONE;
    raw[j] = ok[j] ? thr[i] : 0.0;
    if (ok[j]) m = fmax(m, raw[j]);
  }
  // exclusive scan of per-thread maxima across the CTA
  double incl = m;
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl = fmax(incl, y);
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  double before = tile_base[blockIdx.x];
  for (int w = 0; w < wid; ++w) before = fmax(before, warp_tot[w]);
  double excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane > 0) before = fmax(before, excl);
  double b = before;
#pragma unroll
  for (int j = 0; j < kScanPerThread; ++j) {
    const int64_t i = base + j;
    if (i < n) {
      if (ok[j]) {
        reward[i] = alpha * raw[j] + beta * (raw[j] - b);
        if (raw[j] > b) b = raw[j];
      } else {
        reward[i] = penalty;
      }
    }
  }
}

// ---------------------------------------------------------------- top-k

struct Rec {
  double key, raw;
  int64_t idx;
  uint64_t code;
};

__device__ __forceinline__ bool better(double ka, int64_t ia, double kb, int64_t ib) {
  return ka > kb || (ka == kb && ia < ib);
}

// A sorted (best first) list of at most k <= 64 distinct records in shared
// memory, operated on by one full warp.
struct WarpList {
  double* key;
  double* raw;
  int64_t* idx;
  uint64_t* code;
  int* count;

  // Warp-cooperative insert of r (all lanes pass the same r).
  __device__ void insert(const Rec& r, int k) {
    const int lane = threadIdx.x & 31;
    const int cnt = *count;
    // duplicate vector already listed?
    int dup = -1;
    for (int j = lane; j < cnt; j += 32)
      if (code[j] == r.code) dup = j;
    for (int o = 16; o > 0; o >>= 1) dup = max(dup, __shfl_xor_sync(0xffffffffu, dup, o));
    int n = cnt;
    if (dup >= 0) {
      if (!better(r.key, r.idx, key[dup], idx[dup])) return;
      remove_at(dup, n);
      --n;
    } else if (n == k) {
      if (!better(r.key, r.idx, key[k - 1], idx[k - 1])) return;
      --n;  // drop the worst
    }
    // insertion position = number of entries ranked before r
    int before = 0;
    for (int j = lane; j < n; j += 32) before += better(key[j], idx[j], r.key, r.idx) ? 1 : 0;
    for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
    // shift [before, n) down by one: read all, then write
    double kk[2], rr[2];
    int64_t ii[2];
    uint64_t cc[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int j = lane + 32 * s;
      if (j >= before && j < n) {
        kk[s] = key[j];
        rr[s] = raw[j];
        ii[s] = idx[j];
        cc[s] = code[j];
      }
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int j = lane + 32 * s;
      if (j >= before && j < n) {
        key[j + 1] = kk[s];
        raw[j + 1] = rr[s];
        idx[j + 1] = ii[s];
        code[j + 1] = cc[s];
      }
    }
    if (lane == 0) {
      key[before] = r.key;
      raw[before] = r.raw;
      idx[before] = r.idx;
      code[before] = r.code;
      *count = n + 1;
    }
    __syncwarp();
  }

  __device__ void remove_at(int pos, int n) {
    const int lane = threadIdx.x & 31;
    double kk[2], rr[2];
    int64_t ii[2];
    uint64_t cc[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int j = lane + 32 * s;
      if (j > pos && j < n) {
        kk[s] = key[j];
        rr[s] = raw[j];
        ii[s] = idx[j];
        cc[s] = code[j];
      }
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int j = lane + 32 * s;
      if (j > pos && j < n) {
        key[j - 1] = kk[s];
        raw[j - 1] = rr[s];
        idx[j - 1] = ii[s];
        code[j - 1] = cc[s];
      }
    }
    __syncwarp();
  }

  // Would r enter the list (ignoring duplicates)? Cheap pre-filter.
  __device__ __forceinline__ bool admits(double k_, int64_t i_, int k) const {
    const int cnt = *count;
    return cnt < k || better(k_, i_, key[k - 1], idx[k - 1]);
  }
};

constexpr int kTopkThreads = 256;
constexpr int kTopkWarps = kTopkThreads / 32;

struct ListSmem {
  double key[kTopkWarps][64];
  double raw[kTopkWarps][64];
  int64_t idx[kTopkWarps][64];
  uint64_t code[kTopkWarps][64];
  int count[kTopkWarps];
};

__device__ __forceinline__ WarpList warp_list(ListSmem& s, int w) {
  WarpList l;
  l.key = s.key[w];
  l.raw = s.raw[w];
  l.idx = s.idx[w];
  l.code = s.code[w];
  l.count = &s.count[w];
  return l;
}

// Offer a stream of records, 32 at a time, to warp list `wl`.
__device__ __forceinline__ void offer_lanes(WarpList& wl, bool have, const Rec& mine, int k) {
  const bool cand = have && wl.admits(mine.key, mine.idx, k);
  unsigned mask = __ballot_sync(0xffffffffu, cand);
  while (mask) {
    const int src = __ffs(mask) - 1;
    mask &= mask - 1;
    Rec r;
    r.key = __shfl_sync(0xffffffffu, mine.key, src);
    r.raw = __shfl_sync(0xffffffffu, mine.raw, src);
    r.idx = __shfl_sync(0xffffffffu, mine.idx, src);
    r.code = __shfl_sync(0xffffffffu, mine.code, src);
    wl.insert(r, k);
  }
}

// Write the CTA's merged list (warp 0 list after merging the others).
__device__ void merge_warps_and_emit(ListSmem& s, int k, ls_elite_rec* out, int32_t* count_out) {
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w == 0) {
    WarpList l0 = warp_list(s, 0);
    for (int src = 1; src < kTopkWarps; ++src) {
      const int cnt = s.count[src];
      for (int j0 = 0; j0 < cnt; j0 += 32) {
        const int j = j0 + lane;
        Rec r;
        const bool have = j < cnt;
        if (have) {
          r.key = s.key[src][j];
          r.raw = s.raw[src][j];
          r.idx = s.idx[src][j];
          r.code = s.code[src][j];
        } else {
          r.key = 0;
          r.raw = 0;
          r.idx = 0;
          r.code = 0;
        }
        offer_lanes(l0, have, r, k);
      }
    }
    const int cnt = s.count[0];
    for (int j = lane; j < cnt; j += 32) {
      ls_elite_rec o;
      o.key = s.key[0][j];
      o.raw = s.raw[0][j];
      o.index = s.idx[0][j];
      o.code = s.code[0][j];
      out[j] = o;
    }
    if (lane == 0) *count_out = cnt;
  }
}

__global__ void __launch_bounds__(kTopkThreads) topk_local_kernel(const TopkMeta tm, const uint8_t* __restrict__ planes,
                                                                  int64_t stride, const uint8_t* __restrict__ reason,
                                                                  const double* __restrict__ thr,
                                                                  const double* __restrict__ key, int64_t n, int k,
                                                                  int64_t index_base, ls_elite_rec* __restrict__ out,
                                                                  int32_t* __restrict__ counts) {
  __shared__ ListSmem s;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) s.count[w] = 0;
  __syncwarp();
  WarpList wl = warp_list(s, w);
  // contiguous chunk per CTA, split into contiguous sub-chunks per warp
  const int64_t per_cta = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * per_cta;
  const int64_t hi = min(n, lo + per_cta);
  const int64_t per_warp = (hi - lo + kTopkWarps - 1) / kTopkWarps;
  const int64_t wlo = lo + (int64_t)w * per_warp;
  const int64_t whi = min(hi, wlo + per_warp);
  for (int64_t base = wlo; base < whi; base += 32) {
    const int64_t i = base + lane;
    const bool have = i < whi && reason[i] == LS_REASON_NONE;
    Rec r;
    r.key = have ? key[i] : 0.0;
    r.raw = have ? thr[i] : 0.0;
    r.idx = index_base + i;
    r.code = 0;
    const bool cand = have && wl.admits(r.key, r.idx, k);
    if (cand) {
      uint64_t c = 0;
      for (int h = 0; h < tm.A; ++h) c += (uint64_t)planes[(int64_t)h * stride + i] * (uint64_t)tm.code_stride[h];
      r.code = c;
    }
    offer_lanes(wl, cand, r, k);
  }
  merge_warps_and_emit(s, k, out + (int64_t)blockIdx.x * k, counts + blockIdx.x);
}

// Merge m lists of up to k_in records each into one list of k. One CTA.
__global__ void __launch_bounds__(kTopkThreads) topk_merge_kernel(const ls_elite_rec* __restrict__ recs,
                                                                  const int32_t* __restrict__ counts, int m, int k_in,
                                                                  int k, ls_elite_rec* __restrict__ out,
                                                                  int32_t* __restrict__ count_out) {
  __shared__ ListSmem s;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) s.count[w] = 0;
  __syncwarp();
  WarpList wl = warp_list(s, w);
  for (int list = w; list < m; list += kTopkWarps) {
    const int cnt = min(counts[list], k_in);
    for (int j0 = 0; j0 < cnt; j0 += 32) {
      const int j = j0 + lane;
      const bool have = j < cnt;
      Rec r;
      if (have) {
        const ls_elite_rec& e = recs[(int64_t)list * k_in + j];
        r.key = e.key;
        r.raw = e.raw;
        r.idx = e.index;
        r.code = e.code;
      } else {
        r.key = r.raw = 0.0;
        r.idx = 0;
        r.code = 0;
      }
      offer_lanes(wl, have, r, k);
    }
  }
  merge_warps_and_emit(s, k, out, count_out);
}

}  // namespace

size_t scan_scratch_bytes(int64_t n) {
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  return (size_t)(2 * (tiles > 0 ? tiles : 1)) * sizeof(double);
}

cudaError_t launch_reward_scan(const uint8_t* reason, const double* thr, int64_t n, double b0, double alpha,
                               double beta, double penalty, double* reward, double* best_out, void* scratch,
                               int num_sms, cudaStream_t s) {
  (void)num_sms;
  if (n <= 0) {
    if (best_out) cudaMemcpyAsync(best_out, &b0, sizeof(double), cudaMemcpyHostToDevice, s);
    return cudaGetLastError();
  }
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  double* tile_max = static_cast<double*>(scratch);
  double* tile_base = tile_max + tiles;
  tile_max_kernel<<<(unsigned)tiles, kScanThreads, 0, s>>>(reason, thr, n, tile_max);
  tile_scan_kernel<<<1, 1024, 0, s>>>(tile_max, tiles, b0, tile_base, best_out);
  reward_kernel<<<(unsigned)tiles, kScanThreads, 0, s>>>(reason, thr, n, tile_base, alpha, beta, penalty, reward);
  return cudaGetLastError();
}

static int topk_ctas(int64_t n, int num_sms) {
  (void)num_sms;
  int64_t c = (n + 8191) / 8192;
  const int64_t cap = 296;  // two CTAs per B200 SM
  if (c > cap) c = cap;
  if (c < 1) c = 1;
  return (int)c;
}

size_t topk_scratch_bytes(int64_t n, int k, int num_sms) {
  const int c = topk_ctas(n, num_sms);
  return (size_t)c * k * sizeof(ls_elite_rec) + (size_t)c * sizeof(int32_t) + 16;
}

cudaError_t launch_topk(const TopkMeta& tm, const uint8_t* planes, int64_t stride, const uint8_t* reason,
                        const double* thr, const double* key, int64_t n, int k, int64_t index_base,
                        ls_elite_rec* out, int32_t* count_out, void* scratch, int num_sms, cudaStream_t s) {
  const int c = topk_ctas(n, num_sms);
  ls_elite_rec* part = static_cast<ls_elite_rec*>(scratch);
  int32_t* counts = reinterpret_cast<int32_t*>(part + (size_t)c * k);
  topk_local_kernel<<<c, kTopkThreads, 0, s>>>(tm, planes, stride, reason, thr, key, n > 0 ? n : 0, k, index_base,
                                               part, counts);
  topk_merge_kernel<<<1, kTopkThreads, 0, s>>>(part, counts, c, k, k, out, count_out);
  return cudaGetLastError();
}

cudaError_t launch_topk_merge(const ls_elite_rec* recs, const int32_t* counts, int m, int k_in, int k,
                              ls_elite_rec* out, int32_t* count_out, cudaStream_t s) {
  topk_merge_kernel<<<1, kTopkThreads, 0, s>>>(recs, counts, m, k_in, k, out, count_out);
  return cudaGetLastError();
}

}  // namespace ls
