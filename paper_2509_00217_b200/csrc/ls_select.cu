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
#include "ls_topk.cuh"

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

constexpr int kTopkThreads = 256;
constexpr int kTopkWarps = kTopkThreads / 32;
constexpr int kTopkPerLane = 16;  // candidates per lane per chunk (one 16-byte reason load)

// Per-warp list storage: RegList (k <= 32, registers) or WarpList (k <= 64,
// shared memory); both merge across warps through Rec slots.
struct TopkSmem {
  double lists[kTopkWarps][4 * 64];  // WarpList storage (k > 32 only)
  Rec slots[kTopkWarps][64];         // cross-warp merge
  int count[kTopkWarps];
  int slot_count[kTopkWarps];
};

template <class List>
__device__ __forceinline__ void list_init(List& l, TopkSmem& s, int w);
template <>
__device__ __forceinline__ void list_init<RegList>(RegList& l, TopkSmem&, int) {
  l.init();
}
template <>
__device__ __forceinline__ void list_init<WarpList>(WarpList& l, TopkSmem& s, int w) {
  if ((threadIdx.x & 31) == 0) s.count[w] = 0;
  __syncwarp();
  l.bind(s.lists[w], 64, &s.count[w]);
}

// Merge the CTA's warp lists into warp 0's and write it out.
template <class List>
__device__ void merge_and_emit(List& l, TopkSmem& s, int k, double floor, ls_elite_rec* out, int32_t* count_out,
                               int64_t floor_idx = INT64_MAX) {
  const int w = threadIdx.x >> 5;
  l.store(s.slots[w], &s.slot_count[w]);
  __syncthreads();
  if (w == 0) {
    for (int o = 1; o < kTopkWarps; ++o) l.absorb(s.slots[o], s.slot_count[o], k, floor, floor_idx);
    l.emit(out, count_out);
  }
}

__device__ __forceinline__ uint64_t vector_code(const TopkMeta& tm, const uint8_t* planes, int64_t stride, int64_t i) {
  uint64_t c = 0;
  for (int h = 0; h < tm.A; ++h) c += (uint64_t)planes[(int64_t)h * stride + i] * (uint64_t)tm.code_stride[h];
  return c;
}

// Per-CTA top-k of valid candidates over a contiguous slice of the batch.
template <class List>
__global__ void __launch_bounds__(kTopkThreads) topk_local_kernel(const TopkMeta tm, const uint8_t* __restrict__ planes,
                                                                  int64_t stride, const uint8_t* __restrict__ reason,
                                                                  const double* __restrict__ thr,
                                                                  const double* __restrict__ key, int64_t n, int k,
                                                                  int64_t index_base, ls_elite_rec* __restrict__ out,
                                                                  int32_t* __restrict__ counts) {
  __shared__ TopkSmem s;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  List wl;
  list_init(wl, s, w);
  const int64_t chunk = 32 * kTopkPerLane;
  const int64_t nchunks = (n + chunk - 1) / chunk;
  const bool vec = ((uintptr_t)reason % 16) == 0;
  for (int64_t ch = (int64_t)blockIdx.x * kTopkWarps + w; ch < nchunks; ch += (int64_t)gridDim.x * kTopkWarps) {
    const int64_t base = ch * chunk + (int64_t)lane * kTopkPerLane;
    uint32_t pending = 0;
    if (vec && base + kTopkPerLane <= n) {
      const uint4 r = *reinterpret_cast<const uint4*>(reason + base);
      const uint32_t words[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (((words[q] >> (8 * b)) & 0xffu) == LS_REASON_NONE) pending |= 1u << (4 * q + b);
    } else {
      for (int j = 0; j < kTopkPerLane; ++j)
        if (base + j < n && reason[base + j] == LS_REASON_NONE) pending |= 1u << j;
    }
    while (__any_sync(0xffffffffu, pending != 0)) {
      Rec r{0.0, 0.0, 0, 0};
      bool have = false;
      if (pending) {
        const int j = __ffs(pending) - 1;
        pending &= pending - 1;
        const int64_t i = base + j;
        r.key = key[i];
        r.raw = thr[i];
        r.idx = index_base + i;
        have = wl.admits(r.key, r.idx, k);
        if (have) r.code = vector_code(tm, planes, stride, i);
      }
      wl.offer(have, r, k);
    }
  }
  merge_and_emit(wl, s, k, -1.0e308, out + (int64_t)blockIdx.x * k, counts + blockIdx.x);
}

// Merge m lists of up to k_in records each into one list of k. One CTA.
// `floor` (raw-keyed reductions only) prunes records k distinct vectors beat.
template <class List>
__global__ void __launch_bounds__(kTopkThreads) topk_merge_kernel(const ls_elite_rec* __restrict__ recs,
                                                                  const int32_t* __restrict__ counts, int m, int k_in,
                                                                  int k, const unsigned long long* floor,
                                                                  ls_elite_rec* __restrict__ out,
                                                                  int32_t* __restrict__ count_out) {
  __shared__ TopkSmem s;
  __shared__ double s_fk[kTopkWarps];
  __shared__ int64_t s_fi[kTopkWarps];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Exact floor (key, index): the best k-th entry of any full input list.
  // That list holds k distinct vectors at least as good, so every record
  // strictly worse cannot be in the merged top-k (or is not its vector's best
  // occurrence). Unlike a key-only floor it also prunes ties on the key.
  double fk = floor ? read_floor(floor) : -1.0e308;
  int64_t fi = INT64_MAX;
  if (k <= k_in)
    for (int t = threadIdx.x; t < m; t += kTopkThreads)
      if (counts[t] >= k) {
        const ls_elite_rec& e = recs[(int64_t)t * k_in + k - 1];
        if (better(e.key, e.index, fk, fi)) {
          fk = e.key;
          fi = e.index;
        }
      }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ok = __shfl_xor_sync(0xffffffffu, fk, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, fi, o);
    if (better(ok, oi, fk, fi)) {
      fk = ok;
      fi = oi;
    }
  }
  if (lane == 0) {
    s_fk[w] = fk;
    s_fi[w] = fi;
  }
  __syncthreads();
  for (int o = 0; o < kTopkWarps; ++o)
    if (better(s_fk[o], s_fi[o], fk, fi)) {
      fk = s_fk[o];
      fi = s_fi[o];
    }
  List wl;
  list_init(wl, s, w);
  // records flattened across lists, 32 per warp step: independent loads, so
  // the single CTA is bound by a few L2 round trips, not by m sequential lists
  const int total = m * k_in;
  for (int base = w * 32; base < total; base += kTopkWarps * 32) {
    const int i = base + lane;
    Rec r{0.0, 0.0, 0, 0};
    bool have = false;
    if (i < total) {
      const int list = i / k_in, j = i - list * k_in;
      if (j < counts[list]) {
        const ls_elite_rec& e = recs[i];
        r.key = e.key;
        r.raw = e.raw;
        r.idx = e.index;
        r.code = e.code;
        have = at_least(r.key, r.idx, fk, fi);
      }
    }
    wl.offer(have, r, k);
  }
  merge_and_emit(wl, s, k, fk, out, count_out, fi);
}

// Fast merge of m short lists (k <= 32, register lists), one CTA of 1024
// threads. It is latency-bound, so it runs as a few rounds of independent
// loads instead of a walk over the lists:
//   1. every thread loads the counts of a few lists and the k-th record of
//      each full one; a block reduction gives the exact (key, index) floor —
//      the best k-th entry of any full list (see at_least());
//   2. lane l of a warp takes list l of a 32-list group and loads its
//      records two at a time; records at least as good as the floor (usually
//      a handful: the lists of the fused evaluate are already pruned by the
//      global key floor) are offered to the warp's register list;
//   3. the 32 warp lists merge in a 5-level tree.
constexpr int kMergeThreads = 1024;
constexpr int kMergeWarps = kMergeThreads / 32;

// ROWS: list l's count is the int32 at the start of record k of that list (the
// exchange block layout: k records + a count row) instead of counts[l]; block b
// merges the lists starting at recs + b * step_stride into out + b * k,
// count_out[b] (one launch for a group of steps).
template <bool ROWS>
__global__ void __launch_bounds__(kMergeThreads) topk_merge_fast_kernel(const ls_elite_rec* __restrict__ recs,
                                                                        const int32_t* __restrict__ counts, int m,
                                                                        int k_in, int k,
                                                                        const unsigned long long* floor,
                                                                        ls_elite_rec* __restrict__ out,
                                                                        int32_t* __restrict__ count_out,
                                                                        int64_t step_stride = 0, uint32_t seq0 = 0,
                                                                        int32_t* err = nullptr) {
  __shared__ Rec slots[kMergeWarps][32];
  __shared__ int s_counts[ROWS ? 1024 : 1];
  if (ROWS) {
    recs += (int64_t)blockIdx.x * step_stride;
    out += (int64_t)blockIdx.x * k;
    count_out += blockIdx.x;
    if (seq0) {  // peer-memory exchange: wait until every rank's block of this step carries its seq
      const uint32_t want = seq0 + blockIdx.x;
      for (int l = threadIdx.x; l < m; l += kMergeThreads) {
        const unsigned long long* w = reinterpret_cast<const unsigned long long*>(recs + (int64_t)l * k_in + k);
        const long long t0 = clock64();
        for (;;) {
          unsigned long long v;
          asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(w) : "memory");
          if ((uint32_t)(v >> 32) == want) break;
          if (clock64() - t0 > 20000000000ll) {  // ~10 s: a rank stopped producing
            if (err) atomicExch(err, 1);
            break;
          }
          __nanosleep(200);
        }
      }
      __syncthreads();
    }
    for (int l = threadIdx.x; l < m; l += kMergeThreads)
      s_counts[l] = *reinterpret_cast<const int32_t*>(recs + (int64_t)l * k_in + k);
    __syncthreads();
    counts = s_counts;
  }
  __shared__ int slot_count[kMergeWarps];
  __shared__ double s_fk[kMergeWarps];
  __shared__ int64_t s_fi[kMergeWarps];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // 1. the (key, index) floor
  double fk = floor ? read_floor(floor) : -1.0e308;
  int64_t fi = INT64_MAX;
  for (int l = threadIdx.x; l < m; l += kMergeThreads)
    if ((ROWS ? counts[l] : __ldg(counts + l)) >= k && k <= k_in) {
      const ls_elite_rec& e = recs[(int64_t)l * k_in + k - 1];
      if (better(e.key, e.index, fk, fi)) {
        fk = e.key;
        fi = e.index;
      }
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ok = __shfl_xor_sync(0xffffffffu, fk, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, fi, o);
    if (better(ok, oi, fk, fi)) {
      fk = ok;
      fi = oi;
    }
  }
  if (lane == 0) {
    s_fk[w] = fk;
    s_fi[w] = fi;
  }
  __syncthreads();
  for (int o = 0; o < kMergeWarps; ++o)
    if (better(s_fk[o], s_fi[o], fk, fi)) {
      fk = s_fk[o];
      fi = s_fi[o];
    }

  // 2. lane-per-list offers, four records per lane per round
  RegList wl;
  wl.init();
  for (int l0 = w * 32; l0 < m; l0 += kMergeThreads) {
    const int l = l0 + lane;
    const int c = l < m ? min(ROWS ? counts[l] : __ldg(counts + l), k_in) : 0;
    int cmax = c;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
    const ls_elite_rec* base = recs + (int64_t)l * k_in;
    for (int j0 = 0; j0 < cmax; j0 += 2) {
      Rec r[2];
      bool have[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        have[u] = j0 + u < c;
        r[u] = Rec{0.0, 0.0, 0, 0};
        if (have[u]) {
          const ls_elite_rec& e = base[j0 + u];
          r[u] = Rec{e.key, e.raw, e.index, e.code};
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) wl.offer(have[u] && at_least(r[u].key, r[u].idx, fk, fi), r[u], k);
    }
  }

  // 3. tree merge of the warp lists
  wl.store(slots[w], &slot_count[w]);
  __syncthreads();
  for (int st = 1; st < kMergeWarps; st <<= 1) {
    if ((w & (2 * st - 1)) == 0 && slot_count[w + st] > 0) {
      wl.absorb(slots[w + st], slot_count[w + st], k, fk, fi);
      wl.store(slots[w], &slot_count[w]);
    }
    __syncthreads();
  }
  if (w == 0) wl.emit(out, count_out);
}

// ---- valid-raw compaction (compact host results) --------------------------
// SearchEnv.step keeps only reason and raw (env.py:165-172), and raw is 0 for
// every invalid candidate, so a host result is complete as the reason bytes
// plus the raws of the valid candidates in index order (the host recovers
// their positions from the reason bytes). Two passes over the reason bytes:
// per-tile valid counts, then every tile sums the counts before it (<= a few
// thousand L2-resident ints) and writes its valid raws at that offset.
constexpr int kCmpThreads = 256;
constexpr int kCmpPer = 16;  // reason bytes per thread (one 16-byte load)
constexpr int kCmpTile = kCmpThreads * kCmpPer;

__device__ __forceinline__ uint32_t zero_bytes4(uint32_t w) { return __vcmpeq4(w, 0u) & 0x01010101u; }

// lane's valid count over its 16 bytes (bytes past n count as invalid)
__device__ __forceinline__ uint32_t load16(const uint8_t* __restrict__ reason, int64_t i0, int64_t n, uint4& w) {
  if (i0 + 16 <= n && ((uintptr_t)(reason + i0) & 15) == 0) {
    w = *reinterpret_cast<const uint4*>(reason + i0);
  } else {
    uint32_t b[4] = {0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u};
    for (int j = 0; j < 16; ++j)
      if (i0 + j < n) b[j >> 2] = (b[j >> 2] & ~(0xffu << (8 * (j & 3)))) | ((uint32_t)reason[i0 + j] << (8 * (j & 3)));
    w = make_uint4(b[0], b[1], b[2], b[3]);
  }
  const uint32_t z = zero_bytes4(w.x) + zero_bytes4(w.y) + zero_bytes4(w.z) + zero_bytes4(w.w);
  return (z * 0x01010101u) >> 24;
}

__device__ __forceinline__ int block_excl_scan(int x, int* warp_sums, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = x;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int t = lane < kCmpThreads / 32 ? warp_sums[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_sums[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  total = warp_sums[kCmpThreads / 32 - 1];
  return incl - x + (wid ? warp_sums[wid - 1] : 0);
}

__global__ void __launch_bounds__(kCmpThreads) valid_count_kernel(const uint8_t* __restrict__ reason, int64_t n,
                                                                   int* __restrict__ tile_count) {
  __shared__ int ws[32];
  uint4 w;
  const int c = (int)load16(reason, (int64_t)blockIdx.x * kCmpTile + 16 * threadIdx.x, n, w);
  int total;
  block_excl_scan(c, ws, total);
  if (threadIdx.x == 0) tile_count[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kCmpThreads) valid_compact_kernel(const uint8_t* __restrict__ reason,
                                                                     const double* __restrict__ thr, int64_t n,
                                                                     const int* __restrict__ tile_count,
                                                                     double* __restrict__ out, int64_t* count_out) {
  __shared__ int ws[32];
  __shared__ int s_base;
  // offset of this tile: the counts of every tile before it
  int part = 0;
  for (int t = threadIdx.x; t < (int)blockIdx.x; t += kCmpThreads) part += tile_count[t];
  int tot_before;
  block_excl_scan(part, ws, tot_before);
  if (threadIdx.x == 0) s_base = tot_before;
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.x * kCmpTile + 16 * threadIdx.x;
  uint4 w;
  const int c = (int)load16(reason, i0, n, w);
  int total;
  int pos = s_base + block_excl_scan(c, ws, total);
  if (c) {
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
    for (int j = 0; j < 16; ++j)
      if (((ww[j >> 2] >> (8 * (j & 3))) & 0xffu) == 0 && i0 + j < n) out[pos++] = thr[i0 + j];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *count_out = s_base + total;
}

}  // namespace

size_t compact_scratch_bytes(int64_t n) { return sizeof(int) * (size_t)((n + kCmpTile - 1) / kCmpTile + 1); }

cudaError_t launch_valid_compact(const uint8_t* reason, const double* thr, int64_t n, double* out, int64_t* count_out,
                                 void* scratch, cudaStream_t s) {
  if (n <= 0) return cudaMemsetAsync(count_out, 0, sizeof(int64_t), s);
  const int64_t tiles = (n + kCmpTile - 1) / kCmpTile;
  int* tc = static_cast<int*>(scratch);
  valid_count_kernel<<<(unsigned)tiles, kCmpThreads, 0, s>>>(reason, n, tc);
  valid_compact_kernel<<<(unsigned)tiles, kCmpThreads, 0, s>>>(reason, thr, n, tc, out, count_out);
  return cudaGetLastError();
}

cudaError_t launch_topk_merge_steps(const ls_elite_rec* blocks, int world, int steps, int k, ls_elite_rec* out,
                                    int32_t* counts_out, cudaStream_t s, int rank_stride, uint32_t seq0,
                                    int32_t* err) {
  // rank r's block of step j: blocks + (r * rank_stride + j) * (k + 1) records (rank_stride 0: = steps)
  const int rs = rank_stride > 0 ? rank_stride : steps;
  topk_merge_fast_kernel<true><<<steps, kMergeThreads, 0, s>>>(blocks, nullptr, world, rs * (k + 1), k, nullptr, out,
                                                              counts_out, (int64_t)(k + 1), seq0, err);
  return cudaGetLastError();
}

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
  int64_t c = (n + 65535) / 65536;
  const int64_t cap = 148 * 4;  // four CTAs per B200 SM
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
  if (k <= 32) {
    topk_local_kernel<RegList><<<c, kTopkThreads, 0, s>>>(tm, planes, stride, reason, thr, key, n > 0 ? n : 0, k,
                                                          index_base, part, counts);
    topk_merge_fast_kernel<false><<<1, kMergeThreads, 0, s>>>(part, counts, c, k, k, nullptr, out, count_out);
  } else {
    topk_local_kernel<WarpList><<<c, kTopkThreads, 0, s>>>(tm, planes, stride, reason, thr, key, n > 0 ? n : 0, k,
                                                           index_base, part, counts);
    topk_merge_kernel<WarpList><<<1, kTopkThreads, 0, s>>>(part, counts, c, k, k, nullptr, out, count_out);
  }
  return cudaGetLastError();
}

cudaError_t launch_topk_merge(const ls_elite_rec* recs, const int32_t* counts, int m, int k_in, int k,
                              const unsigned long long* floor,
                              ls_elite_rec* out, int32_t* count_out, cudaStream_t s) {
  if (k <= 32)
    topk_merge_fast_kernel<false><<<1, kMergeThreads, 0, s>>>(recs, counts, m, k_in, k, floor, out, count_out);
  else
    topk_merge_kernel<WarpList><<<1, kTopkThreads, 0, s>>>(recs, counts, m, k_in, k, floor, out, count_out);
  return cudaGetLastError();
}

}  // namespace ls
