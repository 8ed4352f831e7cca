// ls_topk.cuh — warp-cooperative elite list (shared by the evaluate and
// select kernels).
//
// EliteBuffer.offer (policy.py:86-102) keeps the best `capacity` DISTINCT
// vectors, older first among equal rewards; build_report(by_raw)
// (ppo.py:441-447) keeps the earliest best raw. For an empty start both are
// "top-k over distinct vectors by (key desc, index asc), each vector ranked
// by its best occurrence". A WarpList holds such a
// list in shared memory; its insert rule — a duplicate vector is replaced
// only by a better occurrence, the worst entry is evicted when full — keeps
// the invariant "list == top-k distinct of everything offered" for ANY
// arrival order, so per-warp lists, per-CTA merges and the cross-GPU merge of
// all-gathered per-rank lists all compose exactly.
#pragma once
#include <stdint.h>

#include "../../include/ls_eval.h"

namespace ls {

struct Rec {
  double key, raw;
  int64_t idx;
  uint64_t code;
};

__device__ __forceinline__ bool better(double ka, int64_t ia, double kb, int64_t ib) {
  return ka > kb || (ka == kb && ia < ib);
}
// (ka, ia) is the floor record or better than it. A floor (key, idx) taken
// from a full list's k-th entry is beaten by k distinct vectors; with
// idx = INT64_MAX it is the key-only floor (key >= floor).
__device__ __forceinline__ bool at_least(double ka, int64_t ia, double kf, int64_t i_f) {
  return ka > kf || (ka == kf && ia <= i_f);
}

// Sorted (best first) list of at most k <= 64 distinct records in shared
// memory, operated on by one full warp.
struct WarpList {
  double* key;
  double* raw;
  int64_t* idx;
  uint64_t* code;
  int* count;

  __device__ void bind(void* base, int cap, int* cnt) {
    key = static_cast<double*>(base);
    raw = key + cap;
    idx = reinterpret_cast<int64_t*>(raw + cap);
    code = reinterpret_cast<uint64_t*>(idx + cap);
    count = cnt;
  }

  __device__ void move_range(int from, int to_shift, int lo, int n) {
    // entries j in [lo, n) move to j + to_shift (to_shift = +1 or -1)
    const int lane = threadIdx.x & 31;
    double kk[2], rr[2];
    int64_t ii[2];
    uint64_t cc[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int j = lane + 32 * s;
      if (j >= lo && j < n) {
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
      if (j >= lo && j < n) {
        key[j + to_shift] = kk[s];
        raw[j + to_shift] = rr[s];
        idx[j + to_shift] = ii[s];
        code[j + to_shift] = cc[s];
      }
    }
    __syncwarp();
    (void)from;
  }

  // Warp-cooperative insert of r (all lanes pass the same r).
  __device__ void insert(const Rec& r, int k) {
    const int lane = threadIdx.x & 31;
    const int cnt = *count;
    int dup = -1;
    for (int j = lane; j < cnt; j += 32)
      if (code[j] == r.code) dup = j;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dup = max(dup, __shfl_xor_sync(0xffffffffu, dup, o));
    int n = cnt;
    if (dup >= 0) {
      if (!better(r.key, r.idx, key[dup], idx[dup])) return;
      move_range(0, -1, dup + 1, n);
      --n;
    } else if (n == k) {
      if (!better(r.key, r.idx, key[k - 1], idx[k - 1])) return;
      --n;  // drop the worst
    }
    int before = 0;
    for (int j = lane; j < n; j += 32) before += better(key[j], idx[j], r.key, r.idx) ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
    move_range(0, +1, before, n);
    if (lane == 0) {
      key[before] = r.key;
      raw[before] = r.raw;
      idx[before] = r.idx;
      code[before] = r.code;
      *count = n + 1;
    }
    __syncwarp();
  }

  // Could r enter the list (ignoring duplicates)? Cheap pre-filter.
  __device__ __forceinline__ bool admits(double k_, int64_t i_, int k) const {
    return *count < k || better(k_, i_, key[k - 1], idx[k - 1]);
  }

  // Key of the k-th entry once the list is full (else -inf): any record
  // with a strictly smaller key is beaten by k distinct vectors already.
  __device__ __forceinline__ double floor_key(int k) const { return *count < k ? -1.0e308 : key[k - 1]; }

  // Offer one record per lane (lanes with have == false offer nothing).
  __device__ void offer(bool have, const Rec& mine, int k) {
    const bool cand = have && admits(mine.key, mine.idx, k);
    unsigned mask = __ballot_sync(0xffffffffu, cand);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      Rec r;
      r.key = __shfl_sync(0xffffffffu, mine.key, src);
      r.raw = __shfl_sync(0xffffffffu, mine.raw, src);
      r.idx = __shfl_sync(0xffffffffu, mine.idx, src);
      r.code = __shfl_sync(0xffffffffu, mine.code, src);
      insert(r, k);
    }
  }

  // Offer every record of another list (any order is exact). Records with a
  // key strictly below `floor` are skipped: k distinct vectors beat them.
  __device__ void absorb(const WarpList& o, int k, double floor = -1.0e308) {
    const int lane = threadIdx.x & 31;
    const int cnt = *o.count;
    for (int j0 = 0; j0 < cnt; j0 += 32) {
      const int j = j0 + lane;
      Rec r{0.0, 0.0, 0, 0};
      const bool have = j < cnt && o.key[j] >= floor;
      if (have) {
        r.key = o.key[j];
        r.raw = o.raw[j];
        r.idx = o.idx[j];
        r.code = o.code[j];
      }
      offer(have, r, k);
    }
  }

  // Same interface as RegList for cross-warp merges through Rec slots.
  __device__ void store(Rec* slots, int* cnt) const {
    const int lane = threadIdx.x & 31;
    const int c = *count;
    for (int j = lane; j < c; j += 32) slots[j] = Rec{key[j], raw[j], idx[j], code[j]};
    if (lane == 0) *cnt = c;
  }
  __device__ void absorb(const Rec* slots, int n, int k, double floor = -1.0e308,
                         int64_t floor_idx = INT64_MAX) {
    const int lane = threadIdx.x & 31;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      Rec r{0.0, 0.0, 0, 0};
      bool have = false;
      if (j < n) {
        r = slots[j];
        have = at_least(r.key, r.idx, floor, floor_idx);
      }
      offer(have, r, k);
    }
  }

  __device__ void emit(ls_elite_rec* out, int32_t* count_out) const {
    const int lane = threadIdx.x & 31;
    const int cnt = *count;
    for (int j = lane; j < cnt; j += 32) {
      ls_elite_rec e;
      e.key = key[j];
      e.raw = raw[j];
      e.index = idx[j];
      e.code = code[j];
      out[j] = e;
    }
    if (lane == 0) *count_out = cnt;
  }
};

// Register-resident variant for k <= 32: lane j holds entry j, so an insert
// is a handful of ballots and one shuffle — no shared memory, no syncwarp.
// Same ordering, dedupe and eviction rule as WarpList.
struct RegList {
  double key, raw;
  int64_t idx;
  uint64_t code;
  int count;         // warp-uniform
  double kth_key;    // warp-uniform copy of entry k-1 (valid when count == k)
  int64_t kth_idx;

  __device__ __forceinline__ void init() {
    key = raw = 0.0;
    idx = 0;
    code = 0;
    count = 0;
    kth_key = -1.0e308;
    kth_idx = 0;
  }

  // Shuffle-free, so it may be called from divergent code.
  __device__ __forceinline__ bool admits(double k_, int64_t i_, int k) const {
    return count < k || better(k_, i_, kth_key, kth_idx);
  }

  __device__ __forceinline__ double floor_key(int k) const { return count < k ? -1.0e308 : kth_key; }

  // Warp-cooperative insert of r (all lanes pass the same r).
  __device__ void insert(const Rec& r, int k) {
    const int lane = threadIdx.x & 31;
    const unsigned dup = __ballot_sync(0xffffffffu, lane < count && code == r.code);
    if (dup) {
      const int d = __ffs(dup) - 1;
      const double dk = __shfl_sync(0xffffffffu, key, d);
      const int64_t di = __shfl_sync(0xffffffffu, idx, d);
      if (!better(r.key, r.idx, dk, di)) return;
      // remove entry d: lanes >= d take their right neighbour
      const double k2 = __shfl_down_sync(0xffffffffu, key, 1), r2 = __shfl_down_sync(0xffffffffu, raw, 1);
      const int64_t i2 = __shfl_down_sync(0xffffffffu, idx, 1);
      const uint64_t c2 = __shfl_down_sync(0xffffffffu, code, 1);
      if (lane >= d) {
        key = k2;
        raw = r2;
        idx = i2;
        code = c2;
      }
      --count;
    } else if (count == k) {
      if (!better(r.key, r.idx, kth_key, kth_idx)) return;
      --count;  // drop the worst
    }
    const int pos = __popc(__ballot_sync(0xffffffffu, lane < count && better(key, idx, r.key, r.idx)));
    const double k1 = __shfl_up_sync(0xffffffffu, key, 1), r1 = __shfl_up_sync(0xffffffffu, raw, 1);
    const int64_t i1 = __shfl_up_sync(0xffffffffu, idx, 1);
    const uint64_t c1 = __shfl_up_sync(0xffffffffu, code, 1);
    if (lane > pos) {
      key = k1;
      raw = r1;
      idx = i1;
      code = c1;
    } else if (lane == pos) {
      key = r.key;
      raw = r.raw;
      idx = r.idx;
      code = r.code;
    }
    ++count;
    kth_key = __shfl_sync(0xffffffffu, key, k - 1);
    kth_idx = __shfl_sync(0xffffffffu, idx, k - 1);
  }

  // Offer one record per lane (lanes with have == false offer nothing).
  __device__ void offer(bool have, const Rec& mine, int k) {
    const bool cand = have && admits(mine.key, mine.idx, k);
    unsigned mask = __ballot_sync(0xffffffffu, cand);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      Rec r;
      r.key = __shfl_sync(0xffffffffu, mine.key, src);
      r.raw = __shfl_sync(0xffffffffu, mine.raw, src);
      r.idx = __shfl_sync(0xffffffffu, mine.idx, src);
      r.code = __shfl_sync(0xffffffffu, mine.code, src);
      insert(r, k);
    }
  }

  // Spill to / fill from shared memory (lane j <-> slot j) for cross-warp merges.
  __device__ void store(Rec* slots, int* cnt) const {
    const int lane = threadIdx.x & 31;
    if (lane < count) slots[lane] = Rec{key, raw, idx, code};
    if (lane == 0) *cnt = count;
  }

  // Offer n records held in shared memory slots (any order is exact).
  __device__ void absorb(const Rec* slots, int n, int k, double floor = -1.0e308,
                         int64_t floor_idx = INT64_MAX) {
    const int lane = threadIdx.x & 31;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      Rec r{0.0, 0.0, 0, 0};
      bool have = false;
      if (j < n) {
        r = slots[j];
        have = at_least(r.key, r.idx, floor, floor_idx);
      }
      offer(have, r, k);
    }
  }

  // Emit only the entries with key >= floor (a prefix: the list is sorted).
  __device__ void emit_from(double floor, ls_elite_rec* out, int32_t* count_out) const {
    const int lane = threadIdx.x & 31;
    const int c = __popc(__ballot_sync(0xffffffffu, lane < count && key >= floor));
    if (lane < c) {
      ls_elite_rec e;
      e.key = key;
      e.raw = raw;
      e.index = idx;
      e.code = code;
      out[lane] = e;
    }
    if (lane == 0) *count_out = c;
  }

  __device__ void emit(ls_elite_rec* out, int32_t* count_out) const {
    const int lane = threadIdx.x & 31;
    if (lane < count) {
      ls_elite_rec e;
      e.key = key;
      e.raw = raw;
      e.index = idx;
      e.code = code;
      out[lane] = e;
    }
    if (lane == 0) *count_out = count;
  }
};

// Global pruning floor shared by every list of one reduction: the largest
// k-th key any full list has reached. Keys are non-negative doubles (raw
// throughput), whose IEEE bit patterns order like unsigned integers, so the
// floor is an atomicMax on the bits. A record strictly below it cannot make
// the final top-k (k distinct vectors beat it), for any arrival order.
__device__ __forceinline__ void raise_floor(unsigned long long* floor, double k_) {
  if (floor && k_ >= 0.0) atomicMax(floor, (unsigned long long)__double_as_longlong(k_));
}
__device__ __forceinline__ double read_floor(const unsigned long long* floor) {
  if (!floor) return -1.0e308;
  unsigned long long v;  // relaxed, GPU scope (a volatile load would be a system-scope strong load)
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(floor) : "memory");
  return __longlong_as_double((long long)v);
}

// Bytes of one WarpList of capacity cap.
__host__ __device__ constexpr int warp_list_bytes(int cap) { return cap * 32; }

}  // namespace ls
