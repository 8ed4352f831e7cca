// ls_evaluate.cu — the batched strategy-evaluation kernels.
//
// eval_ws_kernel — the hot path (16-byte aligned SoA planes, A <= 16).
// Persistent, warp-specialized CTAs with three roles and no CTA-wide barrier
// in the steady state:
//   * producer warp — its elected lane bulk-copies (TMA, cp.async.bulk) the
//     workload's gate tables into shared memory once, then keeps a 4-stage
//     ring of 1024-candidate tiles in flight (one 1 KB slice per head plane
//     per tile), synchronised through full/empty mbarriers;
//   * 8 gate warps — each owns 128 candidates of a stage (4 per lane, one
//     32-bit shared load per head plane), releases the stage, decodes its 4
//     candidates with SWAR byte arithmetic (range checks and the packed axis
//     word for all 4 at once) and runs gate(): budget and layout bitmasks and
//     the memory model. The ~98% of a uniform batch that is gated out is
//     finished here with coalesced 32-bit / 128-bit stores. Survivors are
//     compacted into the warp's queue (ballot + popc) and handed off 32 at a
//     time through a 2-slot shared-memory mailbox;
//   * 2 fp64 warps — drain the mailboxes: the fp64 cost model (full_path())
//     on 32 survivors at once, verdict stores, and (fused sweep) the offer to
//     the warp's elite list. Gate warps never wait on fp64 latency; when a
//     mailbox is full (survivor-heavy batches) the gate warp scores its own
//     batch instead, so the pipeline degrades to compute-bound, never stalls.
// eval_generic_kernel covers everything else (any alignment, A <= 64), one
// candidate per thread.
#include <cuda_runtime.h>

#include "ls_evaluate.cuh"
#include "ls_kernels.h"
#include "ls_topk.cuh"

namespace ls {

namespace {

#ifdef LS_DIAG_TIMES
// diagnostic build only: per-CTA phase stamps (globaltimer ns), read by ls_diag_times()
// rows: 256 per launch, four launches in a row (launch = CTAs entered / grid)
__device__ unsigned long long g_diag_t[1024][16];
__device__ unsigned int g_diag_entries;
__shared__ int s_diag_launch;
__device__ __forceinline__ void diag_enter() {
  if (threadIdx.x == 0) s_diag_launch = (int)(atomicAdd(&g_diag_entries, 1u) / gridDim.x);
  __syncthreads();
}
__device__ __forceinline__ void diag_stamp(int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_diag_t[((blockIdx.x & 255) + 256 * s_diag_launch) & 1023][slot] = t;
}
#define LS_STAMP(slot) diag_stamp(slot)
#else
#define LS_STAMP(slot) ((void)0)
#endif

// Role counts and ring size (LS_* overrides are for tuning builds only).
#ifndef LS_GATE_WARPS
#define LS_GATE_WARPS 16
#endif
// 16 + 3 + the producer = 20 warps, 5 per SM sub-partition: the 64K-register
// file then allows 96 registers per thread (21 warps capped it at 80, and the
// hot loops rematerialised values to fit); 3 fp64 warps keep up with the
// survivors of a uniform batch.
#ifndef LS_FP_WARPS
#define LS_FP_WARPS 3
#endif
#ifndef LS_RING_KB
#define LS_RING_KB 96
#endif
#ifndef LS_MIN_BLOCKS
#define LS_MIN_BLOCKS 1
#endif
#ifndef LS_LATE_CTAS
#define LS_LATE_CTAS 1  // CTAs (highest indices) without a static first tile group
#endif
#ifndef LS_CLAIM_GROUP
#define LS_CLAIM_GROUP 2  // tiles per dynamic claim of the fused kernels
#endif
#ifndef LS_BACKOFF_MAX
#define LS_BACKOFF_MAX 512
#endif
constexpr int kGateWarps = LS_GATE_WARPS;
constexpr int kFpWarps = LS_FP_WARPS;
constexpr int kWorkWarps = kGateWarps + kFpWarps;
constexpr int kThreads = 32 * (kWorkWarps + 1);  // + producer warp
constexpr int kWarpCands = 128;
constexpr int kTile = kGateWarps * kWarpCands;  // candidates per stage
constexpr int kWarpQueue = 160;  // < 32 left over + 128 from one tile
constexpr int kSlots = 2;        // mailbox slots per gate warp
static_assert(kGateWarps / kFpWarps * kSlots <= 32, "mailbox bits per fp64 warp");
constexpr int kGenericThreads = 256;
constexpr int kFusedK = 32;  // max elite size of the fused evaluate + top-k path
constexpr uint32_t kStageBytes = 16 * kTile;  // 16 plane slices per stage (planes >= A stay zero)
constexpr uint32_t kRingBytes = LS_RING_KB * 1024;
static_assert(kRingBytes / kStageBytes >= 2, "ring holds two plane stages");
// packed words are 8 B per candidate: the same ring holds twice the stages,
// keeping the bytes in flight per SM (and so the HBM pipe) as full as for planes
constexpr int kMaxStages = kRingBytes / (8 * kTile);
template <int MODE>
struct Ring {
  static constexpr uint32_t stage_bytes = MODE == GEN_WORDS ? 8u * kTile : kStageBytes;
  static constexpr int stages = (int)(kRingBytes / stage_bytes);
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void lds_u64x2(uint32_t addr, uint64_t& x, uint64_t& y) {
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(addr));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
__device__ __forceinline__ void mbar_arrive_a(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
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
// The same for candidate tiles, read exactly once: L2 evict-first (LS_EVICT_FIRST tuning builds).
__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
#ifdef LS_EVICT_FIRST
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
#else
  bulk_g2s(dst, src, bytes, bar);
#endif
}

__device__ __forceinline__ uint64_t pack_key(int64_t idx, const Decoded& c) {
  return (uint64_t)idx | ((uint64_t)c.t << 40) | ((uint64_t)c.e << 46) | ((uint64_t)c.p << 52) |
         ((uint64_t)c.b << 58);
}
__device__ __forceinline__ void unpack_key(uint64_t k, uint32_t Y, int64_t& idx, Decoded& c) {
  idx = (int64_t)(k & ((1ull << 40) - 1));
  c.t = (int)((k >> 40) & 63);
  c.e = (int)((k >> 46) & 63);
  c.p = (int)((k >> 52) & 63);
  c.b = (int)((k >> 58) & 63);
  c.Y = Y;
}

// Verdict stores are written once and never re-read by the kernel: streaming
// (evict-first) stores when LS_STCS is set (tuning builds).
__device__ __forceinline__ void st2(double* base, int64_t i, double x, double y) {
#ifdef LS_STCS
  __stcs(reinterpret_cast<double2*>(base + i), make_double2(x, y));
#else
  *reinterpret_cast<double2*>(base + i) = make_double2(x, y);
#endif
}
__device__ __forceinline__ void st_reason4(uint8_t* p, uint32_t v) {
#ifdef LS_STCS
  __stcs(reinterpret_cast<unsigned int*>(p), v);
#else
  *reinterpret_cast<uint32_t*>(p) = v;
#endif
}

template <bool FULL>
__device__ __forceinline__ void write_verdict(const EvalArgs& a, int64_t idx, const Verdict& v) {
  a.reason[idx] = (uint8_t)v.reason;
  if (a.thr) a.thr[idx] = v.thr;
  if (FULL) {
    if (a.tpot) a.tpot[idx] = v.tpot;
    if (a.comp) a.comp[idx] = v.comp;
    if (a.comm) a.comm[idx] = v.comm;
    if (a.pipe) a.pipe[idx] = v.pipe;
  }
}

// SWAR decode of 4 candidates packed byte-wise in w[h] (candidate j in byte
// j). Returns per-byte "bad" flags (head out of range, strategy.py:247-254)
// and q[3]: for axis heads 4..15, 2-bit fields four heads per byte.
__device__ __forceinline__ uint32_t swar_decode(const uint32_t* w, const EvalMeta& M, uint32_t* q) {
  uint32_t badb = 0;
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const uint32_t s4 = (uint32_t)M.head_size[h] * 0x01010101u;
    const uint32_t r = (w[h] | 0x80808080u) - s4;  // per byte: high bit set iff (x & 0x7f) >= size
    badb |= (r | w[h]) & 0x80808080u;
  }
  uint32_t orv = 0, three = 0;
#pragma unroll
  for (int g = 0; g < 3; ++g) {
    const uint32_t a = w[4 + 4 * g], b = w[5 + 4 * g], c = w[6 + 4 * g], d = w[7 + 4 * g];
    orv |= a | b | c | d;
    const uint32_t m = 0x03030303u;
    const uint32_t qq = (a & m) | ((b & m) << 2) | ((c & m) << 4) | ((d & m) << 6);
    three |= qq & (qq >> 1) & 0x55555555u;  // a field holding 3
    q[g] = qq;
  }
  return badb | (orv & 0xfcfcfcfcu) | three;
}

// Candidate j of a lane: byte j of the coarse planes and of the q words
// (byte permutes; j is a compile-time constant after unrolling).
__device__ __forceinline__ void extract(const uint32_t* w, const uint32_t* q, int j, Decoded& c) {
  const uint32_t sel = 0x4440u | (uint32_t)j;  // byte j into byte 0, zeros above
  c.t = (int)__byte_perm(w[0], 0, sel);
  c.e = (int)__byte_perm(w[1], 0, sel);
  c.p = (int)__byte_perm(w[2], 0, sel);
  c.b = (int)__byte_perm(w[3], 0, sel);
  // Y = q0.byte j | q1.byte j << 8 | q2.byte j << 16
  const uint32_t y01 = __byte_perm(q[0], q[1], 0x4440u | ((4u + j) << 4) | (uint32_t)j);
  c.Y = __byte_perm(y01, q[2], 0x4000u | ((4u + j) << 8) | 0x10u) & 0x00ffffffu;
}

// Packed candidate word -> (coarse rank, Y); nonzero return: malformed word
// (bits past the rank, axis bits past head A, an axis field of 3, a rank past
// the coarse space) — the planes path's decode error, strategy.py:247-254.
__device__ __forceinline__ uint32_t word_decode(uint64_t w, const PackMeta& pk, uint32_t& rank, uint32_t& Y) {
  Y = (uint32_t)w & 0xffffffu;
  rank = (uint32_t)(w >> 24) & 0xffffffu;
  // branch-free: any bit past the rank, an axis bit past head A, a field of 3,
  // or rank >= ncoarse (both < 2^24: the sign of ncoarse - 1 - rank)
  const uint32_t bad = (uint32_t)(w >> 48) | (Y & ~pk.axis_mask) | (Y & (Y >> 1) & 0x555555u) |
                       ((pk.ncoarse - 1u - rank) & 0x80000000u);
  return bad != 0 ? 1u : 0u;
}

// ---- on-device candidate streams (ls_sweep) ----------------------------
// Counter-based 64-bit mix (splitmix64 finaliser); host twin: generator.py.
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
// floor(x / d) via a 64-bit reciprocal: exact whenever x * d < 2^64.
__device__ __forceinline__ uint64_t divq(uint64_t x, uint64_t magic, uint64_t d) {
  return d == 1 ? x : __umul64hi(x, magic);
}
// Coarse rank -> (t, e, p, b) (mixed radix, batch fastest).
__device__ __forceinline__ void rank_split(uint32_t rank, const PackMeta& pk, Decoded& c) {
  const uint64_t q1 = divq(rank, pk.m_b, pk.nb);
  c.b = (int)(rank - q1 * pk.nb);
  const uint64_t q2 = divq(q1, pk.m_p, pk.np);
  c.p = (int)(q1 - q2 * pk.np);
  const uint64_t q3 = divq(q2, pk.m_e, pk.ne);
  c.e = (int)(q2 - q3 * pk.ne);
  c.t = (int)q3;
}

// Stream index -> decoded candidate. GEN_UNIFORM: i.i.d. uniform over every
// head (baselines.uniform_vector semantics, baselines.py:50-54) from two
// counter-based draws; GEN_ENUM / GEN_ENUM_ADMISSIBLE: the index-th vector of
// itertools.product over the head domains (all axes / admissible axes only),
// head 0 most significant — the order of the reference's exhaustive sweeps.
template <int MODE>
__device__ __forceinline__ void gen_candidate(const GenMeta& g, uint64_t gidx, Decoded& c) {
  uint64_t coarse, axis;
  if (MODE == GEN_UNIFORM) {
    const uint64_t r1 = splitmix64(g.seed ^ (2 * gidx)), r2 = splitmix64(g.seed ^ (2 * gidx + 1));
    coarse = __umul64hi(r1, g.coarse_size);
    axis = __umul64hi(r2, g.axis_size);
  } else {
    coarse = divq(gidx, g.m_axis, g.axis_size);
    axis = gidx - coarse * g.axis_size;
  }
  const uint64_t hi = divq(axis, g.m_lo, g.lo_size), lo = axis - hi * g.lo_size;
  c.Y = __ldg(g.hi_tab + hi) | __ldg(g.lo_tab + lo);
  const uint64_t q1 = divq(coarse, g.m_b, g.nb);
  c.b = (int)(coarse - q1 * g.nb);
  const uint64_t q2 = divq(q1, g.m_p, g.np);
  c.p = (int)(q1 - q2 * g.np);
  const uint64_t q3 = divq(q2, g.m_e, g.ne);
  c.e = (int)(q2 - q3 * g.ne);
  c.t = (int)q3;
}

// Dynamic shared memory of eval_ws_kernel: TMA ring, gate tables, per-gate
// warp survivor queues, mailboxes and the work warps' elite lists.
struct WsSmem {
  uint8_t* ring;
  uint64_t* gate;
  uint64_t* qkey;  // [kGateWarps][kWarpQueue]
  uint32_t* qy;
  uint64_t* mkey;  // mailboxes [kGateWarps][kSlots][32]
  uint32_t* my;
  uint8_t* lists;  // [kWorkWarps] elite lists (end-of-kernel merge, aliases the ring)
};

// words staged into shared memory: the coarse words in raw mode, else the gate segment
// words staged into shared memory: the whole table (gate words, coarse
// words and every fp64 segment), so neither pass touches L1 or L2 for tables
__host__ __device__ inline int stage_words(const TabLayout& L) { return L.words; }

inline size_t ws_dynamic_bytes(int A, int gate_words, bool smem_gate) {
  return (size_t)kRingBytes + (smem_gate ? (size_t)gate_words * 8 : 0) +
         (size_t)kGateWarps * kWarpQueue * 12 + (size_t)kGateWarps * kSlots * 32 * 12;
}

// fp64 pass over n <= 32 survivors (lane i takes entry i of keys/ys), with
// verdict stores and the optional elite offer. Called by whole warps.
template <bool NEU, bool FULL, bool TOPK, int MODE, bool SMEM_TAB, bool F32 = false>
__device__ __forceinline__ void fp64_batch(const uint64_t* __restrict__ gtab, const TabLayout& L, const EvalMeta& M,
                                        const EvalArgs& a, const TopkArgs& tk, const uint64_t* keys,
                                        const uint32_t* ys, int n, RegList& wl, double& gfloor, double& gpend,
                                        const PackMeta& pk, const float* Tf = nullptr) {
  const int lane = threadIdx.x & 31;
  int64_t idx = 0;
  Decoded c;
  Verdict v;
  v.reason = LS_REASON_DECODE_ERROR;
  v.thr = 0.0;
  if (lane < n) {
    if (MODE == GEN_WORDS && !FULL) {  // raw-mode packed words queue (idx, coarse rank)
      idx = (int64_t)(keys[lane] & ((1ull << 40) - 1));
      rank_split((uint32_t)(keys[lane] >> 40), pk, c);
      c.Y = ys[lane];
    } else {
      unpack_key(keys[lane], ys[lane], idx, c);
    }
    full_path<NEU, !SMEM_TAB, F32>(gtab, L, M, c, v, Tf);  // gtab: the shared-memory copy when SMEM_TAB
    if (a.reason) write_verdict<FULL>(a, idx, v);
  }
  if (TOPK) {  // fused elite: valid survivors offered to this warp's list
    gfloor = fmax(gfloor, gpend);  // the global floor loaded after the previous offer
    Rec r{v.thr, v.thr, tk.index_base + idx, 0};
    const bool ok = lane < n && v.reason == LS_REASON_NONE && r.key >= gfloor && wl.admits(r.key, r.idx, tk.k);
    if (ok) {
      uint64_t code = (uint64_t)c.t * M.code_stride[0] + (uint64_t)c.e * M.code_stride[1] +
                      (uint64_t)c.p * M.code_stride[2] + (uint64_t)c.b * M.code_stride[3];
      for (int h = 4; h < M.A; ++h) code += (uint64_t)((c.Y >> (2 * (h - 4))) & 3u) * M.code_stride[h];
      r.code = code;
    }
    wl.offer(ok, r, tk.k);
    if (__any_sync(0xffffffffu, ok)) {  // the list may have moved: share / refresh the pruning floor
      const double mine = wl.floor_key(tk.k);
      if (lane == 0 && mine > gfloor) raise_floor(tk.floor, mine);
      gfloor = fmax(gfloor, mine);
      gpend = read_floor(tk.floor);  // consumed by the next batch: the L2 round trip overlaps other work
    }
  }
}

// Named barrier 1 over the NW work warps (in eval_ws_kernel the producer warp
// has exited; the sweep kernel has no other warps).
template <int NW>
__device__ __forceinline__ void bar_n() { asm volatile("bar.sync 1, %0;" ::"n"(32 * NW) : "memory"); }
__device__ __forceinline__ void bar_work() { bar_n<kWorkWarps>(); }

// Tree merge of the work warps' register lists through shared slots
// ([NW][32] Rec): log2(NW) levels, warp 0 ends with the merged list. Records
// below the floor (fk, fi) are skipped (at_least()).
template <int NW>
__device__ __forceinline__ void tree_merge(RegList& wl, Rec* slots, int* cnt, int warp, int k, double fk,
                                           int64_t fi = INT64_MAX) {
  wl.store(slots + warp * 32, &cnt[warp]);
  bar_n<NW>();
#pragma unroll 1
  for (int st = 1; st < NW; st <<= 1) {
    if ((warp & (2 * st - 1)) == 0 && warp + st < NW && cnt[warp + st] > 0) {
      wl.absorb(slots + (warp + st) * 32, cnt[warp + st], k, fk, fi);
      wl.store(slots + warp * 32, &cnt[warp]);
    }
    bar_n<NW>();
  }
}

// Exact warp argmax of (key desc, index asc) over the lanes with have set, in
// a handful of REDUX steps instead of a shuffle butterfly: keys are raws
// (finite, > 0), so their IEEE bit patterns order like their values; the
// index (>= 0, unique per record) breaks key ties. Returns the winning lane,
// or -1 when no lane has a record.
__device__ __forceinline__ int warp_argbest(bool have, double key, int64_t idx) {
  constexpr unsigned kAll = 0xffffffffu;
  unsigned c = __ballot_sync(kAll, have);
  if (!c) return -1;
  const unsigned long long kb = (unsigned long long)__double_as_longlong(key);
  const unsigned hi = have ? (unsigned)(kb >> 32) : 0u;
  const unsigned mh = __reduce_max_sync(kAll, hi);
  const bool in1 = have && hi == mh;
  const unsigned lo = in1 ? (unsigned)kb : 0u;
  const unsigned ml = __reduce_max_sync(kAll, lo);
  const bool in2 = in1 && lo == ml;
  c = __ballot_sync(kAll, in2);
  if (__popc(c) == 1) return __ffs(c) - 1;
  const unsigned ih = in2 ? (unsigned)((unsigned long long)idx >> 32) : 0xffffffffu;
  const unsigned mih = __reduce_min_sync(kAll, ih);
  const bool in3 = in2 && ih == mih;
  const unsigned il = in3 ? (unsigned)idx : 0xffffffffu;
  const unsigned mil = __reduce_min_sync(kAll, il);
  return __ffs(__ballot_sync(kAll, in3 && il == mil)) - 1;
}

// One warp merges m staged lists (win[l * stride + j], j < wcnt[l], each
// best-first and free of duplicate vectors) by repeated argmax over the list
// heads: lane l & 31 owns list l and keeps the best head of its lists in
// registers; the winner is emitted unless its vector already was (its best
// occurrence came first), and only the owner lane re-reads its heads.
// k <= 32: lane j holds the code of the j-th emitted record for the dedupe.
__device__ __forceinline__ void warp_merge_lists(const Rec* win, int stride, const int* wcnt, int m, int k,
                                                 ls_elite_rec* out, int32_t* count_out, int* cur, double* hk,
                                                 int64_t* hx, bool stamp = false) {
  const int lane = threadIdx.x & 31;
  // list heads as shared SoA (key, index): a rescan is independent loads
  for (int l = lane; l < m; l += 32) {
    cur[l] = 0;
    const bool h = wcnt[l] > 0;
    hk[l] = h ? win[l * stride].key : -1.0e308;
    hx[l] = h ? win[l * stride].idx : INT64_MAX;
  }
  __syncwarp();
  double bk = -1.0e308;
  int64_t bi = INT64_MAX;
  int bl = -1;
  auto rescan = [&]() {
    bk = -1.0e308;
    bi = INT64_MAX;
    bl = -1;
#pragma unroll 4
    for (int l = lane; l < m; l += 32) {
      const double k_ = hk[l];
      const int64_t i_ = hx[l];
      if (k_ != -1.0e308 && (bl < 0 || better(k_, i_, bk, bi))) {
        bk = k_;
        bi = i_;
        bl = l;
      }
    }
  };
  rescan();
  if (lane == 0 && stamp) LS_STAMP(9);
  uint64_t mine = 0;
  int emitted = 0;
#ifdef LS_DIAG_TIMES
  int rounds = 0;
#endif
  while (emitted < k) {
#ifdef LS_DIAG_TIMES
    ++rounds;
#endif
    const int win_lane = warp_argbest(bl >= 0, bk, bi);
    if (win_lane < 0) break;  // every list is exhausted (warp-uniform)
    const int wl = __shfl_sync(0xffffffffu, bl, win_lane);
    const Rec r = win[wl * stride + cur[wl]];
    if (!__any_sync(0xffffffffu, lane < emitted && mine == r.code)) {
      if (lane == emitted) mine = r.code;
      if (lane == 0) out[emitted] = ls_elite_rec{r.key, r.raw, r.idx, r.code};
      ++emitted;
    }
    __syncwarp();
    if ((wl & 31) == lane) {  // the owner lane advances list wl and rescans its lists
      const int c = cur[wl] + 1;
      cur[wl] = c;
      const bool h = c < wcnt[wl];
      hk[wl] = h ? win[wl * stride + c].key : -1.0e308;
      hx[wl] = h ? win[wl * stride + c].idx : INT64_MAX;
      rescan();
    }
    __syncwarp();
  }
  if (lane == 0) *count_out = emitted;
#ifdef LS_DIAG_TIMES
  if (lane == 0 && stamp) {
    LS_STAMP(10);
    g_diag_t[((blockIdx.x & 255) + 256 * s_diag_launch) & 1023][11] = rounds;
  }
#endif
}

// Final merge of the gridDim.x CTA lists by the last CTA's work warps: lists
// are staged into shared memory a window at a time (one round of coalesced
// L2 loads for the counts, one for the records). When everything fits in one
// window a single warp merges the lists (warp_merge_lists); otherwise the
// window is cut by the exact (key, index) floor, every warp offers its share
// to its own list and the warp lists tree-merge into tk.out.
// NW work warps; smem: REGION bytes of shared memory free for the merge.
template <int NW, uint32_t REGION>
__device__ __forceinline__ void final_merge(RegList& wl, uint8_t* smem, int* cnt, int warp, const TopkArgs& tk) {
  constexpr int kThr = 32 * NW;
  const int lane = threadIdx.x & 31, tid = warp * 32 + lane, k = tk.k, m = (int)gridDim.x;
  Rec* slots = reinterpret_cast<Rec*>(smem);  // [NW][32]
  int* wcnt = reinterpret_cast<int*>(smem + NW * 32 * sizeof(Rec));
  Rec* win = reinterpret_cast<Rec*>(smem + NW * 32 * sizeof(Rec) + 512 * sizeof(int));
  const int cap = (int)((REGION - NW * 32 * sizeof(Rec) - 512 * sizeof(int)) / sizeof(Rec));
  const int lists_per_win = cap / k < 512 ? cap / k : 512;
  __shared__ double s_fk[NW];
  __shared__ int64_t s_fi[NW];
  double fk = m <= lists_per_win ? 0.0 : read_floor(tk.floor);
  int64_t fi = INT64_MAX;
  wl.init();
  for (int l0 = 0; l0 < m; l0 += lists_per_win) {
    const int nl = m - l0 < lists_per_win ? m - l0 : lists_per_win;
    for (int i = tid; i < nl; i += kThr) wcnt[i] = __ldcg(tk.part_counts + l0 + i);
    bar_n<NW>();
    for (int i = tid; i < nl * k; i += kThr) {
      const int l = i / k, j = i - l * k;
      Rec r{-1.0e308, 0.0, INT64_MAX, 0};
      if (j < wcnt[l]) {
        const ls_elite_rec* e = tk.part + (int64_t)(l0 + l) * k + j;
        const double2 kr = __ldcg(reinterpret_cast<const double2*>(e));
        const longlong2 ic = __ldcg(reinterpret_cast<const longlong2*>(e) + 1);
        r = Rec{kr.x, kr.y, (int64_t)ic.x, (uint64_t)ic.y};
      }
      win[i] = r;
    }
    bar_n<NW>();
    if (nl == m) {  // every list is staged: one warp merges them, no block-wide rounds
      if (tid == 0) LS_STAMP(8);
      if (warp == 0) {  // scratch for the heads: the (unused) warp-slot area
        int* cur = reinterpret_cast<int*>(slots);
        double* hk = reinterpret_cast<double*>(smem + 512 * sizeof(int));
        int64_t* hx = reinterpret_cast<int64_t*>(smem + 512 * (sizeof(int) + sizeof(double)));
        warp_merge_lists(win, k, wcnt, m, k, tk.out, tk.count_out, cur, hk, hx, true);
      }
      return;
    }
    // exact (key, index) floor: the best k-th entry of any full list (ties on
    // the key are common — equivalent strategies — and a key-only floor
    // would let them all through to the serial inserts)
    for (int l = tid; l < nl; l += kThr)
      if (wcnt[l] >= k) {
        const Rec& e = win[l * k + k - 1];
        if (better(e.key, e.idx, fk, fi)) {
          fk = e.key;
          fi = e.idx;
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
      s_fk[warp] = fk;
      s_fi[warp] = fi;
    }
    bar_n<NW>();
    for (int o = 0; o < NW; ++o)
      if (better(s_fk[o], s_fi[o], fk, fi)) {
        fk = s_fk[o];
        fi = s_fi[o];
      }
    for (int b = warp * 32; b < nl * k; b += kThr) {
      const int i = b + lane;
      Rec r{0.0, 0.0, 0, 0};
      bool have = false;
      if (i < nl * k) {
        r = win[i];
        have = at_least(r.key, r.idx, fk, fi);  // unused slots carry -inf
      }
      wl.offer(have, r, k);
    }
    bar_n<NW>();
  }
  tree_merge<NW>(wl, slots, cnt, warp, k, fk, fi);
  if (warp == 0) wl.emit(tk.out, tk.count_out);
}


// The final elite block to every sink (the multi-GPU exchange over peer
// memory: each rank's ring slot for this step, peers' rings mapped by CUDA
// IPC): lane j copies record j, then — after a system-scope fence — lane r
// publishes sink r's count | seq << 32 word with a release store, so a reader
// that acquires the word sees the records. Called by warp 0 of the last CTA.
__device__ __noinline__ void sink_copy(const TopkArgs tk) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  __threadfence();
  const int cnt = __ldcg(tk.count_out);
  for (int r = 0; r < tk.nsinks; ++r) {
    uint8_t* dst = tk.sinks[r];
    if (lane < cnt) {
      const int4* src = reinterpret_cast<const int4*>(tk.out + lane);
      int4* d = reinterpret_cast<int4*>(dst + 32 * lane);
      d[0] = __ldcg(src);
      d[1] = __ldcg(src + 1);
    }
  }
  __threadfence_system();
  __syncwarp();
  if (lane < tk.nsinks) {
    const unsigned long long w = (unsigned long long)(uint32_t)cnt | ((unsigned long long)tk.seq << 32);
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(tk.sinks[lane] + 32 * tk.k), "l"(w) : "memory");
  }
}

// End of a fused evaluate + elite kernel (all NW work warps call it): every
// warp's list to shared memory, warp 0 merges them into this CTA's list and
// publishes it; the last CTA to finish merges every CTA's list into tk.out
// and zeroes the sync words for the next call on this scratch.
template <int NW, uint32_t REGION>
__device__ __forceinline__ void elite_epilogue(RegList& wl, uint8_t* region, int* list_count, int warp,
                                               const TopkArgs& tk) {
  Rec* slots = reinterpret_cast<Rec*>(region);
  wl.store(slots + warp * 32, &list_count[warp]);
  bar_n<NW>();
  __shared__ int s_cur[NW];
  __shared__ double s_hk[NW];
  __shared__ int64_t s_hx[NW];
  __shared__ int s_last;
  if (warp == 0) {
    warp_merge_lists(slots, 32, list_count, NW, tk.k, tk.part + (int64_t)blockIdx.x * tk.k,
                     tk.part_counts + blockIdx.x, s_cur, s_hk, s_hx);
    if ((threadIdx.x & 31) == 0) LS_STAMP(5);
    __threadfence();  // this CTA's list is visible device-wide before it is counted
    unsigned t = 0;
    if ((threadIdx.x & 31) == 0) t = atomicAdd(tk.done, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if ((threadIdx.x & 31) == 0) s_last = t == gridDim.x - 1;
  }
  bar_n<NW>();
#ifdef LS_DIAG_NOFINAL
  if (false) {
#else
  if (s_last) {  // the last CTA merges every CTA's list (L2-resident, no second launch)
#endif
    if (warp == 0 && (threadIdx.x & 31) == 0) LS_STAMP(6);
    __threadfence();
    final_merge<NW, REGION>(wl, region, list_count, warp, tk);
    if (tk.nsinks > 0 && warp == 0) sink_copy(tk);
    if (warp == 0 && (threadIdx.x & 31) == 0) {
      LS_STAMP(7);
      // every other CTA is past its last floor read and done increment:
      // leave the sync words zero for the next call on this scratch
      *tk.floor = 0ull;
      *tk.done = 0u;
      if (tk.tile_ctr) *tk.tile_ctr = 0u;
      if (tk.signal) {  // the elite is complete: release it (the word may be host-mapped memory)
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(tk.signal), "r"(tk.seq) : "memory");
      }
    }
  }
}

template <bool NEU, bool FULL, bool SMEM_GATE, bool TOPK, int MODE>
__global__ void __launch_bounds__(kThreads, LS_MIN_BLOCKS)
    eval_ws_kernel(const uint64_t* __restrict__ gtab, const TabLayout L, const EvalMeta M, const EvalArgs a,
                   const int64_t ntiles, const TopkArgs tk, const GenMeta gm) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int NST = Ring<MODE>::stages;
  constexpr uint32_t STB = Ring<MODE>::stage_bytes;
  __shared__ __align__(8) uint64_t full_bar[kMaxStages];
  __shared__ __align__(8) uint64_t empty_bar[kMaxStages];
  __shared__ __align__(8) uint64_t gate_bar;
  __shared__ volatile int64_t stage_tile[kMaxStages];  // tile in each ring stage; -1 ends the stream
  __shared__ int mb_n[kGateWarps][kSlots];
  __shared__ volatile int mb_state[kGateWarps][kSlots];  // 0 empty, 1 full
  __shared__ volatile int gates_done;
  __shared__ int list_count[kWorkWarps];
  __shared__ volatile uint32_t mb_pending[kFpWarps];  // full mailboxes per fp64 warp (bitmask)
  const int A = M.A;
  const uint32_t stage_bytes = (uint32_t)A * kTile;  // bytes the producer copies per stage
  WsSmem S;
  S.ring = smem;
  S.gate = reinterpret_cast<uint64_t*>(smem + kRingBytes);
  S.qkey = SMEM_GATE ? S.gate + stage_words(L) : S.gate;
  const uint64_t* T = SMEM_GATE ? S.gate : gtab;  // the table the fp64 pass reads
  const bool coarse = !FULL && L.coarse_words > 0;
  const uint32_t* Cg = reinterpret_cast<const uint32_t*>((SMEM_GATE ? S.gate : gtab) + L.coarse);
  S.qy = reinterpret_cast<uint32_t*>(S.qkey + kGateWarps * kWarpQueue);
  S.mkey = reinterpret_cast<uint64_t*>(S.qy + kGateWarps * kWarpQueue);
  S.my = reinterpret_cast<uint32_t*>(S.mkey + kGateWarps * kSlots * 32);
  S.lists = S.ring;  // end-of-kernel elite merges reuse the drained ring
  static_assert(kWorkWarps * 32 * sizeof(Rec) + 512 * sizeof(int) + 64 * sizeof(Rec) <= kRingBytes,
                "elite slots and a merge window fit in the ring");
  const uint64_t* Gt = SMEM_GATE ? S.gate : gtab;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const uint32_t ring_base = smem_u32(S.ring);
  // plane slices >= A are never written by the TMA: zero them once so the
  // gate warps can load all 16 unconditionally (zero = in range, UNSHARDED)
  if (MODE == GEN_PLANES)
    for (int s = 0; s < NST; ++s)
      for (int o = A * kTile + 16 * (int)threadIdx.x; o < (int)kStageBytes; o += 16 * kThreads)
        *reinterpret_cast<uint4*>(S.ring + s * kStageBytes + o) = make_uint4(0, 0, 0, 0);
  if (threadIdx.x < kGateWarps * kSlots) mb_state[threadIdx.x / kSlots][threadIdx.x % kSlots] = 0;
  if (threadIdx.x < kFpWarps) mb_pending[threadIdx.x] = 0;
  if (threadIdx.x < kWorkWarps) list_count[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    gates_done = 0;
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kGateWarps);
    }
    mbar_init(&gate_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
#ifdef LS_DIAG_TIMES
  diag_enter();
#endif
  if (threadIdx.x == 0) LS_STAMP(0);

  if (warp == kWorkWarps) {  // ---------------- producer warp
    if (lane == 0) {
      if (SMEM_GATE) {
        const uint32_t bytes = (uint32_t)stage_words(L) * 8u;
        mbar_expect_tx(&gate_bar, bytes);
        bulk_g2s(S.gate, gtab, bytes, &gate_bar);
      }
      // tiles 0..ntiles-1 are whole (TMA); tile ntiles is the ragged tail
      // (< kTile candidates, read by the gate warps directly). Each CTA takes
      // tile blockIdx.x first; later tiles come from the launch's claim
      // counter (tk.tile_ctr: a CTA that starts late — e.g. behind the
      // previous launch's final merge under PDL — simply claims fewer) or,
      // without one, every gridDim.x-th tile. Stage tile -1 ends the stream.
      // Claims are groups of G consecutive tiles (G = 2 with the counter, so
      // one atomic round trip hides behind ~1.7 µs of streaming), and the next
      // group's claim is issued when the current group starts.
      const int64_t last = a.n > ntiles * kTile ? ntiles : ntiles - 1;
      // The last LS_LATE_CTAS CTAs claim even their first group: under PDL the
      // highest block indices are dispatched last, onto the SMs the previous
      // launch frees last (its final merge), and a static group there would
      // finish last in a short launch.
      const int G = tk.tile_ctr ? LS_CLAIM_GROUP : 1;
      const int64_t nstat = !tk.tile_ctr ? (int64_t)gridDim.x
                                         : gridDim.x > LS_LATE_CTAS ? (int64_t)gridDim.x - LS_LATE_CTAS : 0;
      int64_t grp = blockIdx.x < nstat ? (int64_t)blockIdx.x : nstat + atomicAdd(tk.tile_ctr, 1u);
      int64_t nxt = tk.tile_ctr ? nstat + atomicAdd(tk.tile_ctr, 1u) : grp + gridDim.x;
      int j = 0;
      for (int i = 0; MODE == GEN_PLANES || MODE == GEN_WORDS; ++i) {
        const int s = i % NST, k = i / NST;
        if (k > 0) mbar_wait(&empty_bar[s], (uint32_t)((k - 1) & 1));
        const int64_t tile = grp * G + j;
        const bool valid = tile <= last;
        stage_tile[s] = valid ? tile : -1;
        if (!valid || tile == ntiles) {  // end marker or the ragged tail: no copy
          mbar_arrive(&full_bar[s]);
          if (!valid) break;
        } else if (MODE == GEN_WORDS) {  // one contiguous 16 KB tile of candidate words
          mbar_expect_tx(&full_bar[s], 8u * kTile);
          bulk_g2s_stream(S.ring + s * STB, a.words + tile * kTile, 8u * kTile, &full_bar[s]);
        } else {
          mbar_expect_tx(&full_bar[s], stage_bytes);
          const uint8_t* src = a.planes + tile * kTile;
          uint8_t* dst = S.ring + s * STB;
          for (int h = 0; h < A; ++h) bulk_g2s(dst + h * kTile, src + (int64_t)h * a.stride, kTile, &full_bar[s]);
        }
        if (++j == G || tile == last) {  // next group (its claim was issued a group ago)
          j = 0;
          grp = nxt;
          nxt = tk.tile_ctr ? nstat + atomicAdd(tk.tile_ctr, 1u) : grp + gridDim.x;
        }
      }
    }
    return;
  }

  RegList wl;  // this warp's elite list, one entry per lane
  wl.init();
  double gfloor = -1.0e308;  // cached global pruning floor (raw keys are >= 0)
  double gpend = -1.0e308;   // in-flight read of the global floor

  if (warp >= kGateWarps) {  // ---------------- fp64 warps: drain the mailboxes
    const int f = warp - kGateWarps;
    if (SMEM_GATE) mbar_wait(&gate_bar, 0);  // the staged table they read
    unsigned backoff = LS_BACKOFF_MAX < 128 ? LS_BACKOFF_MAX : 128;  // ns; idle fp64 warps back off so gate warps keep the issue slots
    for (;;) {
      // one shared word per fp64 warp: bit (g / kFpWarps) * kSlots + slot set
      // for every full mailbox of its gate warps g = f, f + kFpWarps, ...
      uint32_t pend = __shfl_sync(0xffffffffu, mb_pending[f], 0);
      if (pend) {
        __threadfence_block();
        while (pend) {
          const int bit = __ffs(pend) - 1;
          pend &= pend - 1;
          // claim the batch (its gate warp may take it back once it is done)
          uint32_t old = 0;
          if (lane == 0) old = atomicAnd((uint32_t*)&mb_pending[f], ~(1u << bit));
          if (!((__shfl_sync(0xffffffffu, old, 0) >> bit) & 1u)) continue;
          const int g = f + kFpWarps * (bit / kSlots), sl = bit % kSlots;
          const int base = (g * kSlots + sl) * 32;
          fp64_batch<NEU, FULL, TOPK, MODE, SMEM_GATE>(T, L, M, a, tk, S.mkey + base, S.my + base, mb_n[g][sl], wl,
                                                       gfloor, gpend, gm.pk);
          __syncwarp();
          if (lane == 0) {
            __threadfence_block();
            mb_state[g][sl] = 0;
          }
          __syncwarp();
        }
        backoff = LS_BACKOFF_MAX < 128 ? LS_BACKOFF_MAX : 128;
      } else if (gates_done == kGateWarps) {
        __threadfence_block();  // gate warps finished: one last look at the mailboxes
        if (__shfl_sync(0xffffffffu, mb_pending[f], 0) == 0) {
          if (f == 0 && lane == 0) LS_STAMP(3);
          break;
        }
      } else {
        __nanosleep(backoff);
        backoff = backoff < LS_BACKOFF_MAX ? 2 * backoff : LS_BACKOFF_MAX;
      }
    }
  } else {  // ---------------- gate warps
    uint64_t* qkey = S.qkey + warp * kWarpQueue;
    uint32_t* qy = S.qy + warp * kWarpQueue;
    int qcount = 0;  // warp-uniform
    if (SMEM_GATE) mbar_wait(&gate_bar, 0);
    if (threadIdx.x == 0) LS_STAMP(1);

    // hand the newest n (<= 32) queue entries to a free mailbox slot, or
    // score them here when both slots are still busy
    auto flush = [&](int n) {
      __syncwarp();
      const int pos0 = qcount - n;
      int slot = -1;
      for (int sl = 0; sl < kSlots && slot < 0; ++sl)
        if (mb_state[warp][sl] == 0) slot = sl;
      if (slot >= 0) {
        __threadfence_block();
        const int base = (warp * kSlots + slot) * 32;
        if (lane < n) {
          S.mkey[base + lane] = qkey[pos0 + lane];
          S.my[base + lane] = qy[pos0 + lane];
        }
        __syncwarp();
        if (lane == 0) {
          mb_n[warp][slot] = n;
          __threadfence_block();
          mb_state[warp][slot] = 1;
          atomicOr((uint32_t*)&mb_pending[warp % kFpWarps], 1u << ((warp / kFpWarps) * kSlots + slot));
        }
      } else {
        fp64_batch<NEU, FULL, TOPK, MODE, SMEM_GATE>(T, L, M, a, tk, qkey + pos0, qy + pos0, n, wl, gfloor, gpend, gm.pk);
      }
      qcount -= n;
      __syncwarp();
    };

    // gate pass over this lane's 4 decoded candidates (stream indices base..)
    // ranks: coarse ranks of the 4 candidates when the candidates came as
    // packed words (t, e, p, b then split only where needed)
    // whole: a full tile (every lane of the warp has count 4)
    auto pass_a = [&](Decoded* cs, uint32_t badb, int64_t base, int count, const uint32_t* ranks, bool whole) {
      uint32_t r4 = 0, reason[4];
      double m[4];
      // the 4 gate evaluations are independent: issue them back to back (ILP)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool dbad = ((badb >> (8 * j)) & 0xffu) != 0;
        if (MODE == GEN_WORDS) {
          const uint32_t rk = dbad ? 0u : ranks[j];  // keep the branch-free lookups in range
          if (coarse) {
            reason[j] = gate_rank(Cg, M, rk, cs[j].Y);
            m[j] = 0.0;
          } else {
            rank_split(rk, gm.pk, cs[j]);
            reason[j] = gate(Gt, L, M, cs[j], m[j]);
          }
        } else {
          if (dbad) cs[j].t = cs[j].e = cs[j].p = cs[j].b = 0;  // keep the branch-free lookups in range
          if (coarse) {
            reason[j] = gate_coarse(Cg, L, M, cs[j]);
            m[j] = 0.0;
          } else {
            reason[j] = gate(Gt, L, M, cs[j], m[j]);
          }
        }
        if (dbad) {
          reason[j] = LS_REASON_DECODE_ERROR;
          m[j] = 0.0;
        }
        r4 |= reason[j] << (8 * j);
      }
      // then compact the survivors (~1% of a uniform batch) into the warp
      // queue: the lane's survivor count 0..4 as three ballots gives every
      // lane its queue position and the warp total in one step
      // survivors = zero reason bytes of r4 (SWAR), within the lane's count
      const uint32_t zb = __vcmpeq4(r4, 0u) & (count >= 4 ? 0xffffffffu : (1u << (8 * count)) - 1u);
      const uint32_t nsv = __popc(zb) >> 3;
      const uint32_t b0 = __ballot_sync(0xffffffffu, nsv & 1u), b1 = __ballot_sync(0xffffffffu, nsv & 2u),
                     b2 = __ballot_sync(0xffffffffu, nsv & 4u);
      if (b0 | b1 | b2) {
        const uint32_t lt = (1u << lane) - 1u;
        int pos = qcount + __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (zb & (1u << (8 * j))) {
            qkey[pos] = (MODE == GEN_WORDS && !FULL) ? (uint64_t)(base + j) | ((uint64_t)ranks[j] << 40)
                                                     : pack_key(base + j, cs[j]);
            qy[pos] = cs[j].Y;
            ++pos;
          }
        qcount += __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
      }
      if (!a.reason) {
        // sweep mode: no per-candidate verdicts, only the fused elite
      } else if (whole) {
        st_reason4(a.reason + base, r4);
        // zero fields: the warp's 128 consecutive doubles as two fully
        // coalesced 512-byte stores (every lane of a full tile has count 4;
        // survivors' values are stored later by the fp64 pass)
        const int64_t wz = base - 4 * lane + 2 * lane;
        if (a.thr && !a.sparse_thr) {
          st2(a.thr, wz, 0.0, 0.0);
          st2(a.thr, wz + 64, 0.0, 0.0);
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
              st2(zf[f], wz, 0.0, 0.0);
              st2(zf[f], wz + 64, 0.0, 0.0);
            }
        }
      } else {
        for (int j = 0; j < count; ++j) {
          a.reason[base + j] = (uint8_t)(r4 >> (8 * j));
          if (a.thr && !a.sparse_thr) a.thr[base + j] = 0.0;
          if (FULL) {
            if (a.mem) a.mem[base + j] = m[j];
            if (a.tpot) a.tpot[base + j] = 0.0;
            if (a.comp) a.comp[base + j] = 0.0;
            if (a.comm) a.comm[base + j] = 0.0;
            if (a.pipe) a.pipe[base + j] = 0.0;
          }
        }
      }
      while (qcount >= 32) flush(32);
    };

    const int lane_off = warp * kWarpCands + 4 * lane;
    bool tail = false;  // this CTA drew the ragged tail tile
    if (MODE == GEN_PLANES) {
      for (int i = 0;; ++i) {
        const int s = i % NST;
        mbar_wait(&full_bar[s], (uint32_t)((i / NST) & 1));
        const int64_t tile = stage_tile[s];
        if (tile < 0) break;
        if (tile == ntiles) {  // ragged tail: processed after the stream (cold code off the hot loop)
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_bar[s]);
          tail = true;
          continue;
        }
        uint32_t w[16];
        const uint32_t st = ring_base + (uint32_t)s * STB + (uint32_t)lane_off;
#pragma unroll
        for (int h = 0; h < 16; ++h) w[h] = lds_u32(st + h * kTile);  // planes >= A are zero-filled
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[s]);
        uint32_t q[3];
        const uint32_t badb = swar_decode(w, M, q);
        Decoded cs[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) extract(w, q, j, cs[j]);
        pass_a(cs, badb, tile * kTile + lane_off, 4, nullptr, true);
      }
      if (tail) {  // ragged tail (< one tile), read directly
        const int64_t base = ntiles * kTile + lane_off;
        const int count = base < a.n ? (a.n - base < 4 ? (int)(a.n - base) : 4) : 0;
        uint32_t w[16];
#pragma unroll
        for (int h = 0; h < 16; ++h) {
          w[h] = 0;
          if (h < A)
            for (int j = 0; j < count; ++j) w[h] |= (uint32_t)a.planes[(int64_t)h * a.stride + base + j] << (8 * j);
        }
        uint32_t q[3];
        const uint32_t badb = swar_decode(w, M, q);
        Decoded cs[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) extract(w, q, j, cs[j]);
        pass_a(cs, badb, base, count, nullptr, false);
      }
    } else if (MODE == GEN_WORDS) {  // 4 consecutive 8-byte candidate words per lane
      // shared addresses hoisted out of the loop (barriers are 8 B apart)
      const uint32_t st0 = ring_base + 8u * (uint32_t)lane_off;
      const uint32_t fb0 = smem_u32(&full_bar[0]), eb0 = smem_u32(&empty_bar[0]);
      for (int i = 0;; ++i) {
        const uint32_t s = (uint32_t)(i % NST);
        mbar_wait_a(fb0 + 8u * s, (uint32_t)((i / NST) & 1));
        const int64_t tile = stage_tile[s];
        if (tile < 0) break;
        if (tile == ntiles) {  // ragged tail: processed after the stream (cold code off the hot loop)
          __syncwarp();
          if (lane == 0) mbar_arrive_a(eb0 + 8u * s);
          tail = true;
          continue;
        }
        uint64_t w[4];
        const uint32_t st = st0 + s * STB;
        lds_u64x2(st, w[0], w[1]);
        lds_u64x2(st + 16, w[2], w[3]);
        __syncwarp();
        if (lane == 0) mbar_arrive_a(eb0 + 8u * s);
        Decoded cs[4];
        uint32_t badb = 0, rk[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) badb |= word_decode(w[j], gm.pk, rk[j], cs[j].Y) << (8 * j);
        pass_a(cs, badb, tile * kTile + lane_off, 4, rk, true);
      }
      if (tail) {  // ragged tail (< one tile), read directly
        const int64_t base = ntiles * kTile + lane_off;
        const int count = base < a.n ? (a.n - base < 4 ? (int)(a.n - base) : 4) : 0;
        Decoded cs[4];
        uint32_t badb = 0, rk[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          badb |= word_decode(j < count ? a.words[base + j] : 0ull, gm.pk, rk[j], cs[j].Y) << (8 * j);
        pass_a(cs, badb, base, count, rk, false);
      }
    } else {  // candidates generated in registers: nothing read from HBM
      const int64_t gtiles = (a.n + kTile - 1) / kTile;
      for (int64_t tile = blockIdx.x; tile < gtiles; tile += gridDim.x) {
        const int64_t base = tile * kTile + lane_off;
        const int count = base < a.n ? (a.n - base < 4 ? (int)(a.n - base) : 4) : 0;
        Decoded cs[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)  // past-the-end lanes regenerate the last valid index (never enqueued)
          gen_candidate<MODE>(gm, (uint64_t)(gm.start + (base + j < a.n ? base + j : a.n - 1)), cs[j]);
        pass_a(cs, 0u, base, count, nullptr, false);
      }
    }
    if (qcount > 0) flush(qcount);
    __syncwarp();
    // take back this warp's mailbox batches no fp64 warp has claimed yet, so
    // the end-of-stream backlog is shared by all work warps
    for (int sl = 0; sl < kSlots; ++sl) {
      const int bit = (warp / kFpWarps) * kSlots + sl;
      uint32_t old = 0;
      if (lane == 0) old = atomicAnd((uint32_t*)&mb_pending[warp % kFpWarps], ~(1u << bit));
      if ((__shfl_sync(0xffffffffu, old, 0) >> bit) & 1u) {
        const int base = (warp * kSlots + sl) * 32;
        fp64_batch<NEU, FULL, TOPK, MODE, SMEM_GATE>(T, L, M, a, tk, S.mkey + base, S.my + base, mb_n[warp][sl], wl,
                                                     gfloor, gpend, gm.pk);
        __syncwarp();
        if (lane == 0) mb_state[warp][sl] = 0;
        __syncwarp();
      }
    }
    if (threadIdx.x == 0) LS_STAMP(2);
    if (lane == 0) {
      __threadfence_block();
      atomicAdd((int*)&gates_done, 1);
    }
  }

  if (TOPK) {
    // (named barrier 1 over the work warps: the producer warp is gone)
    Rec* slots = reinterpret_cast<Rec*>(S.lists);
    // the lists live in the ring: every gate warp must be past its last stage
    bar_work();
    if (threadIdx.x == 0) LS_STAMP(4);
    // every warp's list (best-first, distinct vectors) to shared memory; warp 0
    // merges the kWorkWarps lists into this CTA's list (one list per lane)
    (void)slots;
    // Programmatic dependent launch: this CTA's verdicts are written; the
    // next launch on the stream (the next step) may start on SMs as they
    // free up. Before its elite epilogue each CTA waits for the previous
    // launch to complete (its last CTA's merge and tk.out writes, which may
    // share buffers with this one). Both are no-ops without PDL.
    __threadfence();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    elite_epilogue<kWorkWarps, kRingBytes>(wl, S.ring, list_count, warp, tk);
  }
}

// ---- sweep_kernel: on-device candidate streams -> elite --------------------
// The generated-candidate sweeps (ls_sweep: uniform stream, full and
// admissible enumeration) read nothing per candidate, and in the enumeration
// modes most candidates survive the gates (~60% of the admissible space takes
// the full fp64 plan walk), so the warp-specialised streaming design of
// eval_ws_kernel (TMA ring, gate warps handing survivors to a few fp64 warps
// through mailboxes) does not fit. Here every warp does everything: it
// generates 32 consecutive stream positions at a time (one per lane), gates
// them from the shared-memory coarse words, appends the survivors to its own
// shared-memory queue and scores 32 queued survivors at once in place
// (full_path from the shared-memory table), offering the valid ones to its
// register elite list. No ring, no mailboxes, no idle roles; one CTA of
// sw_warps<MODE>() warps per SM.
#ifndef LS_SWEEP_WARPS
#define LS_SWEEP_WARPS 24  // admissible enumeration: survivor-heavy, registers matter
#endif
#ifndef LS_SWEEP_WARPS_SPARSE
#define LS_SWEEP_WARPS_SPARSE 32  // uniform / full enumeration: most candidates fail the gates
#endif
#ifndef LS_SWEEP_CTAS
#define LS_SWEEP_CTAS 1  // CTAs per SM (each stages its own tables)
#endif
// Warps per sweep CTA by stream: 24 (80 registers) for the admissible
// enumeration, where ~60 % of positions take the fp64 walk; 32 (64 registers)
// for the uniform stream and the full enumeration, where most positions fail
// the gates and more warps hide more latency (1.2T: admissible 0.482 vs 0.503
// ms, full 5.95 vs 6.27 ms, uniform 2^30 8.17 vs 8.25 ms).
template <int MODE>
__host__ __device__ constexpr int sw_warps() {
  return MODE == GEN_ENUM_ADMISSIBLE ? LS_SWEEP_WARPS : LS_SWEEP_WARPS_SPARSE;
}
constexpr int kSwWarpsMax = LS_SWEEP_WARPS > LS_SWEEP_WARPS_SPARSE ? LS_SWEEP_WARPS : LS_SWEEP_WARPS_SPARSE;
inline int sw_warps_of(int mode) {
  return mode == GEN_ENUM_ADMISSIBLE ? sw_warps<GEN_ENUM_ADMISSIBLE>() : sw_warps<GEN_ENUM>();
}
constexpr int kSwChunk = 256;  // consecutive stream positions per warp chunk
constexpr int kSwQueue = 64;   // survivor queue per warp (< 32 left over + 32 new)
constexpr uint32_t kSwMergeBytes = 64 * 1024;  // shared memory the end-of-kernel merges use (aliases the tables)
static_assert(kSwWarpsMax * 32 * sizeof(Rec) + 512 * sizeof(int) + 64 * sizeof(Rec) <= kSwMergeBytes, "merge region");

// Shared-memory layout of sweep_kernel: workload table, the stream's two
// axis tables, per-warp survivor queues.
struct SwLayout {
  uint32_t tab, tabf, gen_hi, gen_lo, qkey, qy, bytes;
};
// f32: the fp32 fast mode also stages the fp32 copy of the tables
__host__ __device__ inline uint32_t tabf_bytes(const TabLayout& L) { return ((uint32_t)L.words * 4u + 15u) & ~15u; }
__host__ __device__ inline SwLayout sw_layout(const TabLayout& L, uint32_t hi_size, uint32_t lo_size, int nw,
                                              bool f32 = false) {
  SwLayout o;
  o.tab = 0;
  o.tabf = (uint32_t)L.words * 8u;
  o.gen_hi = o.tabf + (f32 ? tabf_bytes(L) : 0u);
  o.gen_lo = o.gen_hi + 4u * hi_size;
  o.qkey = (o.gen_lo + 4u * lo_size + 15u) & ~15u;
  o.qy = o.qkey + 8u * (uint32_t)nw * kSwQueue;
  o.bytes = o.qy + 4u * (uint32_t)nw * kSwQueue;
  if (o.bytes < kSwMergeBytes) o.bytes = kSwMergeBytes;
  return o;
}

// Coarse rank -> (t, e, p, b) with the stream's divisors (batch fastest).
__device__ __forceinline__ void rank_split_g(const GenMeta& g, uint64_t coarse, Decoded& c) {
  const uint64_t q1 = divq(coarse, g.m_b, g.nb);
  c.b = (int)(coarse - q1 * g.nb);
  const uint64_t q2 = divq(q1, g.m_p, g.np);
  c.p = (int)(q1 - q2 * g.np);
  const uint64_t q3 = divq(q2, g.m_e, g.ne);
  c.e = (int)(q2 - q3 * g.ne);
  c.t = (int)q3;
}

// gen_candidate with the axis tables in shared memory.
template <int MODE>
__device__ __forceinline__ void gen_candidate_s(const GenMeta& g, const uint32_t* hi_tab, const uint32_t* lo_tab,
                                                uint64_t gidx, Decoded& c) {
  uint64_t coarse, axis;
  if (MODE == GEN_UNIFORM) {
    const uint64_t r1 = splitmix64(g.seed ^ (2 * gidx)), r2 = splitmix64(g.seed ^ (2 * gidx + 1));
    coarse = __umul64hi(r1, g.coarse_size);
    axis = __umul64hi(r2, g.axis_size);
  } else {
    coarse = divq(gidx, g.m_axis, g.axis_size);
    axis = gidx - coarse * g.axis_size;
  }
  const uint64_t hi = divq(axis, g.m_lo, g.lo_size), lo = axis - hi * g.lo_size;
  c.Y = hi_tab[hi] | lo_tab[lo];
  const uint64_t q1 = divq(coarse, g.m_b, g.nb);
  c.b = (int)(coarse - q1 * g.nb);
  const uint64_t q2 = divq(q1, g.m_p, g.np);
  c.p = (int)(q1 - q2 * g.np);
  const uint64_t q3 = divq(q2, g.m_e, g.ne);
  c.e = (int)(q2 - q3 * g.ne);
  c.t = (int)q3;
}

template <bool NEU, int MODE, bool F32>
__global__ void __launch_bounds__(32 * sw_warps<MODE>(), LS_SWEEP_CTAS)
    sweep_kernel(const uint64_t* __restrict__ gtab, const TabLayout L, const EvalMeta M, const int64_t n,
                 const TopkArgs tk, const GenMeta gm, const SwLayout SL, const float* __restrict__ gtabf) {
  constexpr int kSwWarps = sw_warps<MODE>();
  constexpr int kSwThreads = 32 * kSwWarps;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t tab_bar;
  __shared__ int list_count[kSwWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* T = reinterpret_cast<uint64_t*>(smem + SL.tab);
  float* Tf = F32 ? reinterpret_cast<float*>(smem + SL.tabf) : nullptr;
  uint32_t* hi_s = reinterpret_cast<uint32_t*>(smem + SL.gen_hi);
  uint32_t* lo_s = reinterpret_cast<uint32_t*>(smem + SL.gen_lo);
  uint64_t* qkey = reinterpret_cast<uint64_t*>(smem + SL.qkey) + warp * kSwQueue;
  uint32_t* qy = reinterpret_cast<uint32_t*>(smem + SL.qy) + warp * kSwQueue;
  if (threadIdx.x == 0) {
    mbar_init(&tab_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint32_t bytes = (uint32_t)L.words * 8u;
    mbar_expect_tx(&tab_bar, bytes + (F32 ? tabf_bytes(L) : 0u));
    bulk_g2s(T, gtab, bytes, &tab_bar);
    if (F32) bulk_g2s(Tf, gtabf, tabf_bytes(L), &tab_bar);
  }
  if (threadIdx.x < kSwWarps) list_count[threadIdx.x] = 0;
  const uint32_t hi_size = (uint32_t)(gm.axis_size / gm.lo_size);
  for (uint32_t i = threadIdx.x; i < hi_size; i += kSwThreads) hi_s[i] = gm.hi_tab[i];
  for (uint32_t i = threadIdx.x; i < (uint32_t)gm.lo_size; i += kSwThreads) lo_s[i] = gm.lo_tab[i];
  __syncthreads();
  mbar_wait(&tab_bar, 0);
  if (threadIdx.x == 0) LS_STAMP(1);

  const uint32_t* Cg = reinterpret_cast<const uint32_t*>(T + L.coarse);
  const bool coarse = L.coarse_words > 0;
  EvalArgs a{};  // no per-candidate verdicts: only the elite leaves the SM
  RegList wl;
  wl.init();
  double gfloor = -1.0e308, gpend = -1.0e308;
  int qcount = 0;  // warp-uniform
  const uint32_t lt = (1u << lane) - 1u;
  const int64_t nchunks = (n + kSwChunk - 1) / kSwChunk;
  const uint32_t lo_size = (uint32_t)gm.lo_size;
  // chunks: each warp's first one static, the rest claimed from the launch's
  // counter (survivor-heavy chunks cost several times the others, so a static
  // deal leaves SMs idle at the end); the next claim is issued a chunk ahead
  const int64_t nwarps = (int64_t)gridDim.x * kSwWarps;
  uint32_t claim = 0;  // lane 0: the claim in flight (read a whole chunk later)
  if (lane == 0) claim = atomicAdd(tk.tile_ctr, 1u);
  for (int64_t ch = (int64_t)blockIdx.x * kSwWarps + warp; ch < nchunks;) {
    const int64_t base = ch * kSwChunk;
    // enumeration: decode the lane's first position once, then step the
    // mixed-radix digits (coarse rank, high / low axis rank) by 32 per round
    uint64_t crank = 0;
    uint32_t ahi = 0, alo = 0;
    Decoded c;
    if (MODE != GEN_UNIFORM) {
      const int64_t i0 = base + lane < n ? base + lane : n - 1;
      const uint64_t g0 = (uint64_t)(gm.start + i0);
      crank = divq(g0, gm.m_axis, gm.axis_size);
      const uint64_t axis = g0 - crank * gm.axis_size;
      const uint64_t hi = divq(axis, gm.m_lo, gm.lo_size);
      ahi = (uint32_t)hi;
      alo = (uint32_t)(axis - hi * gm.lo_size);
      rank_split_g(gm, crank, c);
    }
#pragma unroll 1
    for (int j = 0; j < kSwChunk / 32; ++j) {
      const int64_t i = base + j * 32 + lane;
      const bool in = i < n;
      if (MODE == GEN_UNIFORM) {
        if (coarse) {  // the coarse rank indexes the gate words directly: (t, e, p, b) only for survivors
          const uint64_t gi = (uint64_t)(gm.start + (in ? i : n - 1));
          const uint64_t r1 = splitmix64(gm.seed ^ (2 * gi)), r2 = splitmix64(gm.seed ^ (2 * gi + 1));
          crank = __umul64hi(r1, gm.coarse_size);
          const uint64_t axis = __umul64hi(r2, gm.axis_size);
          const uint64_t hi = divq(axis, gm.m_lo, gm.lo_size);
          c.Y = hi_s[hi] | lo_s[axis - hi * gm.lo_size];
        } else {
          gen_candidate_s<MODE>(gm, hi_s, lo_s, (uint64_t)(gm.start + (in ? i : n - 1)), c);
        }
      } else {
        if (j > 0 && in) {  // advance by 32 positions (past-the-end lanes keep their last candidate)
          alo += 32;
          while (alo >= lo_size) {
            alo -= lo_size;
            if (++ahi * gm.lo_size >= gm.axis_size) {
              ahi = 0;
              rank_split_g(gm, ++crank, c);
            }
          }
        }
        c.Y = hi_s[ahi] | lo_s[alo];
      }
      uint32_t reason;
      if (coarse) {
        reason = gate_rank(Cg, M, (uint32_t)crank, c.Y);
      } else {
        double m;
        reason = gate(T, L, M, c, m);
      }
      const bool sv = in && reason == LS_REASON_NONE;
      const uint32_t b = __ballot_sync(0xffffffffu, sv);
      if (b) {
        if (sv) {
          if (MODE == GEN_UNIFORM && coarse) rank_split_g(gm, crank, c);
          const int pos = qcount + __popc(b & lt);
          qkey[pos] = pack_key(i, c);
          qy[pos] = c.Y;
        }
        qcount += __popc(b);
        if (qcount >= 32) {  // score the newest 32 in place
          __syncwarp();
          qcount -= 32;
          fp64_batch<NEU, false, true, MODE, true, F32>(T, L, M, a, tk, qkey + qcount, qy + qcount, 32, wl, gfloor,
                                                       gpend, gm.pk, Tf);
          __syncwarp();
        }
      }
    }
    ch = nwarps + __shfl_sync(0xffffffffu, claim, 0);
    if (ch < nchunks && lane == 0) claim = atomicAdd(tk.tile_ctr, 1u);
  }
  if (qcount > 0) {
    __syncwarp();
    fp64_batch<NEU, false, true, MODE, true, F32>(T, L, M, a, tk, qkey, qy, qcount, wl, gfloor, gpend, gm.pk, Tf);
  }
  if (threadIdx.x == 0) LS_STAMP(2);
  bar_n<kSwWarps>();  // the merge region aliases the tables every warp reads until here
  elite_epilogue<kSwWarps, kSwMergeBytes>(wl, smem, list_count, warp, tk);
}

template <bool NEU, int MODE>
void launch_sweep_t(const LaunchPlan& lp, const uint64_t* tab, const TabLayout& L, const EvalMeta& M, int64_t n,
                    const TopkArgs& tk, const GenMeta& gm, cudaStream_t s) {
  const bool f32 = lp.tabf != nullptr;
  constexpr int NT = 32 * sw_warps<MODE>();
  const SwLayout SL = sw_layout(L, (uint32_t)(gm.axis_size / gm.lo_size), (uint32_t)gm.lo_size, sw_warps<MODE>(), f32);
  const int64_t blocks = sweep_grid(lp, n, MODE);
  if (f32)  // plain fp32 sums: the NEU flag does not apply
    sweep_kernel<false, MODE, true><<<(unsigned)blocks, NT, SL.bytes, s>>>(tab, L, M, n, tk, gm, SL, lp.tabf);
  else
    sweep_kernel<NEU, MODE, false><<<(unsigned)blocks, NT, SL.bytes, s>>>(tab, L, M, n, tk, gm, SL, nullptr);
}

// One candidate per thread, any alignment, any A <= LS_MAX_HEADS.
template <bool NEU>
__global__ void __launch_bounds__(kGenericThreads) eval_generic_kernel(const uint64_t* __restrict__ gtab,
                                                                       const TabLayout L, const EvalMeta M,
                                                                       const EvalArgs a) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t bad = 0, Y = 0;
    int idx[4] = {0, 0, 0, 0};
    for (int h = 0; h < M.A; ++h) {
      const uint32_t byte = a.planes[(int64_t)h * a.stride + i];
      bad |= byte >= M.head_size[h];
      if (h < 4) {
        idx[h & 3] = (int)byte;
      } else {
        const int slot = M.head_slot[h];
        if (slot >= 0) Y |= (byte & 3u) << (2 * slot);
      }
    }
    Decoded c;
    c.t = idx[0];
    c.e = idx[1];
    c.p = idx[2];
    c.b = idx[3];
    c.Y = Y;
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
  const int b = (int)smem;
  cudaFuncSetAttribute(eval_ws_kernel<NEU, FULL, SG, false, GEN_PLANES>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(eval_ws_kernel<NEU, FULL, SG, true, GEN_PLANES>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(eval_ws_kernel<NEU, FULL, SG, false, GEN_WORDS>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(eval_ws_kernel<NEU, FULL, SG, true, GEN_WORDS>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  if (!FULL) {
    cudaFuncSetAttribute(eval_ws_kernel<NEU, false, SG, true, GEN_UNIFORM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         b);
    cudaFuncSetAttribute(eval_ws_kernel<NEU, false, SG, true, GEN_ENUM>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    cudaFuncSetAttribute(eval_ws_kernel<NEU, false, SG, true, GEN_ENUM_ADMISSIBLE>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  }
}

template <bool NEU, bool FULL, bool TOPK, int MODE = GEN_PLANES>
void launch_ws_t(const LaunchPlan& lp, const uint64_t* tab, const TabLayout& L, const EvalMeta& M, const EvalArgs& a,
                 const TopkArgs& tk, cudaStream_t s, const GenMeta& gm = GenMeta{}) {
  const int64_t ntiles = (MODE == GEN_PLANES || MODE == GEN_WORDS) ? a.n / kTile : (a.n + kTile - 1) / kTile;
  const size_t smem = ws_dynamic_bytes(M.A, stage_words(L), lp.smem_gate);
  const int64_t blocks = ws_grid(lp, a.n, MODE);
  auto kern = lp.smem_gate ? eval_ws_kernel<NEU, FULL, true, TOPK, MODE> : eval_ws_kernel<NEU, FULL, false, TOPK, MODE>;
  // the streaming kernel walks the layer sums from its shared-memory table: its
  // 4 fp64 warps are latency-bound, and dependent L2 reads of the memo slowed
  // the HBM-bound step by 2%
  EvalMeta Mw = M;
  Mw.memo = nullptr;
  if (TOPK && (MODE == GEN_WORDS || MODE == GEN_PLANES) && lp.pdl) {
    // fused steps on one stream overlap: the next launch starts while this
    // one's last CTAs merge (eval_ws_kernel's griddepcontrol)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, tab, L, Mw, a, ntiles, tk, gm);
  } else {
    kern<<<(unsigned)blocks, kThreads, smem, s>>>(tab, L, Mw, a, ntiles, tk, gm);
  }
}

// Write the generated stream as SoA planes (tests, users who want the vectors).
template <int MODE>
__global__ void generate_kernel(const GenMeta gm, int64_t n, int A, const EvalMeta M, uint8_t* planes,
                                int64_t stride) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    Decoded c;
    gen_candidate<MODE>(gm, (uint64_t)(gm.start + i), c);
    planes[i] = (uint8_t)c.t;
    planes[stride + i] = (uint8_t)c.e;
    planes[2 * stride + i] = (uint8_t)c.p;
    planes[3 * stride + i] = (uint8_t)c.b;
    for (int h = 4; h < A; ++h) planes[(int64_t)h * stride + i] = (uint8_t)((c.Y >> (2 * (h - 4))) & 3u);
  }
}

template <bool TOPK>
void launch_ws(const LaunchPlan& lp, bool neumaier, bool full, const uint64_t* tab, const TabLayout& L,
               const EvalMeta& M, const EvalArgs& a, const TopkArgs& tk, cudaStream_t s, const PackMeta* pk) {
  if (pk) {
    GenMeta gm{};
    gm.pk = *pk;
    if (neumaier) {
      if (full) launch_ws_t<true, true, TOPK, GEN_WORDS>(lp, tab, L, M, a, tk, s, gm);
      else launch_ws_t<true, false, TOPK, GEN_WORDS>(lp, tab, L, M, a, tk, s, gm);
    } else {
      if (full) launch_ws_t<false, true, TOPK, GEN_WORDS>(lp, tab, L, M, a, tk, s, gm);
      else launch_ws_t<false, false, TOPK, GEN_WORDS>(lp, tab, L, M, a, tk, s, gm);
    }
    return;
  }
  if (neumaier) {
    if (full) launch_ws_t<true, true, TOPK>(lp, tab, L, M, a, tk, s);
    else launch_ws_t<true, false, TOPK>(lp, tab, L, M, a, tk, s);
  } else {
    if (full) launch_ws_t<false, true, TOPK>(lp, tab, L, M, a, tk, s);
    else launch_ws_t<false, false, TOPK>(lp, tab, L, M, a, tk, s);
  }
}

// SoA planes -> packed candidate words (A <= 16). Out-of-range heads give an
// all-ones (malformed) word, so they still evaluate to LS_REASON_DECODE_ERROR.
__global__ void pack_kernel(const PackMeta pk, int A, const uint8_t* __restrict__ planes, int64_t stride, int64_t n,
                            uint64_t* __restrict__ words) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t t = planes[i], e = planes[stride + i], p = planes[2 * stride + i], b = planes[3 * stride + i];
    bool bad = t >= pk.nt || e >= pk.ne || p >= pk.np || b >= pk.nb;
    uint64_t y = 0;
    for (int h = 4; h < A; ++h) {
      const uint32_t v = planes[(int64_t)h * stride + i];
      bad |= v > 2;
      y |= (uint64_t)(v & 3u) << (2 * (h - 4));
    }
    const uint64_t rank = ((uint64_t)(t * pk.ne + e) * pk.np + p) * pk.nb + b;
    words[i] = bad ? ~0ull : (y | rank << 24);
  }
}

// Four candidates per thread from 32-bit plane loads (planes 4-byte aligned,
// stride % 4 == 0): coalesced 128 B per plane per warp, two 16-byte stores.
__global__ void pack4_kernel(const PackMeta pk, int A, const uint8_t* __restrict__ planes, int64_t stride, int64_t n4,
                             uint64_t* __restrict__ words) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w[16];
#pragma unroll
    for (int h = 0; h < 16; ++h)
      w[h] = h < A ? __ldg(reinterpret_cast<const uint32_t*>(planes + (int64_t)h * stride) + q) : 0u;
    uint64_t out[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t t = (w[0] >> (8 * j)) & 0xffu, e = (w[1] >> (8 * j)) & 0xffu;
      const uint32_t p = (w[2] >> (8 * j)) & 0xffu, b = (w[3] >> (8 * j)) & 0xffu;
      bool bad = t >= pk.nt || e >= pk.ne || p >= pk.np || b >= pk.nb;
      uint64_t y = 0;
#pragma unroll
      for (int h = 4; h < 16; ++h) {
        const uint32_t v = (w[h] >> (8 * j)) & 0xffu;  // heads >= A load as 0
        bad |= v > 2;
        y |= (uint64_t)(v & 3u) << (2 * (h - 4));
      }
      const uint64_t rank = ((uint64_t)(t * pk.ne + e) * pk.np + p) * pk.nb + b;
      out[j] = bad ? ~0ull : (y | rank << 24);
    }
    uint4* dst = reinterpret_cast<uint4*>(words + 4 * q);
    dst[0] = make_uint4((uint32_t)out[0], (uint32_t)(out[0] >> 32), (uint32_t)out[1], (uint32_t)(out[1] >> 32));
    dst[1] = make_uint4((uint32_t)out[2], (uint32_t)(out[2] >> 32), (uint32_t)out[3], (uint32_t)(out[3] >> 32));
  }
}

}  // namespace

size_t tma_smem_budget(const cudaDeviceProp& prop) {
  const size_t per_cta = (size_t)prop.sharedMemPerMultiprocessor / LS_MIN_BLOCKS - 2048;
  return per_cta < (size_t)prop.sharedMemPerBlockOptin ? per_cta : (size_t)prop.sharedMemPerBlockOptin;
}

size_t tma_smem_bytes(const TabLayout& L, int A, bool smem_gate) {
  return ws_dynamic_bytes(A, stage_words(L), smem_gate);
}

bool tma_eligible(const EvalArgs& a, int A) {
  const bool al16 = a.words ? ((uintptr_t)a.words % 16) == 0
                            : ((uintptr_t)a.planes % 16) == 0 && a.stride % 16 == 0;
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
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, eval_ws_kernel<true, false, true, true, GEN_PLANES>, kThreads,
                                                  smem);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, eval_ws_kernel<true, false, false, true, GEN_PLANES>, kThreads,
                                                  smem);
  return nb;
}

int generic_blocks_per_sm() {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, eval_generic_kernel<true>, kGenericThreads, 0);
  return nb;
}

int sweep_ctas_per_sm() { return LS_SWEEP_CTAS; }

int64_t sweep_grid(const LaunchPlan& lp, int64_t n, int mode) {
  const int64_t chunks = (n + kSwChunk - 1) / kSwChunk;
  const int nw = sw_warps_of(mode);
  int64_t blocks = (chunks + nw - 1) / nw;
  if (blocks < 1) blocks = 1;
  // one CTA per SM: the cap counts the eval_ws_kernel's CTAs per SM, the same or more
  return blocks > lp.max_blocks ? lp.max_blocks : blocks;
}

size_t sweep_smem_bytes(const TabLayout& L, uint64_t hi_size, uint64_t lo_size, int mode, bool f32) {
  return sw_layout(L, (uint32_t)hi_size, (uint32_t)lo_size, sw_warps_of(mode), f32).bytes;
}

// Opt every sweep kernel into the largest dynamic shared memory the device
// allows beside its static shared memory; returns that dynamic budget.
size_t prepare_sweep_kernels(size_t optin) {
  size_t st = 0;  // the largest static shared memory of the instances (their warp counts differ)
  auto stat = [&st](auto kern) {
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess && fa.sharedSizeBytes > st) st = fa.sharedSizeBytes;
  };
  stat(sweep_kernel<true, GEN_ENUM_ADMISSIBLE, false>);
  stat(sweep_kernel<true, GEN_ENUM, false>);
  stat(sweep_kernel<true, GEN_UNIFORM, false>);
  const size_t budget = optin > st + 1024 ? optin - st - 1024 : 0;
  const int b = (int)budget;
  auto set = [b](auto kern) { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, b); };
  set(sweep_kernel<true, GEN_UNIFORM, false>);
  set(sweep_kernel<true, GEN_ENUM, false>);
  set(sweep_kernel<true, GEN_ENUM_ADMISSIBLE, false>);
  set(sweep_kernel<false, GEN_UNIFORM, false>);
  set(sweep_kernel<false, GEN_ENUM, false>);
  set(sweep_kernel<false, GEN_ENUM_ADMISSIBLE, false>);
  set(sweep_kernel<false, GEN_UNIFORM, true>);  // fp32 fast mode: no compensation (NEU irrelevant)
  set(sweep_kernel<false, GEN_ENUM, true>);
  set(sweep_kernel<false, GEN_ENUM_ADMISSIBLE, true>);
  return cudaGetLastError() == cudaSuccess ? budget : 0;
}

int64_t ws_grid(const LaunchPlan& lp, int64_t n, int mode) {
  // memory-fed modes: whole tiles (the ragged tail rides on one CTA); generated: ceil
  const int64_t ntiles = (mode == GEN_PLANES || mode == GEN_WORDS) ? n / kTile : (n + kTile - 1) / kTile;
  const int64_t blocks = ntiles > 0 ? ntiles : 1;
  return blocks > lp.max_blocks ? lp.max_blocks : blocks;
}

int fused_k_max() { return kFusedK; }

cudaError_t launch_pack(const PackMeta& pk, int A, const uint8_t* planes, int64_t stride, int64_t n, uint64_t* words,
                        cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int64_t done = 0;
  if (A <= 16 && ((uintptr_t)planes % 4) == 0 && stride % 4 == 0 && ((uintptr_t)words % 16) == 0 && n >= 4) {
    const int64_t n4 = n / 4;
    int64_t blocks = (n4 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    pack4_kernel<<<(unsigned)blocks, 256, 0, s>>>(pk, A, planes, stride, n4, words);
    done = 4 * n4;
  }
  if (done < n) {  // unaligned input or the < 4 tail: one candidate per thread
    int64_t blocks = (n - done + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    pack_kernel<<<(unsigned)blocks, 256, 0, s>>>(pk, A, planes + done, stride, n - done, words + done);
  }
  return cudaGetLastError();
}

cudaError_t launch_evaluate(const LaunchPlan& lp, bool neumaier, const uint64_t* tab, const TabLayout& L,
                            const EvalMeta& M, const EvalArgs& a, cudaStream_t s, const PackMeta* pk) {
  if (a.n <= 0) return cudaSuccess;
  const bool full = a.tpot || a.mem || a.comp || a.comm || a.pipe;
  if (lp.tma || pk) {
    launch_ws<false>(lp, neumaier, full, tab, L, M, a, TopkArgs{}, s, pk);
  } else {
    int64_t blocks = (a.n + kGenericThreads - 1) / kGenericThreads;
    if (blocks > lp.max_blocks) blocks = lp.max_blocks;
    if (neumaier) eval_generic_kernel<true><<<(unsigned)blocks, kGenericThreads, 0, s>>>(tab, L, M, a);
    else eval_generic_kernel<false><<<(unsigned)blocks, kGenericThreads, 0, s>>>(tab, L, M, a);
  }
  return cudaGetLastError();
}

cudaError_t launch_evaluate_topk(const LaunchPlan& lp, bool neumaier, const uint64_t* tab, const TabLayout& L,
                                 const EvalMeta& M, const EvalArgs& a, const TopkArgs& tk, cudaStream_t s,
                                 const PackMeta* pk) {
  const bool full = a.reason && (a.tpot || a.mem || a.comp || a.comm || a.pipe);
  launch_ws<true>(lp, neumaier, full, tab, L, M, a, tk, s, pk);
  return cudaGetLastError();
}

cudaError_t launch_sweep(const LaunchPlan& lp, bool neumaier, int mode, const uint64_t* tab, const TabLayout& L,
                         const EvalMeta& M, int64_t n, const TopkArgs& tk, const GenMeta& gm, cudaStream_t s) {
  EvalArgs a{};
  a.n = n;  // no planes, no per-candidate verdicts: only the fused elite leaves the SMs
  (void)a;
  auto go = [&](auto neu) {
    constexpr bool NEU = decltype(neu)::value;
#ifndef LS_SWEEP_WS  // LS_SWEEP_WS: A/B builds of the streaming kernel's generator modes
    if (!lp.sweep_fits)
#endif
    {
    if (mode == GEN_UNIFORM) launch_ws_t<NEU, false, true, GEN_UNIFORM>(lp, tab, L, M, a, tk, s, gm);
    else if (mode == GEN_ENUM) launch_ws_t<NEU, false, true, GEN_ENUM>(lp, tab, L, M, a, tk, s, gm);
    else launch_ws_t<NEU, false, true, GEN_ENUM_ADMISSIBLE>(lp, tab, L, M, a, tk, s, gm);
    return;
    }
#ifndef LS_SWEEP_WS
    if (mode == GEN_UNIFORM) launch_sweep_t<NEU, GEN_UNIFORM>(lp, tab, L, M, n, tk, gm, s);
    else if (mode == GEN_ENUM) launch_sweep_t<NEU, GEN_ENUM>(lp, tab, L, M, n, tk, gm, s);
    else launch_sweep_t<NEU, GEN_ENUM_ADMISSIBLE>(lp, tab, L, M, n, tk, gm, s);

#endif
  };
  if (neumaier && !lp.tabf) go(std::true_type{});  // fp32 fast mode sums plainly: one instantiation
  else go(std::false_type{});
  return cudaGetLastError();
}

cudaError_t launch_generate(int mode, const GenMeta& gm, int64_t n, int A, uint8_t* planes, int64_t stride,
                            cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int threads = 256;
  int64_t blocks = (n + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  EvalMeta dummy{};
  if (mode == GEN_UNIFORM) generate_kernel<GEN_UNIFORM><<<(unsigned)blocks, threads, 0, s>>>(gm, n, A, dummy, planes, stride);
  else if (mode == GEN_ENUM) generate_kernel<GEN_ENUM><<<(unsigned)blocks, threads, 0, s>>>(gm, n, A, dummy, planes, stride);
  else generate_kernel<GEN_ENUM_ADMISSIBLE><<<(unsigned)blocks, threads, 0, s>>>(gm, n, A, dummy, planes, stride);
  return cudaGetLastError();
}

}  // namespace ls

#ifdef LS_DIAG_TIMES
extern "C" int ls_diag_times(unsigned long long* host, int rows) {
  const unsigned zero = 0;
  cudaMemcpyToSymbol(ls::g_diag_entries, &zero, sizeof(zero));
  return (int)cudaMemcpyFromSymbol(host, ls::g_diag_t, sizeof(unsigned long long) * 16 * (rows < 1024 ? rows : 1024));
}
#endif
