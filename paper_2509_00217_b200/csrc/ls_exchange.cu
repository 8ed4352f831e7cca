// ls_exchange.cu — cross-rank elite exchange over peer memory (NVLink 5 /
// NVSwitch), fused with the merge.
//
// the only exchange of the sharded sweep is each rank's
// top-k (k records + count). Instead of an NCCL all-gather followed by a
// merge launch, one single-CTA kernel per rank
//   1. stores its block into slot `rank` of EVERY rank's symmetric buffer
//      with P2P stores over NVLink, in the low-latency ("LL") format: every
//      4-byte data word travels in one 8-byte store together with the step's
//      sequence number, so a reader knows a word has arrived when its tag
//      matches — no flags and no system-scope fences (a membar.sys costs tens
//      of microseconds here);
//   2. polls (bounded) the world slots of its own buffer until every word
//      carries this step's tag;
//   3. merges the world blocks into the global top-k with the same order
//      and dedupe rule as every other merge.
// Symmetric buffer layout (identical offsets on every rank; zeroed once):
//   [2 parities][world][(k + 1) * 8 words] uint64 = data word | seq << 32
//   (k record rows of 32 B, then a row whose first word is the count).
// The parity (seq & 1) double-buffers consecutive steps: a rank can run at
// most one step ahead of any peer, because finishing step s needs every
// peer's step-s words.
#include <cuda_runtime.h>

#include "ls_kernels.h"
#include "ls_topk.cuh"

namespace ls {

namespace {

constexpr int kExThreads = 256;
#ifndef LS_EX_SLEEP
#define LS_EX_SLEEP 20  // ns between polls of a word that has not arrived
#endif
constexpr int kExMaxRecs = 8 * 32;  // world <= 8, k <= 32

__global__ void __launch_bounds__(kExThreads) elite_exchange_kernel(const uint4* __restrict__ block,
                                                                    const uint64_t* __restrict__ peer_bases,
                                                                    uint8_t* local_base, int rank, int world, int k,
                                                                    uint32_t seq, long long timeout_cycles,
                                                                    ls_elite_rec* __restrict__ out,
                                                                    int32_t* __restrict__ count_out) {
  __shared__ __align__(16) uint8_t sbuf[8 * 33 * 8 * 4];  // staged LL data words, then the records
  Rec* recs = reinterpret_cast<Rec*>(sbuf);
  static_assert(kExMaxRecs * sizeof(Rec) <= sizeof(sbuf), "records fit the staging buffer");
  __shared__ double s_k[kExThreads / 32];
  __shared__ int64_t s_i[kExThreads / 32];
  __shared__ int s_slot[kExThreads / 32];
  __shared__ int s_timeout;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int parity = (int)(seq & 1u);
  if (tid == 0) s_timeout = 0;
  __syncthreads();

  // 1. push this rank's block, LL-tagged, into slot [parity][rank] of every rank
  const int words = (k + 1) * 8;
  const uint32_t* src = reinterpret_cast<const uint32_t*>(block);
  for (int i = tid; i < world * words; i += kExThreads) {
    const int q = i / words, w = i - q * words;
    volatile uint64_t* dst = reinterpret_cast<volatile uint64_t*>(peer_bases[q]) +
                             ((size_t)parity * world + rank) * words + w;
    *dst = (uint64_t)src[w] | ((uint64_t)seq << 32);
  }
  // 2. every word of every rank's block of this step, from this rank's buffer
  uint32_t* stage = reinterpret_cast<uint32_t*>(sbuf);  // world * words data words
  const volatile uint64_t* mine = reinterpret_cast<const volatile uint64_t*>(local_base) +
                                  (size_t)parity * world * words;
  const long long t0 = clock64();
  for (int i = tid; i < world * words; i += kExThreads) {
    uint64_t v = mine[i];
    while ((uint32_t)(v >> 32) != seq) {
      if (clock64() - t0 > timeout_cycles) {
        s_timeout = 1;
        break;
      }
      __nanosleep(LS_EX_SLEEP);
      v = mine[i];
    }
    stage[i] = (uint32_t)v;
  }
  __syncthreads();
  if (s_timeout) {
    if (tid == 0) *count_out = -1;  // a peer never arrived: reported by the caller
    return;
  }

  // 3. merge: records out of the staged words, then k rounds of block-wide
  //    argmax (each round emits the best remaining record and retires every
  //    record of the same vector)
  const int total = world * k;
  Rec r_mine[(kExMaxRecs + kExThreads - 1) / kExThreads];
  int nm = 0;
  for (int i = tid; i < total; i += kExThreads, ++nm) {
    const int q = i / k, j = i - q * k;
    const uint32_t* b = stage + (size_t)q * words;
    const int cnt = (int)b[k * 8];
    Rec r{-1.0e308, 0.0, INT64_MAX, 0};
    if (j < cnt) {
      const uint32_t* w = b + j * 8;
      r.key = __hiloint2double((int)w[1], (int)w[0]);
      r.raw = __hiloint2double((int)w[3], (int)w[2]);
      r.idx = (int64_t)(((uint64_t)w[5] << 32) | w[4]);
      r.code = ((uint64_t)w[7] << 32) | w[6];
    }
    r_mine[nm] = r;
  }
  __syncthreads();  // the staged words are read; recs[] may now be overwritten
  nm = 0;
  for (int i = tid; i < total; i += kExThreads, ++nm) recs[i] = r_mine[nm];
  __syncthreads();
  int emitted = 0;
  for (int r = 0; r < k; ++r) {
    double bk = -1.0e308;
    int64_t bi = INT64_MAX;
    int bs = -1;
    for (int i = tid; i < total; i += kExThreads)
      if (recs[i].key != -1.0e308 && better(recs[i].key, recs[i].idx, bk, bi)) {
        bk = recs[i].key;
        bi = recs[i].idx;
        bs = i;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      const int os = __shfl_xor_sync(0xffffffffu, bs, o);
      if (better(ok, oi, bk, bi)) {
        bk = ok;
        bi = oi;
        bs = os;
      }
    }
    if (lane == 0) {
      s_k[warp] = bk;
      s_i[warp] = bi;
      s_slot[warp] = bs;
    }
    __syncthreads();
    for (int o = 0; o < kExThreads / 32; ++o)
      if (better(s_k[o], s_i[o], bk, bi)) {
        bk = s_k[o];
        bi = s_i[o];
        bs = s_slot[o];
      }
    if (bs < 0) break;  // block-uniform: nothing left
    const Rec best = recs[bs];
    if (tid == 0) out[r] = ls_elite_rec{best.key, best.raw, best.idx, best.code};
    ++emitted;
    __syncthreads();
    for (int i = tid; i < total; i += kExThreads)
      if (recs[i].code == best.code) recs[i].key = -1.0e308;
    __syncthreads();
  }
  if (tid == 0) *count_out = emitted;
}

}  // namespace

size_t elite_exchange_bytes(int world, int k) {
  return 2 * (size_t)world * (size_t)(k + 1) * 8 * sizeof(uint64_t);  // LL words: 8 B per 4 data bytes
}

cudaError_t launch_elite_exchange(const void* block, const uint64_t* peer_bases, void* local_base, int rank,
                                  int world, int k, uint32_t seq, long long timeout_cycles, ls_elite_rec* out,
                                  int32_t* count_out, cudaStream_t s) {
  elite_exchange_kernel<<<1, kExThreads, 0, s>>>(static_cast<const uint4*>(block), peer_bases,
                                                 static_cast<uint8_t*>(local_base), rank, world, k, seq,
                                                 timeout_cycles, out, count_out);
  return cudaGetLastError();
}

}  // namespace ls
