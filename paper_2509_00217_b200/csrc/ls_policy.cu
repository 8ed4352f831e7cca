// ls_policy.cu — the reference's policy network and PPO update as fused
// float64 device kernels (policy.py:213-499, ppo.py:170-359).
//
// The policy is tiny (R = n_steps * history_len <= 16 observation rows,
// width 256) so every stage is latency-bound: the design goal is few
// launches per PPO round, each reading its weight slice once, with the
// whole round capturable in one CUDA graph. A forward is five column-tiled
// kernels (each CTA recomputes the small row-wise prologue it needs — the
// embedding, attention, a LayerNorm — instead of waiting for another
// launch), then one single-CTA kernel for the masked softmax heads that
// also samples, runs the env step (ls_envstep.cuh) or builds the loss
// gradient. The backward is six row-tiled kernels (warp per output
// feature, lanes along the contiguous weight row). Adam computes every
// weight gradient on the fly from the saved (input, output-gradient) rows —
// a <= 16-term outer-product sum per element — so no gradient tensor is
// ever materialised.
//
// Activation rows r = s * T + t (sample s, observation row t). Samples of a
// round live in fixed slots, so the epoch-1 update reuses the activations of
// the sampling forwards (same parameters), and the confidence forward after
// the update doubles as the next round's first sampling forward.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cstring>

#include "../../include/ls_eval.h"
#include "ls_envstep.cuh"
#include "ls_kernels.h"

namespace ls {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRowsMax = 16;
constexpr size_t kSmemMax = 200 * 1024;
constexpr double kMasked = -1e30;  // policy.py:36 MASKED_LOGIT
constexpr double kLnEps = 1e-5;

// Workspace: activations and their gradients (doubles).
struct Work {
  double *E, *QKV, *ATTW, *CTX, *RES1, *N1, *IS1, *H1, *ACT, *RES2, *N2, *IS2, *POOL, *LRAW, *VH;
  double *DL, *DVAL, *DVPRE, *DPOOL, *DRES2, *DPRE, *DH1, *DRES1, *DCTX, *DQKV, *DEMB, *HYP;
};

struct Seg {
  int blk0, colblocks;      // first CTA of the segment, CTAs per row
  int64_t off, rows, cols;  // rows = 0: vector segment of length cols
  int kind;                 // 0 matrix x^T dy, 1 bias sum dy, 2 LN gain sum dy*x
  int nrows;                // summed rows
  const double* x;
  int64_t ldx;
  const double* dy;
  int64_t lddy;
  int row_div;  // dy row = r / row_div
  double div;   // dy value = dy / div
};

struct Args {
  int A, d, f, T, H, K, HK, RM, SM;
  const double *We, *be, *Wqkv, *bqkv, *Wo, *bo, *g1, *c1, *W1, *b1, *W2, *b2, *g2, *c2, *Wh, *bh, *Wv1, *bv1, *Wv2,
      *bv2;
  double *P, *Mo, *Vo, *G;
  int64_t total;
  Work w;
  double* X;
  const uint8_t* blocked;
  const int32_t* head_size;
  const double* denom;
  ls_search_state env;
  const double* uniforms;
  const double* lr_table;
  int64_t* spent;
  int64_t* adam_step;
  int32_t* status;
  int64_t* b_act;
  double *b_logp, *b_val, *b_rew;
  double tau, clip, vc, ec, beta1, beta2, eps;
  double *out_logp, *out_val;
};

struct SegTable {
  int n, blocks;
  Seg s[LS_PSEG_COUNT];
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;  // xor butterfly: every lane holds the same (commutative) sum
}

// Column tile: out(r, j) = sum_i X[r*ldx + i] * W[i*ldw + j] for the kCols
// columns j0.. of this CTA. Threads are (k group, column): each k group sums
// every kKG-th input row, then the kKG partials are reduced in a fixed order
// (deterministic); finally epi(r, j, sum) for every (r < R, j < N).
constexpr int kCols = 8;
constexpr int kKG = kThreads / kCols;
constexpr int kRedDoubles = kKG * kRowsMax * kCols;

template <class Epi>
__device__ __forceinline__ void xw_tile(const double* X, int64_t ldx, int R, int K, const double* __restrict__ W,
                                        int64_t ldw, int N, int j0, double* red, Epi epi) {
  const int c = threadIdx.x % kCols, kg = threadIdx.x / kCols;
  const int j = j0 + c;
  double acc[kRowsMax];
#pragma unroll
  for (int r = 0; r < kRowsMax; ++r) acc[r] = 0.0;
  if (j < N) {
#pragma unroll 4
    for (int i = kg; i < K; i += kKG) {
      const double wv = __ldg(W + (int64_t)i * ldw + j);
#pragma unroll
      for (int r = 0; r < kRowsMax; ++r)
        if (r < R) acc[r] += X[(int64_t)r * ldx + i] * wv;
    }
  }
#pragma unroll
  for (int r = 0; r < kRowsMax; ++r)
    if (r < R) red[(kg * kRowsMax + r) * kCols + c] = acc[r];
  __syncthreads();
  for (int idx = threadIdx.x; idx < R * kCols; idx += kThreads) {
    const int r = idx / kCols, cc = idx % kCols, jj = j0 + cc;
    if (jj >= N) continue;
    double s = red[r * kCols + cc];
    for (int g = 1; g < kKG; ++g) s += red[(g * kRowsMax + r) * kCols + cc];
    epi(r, jj, s);
  }
}

// Row output (one warp): out(r) = sum_j DY[r*ldd + j] * W[i*ldw + j] over the
// contiguous weight row i; every lane returns all R sums.
__device__ __forceinline__ void dywt_row(const double* DY, int64_t ldd, int R, int N, const double* __restrict__ W,
                                         int64_t ldw, int i, double* out) {
  const int lane = threadIdx.x & 31;
  double acc[kRowsMax];
#pragma unroll
  for (int r = 0; r < kRowsMax; ++r) acc[r] = 0.0;
  const double* wr = W + (int64_t)i * ldw;
#pragma unroll 4
  for (int j = lane; j < N; j += 32) {
    const double wv = __ldg(wr + j);
#pragma unroll
    for (int r = 0; r < kRowsMax; ++r)
      if (r < R) acc[r] += DY[(int64_t)r * ldd + j] * wv;
  }
#pragma unroll
  for (int r = 0; r < kRowsMax; ++r)
    if (r < R) out[r] = warp_sum(acc[r]);
}

// LayerNorm forward of one row by one warp (policy.py:177-185).
__device__ __forceinline__ void ln_row(const double* x, int d, const double* g, const double* b, double* h,
                                       double* nrm_out, double* inv_out) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
#pragma unroll 8
  for (int c = lane; c < d; c += 32) s += x[c];
  const double mean = warp_sum(s) / d;
  double q = 0.0;
#pragma unroll 8
  for (int c = lane; c < d; c += 32) {
    const double cc = x[c] - mean;
    q += cc * cc;
  }
  const double var = warp_sum(q) / d;
  const double inv = 1.0 / sqrt(var + kLnEps);
#pragma unroll 8
  for (int c = lane; c < d; c += 32) {
    const double n = (x[c] - mean) * inv;
    h[c] = g[c] * n + b[c];
    if (nrm_out) nrm_out[c] = n;
  }
  if (inv_out && lane == 0) *inv_out = inv;
}

// LayerNorm backward of one row by one warp (policy.py:188-202, in the
// equivalent form inv * (dn - mean(dn) - n * mean(dn * n)), dn = dh * g).
template <class DH>
__device__ __forceinline__ void ln_back_row(DH dh, int d, const double* g, const double* nrm, double inv, double* dx) {
  const int lane = threadIdx.x & 31;
  double s1 = 0.0, s2 = 0.0;
#pragma unroll 8
  for (int c = lane; c < d; c += 32) {
    const double dn = dh(c) * g[c];
    s1 += dn;
    s2 += dn * nrm[c];
  }
  const double m1 = warp_sum(s1) / d, m2 = warp_sum(s2) / d;
#pragma unroll 8
  for (int c = lane; c < d; c += 32) {
    const double dn = dh(c) * g[c];
    dx[c] = inv * (dn - m1 - nrm[c] * m2);
  }
}

// ---- forward ---------------------------------------------------------------

// embedding (recomputed per CTA) + q/k/v column tile. build: render the
// observation from the device elite buffer (build_observation, policy.py:105-117).
__global__ void __launch_bounds__(kThreads) fwd_embed_qkv(const __grid_constant__ Args a, int row0, int R, int build) {
  extern __shared__ double sm[];
  double* red = sm;
  double* Xs = red + kRedDoubles;
  double* Es = Xs + R * a.A;
  const int A = a.A, d = a.d;
  for (int i = threadIdx.x; i < R * A; i += kThreads) {
    double x;
    if (build) {
      const int t = i / A, h = i % A;
      x = isinf(a.env.elite_reward[t]) ? 0.0 : (double)a.env.elite_vec[(int64_t)t * A + h] / a.denom[h];
      if (blockIdx.x == 0) a.X[(int64_t)row0 * A + i] = x;
    } else {
      x = a.X[(int64_t)row0 * A + i];
    }
    Xs[i] = x;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < R * d; i += kThreads) {
    const int r = i / d, c = i % d;
    double s = 0.0;
#pragma unroll 8
    for (int k = 0; k < A; ++k) s += Xs[r * A + k] * __ldg(a.We + (int64_t)k * d + c);
    const double e = s + a.be[c];
    Es[i] = e;
    if (blockIdx.x == 0) a.w.E[(int64_t)row0 * d + i] = e;
  }
  __syncthreads();
  double* QKV = a.w.QKV + (int64_t)row0 * 3 * d;
  const double* bq = a.bqkv;
  xw_tile(Es, d, R, d, a.Wqkv, 3 * d, 3 * d, blockIdx.x * kCols, red,
          [&](int r, int j, double s) { QKV[(int64_t)r * 3 * d + j] = s + bq[j]; });
}

// attention (recomputed per CTA) + output projection tile + residual.
__global__ void __launch_bounds__(kThreads) fwd_attn_out(const __grid_constant__ Args a, int row0, int R) {
  extern __shared__ double sm[];
  const int d = a.d, T = a.T, S = R / T, TT = T * T;
  double* red = sm;
  double* Ws = red + kRedDoubles;
  double* Cs = Ws + S * TT;
  const double* QKV = a.w.QKV + (int64_t)row0 * 3 * d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double scale = 1.0 / sqrt((double)d);
  for (int p = warp; p < S * TT; p += kWarps) {
    const int s = p / TT, t = (p / T) % T, u = p % T;
    const double* q = QKV + (int64_t)(s * T + t) * 3 * d;
    const double* k = QKV + (int64_t)(s * T + u) * 3 * d + d;
    double acc = 0.0;
#pragma unroll 8
    for (int c = lane; c < d; c += 32) acc += q[c] * k[c];
    acc = warp_sum(acc);
    if (lane == 0) Ws[p] = acc * scale;
  }
  __syncthreads();
  for (int row = threadIdx.x; row < S * T; row += kThreads) {  // row softmax
    double* w = Ws + row * T;
    double mx = w[0];
    for (int u = 1; u < T; ++u) mx = fmax(mx, w[u]);
    double tot = 0.0;
    for (int u = 0; u < T; ++u) {
      w[u] = exp(w[u] - mx);
      tot += w[u];
    }
    for (int u = 0; u < T; ++u) w[u] /= tot;
  }
  __syncthreads();
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < S * TT; i += kThreads) a.w.ATTW[(int64_t)(row0 / T) * TT + i] = Ws[i];
  for (int i = threadIdx.x; i < R * d; i += kThreads) {
    const int r = i / d, c = i % d, s = r / T, t = r % T;
    double acc = 0.0;
#pragma unroll 4
    for (int u = 0; u < T; ++u) acc += Ws[(s * T + t) * T + u] * QKV[(int64_t)(s * T + u) * 3 * d + 2 * d + c];
    Cs[i] = acc;
    if (blockIdx.x == 0) a.w.CTX[(int64_t)row0 * d + i] = acc;
  }
  __syncthreads();
  const double* E = a.w.E + (int64_t)row0 * d;
  double* RES1 = a.w.RES1 + (int64_t)row0 * d;
  const double* bo = a.bo;
  xw_tile(Cs, d, R, d, a.Wo, d, d, blockIdx.x * kCols, red,
          [&](int r, int j, double s) { RES1[(int64_t)r * d + j] = E[(int64_t)r * d + j] + (s + bo[j]); });
}

// LayerNorm 1 (recomputed per CTA) + FFN first layer tile + ReLU.
__global__ void __launch_bounds__(kThreads) fwd_ln1_ffn1(const __grid_constant__ Args a, int row0, int R) {
  extern __shared__ double sm[];
  const int d = a.d, f = a.f;
  double* red = sm;
  double* Hs = red + kRedDoubles;
  const int warp = threadIdx.x >> 5;
  const bool first = blockIdx.x == 0;
  for (int r = warp; r < R; r += kWarps) {
    const int64_t g = (int64_t)(row0 + r) * d;
    ln_row(a.w.RES1 + g, d, a.g1, a.c1, Hs + r * d, first ? a.w.N1 + g : nullptr, first ? a.w.IS1 + row0 + r : nullptr);
  }
  __syncthreads();
  if (first)
    for (int i = threadIdx.x; i < R * d; i += kThreads) a.w.H1[(int64_t)row0 * d + i] = Hs[i];
  double* ACT = a.w.ACT + (int64_t)row0 * f;
  const double* b1 = a.b1;
  xw_tile(Hs, d, R, d, a.W1, f, f, blockIdx.x * kCols, red, [&](int r, int j, double s) {
    const double v = s + b1[j];
    ACT[(int64_t)r * f + j] = v > 0.0 ? v : 0.0;
  });
}

// FFN second layer tile + residual.
__global__ void __launch_bounds__(kThreads) fwd_ffn2(const __grid_constant__ Args a, int row0, int R) {
  extern __shared__ double sm[];
  const int d = a.d, f = a.f;
  const double* H1 = a.w.H1 + (int64_t)row0 * d;
  double* RES2 = a.w.RES2 + (int64_t)row0 * d;
  const double* b2 = a.b2;
  double* As = sm + kRedDoubles;
#pragma unroll 4
  for (int i = threadIdx.x; i < R * f; i += kThreads) As[i] = a.w.ACT[(int64_t)row0 * f + i];
  __syncthreads();
  xw_tile(As, f, R, f, a.W2, d, d, blockIdx.x * kCols, sm,
          [&](int r, int j, double s) { RES2[(int64_t)r * d + j] = H1[(int64_t)r * d + j] + (s + b2[j]); });
}

// LayerNorm 2 + mean pool (recomputed per CTA) + a column tile of the heads
// (first ceil(HK/32) CTAs) or of the value hidden layer (the rest).
__global__ void __launch_bounds__(kThreads) fwd_ln2_heads(const __grid_constant__ Args a, int row0, int R) {
  extern __shared__ double sm[];
  const int d = a.d, T = a.T, S = R / T, slot0 = row0 / T;
  double* red = sm;
  double* Hs = red + kRedDoubles;
  double* Ps = Hs + R * d;
  const int warp = threadIdx.x >> 5;
  const bool first = blockIdx.x == 0;
  for (int r = warp; r < R; r += kWarps) {
    const int64_t g = (int64_t)(row0 + r) * d;
    ln_row(a.w.RES2 + g, d, a.g2, a.c2, Hs + r * d, first ? a.w.N2 + g : nullptr, first ? a.w.IS2 + row0 + r : nullptr);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < S * d; i += kThreads) {
    const int s = i / d, c = i % d;
    double acc = 0.0;
    for (int t = 0; t < T; ++t) acc += Hs[(s * T + t) * d + c];
    Ps[i] = acc / T;
    if (first) a.w.POOL[(int64_t)slot0 * d + i] = Ps[i];
  }
  __syncthreads();
  const int nh = (a.HK + kCols - 1) / kCols;
  if ((int)blockIdx.x < nh) {
    double* L = a.w.LRAW + (int64_t)slot0 * a.HK;
    const double* bh = a.bh;
    const int HK = a.HK;
    xw_tile(Ps, d, S, d, a.Wh, HK, HK, blockIdx.x * kCols, red,
            [&](int r, int j, double s) { L[(int64_t)r * HK + j] = s + bh[j]; });
  } else {
    double* VH = a.w.VH + (int64_t)slot0 * d;
    const double* bv = a.bv1;
    xw_tile(Ps, d, S, d, a.Wv1, d, d, (blockIdx.x - nh) * kCols, red, [&](int r, int j, double s) {
      const double v = s + bv[j];
      VH[(int64_t)r * d + j] = v > 0.0 ? v : 0.0;
    });
  }
}

enum { MODE_SAMPLE = 0, MODE_CONF = 1, MODE_TRAIN = 2, MODE_PROBE = 3 };

// Heads and value on one CTA: masked log-softmax per head (policy.py:168-174),
// value, then per mode — sample + env step, confidence, or the PPO loss
// gradient w.r.t. logits and value (ppo.py:225-283). Every global input is
// first staged into shared memory with independent loads, so the serial
// per-head and per-sample loops run on on-chip data. SMEMTAB: the workload's
// cost tables are staged too, for the env step's single-thread walk.
template <int MODE, bool NEU>
__global__ void __launch_bounds__(kThreads) fwd_final(const __grid_constant__ Args a, int slot0, int S,
                                                      const uint64_t* __restrict__ tab,
                                                      const __grid_constant__ TabLayout L,
                                                      const __grid_constant__ EvalMeta M) {
  extern __shared__ double sm[];
  const int d = a.d, H = a.H, K = a.K, HK = a.HK;
  double* LP = sm;
  double* PR = LP + S * HK;
  double* ENT = PR + S * HK;  // [S*H]
  double* VAL = ENT + S * H;  // [S]
  double* DLP = VAL + S;      // [S] d loss / d logprob
  double* RAW = DLP + S;      // [S*HK] staged logits
  double* MX = RAW + S * HK;  // [S*H] per-head max, then log(total)
  double* TOT = MX + S * H;   // [S*H]
  int64_t* EV = reinterpret_cast<int64_t*>(TOT + S * H);  // elite copy (sample mode)
  double* ER = reinterpret_cast<double*>(EV + a.env.elite_capacity * a.A);
  __shared__ uint8_t blk[LS_MAX_HEADS * 64];
  __shared__ int act[LS_MAX_HEADS];
  __shared__ int all_conf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if constexpr (MODE == MODE_SAMPLE) {  // pull the cost tables into L1 for the env step's serial walk
    for (int i = threadIdx.x * 16; i < L.words; i += kThreads * 16)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(tab + i));
  }
  const double* LR = a.w.LRAW + (int64_t)slot0 * HK;
#pragma unroll 4
  for (int i = threadIdx.x; i < S * HK; i += kThreads) RAW[i] = LR[i];
  for (int i = threadIdx.x; i < HK; i += kThreads) blk[i] = a.blocked[i];
  for (int s = warp; s < S; s += kWarps) {
    const double* vh = a.w.VH + (int64_t)(slot0 + s) * d;
    double acc = 0.0;
#pragma unroll 4
    for (int c = lane; c < d; c += 32) acc += vh[c] * a.Wv2[c];
    acc = warp_sum(acc);
    if (lane == 0) VAL[s] = acc + a.bv2[0];
  }
  __syncthreads();
  // masked log-softmax: per-head max, element-parallel exp, per-head sums in k order
  for (int i = threadIdx.x; i < S * H; i += kThreads) {
    const int s = i / H, h = i % H;
    const double* raw = RAW + s * HK + h * K;
    const uint8_t* bk = blk + h * K;
    double mx = -INFINITY;
    for (int k = 0; k < K; ++k) mx = fmax(mx, bk[k] ? kMasked : raw[k]);
    MX[i] = mx;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < S * HK; i += kThreads) {
    const int s = i / HK, j = i % HK;
    const double sh = (blk[j] ? kMasked : RAW[i]) - MX[s * H + j / K];
    LP[i] = sh;
    PR[i] = exp(sh);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < S * H; i += kThreads) {
    const double* ex = PR + (i / H) * HK + (i % H) * K;
    double tot = 0.0;
    for (int k = 0; k < K; ++k) tot += ex[k];
    TOT[i] = tot;
    MX[i] = log(tot);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < S * HK; i += kThreads) {
    const int hh = (i / HK) * H + (i % HK) / K;
    LP[i] = LP[i] - MX[hh];
    PR[i] = PR[i] / TOT[hh];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < S * H; i += kThreads) {
    const int o = (i / H) * HK + (i % H) * K;
    double e = 0.0;
    for (int k = 0; k < K; ++k) e += PR[o + k] * LP[o + k];
    ENT[i] = -e;
  }
  __syncthreads();

  if constexpr (MODE == MODE_PROBE) {
    for (int i = threadIdx.x; i < S * HK; i += kThreads) a.out_logp[i] = LP[i];
    if (threadIdx.x < S) a.out_val[threadIdx.x] = VAL[threadIdx.x];
  } else if constexpr (MODE == MODE_SAMPLE) {  // sample_categorical per head (policy.py:205-210), then env.step
    const int64_t sp = *a.spent;
    if (threadIdx.x < H) {
      const int h = threadIdx.x;
      const double u = a.uniforms[sp * H + h];
      const double* p = PR + h * K;
      double cdf = 0.0, tot = 0.0;
      for (int k = 0; k < K; ++k) tot += p[k];
      const double draw = u * tot;
      int idx = K;
      for (int k = 0; k < K; ++k) {
        cdf += p[k];
        if (cdf > draw) {
          idx = k;
          break;
        }
      }
      idx = min(idx, a.head_size[h] - 1);
      act[h] = idx;
      a.b_act[(int64_t)slot0 * H + h] = idx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double lp = 0.0;
      for (int h = 0; h < H; ++h) lp += LP[h * K + act[h]];
      a.b_logp[slot0] = lp;
      a.b_val[slot0] = VAL[0];
      *a.spent = sp + 1;
    }
    env_step_block<NEU, true>(tab, L, M, a.env, act, a.b_rew + slot0, EV, ER);
  } else if constexpr (MODE == MODE_CONF) {  // confidence (policy.py:502-504) >= tau on every head
    if (threadIdx.x == 0) all_conf = 1;
    __syncthreads();
    if (threadIdx.x < H) {
      double mx = 0.0;
      for (int k = 0; k < K; ++k) mx = fmax(mx, PR[threadIdx.x * K + k]);
      if (!(mx >= a.tau)) atomicAnd(&all_conf, 0);
    }
    __syncthreads();
    if (threadIdx.x == 0 && all_conf) atomicOr(a.status, 1);
  } else {  // MODE_TRAIN: clipped surrogate + value + entropy (ppo.py:225-283)
    __shared__ int64_t bact[8 * LS_MAX_HEADS];
    for (int i = threadIdx.x; i < S * H; i += kThreads) bact[i] = a.b_act[i];
    __syncthreads();
    if (threadIdx.x == 0) {
      const double n = (double)S, lo = 1.0 - a.clip, hi = 1.0 + a.clip;
      double pl = 0.0, vl = 0.0, et = 0.0;
      bool bad = false;
      for (int s = 0; s < S; ++s) {
        const double rew = a.b_rew[s], vold = a.b_val[s], lold = a.b_logp[s];
        bad |= !(isfinite(rew) && isfinite(vold) && isfinite(lold));
        double lpn = 0.0, ent = 0.0;
        for (int h = 0; h < H; ++h) {
          lpn += LP[s * HK + h * K + (int)bact[s * H + h]];
          ent += ENT[s * H + h];
        }
        const double adv = rew - vold;
        const double ratio = exp(lpn - lold);
        const double unc = ratio * adv;
        const double clp = fmin(fmax(ratio, lo), hi) * adv;
        const double sur = fmin(unc, clp);
        const double d_ratio = unc <= clp ? -adv / n : 0.0;
        const double err = VAL[s] - rew;
        pl += -sur / n;
        vl += a.vc * err * err / n;
        et += ent / n;
        DLP[s] = d_ratio * ratio;
        a.w.DVAL[s] = 2.0 * a.vc * err / n;
      }
      const double total = pl + vl - a.ec * et;
      if (bad || !isfinite(total)) atomicOr(a.status, 2);
      const int64_t step = *a.adam_step + 1;  // Adam.apply (ppo.py:150-152)
      *a.adam_step = step;
      a.w.HYP[0] = a.lr_table[*a.spent - S];
      a.w.HYP[1] = 1.0 - pow(a.beta1, (double)step);
      a.w.HYP[2] = 1.0 - pow(a.beta2, (double)step);
    }
    __syncthreads();
    const double n = (double)S;
    for (int i = threadIdx.x; i < S * HK; i += kThreads) {
      const int s = i / HK, j = i % HK, h = j / K, k = j % K;
      double g = 0.0;
      if (!blk[j]) {
        const double p = PR[i], oh = k == (int)bact[s * H + h] ? 1.0 : 0.0;
        g = DLP[s] * (oh - p);
        g += a.ec * p * (LP[i] + ENT[s * H + h]) / n;
      }
      a.w.DL[i] = g;
    }
  }
}

// ---- backward --------------------------------------------------------------

// d pooled = heads^T dl + value_w1^T d value_pre (policy.py:405-419).
__global__ void __launch_bounds__(kThreads) bwd_pool(const __grid_constant__ Args a, int S) {
  extern __shared__ double sm[];
  const int d = a.d, HK = a.HK;
  double* DLs = sm;
  double* DVP = DLs + S * HK;
#pragma unroll 4
  for (int i = threadIdx.x; i < S * HK; i += kThreads) DLs[i] = a.w.DL[i];
  for (int i = threadIdx.x; i < S * d; i += kThreads) {
    const int s = i / d, k = i % d;
    const double v = a.w.VH[i] > 0.0 ? a.w.DVAL[s] * a.Wv2[k] : 0.0;
    DVP[i] = v;
    if (blockIdx.x == 0) a.w.DVPRE[i] = v;
  }
  __syncthreads();
  const int c = blockIdx.x * kWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (c >= d) return;
  double o1[kRowsMax], o2[kRowsMax];
  dywt_row(DLs, HK, S, HK, a.Wh, HK, c, o1);
  dywt_row(DVP, d, S, d, a.Wv1, d, c, o2);
  for (int s = lane; s < S; s += 32) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kRowsMax; ++q)
      if (q == s) v = o1[q] + o2[q];
    a.w.DPOOL[(int64_t)s * d + c] = v;
  }
}

// LayerNorm 2 backward (recomputed per CTA) + d ffn_pre tile (policy.py:421-430).
__global__ void __launch_bounds__(kThreads) bwd_ln2_ffn2(const __grid_constant__ Args a, int S) {
  extern __shared__ double sm[];
  const int d = a.d, f = a.f, T = a.T, R = S * T;
  double* DR = sm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < R; r += kWarps) {
    const double* dp = a.w.DPOOL + (int64_t)(r / T) * d;
    const double rows = (double)T;
    ln_back_row([&](int c) { return dp[c] / rows; }, d, a.g2, a.w.N2 + (int64_t)r * d, a.w.IS2[r], DR + r * d);
  }
  __syncthreads();
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < R * d; i += kThreads) a.w.DRES2[i] = DR[i];
  const int k = blockIdx.x * kWarps + warp;
  if (k >= f) return;
  double o[kRowsMax];
  dywt_row(DR, d, R, d, a.W2, d, k, o);
  for (int r = lane; r < R; r += 32) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kRowsMax; ++q)
      if (q == r) v = o[q];
    a.w.DPRE[(int64_t)r * f + k] = a.w.ACT[(int64_t)r * f + k] > 0.0 ? v : 0.0;
  }
}

// d hidden1 = d res2 + d ffn_pre W1^T (policy.py:426-433).
__global__ void __launch_bounds__(kThreads) bwd_ffn1(const __grid_constant__ Args a, int S) {
  extern __shared__ double sm[];
  const int d = a.d, f = a.f, R = S * a.T;
  double* DP = sm;
#pragma unroll 4
  for (int i = threadIdx.x; i < R * f; i += kThreads) DP[i] = a.w.DPRE[i];
  __syncthreads();
  const int c = blockIdx.x * kWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (c >= d) return;
  double o[kRowsMax];
  dywt_row(DP, f, R, f, a.W1, f, c, o);
  for (int r = lane; r < R; r += 32) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kRowsMax; ++q)
      if (q == r) v = o[q];
    a.w.DH1[(int64_t)r * d + c] = a.w.DRES2[(int64_t)r * d + c] + v;
  }
}

// LayerNorm 1 backward (recomputed per CTA) + d context = d res1 Wo^T (policy.py:435-442).
__global__ void __launch_bounds__(kThreads) bwd_ln1_wo(const __grid_constant__ Args a, int S) {
  extern __shared__ double sm[];
  const int d = a.d, R = S * a.T;
  double* DR = sm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < R; r += kWarps) {
    const double* dh = a.w.DH1 + (int64_t)r * d;
    ln_back_row([&](int c) { return dh[c]; }, d, a.g1, a.w.N1 + (int64_t)r * d, a.w.IS1[r], DR + r * d);
  }
  __syncthreads();
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < R * d; i += kThreads) a.w.DRES1[i] = DR[i];
  const int c = blockIdx.x * kWarps + warp;
  if (c >= d) return;
  double o[kRowsMax];
  dywt_row(DR, d, R, d, a.Wo, d, c, o);
  for (int r = lane; r < R; r += 32) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kRowsMax; ++q)
      if (q == r) v = o[q];
    a.w.DCTX[(int64_t)r * d + c] = v;
  }
}

// Attention backward (policy.py:444-453): d scores recomputed per CTA, then
// d q, d k, d v per feature column.
__global__ void __launch_bounds__(kThreads) bwd_attn(const __grid_constant__ Args a, int S) {
  extern __shared__ double sm[];
  const int d = a.d, T = a.T, TT = T * T;
  double* dW = sm;
  double* dS = dW + S * TT;
  const double* QKV = a.w.QKV;
  const double* W = a.w.ATTW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int p = warp; p < S * TT; p += kWarps) {
    const int s = p / TT, t = (p / T) % T, u = p % T;
    const double* dc = a.w.DCTX + (int64_t)(s * T + t) * d;
    const double* v = QKV + (int64_t)(s * T + u) * 3 * d + 2 * d;
    double acc = 0.0;
#pragma unroll 8
    for (int c = lane; c < d; c += 32) acc += dc[c] * v[c];
    acc = warp_sum(acc);
    if (lane == 0) dW[p] = acc;
  }
  __syncthreads();
  const double scale = 1.0 / sqrt((double)d);
  for (int row = threadIdx.x; row < S * T; row += kThreads) {
    double sm1 = 0.0;
    for (int u = 0; u < T; ++u) sm1 += dW[row * T + u] * W[row * T + u];
    for (int u = 0; u < T; ++u) dS[row * T + u] = W[row * T + u] * (dW[row * T + u] - sm1) * scale;
  }
  __syncthreads();
  const int c = blockIdx.x * kThreads + threadIdx.x;
  if (c >= d) return;
  for (int s = 0; s < S; ++s) {
    for (int t = 0; t < T; ++t) {
      const int r = s * T + t;
      double dq = 0.0, dk = 0.0, dv = 0.0;
      for (int u = 0; u < T; ++u) {
        const int ru = s * T + u;
        dq += dS[r * T + u] * QKV[(int64_t)ru * 3 * d + d + c];          // d_scores @ k
        dk += dS[(s * T + u) * T + t] * QKV[(int64_t)ru * 3 * d + c];     // d_scores^T @ q
        dv += W[(s * T + u) * T + t] * a.w.DCTX[(int64_t)ru * d + c];     // weights^T @ d_context
      }
      a.w.DQKV[(int64_t)r * 3 * d + c] = dq;
      a.w.DQKV[(int64_t)r * 3 * d + d + c] = dk;
      a.w.DQKV[(int64_t)r * 3 * d + 2 * d + c] = dv;
    }
  }
}

// d embedded = d res1 + d qkv Wqkv^T (policy.py:455-464).
__global__ void __launch_bounds__(kThreads) bwd_embed(const __grid_constant__ Args a, int S) {
  extern __shared__ double sm[];
  const int d = a.d, R = S * a.T;
  double* DQ = sm;
#pragma unroll 4
  for (int i = threadIdx.x; i < R * 3 * d; i += kThreads) DQ[i] = a.w.DQKV[i];
  __syncthreads();
  const int e = blockIdx.x * kWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (e >= d) return;
  double o[kRowsMax];
  dywt_row(DQ, 3 * d, R, 3 * d, a.Wqkv, 3 * d, e, o);
  for (int r = lane; r < R; r += 32) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kRowsMax; ++q)
      if (q == r) v = o[q];
    a.w.DEMB[(int64_t)r * d + e] = a.w.DRES1[(int64_t)r * d + e] + v;
  }
}

// Adam (ppo.py:147-161) with every gradient element computed in place from
// the saved rows; flags non-finite parameters. One CTA per (segment, matrix
// row, 256-column chunk): the row's input values are loaded once, the output
// gradients are coalesced along the row.
__global__ void __launch_bounds__(kThreads) adam_kernel(const __grid_constant__ Args a,
                                                        const __grid_constant__ SegTable st, int S) {
  // segment of this CTA: lanes test one segment start each
  const int lane = threadIdx.x & 31;
  const bool ge = lane < st.n && st.s[lane].blk0 <= (int)blockIdx.x;
  const int q = __popc(__ballot_sync(0xffffffffu, ge)) - 1;
  const Seg& g = st.s[q];
  const int b = blockIdx.x - g.blk0;
  const int i = b / g.colblocks;
  const int j = (b - i * g.colblocks) * kThreads + threadIdx.x;
  if (j >= g.cols) return;
  double grad = 0.0;
  if (g.kind == 0) {
#pragma unroll
    for (int r = 0; r < kRowsMax; ++r) {
      if (r >= g.nrows) break;
      grad += g.x[(int64_t)r * g.ldx + i] * g.dy[(int64_t)r * g.lddy + j];
    }
  } else if (g.row_div == 1) {
#pragma unroll
    for (int r = 0; r < kRowsMax; ++r) {
      if (r >= g.nrows) break;
      const double dy = g.dy[(int64_t)r * g.lddy + j];
      grad += g.kind == 1 ? dy : dy * g.x[(int64_t)r * g.ldx + j];
    }
  } else {  // LayerNorm 2: dy = d pooled / T broadcast over the sample's rows (policy.py:421)
    for (int r = 0; r < g.nrows; ++r) {
      const double dy = g.dy[(int64_t)(r / g.row_div) * g.lddy + j] / g.div;
      grad += g.kind == 1 ? dy : dy * g.x[(int64_t)r * g.ldx + j];
    }
  }
  const int64_t idx = g.off + (int64_t)i * g.cols + j;
  if (a.G) a.G[idx] = grad;
  const double lr = a.w.HYP[0], bias1 = a.w.HYP[1], bias2 = a.w.HYP[2];
  double m = a.Mo[idx], v = a.Vo[idx];
  m = m * a.beta1 + (1.0 - a.beta1) * grad;
  v = v * a.beta2 + (1.0 - a.beta2) * grad * grad;
  const double p = a.P[idx] - lr * (m / bias1) / (sqrt(v / bias2) + a.eps);
  a.Mo[idx] = m;
  a.Vo[idx] = v;
  a.P[idx] = p;
  if (!isfinite(p)) atomicOr(a.status, 2);
}

// ---- host side ---------------------------------------------------------------

int64_t align32(int64_t x) { return (x + 31) & ~int64_t(31); }

bool layout_of(const ls_policy_dims& D, ls_policy_layout& out) {
  if (D.obs_dim < 1 || D.obs_dim > LS_MAX_HEADS || D.width < 1 || D.ffn_width < 1 || D.history_len < 1 ||
      D.num_heads < 1 || D.num_heads > LS_MAX_HEADS || D.kmax < 1 || D.n_steps < 1)
    return false;
  const int64_t A = D.obs_dim, d = D.width, f = D.ffn_width, HK = (int64_t)D.num_heads * D.kmax;
  const int64_t sz[LS_PSEG_COUNT] = {A * d, d, d * 3 * d, 3 * d, d * d, d, d, d, d * f, f, f * d, d, d, d,
                                     d * HK, HK, d * d, d, d, 1};
  int64_t off = 0;
  for (int i = 0; i < LS_PSEG_COUNT; ++i) {
    out.off[i] = off;
    off = align32(off + sz[i]);
  }
  out.total = off;
  return true;
}

struct WsLayout {
  int64_t n[27];
  int64_t total;
};

WsLayout ws_layout(const ls_policy_dims& D) {
  const int64_t d = D.width, f = D.ffn_width, T = D.history_len, SM = D.n_steps, RM = SM * T,
                HK = (int64_t)D.num_heads * D.kmax;
  WsLayout w;
  const int64_t n[27] = {RM * d,  RM * 3 * d, SM * T * T, RM * d,  RM * d,     RM * d, RM,     RM * d,  RM * f,
                         RM * d,  RM * d,     RM,         SM * d,  SM * HK,    SM * d, SM * HK, SM,      SM * d,
                         SM * d,  RM * d,     RM * f,     RM * d,  RM * d,     RM * d, RM * 3 * d, RM * d, 4};
  w.total = 0;
  for (int i = 0; i < 27; ++i) {
    w.n[i] = n[i];
    w.total += align32(n[i]);
  }
  return w;
}

size_t red_bytes() { return sizeof(double) * kRedDoubles; }

// dynamic shared memory per stage
struct Smem {
  size_t embed, attn, ln1, ffn2, ln2, fin, pool, b_ln2, b_ffn1, b_ln1, b_attn, b_embed;
};

Smem smem_of(const ls_policy_dims& D, int R) {
  const size_t d = D.width, f = D.ffn_width, T = D.history_len, A = D.obs_dim, S = R / T,
               HK = (size_t)D.num_heads * D.kmax, H = D.num_heads, db = sizeof(double);
  Smem s;
  s.embed = red_bytes() + db * R * (A + d);
  s.attn = red_bytes() + db * (S * T * T + R * d);
  s.ln1 = red_bytes() + db * R * d;
  s.ffn2 = red_bytes() + db * R * f;
  s.ln2 = red_bytes() + db * (R * d + S * d);
  s.fin = db * (3 * S * HK + 3 * S * H + 2 * S);
  s.pool = db * (S * HK + S * d);
  s.b_ln2 = db * R * d;
  s.b_ffn1 = db * R * f;
  s.b_ln1 = db * R * d;
  s.b_attn = db * 2 * S * T * T;
  s.b_embed = db * R * 3 * d;
  return s;
}

size_t smem_max(const Smem& s) {
  return std::max({s.embed, s.attn, s.ln1, s.ffn2, s.ln2, s.fin, s.pool, s.b_ln2, s.b_ffn1, s.b_ln1, s.b_attn,
                   s.b_embed});
}

bool supported(const ls_policy_dims& D) {
  ls_policy_layout l;
  if (!layout_of(D, l)) return false;
  if ((int64_t)D.n_steps * D.history_len > kRowsMax || D.n_steps > 8 || D.kmax > 64) return false;
  if (D.num_heads != D.obs_dim) return false;
  return smem_max(smem_of(D, D.n_steps * D.history_len)) <= kSmemMax;
}

cudaError_t set_smem_attrs() {
  static bool done = false;
  if (done) return cudaSuccess;
  const int b = (int)kSmemMax;
  cudaFuncSetAttribute(fwd_embed_qkv, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(fwd_attn_out, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(fwd_ln1_ffn1, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(fwd_ffn2, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(fwd_ln2_heads, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(fwd_final<MODE_SAMPLE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(fwd_final<MODE_SAMPLE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(fwd_final<MODE_CONF, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(fwd_final<MODE_TRAIN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(fwd_final<MODE_PROBE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(bwd_pool, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(bwd_ln2_ffn2, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(bwd_ffn1, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(bwd_ln1_wo, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(bwd_attn, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  cudaFuncSetAttribute(bwd_embed, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  done = true;
  return cudaGetLastError();
}

Args make_args(const ls_ppo_plan& p) {
  const ls_policy_dims& D = p.dims;
  ls_policy_layout l;
  layout_of(D, l);
  Args a;
  std::memset(&a, 0, sizeof(a));
  a.A = D.obs_dim;
  a.d = D.width;
  a.f = D.ffn_width;
  a.T = D.history_len;
  a.H = D.num_heads;
  a.K = D.kmax;
  a.HK = D.num_heads * D.kmax;
  a.SM = D.n_steps;
  a.RM = D.n_steps * D.history_len;
  const double* P = p.params;
  a.We = P + l.off[LS_PSEG_EMBED_W];
  a.be = P + l.off[LS_PSEG_EMBED_B];
  a.Wqkv = P + l.off[LS_PSEG_WQKV];
  a.bqkv = P + l.off[LS_PSEG_BQKV];
  a.Wo = P + l.off[LS_PSEG_WO];
  a.bo = P + l.off[LS_PSEG_BO];
  a.g1 = P + l.off[LS_PSEG_LN1_G];
  a.c1 = P + l.off[LS_PSEG_LN1_B];
  a.W1 = P + l.off[LS_PSEG_FFN_W1];
  a.b1 = P + l.off[LS_PSEG_FFN_B1];
  a.W2 = P + l.off[LS_PSEG_FFN_W2];
  a.b2 = P + l.off[LS_PSEG_FFN_B2];
  a.g2 = P + l.off[LS_PSEG_LN2_G];
  a.c2 = P + l.off[LS_PSEG_LN2_B];
  a.Wh = P + l.off[LS_PSEG_HEAD_W];
  a.bh = P + l.off[LS_PSEG_HEAD_B];
  a.Wv1 = P + l.off[LS_PSEG_VALUE_W1];
  a.bv1 = P + l.off[LS_PSEG_VALUE_B1];
  a.Wv2 = P + l.off[LS_PSEG_VALUE_W2];
  a.bv2 = P + l.off[LS_PSEG_VALUE_B2];
  a.P = p.params;
  a.Mo = p.adam_m;
  a.Vo = p.adam_v;
  a.G = p.grad_out;
  a.total = l.total;
  WsLayout wl = ws_layout(D);
  double* base = static_cast<double*>(p.workspace);
  double** ptrs[27] = {&a.w.E,    &a.w.QKV,   &a.w.ATTW, &a.w.CTX,  &a.w.RES1,  &a.w.N1,    &a.w.IS1,
                       &a.w.H1,   &a.w.ACT,   &a.w.RES2, &a.w.N2,   &a.w.IS2,   &a.w.POOL,  &a.w.LRAW,
                       &a.w.VH,   &a.w.DL,    &a.w.DVAL, &a.w.DVPRE, &a.w.DPOOL, &a.w.DRES2, &a.w.DPRE,
                       &a.w.DH1,  &a.w.DRES1, &a.w.DCTX, &a.w.DQKV, &a.w.DEMB, &a.w.HYP};
  for (int i = 0; i < 27; ++i) {
    *ptrs[i] = base;
    base += align32(wl.n[i]);
  }
  a.X = p.batch_obs;
  a.blocked = p.blocked;
  a.head_size = p.head_size;
  a.denom = p.obs_denom;
  a.env = p.env;
  a.uniforms = p.uniforms;
  a.lr_table = p.lr_table;
  a.spent = p.spent;
  a.adam_step = p.adam_step;
  a.status = p.status;
  a.b_act = p.batch_action;
  a.b_logp = p.batch_logp;
  a.b_val = p.batch_value;
  a.b_rew = p.batch_reward;
  a.tau = p.tau;
  a.clip = p.clip_eps;
  a.vc = p.value_coef;
  a.ec = p.entropy_coef;
  a.beta1 = p.beta1;
  a.beta2 = p.beta2;
  a.eps = p.adam_eps;
  return a;
}

SegTable seg_table(const Args& a, const ls_policy_layout& l, int S) {
  const int R = S * a.T;
  const int64_t d = a.d, f = a.f, A = a.A, HK = a.HK;
  SegTable t;
  t.n = LS_PSEG_COUNT;
  auto mat = [&](int q, int64_t rows, int64_t cols, const double* x, int64_t ldx, const double* dy, int64_t lddy,
                 int nrows) { t.s[q] = Seg{0, 0, l.off[q], rows, cols, 0, nrows, x, ldx, dy, lddy, 1, 1.0}; };
  auto vec = [&](int q, int64_t cols, int kind, const double* x, const double* dy, int nrows, int row_div,
                 double div) { t.s[q] = Seg{0, 0, l.off[q], 0, cols, kind, nrows, x, cols, dy, cols, row_div, div}; };
  mat(LS_PSEG_EMBED_W, A, d, a.X, A, a.w.DEMB, d, R);
  vec(LS_PSEG_EMBED_B, d, 1, nullptr, a.w.DEMB, R, 1, 1.0);
  mat(LS_PSEG_WQKV, d, 3 * d, a.w.E, d, a.w.DQKV, 3 * d, R);
  vec(LS_PSEG_BQKV, 3 * d, 1, nullptr, a.w.DQKV, R, 1, 1.0);
  mat(LS_PSEG_WO, d, d, a.w.CTX, d, a.w.DRES1, d, R);
  vec(LS_PSEG_BO, d, 1, nullptr, a.w.DRES1, R, 1, 1.0);
  vec(LS_PSEG_LN1_G, d, 2, a.w.N1, a.w.DH1, R, 1, 1.0);
  vec(LS_PSEG_LN1_B, d, 1, nullptr, a.w.DH1, R, 1, 1.0);
  mat(LS_PSEG_FFN_W1, d, f, a.w.H1, d, a.w.DPRE, f, R);
  vec(LS_PSEG_FFN_B1, f, 1, nullptr, a.w.DPRE, R, 1, 1.0);
  mat(LS_PSEG_FFN_W2, f, d, a.w.ACT, f, a.w.DRES2, d, R);
  vec(LS_PSEG_FFN_B2, d, 1, nullptr, a.w.DRES2, R, 1, 1.0);
  vec(LS_PSEG_LN2_G, d, 2, a.w.N2, a.w.DPOOL, R, a.T, (double)a.T);
  vec(LS_PSEG_LN2_B, d, 1, nullptr, a.w.DPOOL, R, a.T, (double)a.T);
  mat(LS_PSEG_HEAD_W, d, HK, a.w.POOL, d, a.w.DL, HK, S);
  vec(LS_PSEG_HEAD_B, HK, 1, nullptr, a.w.DL, S, 1, 1.0);
  mat(LS_PSEG_VALUE_W1, d, d, a.w.POOL, d, a.w.DVPRE, d, S);
  vec(LS_PSEG_VALUE_B1, d, 1, nullptr, a.w.DVPRE, S, 1, 1.0);
  mat(LS_PSEG_VALUE_W2, d, 1, a.w.VH, d, a.w.DVAL, 1, S);
  vec(LS_PSEG_VALUE_B2, 1, 1, nullptr, a.w.DVAL, S, 1, 1.0);
  int blocks = 0;
  for (int q = 0; q < t.n; ++q) {
    Seg& g = t.s[q];
    g.colblocks = (int)((g.cols + kThreads - 1) / kThreads);
    g.blk0 = blocks;
    blocks += (int)(g.rows ? g.rows : 1) * g.colblocks;
  }
  t.blocks = blocks;
  return t;
}

unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

void forward_rows(const Args& a, const ls_policy_dims& D, int row0, int R, int build, cudaStream_t s) {
  const Smem m = smem_of(D, R);
  fwd_embed_qkv<<<cdiv(3 * a.d, kCols), kThreads, m.embed, s>>>(a, row0, R, build);
  fwd_attn_out<<<cdiv(a.d, kCols), kThreads, m.attn, s>>>(a, row0, R);
  fwd_ln1_ffn1<<<cdiv(a.f, kCols), kThreads, m.ln1, s>>>(a, row0, R);
  fwd_ffn2<<<cdiv(a.d, kCols), kThreads, m.ffn2, s>>>(a, row0, R);
  fwd_ln2_heads<<<cdiv(a.HK, kCols) + cdiv(a.d, kCols), kThreads, m.ln2, s>>>(a, row0, R);
}

template <int MODE>
void final_stage(const Args& a, const ls_policy_dims& D, int slot0, int S, const PpoCtx& c, cudaStream_t s) {
  size_t sm = smem_of(D, S * D.history_len).fin;
  if (MODE == MODE_SAMPLE) {
    sm += sizeof(int64_t) * (size_t)a.env.elite_capacity * (a.A + 1);
    if (!c.neumaier) {
      fwd_final<MODE, false><<<1, kThreads, sm, s>>>(a, slot0, S, c.tab, c.L, c.M);
      return;
    }
  }
  fwd_final<MODE, true><<<1, kThreads, sm, s>>>(a, slot0, S, c.tab, c.L, c.M);
}

void backward_adam(const Args& a, const ls_policy_dims& D, int S, cudaStream_t s) {
  const Smem m = smem_of(D, S * D.history_len);
  ls_policy_layout l;
  layout_of(D, l);
  bwd_pool<<<cdiv(a.d, kWarps), kThreads, m.pool, s>>>(a, S);
  bwd_ln2_ffn2<<<cdiv(a.f, kWarps), kThreads, m.b_ln2, s>>>(a, S);
  bwd_ffn1<<<cdiv(a.d, kWarps), kThreads, m.b_ffn1, s>>>(a, S);
  bwd_ln1_wo<<<cdiv(a.d, kWarps), kThreads, m.b_ln1, s>>>(a, S);
  bwd_attn<<<cdiv(a.d, kThreads), kThreads, m.b_attn, s>>>(a, S);
  bwd_embed<<<cdiv(a.d, kWarps), kThreads, m.b_embed, s>>>(a, S);
  const SegTable st = seg_table(a, l, S);
  adam_kernel<<<(unsigned)st.blocks, kThreads, 0, s>>>(a, st, S);
}

}  // namespace

bool ppo_layout(const ls_policy_dims& D, ls_policy_layout* out) { return layout_of(D, *out); }

size_t ppo_workspace_bytes(const ls_policy_dims& D) {
  if (!supported(D)) return 0;
  return sizeof(double) * (size_t)ws_layout(D).total;
}

cudaError_t ppo_prime(const ls_ppo_plan& p, const PpoCtx& c, cudaStream_t s) {
  cudaError_t e = set_smem_attrs();
  if (e != cudaSuccess) return e;
  const Args a = make_args(p);
  forward_rows(a, p.dims, 0, p.dims.history_len, 1, s);
  return cudaGetLastError();
}

cudaError_t ppo_round(const ls_ppo_plan& p, const PpoCtx& c, int n, cudaStream_t s) {
  cudaError_t e = set_smem_attrs();
  if (e != cudaSuccess) return e;
  const Args a = make_args(p);
  const ls_policy_dims& D = p.dims;
  const int T = D.history_len;
  if ((e = cudaMemsetAsync(p.status, 0, sizeof(int32_t), s)) != cudaSuccess) return e;
  // samples (collect, ppo.py:170-200): slot 0 was primed by the last confidence forward
  final_stage<MODE_SAMPLE>(a, D, 0, 1, c, s);
  for (int j = 1; j < n; ++j) {
    forward_rows(a, D, j * T, T, 1, s);
    final_stage<MODE_SAMPLE>(a, D, j, 1, c, s);
  }
  // ppo_update (ppo.py:297-327): epoch 1 reuses the sampling forwards
  for (int ep = 0; ep < p.epochs; ++ep) {
    if (ep) forward_rows(a, D, 0, n * T, 0, s);
    final_stage<MODE_TRAIN>(a, D, 0, n, c, s);
    backward_adam(a, D, n, s);
  }
  // confidence check (ppo.py:356-358) = next round's first sampling forward
  forward_rows(a, D, 0, T, 1, s);
  final_stage<MODE_CONF>(a, D, 0, 1, c, s);
  return cudaGetLastError();
}

cudaError_t ppo_forward(const ls_ppo_plan& p, const PpoCtx& c, int n, double* logp, double* value, cudaStream_t s) {
  cudaError_t e = set_smem_attrs();
  if (e != cudaSuccess) return e;
  Args a = make_args(p);
  a.out_logp = logp;
  a.out_val = value;
  forward_rows(a, p.dims, 0, n * p.dims.history_len, 0, s);
  final_stage<MODE_PROBE>(a, p.dims, 0, n, c, s);
  return cudaGetLastError();
}

cudaError_t ppo_update(const ls_ppo_plan& p, const PpoCtx& c, int n, cudaStream_t s) {
  cudaError_t e = set_smem_attrs();
  if (e != cudaSuccess) return e;
  const Args a = make_args(p);
  for (int ep = 0; ep < p.epochs; ++ep) {
    forward_rows(a, p.dims, 0, n * p.dims.history_len, 0, s);
    final_stage<MODE_TRAIN>(a, p.dims, 0, n, c, s);
    backward_adam(a, p.dims, n, s);
  }
  return cudaGetLastError();
}

}  // namespace ls
