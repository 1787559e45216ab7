// Attention-LSTM decoder step pieces (operand packing, Bahdanau attention with
// the fp64 attention accumulator + coverage, row log-softmax) and the word-LM
// bookkeeping of the fused engine (speculative <eos> events, word-boundary
// slot plan, row copies).
//
// Model equations: DESIGN.md §3; search semantics:
// decoder.py:419-425 (accumulator), fusion.py:177-223 (LM events).
#include "common.cuh"

#include <cstdlib>

#include <cuda_bf16.h>

namespace fb {

// ---------------------------------------------------------------- packing --
// One warp per output row, 4 consecutive columns per lane (float4 in, 8-byte
// 4 x 16-bit per operand plane out, split_operand) when the segment allows it.
__global__ void __launch_bounds__(256)
pack_rows_kernel(fb_pack_t p, int m_max, const int32_t* __restrict__ m_dev,
                 const int32_t* __restrict__ rows, const int32_t* __restrict__ parent,
                 const int32_t* __restrict__ tokens, const int32_t* __restrict__ ranks,
                 float* __restrict__ out, int64_t ld_out) {
  pdl_entry();
  const int m = row_count(m_max, m_dev);
  const bool split = p.out_mode == 1;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  uint16_t* ob = reinterpret_cast<uint16_t*>(out);
  const int64_t plane = p.plane_rows * ld_out;
  for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < m; i += gridDim.x * wpb) {
    // resolve every segment's source row first (the index loads overlap)
    const int sl = rows ? rows[i] : i;
    const int pr = (parent && (p.nseg > 0)) ? parent[sl] : sl;
    const int tk = tokens ? tokens[sl] : -1;
    const int rk = ranks ? ranks[i] : -1;
    int col = 0;
    for (int s = 0; s <= p.nseg; ++s) {
      const float* src = nullptr;
      int width;
      if (s < p.nseg) {
        const fb_seg_t& sg = p.seg[s];
        if (sg.mode == 5) {                         // columns owned by another writer
          col += sg.width;
          continue;
        }
        int64_t r;
        switch (sg.mode) {
          case 0: r = i; break;
          case 1: r = sl; break;
          case 2: r = pr; break;
          case 3: r = tk < 0 ? p.tok_default : tk; break;
          default: r = rk < 0 ? p.tok_default : rk; break;
        }
        src = sg.src ? sg.src + r * sg.ld : nullptr;
        width = sg.width;
      } else {
        width = p.k_pad - col;                      // zero padding
      }
      const bool vec = ((width & 3) == 0) && ((col & 3) == 0) &&
                       (!src || (reinterpret_cast<uintptr_t>(src) & 15) == 0);
      if (vec) {
        // four float4 per lane in flight before any store
        for (int j0 = lane * 4; j0 < width; j0 += 512) {
          float4 v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int j = j0 + 128 * q;
            v[q] = (src && j < width) ? __ldg(reinterpret_cast<const float4*>(src + j))
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int j = j0 + 128 * q;
            if (j >= width) break;
            const int64_t o = (int64_t)i * ld_out + col + j;
            if (!split) {
              *reinterpret_cast<float4*>(out + o) = v[q];
            } else {
              uint16_t e[4][3], pl[3][4];
              split_operand(v[q].x, e[0]);
              split_operand(v[q].y, e[1]);
              split_operand(v[q].z, e[2]);
              split_operand(v[q].w, e[3]);
#pragma unroll
              for (int pp = 0; pp < kPlanes; ++pp) {
#pragma unroll
                for (int c = 0; c < 4; ++c) pl[pp][c] = e[c][pp];
                *reinterpret_cast<uint2*>(ob + pp * plane + o) = *reinterpret_cast<uint2*>(pl[pp]);
              }
            }
          }
        }
      } else {
        for (int j = lane; j < width; j += 32) {
          const float x = src ? src[j] : 0.f;
          const int64_t o = (int64_t)i * ld_out + col + j;
          if (!split) {
            out[o] = x;
          } else {
            uint16_t e[3];
            split_operand(x, e);
#pragma unroll
            for (int pp = 0; pp < kPlanes; ++pp) ob[pp * plane + o] = e[pp];
          }
        }
      }
      col += width;
    }
  }
}

// ------------------------------------------------------------ log-softmax --
__global__ void log_softmax_kernel(int m_max, const int32_t* __restrict__ m_dev,
                                   const int32_t* __restrict__ rows, const float* __restrict__ x,
                                   int64_t ldx, int n, float* __restrict__ out, int64_t ldo) {
  const int m = row_count(m_max, m_dev);
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < m; i += gridDim.x * wpb) {
    const int r = rows ? rows[i] : i;
    const float* xr = x + (int64_t)r * ldx;
    float mx = -INFINITY;
    for (int j = lane; j < n; j += 32) mx = fmaxf(mx, xr[j]);
    for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    // the normaliser accumulates in fp64: over thousands of outputs an fp32
    // sum drops every term below half an ulp of the running sum, which biases
    // log P upward by ~1e-7 per step -- coherent over a long decode
    double s = 0.0;
    for (int j = lane; j < n; j += 32) s += (double)expf(xr[j] - mx);
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    const double lse = log(s);
    float* o = out + (int64_t)r * ldo;
    for (int j = lane; j < n; j += 32) o[j] = (float)((double)(xr[j] - mx) - lse);
  }
}

// Token-LM log-normaliser in fp64 (oracle: fp64 softmax of the fp32 logits):
// one warp per row, exact fp64 exp of (x - max).
__global__ void row_lse_kernel(int m_max, const int32_t* __restrict__ m_dev,
                               const int32_t* __restrict__ rows, const float* __restrict__ x,
                               int64_t ldx, int n, int skip, double* __restrict__ out) {
  const int m = row_count(m_max, m_dev);
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < m; i += gridDim.x * wpb) {
    const int r = rows ? rows[i] : i;
    const float* xr = x + (int64_t)r * ldx;
    float mx = -INFINITY;
    for (int j = lane; j < n; j += 32)
      if (j != skip) mx = fmaxf(mx, xr[j]);
    for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const double m0 = (double)mx;
    double s = 0.0;
    for (int j = lane; j < n; j += 32)
      if (j != skip) s += exp((double)xr[j] - m0);
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) out[r] = m0 + log(s);
  }
}

// -------------------------------------------------------------- attention --
__device__ __forceinline__ float tanh_fast(float x) {
  // 1 - 2/(e^{2x}+1) with MUFU ex2/rcp: absolute error ~2e-7; the clamp keeps
  // __fdividef in range (tanh(15) == 1 in fp32)
  x = fminf(fmaxf(x, -15.0f), 15.0f);
  const float e = __expf(2.0f * x);
  return 1.0f - __fdividef(2.0f, e + 1.0f);
}


template <typename F>
__device__ double pairwise_sum_d(const double* a, int n, F f) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = dadd(res, f(a[i]));
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = f(a[j]);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = dadd(r[j], f(a[i + j]));
    }
    double res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
    for (; i < n; ++i) res = dadd(res, f(a[i]));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return dadd(pairwise_sum_d(a, n2, f), pairwise_sum_d(a + n2, n - n2, f));
}

// Bahdanau attention in two balanced kernels.
// (A) energies: CTA = (utterance, chunk of 8 x kEnWarps frames); warp = frame
//     t; lanes split the attention dim; every live row's energy for frame t is
//     a warp reduction.  MUFU-bound (ex2 + rcp per tanh).
// (B) softmax / fp64 accumulator / coverage / context: CTA = (utterance, group
//     of RB rows), thread = 4 encoder columns: the encoder output is streamed
//     from HBM once per row group (HBM-bound; it does not fit L2 at c2).


constexpr int kMaxBeam = 512;
constexpr int kCtxMaxThreads = 512;   // context CTA: one thread per 4 encoder columns
// 1 + E_k E_q clamp: tanh is saturated (2/(1+1e18) = 2e-18) and a product of
// two clamped terms (1e36) stays below FLT_MAX
constexpr float kDMax2 = 1.0e18f;
constexpr float kDMax4 = 1.0e9f;      // four-term grouping (FB_ENERGY_QUAD)
#ifndef FB_ENERGY_QUAD
#define FB_ENERGY_QUAD 1
#endif

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// keys arrive as E_k = exp(2 K) (fb_exp2x after the key projection) and the
// query as E_q = exp(2 q) (here), so tanh(k + q) = 1 - 2 / (1 + E_k E_q) and
// e_t = sum_a v_a - 2 sum_a v_a / (1 + E_k E_q).  The constant sum_a v_a
// cancels in the softmax, so the kernel stores e'_t = -2 sum_a v_a / (1 + E_k E_q):
// one FFMA + one MUFU.RCP + one FFMA per (row, frame, a).
// Softmax over frames + fp64 accumulator + coverage (decoder.py:421-425) for
// one row, by one warp: alpha[t] = softmax(e)[t] (e may live in shared memory,
// alpha in global), acc_out = acc_in[parent] + alpha (fp64), coverage.
__device__ __forceinline__ void softmax_row(const fb_search_cfg_t& cfg, int r, int T, int TM,
                                            const float* e, float* alpha, const int32_t* parent,
                                            const double* acc_in, double* acc_out,
                                            double* cov_out, float* attn_out, int64_t ld_attn,
                                            int lane) {
  float mx = -INFINITY;
  for (int t = lane; t < T; t += 32) mx = fmaxf(mx, __ldcg(e + t));
  for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  float sum = 0.f;
  for (int t = lane; t < T; t += 32) sum += expf(__ldcg(e + t) - mx);
  for (int off = 16; off; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
  const float inv = 1.0f / sum;
  const int p = parent ? parent[r] : r;
  const double* a0 = acc_in + (int64_t)p * TM;
  double* a1 = acc_out + (int64_t)r * TM;
  int cnt = 0;
  for (int t = lane; t < T; t += 32) {
    const float a = expf(__ldcg(e + t) - mx) * inv;
    alpha[t] = a;
    const double x = dadd(a0[t], (double)a);
    a1[t] = x;
    cnt += x > cfg.tau1;
    if (attn_out) attn_out[(int64_t)r * ld_attn + t] = a;
  }
  if (cfg.cov_mode != 0) {
    for (int off = 16; off; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
    __syncwarp();
    if (lane == 0) {
      double cov;
      if (cfg.cov_mode == 1) {
        cov = (double)cnt;
      } else {
        const double tau2 = cfg.tau2, mg = cfg.cov_margin;
        const double pen = pairwise_sum_d(a1, T, [=](double x) {
          return x > tau2 ? dsub(dadd(mg, x), tau2) : 0.0;
        });
        cov = dsub((double)cnt, pen);
      }
      cov_out[r] = cov;
    }
  }
}

// Separate softmax pass (utterances longer than one energy CTA): one warp per
// live row; alpha overwrites the energy row in place.
__global__ void __launch_bounds__(256)
att_softmax_kernel(fb_search_cfg_t cfg, const int32_t* __restrict__ active,
                   const int32_t* __restrict__ n_live, const int32_t* __restrict__ t_enc,
                   float* __restrict__ energy, const int32_t* __restrict__ parent,
                   const double* __restrict__ acc_in, double* __restrict__ acc_out,
                   double* __restrict__ cov_out, float* __restrict__ attn_out, int64_t ld_attn) {
  const int u = blockIdx.x;
  if (!active[u]) return;
  const int i = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n_live[u]) return;
  const int r = u * cfg.beam + i;
  float* e = energy + (int64_t)r * cfg.t_max;
  softmax_row(cfg, r, t_enc[u], cfg.t_max, e, e, parent, acc_in, acc_out, cov_out, attn_out,
              ld_attn, threadIdx.x & 31);
}

// packed fp32 pairs (sm_100 FFMA2 / FMUL2: two lanes of work per issue)
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t pk2(float a, float b) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void up2(f2_t x, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x));
}
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
  f2_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) {
  f2_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// (FB_ENERGY_MINB=4: a 64-register cap puts four 8-warp CTAs on an SM -- 9 %
// faster at the all-live c2 shape, 1 % slower over the real c2 decode)
#ifndef FB_ENERGY_MINB
#define FB_ENERGY_MINB 1
#endif
#ifndef FB_ENERGY_PF
#define FB_ENERGY_PF 1   // groups of four key dims in flight ahead of the one in use
#endif
#ifndef FB_ENERGY_MINB8
// 256-frame CTAs with <= 10 rows (c2's main graph set): three CTAs per SM
// (77 registers, no spills) -- c2 163.6 -> 162.9-163.1 ms over three
// alternating A/B rounds; four (64 registers) is slower (166 ms)
#define FB_ENERGY_MINB8 3
#endif
template <int R, int kEnWarps>
__global__ void __launch_bounds__(kEnWarps * 32,
                                  (kEnWarps == 8 && R <= 10) ? FB_ENERGY_MINB8 : FB_ENERGY_MINB)
att_energy_kernel(fb_search_cfg_t cfg, const int32_t* __restrict__ active,
                  const int32_t* __restrict__ n_live, const int32_t* __restrict__ t_enc,
                  const float* __restrict__ ekt, int A, const float* __restrict__ v,
                  const float* __restrict__ q, int64_t ldq, float* __restrict__ energy,
                  int32_t* __restrict__ sync_ws, const int32_t* __restrict__ parent,
                  const double* __restrict__ acc_in, double* __restrict__ acc_out,
                  double* __restrict__ cov_out, float* __restrict__ attn_out, int64_t ld_attn,
                  int parts) {
  // CTA = (utterance, chunk of kEnWarps*32 frames, group of R rows); lane = one
  // frame t, so every energy is a private register sum (no cross-lane
  // reduction).  Keys are read transposed (E_K^T[u][a][t]: coalesced across
  // lanes); E_q (row pairs interleaved) and v are shared-memory broadcasts.
  // Work per (row pair, dim pair) = 4 terms v_a / d_a, d_a = 1 + E_k E_q:
  //   v0/d0 + v1/d1 = (v0 d1 + v1 d0) / (d0 d1)   -- one reciprocal per two
  // terms, rows paired in f32x2 registers (FFMA2/FMUL2); d clamped to kDMax2
  // so the product stays finite (tanh is saturated long before).
  // parts > 1: the attention dims are split over `parts` CTAs (blockIdx.y =
  // chunk * parts + part), each writing its partial sums to its own plane of
  // energy; the last CTA adds the planes in part order before the softmax.
  // (Twice the CTAs of half the work: at c2 one utterance per 8-warp CTA made
  // 1.15 waves, the second one almost empty.)
  static_assert(R % 2 == 0, "rows come in pairs");
  pdl_entry();
  const int u = blockIdx.x;
  if (!active[u]) return;
  const int T = t_enc[u];
  const int part = blockIdx.y % parts;
  const int t0 = (blockIdx.y / parts) * (kEnWarps * 32);
  if (t0 >= T) return;
  const int Ap = A / parts, a0 = part * Ap;
  const int n = n_live[u];
  const int r0 = blockIdx.z * R;
  if (r0 >= n) return;
  const int rows = min(R, n - r0);
  extern __shared__ float sm[];
  const int K = cfg.beam, TM = cfg.t_max;
  float2* vs2 = reinterpret_cast<float2*>(sm);          // [Ap]  (v_a, v_a)
  float2* qs2 = vs2 + Ap;                               // [R/2][Ap] (Eq_r, Eq_r+1)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot0 = u * K + r0;
  for (int rp = 0; rp < R / 2; ++rp) {
    const int ra = 2 * rp, rb = ra + 1;
    const float* qa = q + (int64_t)(slot0 + ra) * ldq + a0;
    const float* qb = q + (int64_t)(slot0 + rb) * ldq + a0;
    for (int a = tid; a < Ap; a += blockDim.x)
      qs2[rp * Ap + a] = make_float2(ra < rows ? qa[a] : 0.f, rb < rows ? qb[a] : 0.f);
  }
  for (int a = tid; a < Ap; a += blockDim.x) vs2[a] = make_float2(v[a0 + a], v[a0 + a]);
  __syncthreads();
  const int t = t0 + warp * 32 + lane;
  const bool valid = t < T;
  if (t0 + warp * 32 < T) {
  const float* kt = ekt + ((int64_t)u * A + a0) * TM + (valid ? t : T - 1);
  const f2_t one2 = pk2(1.0f, 1.0f);
  f2_t e2[R / 2];
#pragma unroll
  for (int rp = 0; rp < R / 2; ++rp) e2[rp] = pk2(0.f, 0.f);
  // keys for dims a..a+3 in registers, the next FB_ENERGY_PF groups of four
  // in flight (A % 4 == 0)
  float kb[FB_ENERGY_PF + 1][4];
#pragma unroll
  for (int p = 0; p <= FB_ENERGY_PF; ++p)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      kb[p][j] = 4 * p + j < Ap ? __ldg(kt + (int64_t)(4 * p + j) * TM) : 0.f;
  for (int a = 0; a < Ap; a += 4) {
    float kc[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) kc[j] = kb[0][j];
#pragma unroll
    for (int p = 0; p < FB_ENERGY_PF; ++p)
#pragma unroll
      for (int j = 0; j < 4; ++j) kb[p][j] = kb[p + 1][j];
    const int an = a + 4 * (FB_ENERGY_PF + 1);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      kb[FB_ENERGY_PF][j] = an + j < Ap ? __ldg(kt + (int64_t)(an + j) * TM) : 0.f;
#if FB_ENERGY_QUAD
    {
      // four dims per reciprocal: sum_a v_a/d_a over a..a+3 =
      //   [(v0 d1 + v1 d0) d2 d3 + (v2 d3 + v3 d2) d0 d1] / (d0 d1 d2 d3),
      // every d clamped to kDMax4 so the product stays below 1e36 (tanh is
      // saturated long before: the clamp moves a term by < 1e-9 |v|)
      const f2_t K0 = pk2(kc[0], kc[0]), K1 = pk2(kc[1], kc[1]);
      const f2_t K2 = pk2(kc[2], kc[2]), K3 = pk2(kc[3], kc[3]);
      const float4 va = *reinterpret_cast<const float4*>(vs2 + a);       // (v0,v0,v1,v1)
      const float4 vb = *reinterpret_cast<const float4*>(vs2 + a + 2);   // (v2,v2,v3,v3)
      const f2_t V0 = pk2(va.x, va.y), V1 = pk2(va.z, va.w);
      const f2_t V2 = pk2(vb.x, vb.y), V3 = pk2(vb.z, vb.w);
#pragma unroll
      for (int rp = 0; rp < R / 2; ++rp) {
        const float4 qa = *reinterpret_cast<const float4*>(qs2 + rp * Ap + a);
        const float4 qb = *reinterpret_cast<const float4*>(qs2 + rp * Ap + a + 2);
        f2_t d0 = fma2(K0, pk2(qa.x, qa.y), one2);
        f2_t d1 = fma2(K1, pk2(qa.z, qa.w), one2);
        f2_t d2 = fma2(K2, pk2(qb.x, qb.y), one2);
        f2_t d3 = fma2(K3, pk2(qb.z, qb.w), one2);
        float x0, y0, x1, y1, x2, y2, x3, y3;
        up2(d0, x0, y0);
        up2(d1, x1, y1);
        up2(d2, x2, y2);
        up2(d3, x3, y3);
        d0 = pk2(fminf(x0, kDMax4), fminf(y0, kDMax4));
        d1 = pk2(fminf(x1, kDMax4), fminf(y1, kDMax4));
        d2 = pk2(fminf(x2, kDMax4), fminf(y2, kDMax4));
        d3 = pk2(fminf(x3, kDMax4), fminf(y3, kDMax4));
        const f2_t p01 = mul2(d0, d1), p23 = mul2(d2, d3);
        const f2_t n01 = fma2(V0, d1, mul2(V1, d0));
        const f2_t n23 = fma2(V2, d3, mul2(V3, d2));
        const f2_t num = fma2(n01, p23, mul2(n23, p01));
        const f2_t den = mul2(p01, p23);
        float dx, dy;
        up2(den, dx, dy);
        e2[rp] = fma2(num, pk2(rcp_approx(dx), rcp_approx(dy)), e2[rp]);
      }
    }
#else
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const f2_t K0 = pk2(kc[2 * h], kc[2 * h]), K1 = pk2(kc[2 * h + 1], kc[2 * h + 1]);
      const float4 vv = *reinterpret_cast<const float4*>(vs2 + a + 2 * h);   // (v0,v0,v1,v1)
      const f2_t V0 = pk2(vv.x, vv.y), V1 = pk2(vv.z, vv.w);
#pragma unroll
      for (int rp = 0; rp < R / 2; ++rp) {
        const float4 qq = *reinterpret_cast<const float4*>(qs2 + rp * Ap + a + 2 * h);
        f2_t d0 = fma2(K0, pk2(qq.x, qq.y), one2);
        f2_t d1 = fma2(K1, pk2(qq.z, qq.w), one2);
        float x0, y0, x1, y1;
        up2(d0, x0, y0);
        up2(d1, x1, y1);
        d0 = pk2(fminf(x0, kDMax2), fminf(y0, kDMax2));
        d1 = pk2(fminf(x1, kDMax2), fminf(y1, kDMax2));
        const f2_t num = fma2(V0, d1, mul2(V1, d0));
        const f2_t den = mul2(d0, d1);
        float dx, dy;
        up2(den, dx, dy);
        e2[rp] = fma2(num, pk2(rcp_approx(dx), rcp_approx(dy)), e2[rp]);
      }
    }
#endif
  }
  if (valid) {
#pragma unroll
    for (int rp = 0; rp < R / 2; ++rp) {
      float ea, eb;
      up2(e2[rp], ea, eb);
      float* eo = energy + (int64_t)(blockIdx.y % parts) * gridDim.x * K * TM;   // part's plane
      if (2 * rp < rows) eo[(int64_t)(slot0 + 2 * rp) * TM + t] = -2.0f * ea;
      if (2 * rp + 1 < rows) eo[(int64_t)(slot0 + 2 * rp + 1) * TM + t] = -2.0f * eb;
    }
  }
  }
  // the last frame chunk of (utterance, row group) to finish runs the softmax,
  // fp64 accumulator and coverage of the group's rows (counter self-resets)
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    int32_t* cnt = sync_ws + (int64_t)u * gridDim.z + blockIdx.z;
    const int chunks = (T + kEnWarps * 32 - 1) / (kEnWarps * 32) * parts;
    const int prev = atomicAdd(cnt, 1);
    s_last = prev + 1 == chunks;
    if (s_last) *cnt = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int i = warp; i < rows; i += kEnWarps) {
    float* er = energy + (int64_t)(slot0 + i) * TM;
    if (parts > 1) {
      for (int tt = lane; tt < T; tt += 32) {
        float e = er[tt];
        for (int p = 1; p < parts; ++p) e += er[(int64_t)p * gridDim.x * K * TM + tt];
        er[tt] = e;
      }
      __syncwarp();
    }
    softmax_row(cfg, slot0 + i, T, TM, er, er, parent, acc_in, acc_out, cov_out, attn_out,
                ld_attn, lane);
  }
}

// E_q = exp(2 q) in place for the live rows of active utterances (once per
// step, instead of once per energy CTA)
__global__ void query_exp_kernel(int num_utts, int beam, const int32_t* __restrict__ active,
                                 const int32_t* __restrict__ n_live, float* __restrict__ q,
                                 int64_t ldq, int nq4) {
  const int64_t total = (int64_t)num_utts * beam * nq4;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / nq4), a4 = (int)(idx - (int64_t)r * nq4);
    const int u = r / beam, i = r - u * beam;
    if (!active[u] || i >= n_live[u]) continue;
    float4* p = reinterpret_cast<float4*>(q + (int64_t)r * ldq) + a4;
    float4 x = *p;
    x.x = expf(2.0f * x.x);
    x.y = expf(2.0f * x.y);
    x.z = expf(2.0f * x.z);
    x.w = expf(2.0f * x.w);
    *p = x;
  }
}

// ekt[u][a][t] = exp(2 k[u][t][a]): the attention keys in the layout the
// energy kernel reads (32 x 32 tiles through shared memory)
__global__ void keys_exp2t_kernel(int t_max, int A, const float* __restrict__ k,
                                  float* __restrict__ ekt) {
  __shared__ float tile[32][33];
  const int u = blockIdx.z;
  const int t0 = blockIdx.x * 32, a0 = blockIdx.y * 32;
  const float* ku = k + (int64_t)u * t_max * A;
  float* eu = ekt + (int64_t)u * A * t_max;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int t = t0 + i, a = a0 + threadIdx.x;
    tile[i][threadIdx.x] = (t < t_max && a < A) ? expf(2.0f * ku[(int64_t)t * A + a]) : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int a = a0 + i, t = t0 + threadIdx.x;
    if (a < A && t < t_max) eu[(int64_t)a * t_max + t] = tile[threadIdx.x][i];
  }
}

__global__ void exp2x_kernel(int64_t n, const float* __restrict__ x, float* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = expf(2.0f * x[i]);
}


#ifndef FB_CTX_TU
#define FB_CTX_TU 8      // encoder frames per thread in flight (float4 each)
#endif
template <int RB>
#ifdef FB_CTX_MAXREG   // register cap for more resident context CTAs
__global__ void __maxnreg__(RB <= 12 ? FB_CTX_MAXREG : 128)
#else
__global__ void __launch_bounds__(kCtxMaxThreads)
#endif
att_context_kernel(fb_search_cfg_t cfg, const int32_t* __restrict__ active,
                   const int32_t* __restrict__ n_live, const int32_t* __restrict__ t_enc,
                   const float* __restrict__ enc, int C, const float* __restrict__ alpha,
                   float* __restrict__ ctx_out, int64_t ld_ctx, uint16_t* __restrict__ planes,
                   int64_t plane_stride, int64_t ld_planes, const int32_t* __restrict__ row_pos) {
  // CTA = (utterance, group of RB rows, column chunk); thread = 4 adjacent
  // encoder columns (float4 loads, register double buffer), alpha tile in smem.
  // planes != NULL: the context is also stored as operand planes at GEMM row
  // row_pos[slot] (the output GEMM's A, which then needs no pack)
  pdl_entry();
  const int u = blockIdx.x;
  if (!active[u]) return;
  const int n = n_live[u];
  const int g0 = blockIdx.y * RB;
  if (g0 >= n) return;
  const int rows = min(RB, n - g0);
  extern __shared__ float sm[];
  const int K = cfg.beam, TM = cfg.t_max;
  const int T = t_enc[u];
  float* at = sm;                                      // [T][RB] alpha, transposed
  const int tid = threadIdx.x;
  const int slot0 = u * K + g0;
  const int col = 4 * (blockIdx.z * blockDim.x + tid);
  const bool has_col = col < C;
  const float* eu = enc + (int64_t)u * TM * C + (has_col ? col : 0);
  constexpr int TU = FB_CTX_TU;
  float4 xn[TU];
  if (has_col && TU <= T) {       // first frames in flight before the alpha tile
#pragma unroll
    for (int j = 0; j < TU; ++j) xn[j] = __ldg(reinterpret_cast<const float4*>(eu + (int64_t)j * C));
  }
  for (int j = tid; j < T * RB; j += blockDim.x) {
    const int r = j / T, t = j - r * T;
    at[t * RB + r] = r < rows ? alpha[(int64_t)(slot0 + r) * TM + t] : 0.f;
  }
  __syncthreads();
  if (!has_col) return;
  float4 acc[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
  int t = 0;
  for (; t + TU <= T; t += TU) {
    float4 x[TU];
#pragma unroll
    for (int j = 0; j < TU; ++j) x[j] = xn[j];
    if (t + 2 * TU <= T) {
#pragma unroll
      for (int j = 0; j < TU; ++j)
        xn[j] = __ldg(reinterpret_cast<const float4*>(eu + (int64_t)(t + TU + j) * C));
    }
#pragma unroll
    for (int j = 0; j < TU; ++j) {
      const float4* a4 = reinterpret_cast<const float4*>(at + (t + j) * RB);
#pragma unroll
      for (int q4 = 0; q4 < RB / 4; ++q4) {
        const float4 w = a4[q4];
        const float wr[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float4& o = acc[4 * q4 + k];
          o.x = fmaf(wr[k], x[j].x, o.x);
          o.y = fmaf(wr[k], x[j].y, o.y);
          o.z = fmaf(wr[k], x[j].z, o.z);
          o.w = fmaf(wr[k], x[j].w, o.w);
        }
      }
    }
  }
  for (; t < T; ++t) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(eu + (int64_t)t * C));
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const float w = at[t * RB + r];
      acc[r].x = fmaf(w, x.x, acc[r].x);
      acc[r].y = fmaf(w, x.y, acc[r].y);
      acc[r].z = fmaf(w, x.z, acc[r].z);
      acc[r].w = fmaf(w, x.w, acc[r].w);
    }
  }
#pragma unroll
  for (int r = 0; r < RB; ++r)
    if (r < rows) *reinterpret_cast<float4*>(ctx_out + (int64_t)(slot0 + r) * ld_ctx + col) = acc[r];
  if (planes != nullptr) {
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      if (r >= rows) continue;
      uint16_t e[4][3], pl[3][4];
      split_operand(acc[r].x, e[0]);
      split_operand(acc[r].y, e[1]);
      split_operand(acc[r].z, e[2]);
      split_operand(acc[r].w, e[3]);
#pragma unroll
      for (int pp = 0; pp < kPlanes; ++pp)
#pragma unroll
        for (int k = 0; k < 4; ++k) pl[pp][k] = e[k][pp];
      uint16_t* o = planes + (int64_t)row_pos[slot0 + r] * ld_planes + col;
#pragma unroll
      for (int pp = 0; pp < kPlanes; ++pp)
        *reinterpret_cast<uint2*>(o + pp * plane_stride) = *reinterpret_cast<uint2*>(pl[pp]);
    }
  }
}

// ---------------------------------------------------------- LM bookkeeping --
__global__ void spec_events_kernel(fb_trie_t trie, int n_max, const int32_t* __restrict__ n_dev,
                                   const int32_t* __restrict__ rows,
                                   const int32_t* __restrict__ tstate,
                                   const int32_t* __restrict__ hslot, int32_t* ev_row,
                                   int32_t* ev_rank, int32_t* ev_slot, int32_t* ev_count,
                                   int32_t* row_ev) {
  const int n = row_count(n_max, n_dev);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int r = row_at(rows, i);
    const int s = tstate[r];
    int e = -1;
    if (s > 0) {
      const int rk = trie.info[4 * s + 2];
      if (rk >= 0) {
        e = atomicAdd(ev_count, 1);
        ev_row[e] = r;
        ev_rank[e] = rk;
        ev_slot[e] = hslot[r];
      }
    }
    row_ev[r] = e;
  }
}

// Single CTA: mark live slots, list free slots in order, hand them to the
// boundary rows in row order.  Rows whose parent ran a speculative LM event
// reuse it now (bnd list); the others become "late" events that the next
// step's LM batch runs first (late lists, written where that batch reads them).
constexpr int kBpRows = 8;      // rows per thread gathered per batch (boundary plan)
__global__ void __launch_bounds__(1024)
boundary_plan_kernel(int n_max, const int32_t* __restrict__ n_dev, const int32_t* __restrict__ rows,
                     const int32_t* __restrict__ parent, const int32_t* __restrict__ brank,
                     const int32_t* __restrict__ row_ev, const int32_t* __restrict__ cur_rows,
                     const int32_t* __restrict__ cur_count, const int32_t* __restrict__ hist_cur,
                     int32_t* __restrict__ hist_next, int num_slots, int32_t* __restrict__ mark,
                     int32_t* __restrict__ bnd_slot, int32_t* __restrict__ bnd_src,
                     int32_t* __restrict__ bnd_count, int32_t* __restrict__ late_slot,
                     int32_t* __restrict__ late_tok, int32_t* __restrict__ late_row,
                     int32_t* __restrict__ late_dst, int32_t* __restrict__ late_count,
                     int late_sink_row) {
  pdl_entry();
  // each thread owns a contiguous run of slots / rows, so one block scan per
  // pass (instead of one per 1024 elements) assigns the ordered positions
  __shared__ int wsum[32];
  __shared__ int wsum2[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  int32_t* freel = mark + num_slots;   // second half of the scratch: free list
  for (int s = tid; s < num_slots; s += blockDim.x) mark[s] = 0;
  __syncthreads();
  const int nc = *cur_count;
  // dependent gathers batched: all index loads of a chunk in flight together
  for (int i0 = tid; i0 < nc; i0 += kBpRows * blockDim.x) {
    int cr[kBpRows];
#pragma unroll
    for (int j = 0; j < kBpRows; ++j) {
      const int i = i0 + j * blockDim.x;
      cr[j] = i < nc ? cur_rows[i] : -1;
    }
    int hs[kBpRows];
#pragma unroll
    for (int j = 0; j < kBpRows; ++j) hs[j] = cr[j] >= 0 ? hist_cur[cr[j]] : -1;
#pragma unroll
    for (int j = 0; j < kBpRows; ++j)
      if (hs[j] >= 0) mark[hs[j]] = 1;
  }
  __syncthreads();
  // exclusive block scan of (a, b) per thread -> (a_before, b_before), totals
  auto scan2 = [&](int a, int b, int& ea, int& eb, int& ta, int& tb) {
    int x = a, y = b;
    for (int off = 1; off < 32; off <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, x, off);
      const int v = __shfl_up_sync(0xffffffffu, y, off);
      if (lane >= off) { x += u; y += v; }
    }
    if (lane == 31) { wsum[warp] = x; wsum2[warp] = y; }
    __syncthreads();
    if (warp == 0) {
      int w = lane < nw ? wsum[lane] : 0;
      int w2 = lane < nw ? wsum2[lane] : 0;
      for (int off = 1; off < 32; off <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, w, off);
        const int v = __shfl_up_sync(0xffffffffu, w2, off);
        if (lane >= off) { w += u; w2 += v; }
      }
      wsum[lane] = w;
      wsum2[lane] = w2;
    }
    __syncthreads();
    ea = (warp ? wsum[warp - 1] : 0) + x - a;
    eb = (warp ? wsum2[warp - 1] : 0) + y - b;
    ta = wsum[nw - 1];
    tb = wsum2[nw - 1];
    __syncthreads();
  };
  {
    const int per = (num_slots + blockDim.x - 1) / blockDim.x;
    const int s0 = tid * per, s1 = min(num_slots, s0 + per);
    int f = 0;
    for (int s = s0; s < s1; ++s) f += mark[s] == 0;
    int pos, dummy, t1, t2;
    scan2(f, 0, pos, dummy, t1, t2);
    for (int s = s0; s < s1; ++s)
      if (mark[s] == 0) freel[pos++] = s;            // k-th free slot, ascending
  }
  __syncthreads();
  const int n = row_count(n_max, n_dev);
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int i0 = tid * per, i1 = min(n, i0 + per);
  // per-row (row, boundary rank, parent, parent's event) for this thread's run,
  // gathered kBpRows at a time with the four dependent loads batched (one
  // latency round each instead of four per row); kept for the second pass
  // when the run fits, else gathered again
  int cr[kBpRows], cb[kBpRows], cp[kBpRows], ce[kBpRows];
  auto gather = [&](int c) {
#pragma unroll
    for (int j = 0; j < kBpRows; ++j) cr[j] = c + j < i1 ? rows[c + j] : -1;
#pragma unroll
    for (int j = 0; j < kBpRows; ++j) cb[j] = cr[j] >= 0 ? brank[cr[j]] : -2;
#pragma unroll
    for (int j = 0; j < kBpRows; ++j) cp[j] = cb[j] >= -1 ? parent[cr[j]] : 0;
#pragma unroll
    for (int j = 0; j < kBpRows; ++j) ce[j] = cb[j] >= 0 ? row_ev[cp[j]] : -1;
  };
  int nb = 0, nl = 0;
  for (int c = i0; c < i1; c += kBpRows) {
    gather(c);
#pragma unroll
    for (int j = 0; j < kBpRows; ++j)
      if (cb[j] >= -1) {
        ++nb;
        nl += (cb[j] == -1 || ce[j] < 0);
      }
  }
  int k, kl, tot_b, tot_l;
  scan2(nb, nl, k, kl, tot_b, tot_l);
  const bool cached = i1 - i0 <= kBpRows;
  for (int c = i0; c < i1; c += kBpRows) {
    if (!cached) gather(c);
#pragma unroll
    for (int j = 0; j < kBpRows; ++j) {
      const int r = cr[j];
      const int br = cb[j];
      if (br < -1) continue;                       // not a boundary (or past the run)
      const int p = cp[j];
      const bool late = br == -1 || ce[j] < 0;
      const int slot = freel[k];                   // k-th boundary in row order
      hist_next[r] = slot;
      if (late) {
        late_slot[kl] = hist_cur[p];
        late_tok[kl] = br;
        late_row[kl] = late_sink_row;
        late_dst[kl] = slot;
        ++kl;
      } else {
        const int ks = k - kl;                     // spec index = k - #late rows before it
        bnd_slot[ks] = slot;
        bnd_src[ks] = ce[j];
      }
      ++k;
    }
  }
  if (tid == 0) { *bnd_count = tot_b - tot_l; *late_count = tot_l; }
}

__global__ void copy_rows_kernel(int n_max, const int32_t* __restrict__ n_dev,
                                 const int32_t* __restrict__ si, const int32_t* __restrict__ di,
                                 const char* __restrict__ src, char* __restrict__ dst,
                                 int64_t row_bytes) {
  pdl_entry();
  const int n = row_count(n_max, n_dev);
  const bool vec = (row_bytes % 16 == 0) && ((uintptr_t)src % 16 == 0) && ((uintptr_t)dst % 16 == 0);
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const char* s = src + (int64_t)(si ? si[i] : i) * row_bytes;
    char* d = dst + (int64_t)(di ? di[i] : i) * row_bytes;
    if (vec) {
      // eight 16-byte loads per thread in flight before any store (one
      // latency round per 32 KB of row instead of one per 4 KB)
      const int64_t nv = row_bytes / 16;
      const int4* s4 = reinterpret_cast<const int4*>(s);
      int4* d4 = reinterpret_cast<int4*>(d);
      for (int64_t j0 = threadIdx.x; j0 < nv; j0 += 8 * (int64_t)blockDim.x) {
        int4 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int64_t j = j0 + q * (int64_t)blockDim.x;
          if (j < nv) v[q] = __ldg(s4 + j);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int64_t j = j0 + q * (int64_t)blockDim.x;
          if (j < nv) d4[j] = v[q];
        }
      }
    } else {
      for (int64_t j = threadIdx.x; j < row_bytes; j += blockDim.x) d[j] = s[j];
    }
  }
}

}  // namespace fb

using namespace fb;

extern "C" int fb_pack_rows(const fb_pack_t* p, int32_t m_max, const int32_t* m_dev,
                            const int32_t* rows, const int32_t* parent, const int32_t* tokens,
                            const int32_t* ranks, float* out, int64_t ld_out, void* stream) {
  FB_CHECK_ARG(p && out && p->nseg >= 1 && p->nseg <= 4, "bad pack description");
  int w = 0;
  for (int s = 0; s < p->nseg; ++s) w += p->seg[s].width;
  FB_CHECK_ARG(w <= p->k_pad && p->k_pad <= ld_out, "pack width exceeds k_pad / ld_out");
  if (m_max <= 0) return FB_OK;
#ifndef FB_PACK_GRID
#define FB_PACK_GRID (kNumSMs * 2)
#endif
  launch_pdl(pack_rows_kernel, dim3(std::min((m_max + 7) / 8, FB_PACK_GRID)), dim3(256), 0,
             (cudaStream_t)stream, *p, m_max, m_dev, rows, parent, tokens, ranks, out, ld_out);
  count_launch();
  return check_launch("pack_rows");
}

extern "C" int fb_log_softmax_rows(int32_t m_max, const int32_t* m_dev, const int32_t* rows,
                                   const float* x, int64_t ldx, int32_t n, float* out,
                                   int64_t ldo, void* stream) {
  FB_CHECK_ARG(x && out && n > 0, "bad log-softmax arguments");
  if (m_max <= 0) return FB_OK;
  log_softmax_kernel<<<std::min((m_max + 7) / 8, kNumSMs * 8), 256, 0, (cudaStream_t)stream>>>(
      m_max, m_dev, rows, x, ldx, n, out, ldo);
  count_launch();
  return check_launch("log_softmax_rows");
}

extern "C" int fb_row_logsumexp(int32_t m_max, const int32_t* m_dev, const int32_t* rows,
                                const float* logits, int64_t l_stride, int32_t n_cols,
                                int32_t skip_col, double* norm_out, void* stream) {
  FB_CHECK_ARG(logits && norm_out && n_cols > 0, "bad logsumexp arguments");
  if (m_max <= 0) return FB_OK;
  row_lse_kernel<<<std::min((m_max + 7) / 8, kNumSMs * 8), 256, 0, (cudaStream_t)stream>>>(
      m_max, m_dev, rows, logits, l_stride, n_cols, skip_col, norm_out);
  count_launch();
  return check_launch("row_logsumexp");
}

// Launch tiling of fb_attention_step (0 = default), read when a launch is
// issued -- a captured graph keeps the tiling it was captured with.
static int g_att_ew = 0, g_att_re = 0, g_att_cq = 0;

extern "C" int fb_set_attention_tiling(int32_t frames_warps, int32_t rows, int32_t quads) {
  FB_CHECK_ARG(frames_warps == 0 || frames_warps == 2 || frames_warps == 4 || frames_warps == 8,
               "frame warps must be 0, 2, 4 or 8");
  FB_CHECK_ARG(rows == 0 || (rows >= 2 && rows <= 16 && rows % 2 == 0), "rows must be 0 or even 2..16");
  FB_CHECK_ARG(quads >= 0, "negative quads");
  g_att_ew = frames_warps;
  g_att_re = rows;
  g_att_cq = quads;
  return FB_OK;
}

extern "C" int fb_attention_step(const fb_search_cfg_t* cfg, int32_t num_utts,
                                 const int32_t* active, const int32_t* n_live,
                                 const int32_t* t_enc, const float* keys, const float* enc,
                                 int32_t att_dim, int32_t ctx_dim, const float* v, float* q,
                                 int64_t ldq, const int32_t* parent, const double* acc_in,
                                 double* acc_out, double* cov_out, float* ctx_out,
                                 int64_t ld_ctx, float* attn_out, int64_t ld_attn,
                                 float* energy_ws, int32_t* sync_ws, int32_t q_is_exp,
                                 void* ctx_planes, int64_t ctx_plane_stride,
                                 int64_t ctx_plane_ld, const int32_t* ctx_row_pos,
                                 void* stream) {
  FB_CHECK_ARG(cfg && keys && enc && v && q && acc_in && acc_out && ctx_out && energy_ws &&
                   sync_ws, "null attention args");
  FB_CHECK_ARG(!ctx_planes || (ctx_row_pos && ctx_plane_ld % 4 == 0 && ctx_plane_stride % 4 == 0 &&
                               (reinterpret_cast<uintptr_t>(ctx_planes) & 7) == 0),
               "context planes need row positions and 8-byte aligned rows");
  FB_CHECK_ARG(cfg->cov_mode == 0 || cov_out, "coverage output required");
  FB_CHECK_ARG(cfg->beam <= kMaxBeam, "beam too large for the attention kernels");
  FB_CHECK_ARG(att_dim % 4 == 0 && ldq % 4 == 0,
               "attention dim and query stride must be multiples of 4");
  if (num_utts <= 0) return FB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  static const int re_env = [] {                      // dev override (experiments)
    const char* e = getenv("FB_ATT_RE");
    return e ? atoi(e) : 0;
  }();
  const int RE = g_att_re > 0 ? g_att_re : re_env > 0 ? re_env
                            : (cfg->beam >= 16 ? 16 : (cfg->beam + 1) & ~1);   // rows per energy CTA
  // attention dims split over two CTAs (energy_ws holds one plane per part)
  static const int split_env = [] {
    const char* e = getenv("FB_ATT_SPLIT");
    return e ? atoi(e) : 2;
  }();
  const int parts = (split_env == 2 && att_dim % 8 == 0) ? 2 : 1;
  const int adim_p = att_dim / parts;
  const size_t sm_e = sizeof(float) * ((size_t)RE * adim_p + 2 * (size_t)adim_p);
  const int RB = cfg->beam <= 4 ? 4 : cfg->beam <= 8 ? 8 : cfg->beam <= 12 ? 12 : 16;
  const size_t sm_c = sizeof(float) * (size_t)RB * cfg->t_max;
  if (sm_e > 200 * 1024 || sm_c > 200 * 1024)
    return fail(FB_ERR_CONFIG, "attention working set exceeds shared memory");
  FB_CHECK_ARG(ctx_dim % 4 == 0 && ctx_dim <= 4 * kCtxMaxThreads && ld_ctx % 4 == 0,
               "context dim must be a multiple of 4 and <= 2048");
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(att_context_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(att_context_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(att_context_kernel<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(att_context_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
#define FB_ATTR(R)                                                                                  \
  cudaFuncSetAttribute(att_energy_kernel<R, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); \
  cudaFuncSetAttribute(att_energy_kernel<R, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); \
  cudaFuncSetAttribute(att_energy_kernel<R, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)
    FB_ATTR(2); FB_ATTR(4); FB_ATTR(6); FB_ATTR(8); FB_ATTR(10); FB_ATTR(12); FB_ATTR(14); FB_ATTR(16);
#undef FB_ATTR
    attr_set = true;
  }
  if (!q_is_exp) {
    const int64_t total = (int64_t)num_utts * cfg->beam * (att_dim / 4);
    query_exp_kernel<<<(int)std::min<int64_t>((total + 255) / 256, kNumSMs * 8), 256, 0, s>>>(
        num_utts, cfg->beam, active, n_live, q, ldq, att_dim / 4);
    count_launch();
  }
  // frames per energy CTA: enough CTAs to fill the GPU a few times over
  static const int ew_env = [] {
    const char* e = getenv("FB_ATT_EW");
    return e ? atoi(e) : 0;
  }();
  // (measured, scripts/bench_attention.py + the c2 decode: 256-frame CTAs win at
  // c2 and c4; smaller chunks add more q staging than they recover in occupancy)
  const int groups_e = (cfg->beam + RE - 1) / RE;
  int EW = 8;
  if (ew_env == 2 || ew_env == 4 || ew_env == 8) EW = ew_env;
  if (g_att_ew > 0) EW = g_att_ew;
  dim3 ge(num_utts, (cfg->t_max + EW * 32 - 1) / (EW * 32) * parts, groups_e);
#define FB_EN2(R, W)                                                                          \
  launch_pdl(att_energy_kernel<R, W>, ge, dim3(W * 32), sm_e, s, *cfg, active, n_live, t_enc,   \
             keys, att_dim,                                                                    \
                                                    v, q, ldq, energy_ws, sync_ws, parent,     \
                                                    acc_in, acc_out, cov_out, attn_out, ld_attn, \
                                                    parts)
#define FB_EN(R) \
  if (EW == 2) FB_EN2(R, 2); else if (EW == 4) FB_EN2(R, 4); else FB_EN2(R, 8)
  switch (RE) {
    case 2: FB_EN(2); break;
    case 4: FB_EN(4); break;
    case 6: FB_EN(6); break;
    case 8: FB_EN(8); break;
    case 10: FB_EN(10); break;
    case 12: FB_EN(12); break;
    case 14: FB_EN(14); break;
    default: FB_EN(16); break;
  }
#undef FB_EN2
#undef FB_EN
  count_launch();
  int rc = check_launch("att_energy");
  if (rc) return rc;
  // column split so that the grid covers the SMs a few times over (the kernel
  // streams the encoder output; more CTAs = more bytes in flight)
  const int groups = (cfg->beam + RB - 1) / RB;
  const int quads = ctx_dim / 4;
  static const int cq_env = [] {
    const char* e = getenv("FB_ATT_CQ");
    return e ? atoi(e) : 0;
  }();
  // quads (4 columns) per context CTA: 160 (whole c2 rows; measured over the
  // c2 decode 64 -> 160: -0.9 ms, and the c4 choice already)
  const int cq = g_att_cq > 0 ? g_att_cq : cq_env > 0 ? cq_env : 160;
  const int csplit = (quads + cq - 1) / cq;
  const int qpc = (quads + csplit - 1) / csplit;
  dim3 gc(num_utts, groups, csplit);
  const int ctx_threads = ((qpc + 31) / 32) * 32;
#define FB_CTX(R)                                                                             \
  launch_pdl(att_context_kernel<R>, gc, dim3(ctx_threads), sm_c, s, *cfg, active, n_live, t_enc, \
             enc, ctx_dim,                                                                      \
                                                      energy_ws, ctx_out, ld_ctx,          \
                                                      (uint16_t*)ctx_planes, ctx_plane_stride, \
                                                      ctx_plane_ld, ctx_row_pos)
  if (RB == 4) FB_CTX(4); else if (RB == 8) FB_CTX(8); else if (RB == 12) FB_CTX(12); else FB_CTX(16);
#undef FB_CTX
  count_launch();
  return check_launch("att_context");
}

extern "C" int fb_spec_events(const fb_trie_t* trie, int32_t n_max, const int32_t* n_dev,
                              const int32_t* rows, const int32_t* trie_state,
                              const int32_t* hist_slot, int32_t* ev_row, int32_t* ev_rank,
                              int32_t* ev_slot, int32_t* ev_count, int32_t* row_ev,
                              void* stream) {
  FB_CHECK_ARG(trie && ev_count && row_ev, "null spec-event arguments");
  cudaMemsetAsync(ev_count, 0, sizeof(int32_t), (cudaStream_t)stream);
  if (n_max <= 0) return check_launch("spec_events");
  spec_events_kernel<<<std::min((n_max + 255) / 256, kNumSMs * 4), 256, 0, (cudaStream_t)stream>>>(
      *trie, n_max, n_dev, rows, trie_state, hist_slot, ev_row, ev_rank, ev_slot, ev_count,
      row_ev);
  count_launch();
  return check_launch("spec_events");
}

extern "C" int fb_boundary_plan(int32_t n_max, const int32_t* n_dev, const int32_t* rows,
                                const int32_t* parent, const int32_t* boundary_rank,
                                const int32_t* row_ev, const int32_t* cur_rows,
                                const int32_t* cur_count, const int32_t* hist_cur,
                                int32_t* hist_next, int32_t num_slots, int32_t* slot_mark,
                                int32_t* bnd_slot, int32_t* bnd_src, int32_t* bnd_count,
                                int32_t* late_slot, int32_t* late_tok, int32_t* late_row,
                                int32_t* late_dst, int32_t* late_count, int32_t late_sink_row,
                                void* stream) {
  FB_CHECK_ARG(rows && parent && boundary_rank && cur_rows && cur_count && hist_cur && hist_next,
               "null boundary-plan arguments");
  launch_pdl(boundary_plan_kernel, dim3(1), dim3(1024), 0, (cudaStream_t)stream,
      n_max, n_dev, rows, parent, boundary_rank, row_ev, cur_rows, cur_count, hist_cur,
      hist_next, num_slots, slot_mark, bnd_slot, bnd_src, bnd_count, late_slot, late_tok,
      late_row, late_dst, late_count, late_sink_row);
  count_launch();
  return check_launch("boundary_plan");
}

extern "C" int fb_copy_rows(int32_t n_max, const int32_t* n_dev, const int32_t* src_idx,
                            const int32_t* dst_idx, const void* src, void* dst, int64_t row_bytes,
                            void* stream) {
  FB_CHECK_ARG(src && dst && row_bytes > 0, "bad copy arguments");
  if (n_max <= 0) return FB_OK;
#ifndef FB_COPY_GRID
#define FB_COPY_GRID (kNumSMs * 8)
#endif
  launch_pdl(copy_rows_kernel, dim3(std::min(n_max, FB_COPY_GRID)), dim3(256), 0,
      (cudaStream_t)stream, n_max, n_dev, src_idx, dst_idx, (const char*)src, (char*)dst, row_bytes);
  count_launch();
  return check_launch("copy_rows");
}

extern "C" int fb_keys_exp2t(int32_t num_utts, int32_t t_max, int32_t att_dim, const float* keys,
                             float* ekt, void* stream) {
  FB_CHECK_ARG(keys && ekt && keys != ekt && num_utts >= 0 && t_max > 0 && att_dim > 0,
               "bad key transpose arguments");
  if (num_utts == 0) return FB_OK;
  dim3 g((t_max + 31) / 32, (att_dim + 31) / 32, num_utts);
  keys_exp2t_kernel<<<g, dim3(32, 8), 0, (cudaStream_t)stream>>>(t_max, att_dim, keys, ekt);
  count_launch();
  return check_launch("keys_exp2t");
}

extern "C" int fb_exp2x(int64_t n, const float* x, float* y, void* stream) {
  FB_CHECK_ARG(x && y && n >= 0, "bad exp2x arguments");
  if (n == 0) return FB_OK;
  exp2x_kernel<<<std::min<int64_t>((n + 255) / 256, kNumSMs * 16), 256, 0, (cudaStream_t)stream>>>(n, x, y);
  count_launch();
  return check_launch("exp2x");
}
