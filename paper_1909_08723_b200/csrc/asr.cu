// Attention-LSTM decoder step pieces (operand packing, Bahdanau attention with
// the fp64 attention accumulator + coverage, row log-softmax) and the word-LM
// bookkeeping of the fused engine (speculative <eos> events, word-boundary
// slot plan, row copies).
//
// Model equations: DESIGN.md §3; search semantics:
// decoder.py:419-425 (accumulator), fusion.py:177-223 (LM events).
#include "common.cuh"

#include <cuda_bf16.h>

namespace fb {

// ---------------------------------------------------------------- packing --
__device__ __forceinline__ void split3(float x, __nv_bfloat16& hi, __nv_bfloat16& mid,
                                       __nv_bfloat16& lo) {
  // x = hi + mid + lo exactly (8+8+8 mantissa bits of the fp32 value)
  hi = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(hi);
  mid = __float2bfloat16_rn(r1);
  lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
}

// One warp per output row, 4 consecutive columns per lane (float4 in, 8-byte
// bf16x4 per plane out) when the segment allows it.
__global__ void __launch_bounds__(256)
pack_rows_kernel(fb_pack_t p, int m_max, const int32_t* __restrict__ m_dev,
                 const int32_t* __restrict__ rows, const int32_t* __restrict__ parent,
                 const int32_t* __restrict__ tokens, const int32_t* __restrict__ ranks,
                 float* __restrict__ out, int64_t ld_out) {
  const int m = row_count(m_max, m_dev);
  const bool split = p.out_mode == 1;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(out);
  const int64_t plane = p.plane_rows * ld_out;
  for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < m; i += gridDim.x * wpb) {
    int col = 0;
    for (int s = 0; s <= p.nseg; ++s) {
      const float* src = nullptr;
      int width;
      if (s < p.nseg) {
        const fb_seg_t& sg = p.seg[s];
        int64_t r;
        switch (sg.mode) {
          case 0: r = i; break;
          case 1: r = rows ? rows[i] : i; break;
          case 2: { const int sl = rows ? rows[i] : i; r = parent ? parent[sl] : sl; break; }
          case 3: { const int sl = rows ? rows[i] : i; const int t = tokens[sl];
                    r = t < 0 ? p.tok_default : t; break; }
          default: { const int t = ranks ? ranks[i] : -1; r = t < 0 ? p.tok_default : t; break; }
        }
        src = sg.src ? sg.src + r * sg.ld : nullptr;
        width = sg.width;
      } else {
        width = p.k_pad - col;                      // zero padding
      }
      const bool vec = ((width & 3) == 0) && ((col & 3) == 0) &&
                       (!src || (reinterpret_cast<uintptr_t>(src) & 15) == 0);
      if (vec) {
        for (int j = lane * 4; j < width; j += 128) {
          const float4 v = src ? *reinterpret_cast<const float4*>(src + j)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
          const int64_t o = (int64_t)i * ld_out + col + j;
          if (!split) {
            *reinterpret_cast<float4*>(out + o) = v;
          } else {
            __nv_bfloat16 h[4], md[4], lo[4];
            split3(v.x, h[0], md[0], lo[0]);
            split3(v.y, h[1], md[1], lo[1]);
            split3(v.z, h[2], md[2], lo[2]);
            split3(v.w, h[3], md[3], lo[3]);
            *reinterpret_cast<uint2*>(ob + o) = *reinterpret_cast<uint2*>(h);
            *reinterpret_cast<uint2*>(ob + plane + o) = *reinterpret_cast<uint2*>(md);
            *reinterpret_cast<uint2*>(ob + 2 * plane + o) = *reinterpret_cast<uint2*>(lo);
          }
        }
      } else {
        for (int j = lane; j < width; j += 32) {
          const float x = src ? src[j] : 0.f;
          const int64_t o = (int64_t)i * ld_out + col + j;
          if (!split) {
            out[o] = x;
          } else {
            __nv_bfloat16 h, md, lo;
            split3(x, h, md, lo);
            ob[o] = h;
            ob[plane + o] = md;
            ob[2 * plane + o] = lo;
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
    float s = 0.f;
    for (int j = lane; j < n; j += 32) s += expf(xr[j] - mx);
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    const float lse = logf(s);
    float* o = out + (int64_t)r * ldo;
    for (int j = lane; j < n; j += 32) o[j] = (xr[j] - mx) - lse;
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
// (B) softmax / fp64 accumulator / coverage / context: CTA = (utterance, chunk
//     of kCtxCols encoder columns); every CTA re-normalises its utterance's
//     rows (cheap) and CTA 0 of the utterance owns the accumulator + coverage.
constexpr int kEnWarps = 8;
constexpr int kEnFrames = 4;          // frames per warp
constexpr int kMaxBeam = 512;
constexpr int kCtxCols = 128;

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
template <int R>
__global__ void __launch_bounds__(kEnWarps * 32)
att_energy_kernel(fb_search_cfg_t cfg, const int32_t* __restrict__ active,
                  const int32_t* __restrict__ n_live, const int32_t* __restrict__ t_enc,
                  const float* __restrict__ ekeys, int A, const float* __restrict__ v,
                  const float* __restrict__ q, int64_t ldq, float* __restrict__ energy) {
  const int u = blockIdx.x;
  if (!active[u]) return;
  const int T = t_enc[u];
  const int t_base = blockIdx.y * (kEnWarps * kEnFrames);
  if (t_base >= T) return;
  extern __shared__ float sm[];
  const int K = cfg.beam, TM = cfg.t_max;
  const int n = n_live[u];
  const int npass = (n + R - 1) / R;
  float* vs = sm;                  // [A]
  float* qs = sm + A;              // [npass*R][A]  E_q = exp(2 q); rows >= n are 0
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot0 = u * K;
  for (int j = tid; j < npass * R * A; j += blockDim.x) {
    const int i = j / A, a = j - i * A;
    qs[j] = i < n ? expf(2.0f * q[(int64_t)(slot0 + i) * ldq + a]) : 0.f;
  }
  for (int a = tid; a < A; a += blockDim.x) vs[a] = v[a];
  __syncthreads();
  const float* ku = ekeys + (int64_t)u * TM * A;
  for (int f = 0; f < kEnFrames; ++f) {
    const int t = t_base + warp * kEnFrames + f;
    if (t >= T) break;
    const float* kt = ku + (int64_t)t * A;
    for (int ps = 0; ps < npass; ++ps) {
      float e[R];
#pragma unroll
      for (int r = 0; r < R; ++r) e[r] = 0.f;
      for (int a = lane; a < A; a += 32) {
        const float ek = __ldg(kt + a);
        const float va = vs[a];
        const float* qa = qs + (ps * R) * A + a;
#pragma unroll
        for (int r = 0; r < R; ++r) e[r] = fmaf(va, rcp_approx(fmaf(ek, qa[r * A], 1.0f)), e[r]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float x = e[r];
        for (int off = 16; off; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
        e[r] = x;
      }
      const int row = ps * R + lane;
      if (lane < R && row < n) {
        float x = 0.f;
#pragma unroll
        for (int r = 0; r < R; ++r) x = lane == r ? e[r] : x;
        energy[(int64_t)(slot0 + row) * TM + t] = -2.0f * x;
      }
    }
  }
}

__global__ void exp2x_kernel(int64_t n, const float* __restrict__ x, float* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = expf(2.0f * x[i]);
}

template <int RB>
__global__ void __launch_bounds__(256)
att_context_kernel(fb_search_cfg_t cfg, const int32_t* __restrict__ active,
                   const int32_t* __restrict__ n_live, const int32_t* __restrict__ t_enc,
                   const float* __restrict__ enc, int C, const float* __restrict__ energy,
                   const int32_t* __restrict__ parent, const double* __restrict__ acc_in,
                   double* __restrict__ acc_out, double* __restrict__ cov_out,
                   float* __restrict__ ctx_out, int64_t ld_ctx, float* __restrict__ attn_out,
                   int64_t ld_attn) {
  const int u = blockIdx.x;
  if (!active[u]) return;
  const int c0 = blockIdx.y * kCtxCols;
  if (c0 >= C) return;
  extern __shared__ float sm[];
  const int K = cfg.beam, TM = cfg.t_max;
  const int n = n_live[u];
  const int T = t_enc[u];
  // per-row softmax statistics only; weights are re-derived from the energy
  // rows (L2-resident) per row group, so shared memory is O(RB * T) for any beam
  constexpr int RBS = RB + 4;      // padded row stride of the transposed group (float4-aligned)
  float* st_mx = sm;                                   // [n]
  float* st_inv = sm + n;                              // [n]
  float* at = sm + ((2 * n + 3) & ~3);                 // [T][RBS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int slot0 = u * K;
  // softmax over frames, one warp per row (every column chunk recomputes it)
  for (int i = warp; i < n; i += nw) {
    const float* e = energy + (int64_t)(slot0 + i) * TM;
    float mx = -INFINITY;
    for (int t = lane; t < T; t += 32) mx = fmaxf(mx, e[t]);
    for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    float s = 0.f;
    for (int t = lane; t < T; t += 32) s += expf(e[t] - mx);
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) {
      st_mx[i] = mx;
      st_inv[i] = 1.0f / s;
    }
  }
  const float* eu = enc + (int64_t)u * TM * C;
  const int col = c0 + 2 * tid;
  for (int g0 = 0; g0 < n; g0 += RB) {
  __syncthreads();
  for (int j = tid; j < T * RB; j += blockDim.x) {
    const int r = j / T, t = j - r * T;
    at[t * RBS + r] = g0 + r < n ? expf(energy[(int64_t)(slot0 + g0 + r) * TM + t] -
                                        st_mx[g0 + r]) * st_inv[g0 + r]
                                 : 0.f;
  }
  __syncthreads();
  // context columns [c0, c0 + kCtxCols): thread = 2 adjacent columns (float2),
  // rows g0..g0+RB; 8 frames of enc in flight per thread
  if (tid < kCtxCols / 2 && col < C) {
    const bool pair = col + 1 < C;
    float acc0[RB], acc1[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) acc0[r] = acc1[r] = 0.f;
    constexpr int TU = 8;
    int t = 0;
    for (; t + TU <= T; t += TU) {
      float2 x[TU];
#pragma unroll
      for (int j = 0; j < TU; ++j)
        x[j] = pair ? __ldg(reinterpret_cast<const float2*>(eu + (int64_t)(t + j) * C + col))
                    : make_float2(__ldg(eu + (int64_t)(t + j) * C + col), 0.f);
#pragma unroll
      for (int j = 0; j < TU; ++j) {
        const float4* a4 = reinterpret_cast<const float4*>(at + (t + j) * RBS);
#pragma unroll
        for (int q4 = 0; q4 < RB / 4; ++q4) {
          const float4 w = a4[q4];
          acc0[4 * q4] = fmaf(w.x, x[j].x, acc0[4 * q4]);
          acc0[4 * q4 + 1] = fmaf(w.y, x[j].x, acc0[4 * q4 + 1]);
          acc0[4 * q4 + 2] = fmaf(w.z, x[j].x, acc0[4 * q4 + 2]);
          acc0[4 * q4 + 3] = fmaf(w.w, x[j].x, acc0[4 * q4 + 3]);
          acc1[4 * q4] = fmaf(w.x, x[j].y, acc1[4 * q4]);
          acc1[4 * q4 + 1] = fmaf(w.y, x[j].y, acc1[4 * q4 + 1]);
          acc1[4 * q4 + 2] = fmaf(w.z, x[j].y, acc1[4 * q4 + 2]);
          acc1[4 * q4 + 3] = fmaf(w.w, x[j].y, acc1[4 * q4 + 3]);
        }
      }
    }
    for (; t < T; ++t) {
      const float x0 = __ldg(eu + (int64_t)t * C + col);
      const float x1 = pair ? __ldg(eu + (int64_t)t * C + col + 1) : 0.f;
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        acc0[r] = fmaf(at[t * RBS + r], x0, acc0[r]);
        acc1[r] = fmaf(at[t * RBS + r], x1, acc1[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      if (g0 + r < n) {
        float* o = ctx_out + (int64_t)(slot0 + g0 + r) * ld_ctx + col;
        o[0] = acc0[r];
        if (pair) o[1] = acc1[r];
      }
    }
  }
  }
  if (blockIdx.y != 0) return;
  // fp64 accumulator + coverage (decoder.py:421-425), one warp per row
  for (int i = warp; i < n; i += nw) {
    const int r = slot0 + i;
    const int p = parent ? parent[r] : r;
    const double* a0 = acc_in + (int64_t)p * TM;
    double* a1 = acc_out + (int64_t)r * TM;
    const float* e = energy + (int64_t)r * TM;
    const float mx = st_mx[i], inv = st_inv[i];
    int cnt = 0;
    for (int t = lane; t < T; t += 32) {
      const float a = expf(e[t] - mx) * inv;
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
  __shared__ int wsum[32];
  __shared__ int wsum2[32];
  __shared__ int carry, carry2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  int32_t* freel = mark + num_slots;   // second half of the scratch: free list
  for (int s = tid; s < num_slots; s += blockDim.x) mark[s] = 0;
  __syncthreads();
  const int nc = *cur_count;
  for (int i = tid; i < nc; i += blockDim.x) mark[hist_cur[cur_rows[i]]] = 1;
  __syncthreads();
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < num_slots; b0 += blockDim.x) {
    const int s = b0 + tid;
    const int f = (s < num_slots && mark[s] == 0) ? 1 : 0;
    int x = f;
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = lane < nw ? wsum[lane] : 0;
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, off);
        if (lane >= off) w += y;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    const int pos = carry + (warp ? wsum[warp - 1] : 0) + x - f;
    if (f) freel[pos] = s;              // k-th free slot, ascending
    __syncthreads();
    if (tid == 0) carry += wsum[nw - 1];
    __syncthreads();
  }
  const int n = row_count(n_max, n_dev);
  if (tid == 0) { carry = 0; carry2 = 0; }
  __syncthreads();
  for (int b0 = 0; b0 < n; b0 += blockDim.x) {
    const int i = b0 + tid;
    int is_b = 0, is_late = 0, r = -1, br = -2;
    if (i < n) {
      r = rows[i];
      br = brank[r];
      is_b = br >= -1;
      is_late = is_b && (br == -1 || row_ev[parent[r]] < 0);
    }
    // prefix counts: all boundaries (slot order), spec-sourced, late
    int x = is_b, y = is_late;
    for (int off = 1; off < 32; off <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, x, off);
      const int b = __shfl_up_sync(0xffffffffu, y, off);
      if (lane >= off) { x += a; y += b; }
    }
    if (lane == 31) { wsum[warp] = x; wsum2[warp] = y; }
    __syncthreads();
    if (warp == 0) {
      int w = lane < nw ? wsum[lane] : 0;
      int w2 = lane < nw ? wsum2[lane] : 0;
      for (int off = 1; off < 32; off <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, w, off);
        const int b = __shfl_up_sync(0xffffffffu, w2, off);
        if (lane >= off) { w += a; w2 += b; }
      }
      wsum[lane] = w;
      wsum2[lane] = w2;
    }
    __syncthreads();
    if (is_b) {
      const int k = carry + (warp ? wsum[warp - 1] : 0) + x - 1;      // k-th boundary
      const int kl = carry2 + (warp ? wsum2[warp - 1] : 0) + y - 1;   // late index if late
      const int slot = freel[k];
      hist_next[r] = slot;
      const int p = parent[r];
      if (is_late) {
        late_slot[kl] = hist_cur[p];
        late_tok[kl] = br;
        late_row[kl] = late_sink_row;
        late_dst[kl] = slot;
      } else {
        const int ks = k - (kl + 1);                 // spec index = k - #late rows before it
        bnd_slot[ks] = slot;
        bnd_src[ks] = row_ev[p];
      }
    }
    __syncthreads();
    if (tid == 0) { carry += wsum[nw - 1]; carry2 += wsum2[nw - 1]; }
    __syncthreads();
  }
  if (tid == 0) { *bnd_count = carry - carry2; *late_count = carry2; }
}

__global__ void copy_rows_kernel(int n_max, const int32_t* __restrict__ n_dev,
                                 const int32_t* __restrict__ si, const int32_t* __restrict__ di,
                                 const char* __restrict__ src, char* __restrict__ dst,
                                 int64_t row_bytes) {
  const int n = row_count(n_max, n_dev);
  const bool vec = (row_bytes % 16 == 0) && ((uintptr_t)src % 16 == 0) && ((uintptr_t)dst % 16 == 0);
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const char* s = src + (int64_t)(si ? si[i] : i) * row_bytes;
    char* d = dst + (int64_t)(di ? di[i] : i) * row_bytes;
    if (vec) {
      for (int64_t j = threadIdx.x; j < row_bytes / 16; j += blockDim.x)
        reinterpret_cast<int4*>(d)[j] = reinterpret_cast<const int4*>(s)[j];
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
  pack_rows_kernel<<<std::min((m_max + 7) / 8, kNumSMs * 8), 256, 0, (cudaStream_t)stream>>>(
      *p, m_max, m_dev, rows, parent, tokens, ranks, out, ld_out);
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

extern "C" int fb_attention_step(const fb_search_cfg_t* cfg, int32_t num_utts,
                                 const int32_t* active, const int32_t* n_live,
                                 const int32_t* t_enc, const float* keys, const float* enc,
                                 int32_t att_dim, int32_t ctx_dim, const float* v, const float* q,
                                 int64_t ldq, const int32_t* parent, const double* acc_in,
                                 double* acc_out, double* cov_out, float* ctx_out,
                                 int64_t ld_ctx, float* attn_out, int64_t ld_attn,
                                 float* energy_ws, void* stream) {
  FB_CHECK_ARG(cfg && keys && enc && v && q && acc_in && acc_out && ctx_out && energy_ws,
               "null attention args");
  FB_CHECK_ARG(cfg->cov_mode == 0 || cov_out, "coverage output required");
  FB_CHECK_ARG(cfg->beam <= kMaxBeam, "beam too large for the attention kernels");
  if (num_utts <= 0) return FB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int RE = cfg->beam >= 16 ? 16 : (cfg->beam + 1) & ~1;   // rows per energy pass
  const int npass = (cfg->beam + RE - 1) / RE;
  const size_t sm_e = sizeof(float) * ((size_t)npass * RE * att_dim + att_dim);
  const int RB = cfg->beam <= 4 ? 4 : cfg->beam <= 8 ? 8 : cfg->beam <= 12 ? 12 : 16;
  const size_t sm_c = sizeof(float) * ((size_t)2 * cfg->beam + 4 + (size_t)(RB + 4) * cfg->t_max);
  if (sm_e > 200 * 1024 || sm_c > 200 * 1024)
    return fail(FB_ERR_CONFIG, "attention working set exceeds shared memory");
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(att_energy_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(att_energy_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(att_energy_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(att_energy_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(att_energy_kernel<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(att_energy_kernel<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(att_energy_kernel<14>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(att_energy_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(att_context_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(att_context_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(att_context_kernel<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(att_context_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  dim3 ge(num_utts, (cfg->t_max + kEnWarps * kEnFrames - 1) / (kEnWarps * kEnFrames));
#define FB_EN(R)                                                                              \
  att_energy_kernel<R><<<ge, kEnWarps * 32, sm_e, s>>>(*cfg, active, n_live, t_enc, keys, att_dim, \
                                                        v, q, ldq, energy_ws)
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
#undef FB_EN
  count_launch();
  int rc = check_launch("att_energy");
  if (rc) return rc;
  dim3 gc(num_utts, (ctx_dim + kCtxCols - 1) / kCtxCols);
#define FB_CTX(R)                                                                             \
  att_context_kernel<R><<<gc, 256, sm_c, s>>>(*cfg, active, n_live, t_enc, enc, ctx_dim,       \
                                              energy_ws, parent, acc_in, acc_out, cov_out,    \
                                              ctx_out, ld_ctx, attn_out, ld_attn)
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
  boundary_plan_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(
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
  copy_rows_kernel<<<std::min(n_max, kNumSMs * 8), 256, 0, (cudaStream_t)stream>>>(
      n_max, n_dev, src_idx, dst_idx, (const char*)src, (char*)dst, row_bytes);
  count_launch();
  return check_launch("copy_rows");
}

extern "C" int fb_exp2x(int64_t n, const float* x, float* y, void* stream) {
  FB_CHECK_ARG(x && y && n >= 0, "bad exp2x arguments");
  if (n == 0) return FB_OK;
  exp2x_kernel<<<std::min<int64_t>((n + 255) / 256, kNumSMs * 16), 256, 0, (cudaStream_t)stream>>>(n, x, y);
  count_launch();
  return check_launch("exp2x");
}
