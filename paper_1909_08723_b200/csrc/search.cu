// Beam-search step kernels: score combine + EOS gate + token-major stable
// top-beam + coverage bonus + finished-set cap + early stop + result pick, and
// the attention-accumulator / coverage update.
//
// Reference semantics: decoder.py:339-480 (loop body :382-456), coverage
// decoder.py:36-48, gate :396-398, finished key :322-323.  All score arithmetic
// is IEEE float64 without FMA contraction so results equal numpy's.
#include "common.cuh"

#include <algorithm>

namespace fb {

constexpr int kSelThreads = 256;

#ifdef FB_SEARCH_TRACE
// dev experiment: phase times (ns, %globaltimer) of utterance 0's last search step
__device__ unsigned long long g_strace[16];
#define STRACE(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) { unsigned long long t_; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_strace[i] = t_; } } while (0)
#else
#define STRACE(i) do {} while (0)
#endif

// numpy's pairwise summation (loops_utils.h pairwise_sum, PW_BLOCKSIZE 128)
// over f(a[i]); reproduces np.sum bit-for-bit for contiguous float64.
template <typename F>
__device__ double pairwise_sum(const double* a, int n, F f) {
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
    double res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])),
                      dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
    for (; i < n; ++i) res = dadd(res, f(a[i]));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return dadd(pairwise_sum(a, n2, f), pairwise_sum(a + n2, n - n2, f));
}

__device__ __forceinline__ double coverage_of(const fb_search_cfg_t& c, const double* acc, int T,
                                              int count_above_tau1) {
  if (c.cov_mode == 1) return (double)count_above_tau1;
  const double tau2 = c.tau2, mg = c.cov_margin;
  const double pen = pairwise_sum(acc, T, [=](double x) {
    return x > tau2 ? dsub(dadd(mg, x), tau2) : 0.0;
  });
  return dsub((double)count_above_tau1, pen);
}

// acc_out[r] = acc_in[parent[r]] + attn[r]; cov_out[r] = coverage(acc_out[r]).
template <typename AT>
__global__ void attend_coverage_kernel(fb_search_cfg_t cfg, int n_max, const int32_t* n_dev,
                                       const int32_t* rows, const int32_t* parent,
                                       const int32_t* t_enc, const double* acc_in,
                                       const AT* attn, int64_t attn_stride, double* acc_out,
                                       double* cov_out) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int n = row_count(n_max, n_dev);
  for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < n; i += gridDim.x * wpb) {
    const int r = row_at(rows, i);
    const int p = parent ? parent[r] : r;
    const int T = t_enc[r / cfg.beam];
    const double* a0 = acc_in + (int64_t)p * cfg.t_max;
    const AT* at = attn + (int64_t)r * attn_stride;
    double* a1 = acc_out + (int64_t)r * cfg.t_max;
    int cnt = 0;
    for (int k = lane; k < T; k += 32) {
      const double v = dadd(a0[k], (double)at[k]);
      a1[k] = v;
      cnt += v > cfg.tau1;
    }
    if (cfg.cov_mode != 0) {
      for (int off = 16; off; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
      __syncwarp();
      if (lane == 0) cov_out[r] = coverage_of(cfg, a1, T, cnt);
    }
    __syncwarp();
  }
}

struct Cand {
  double s;
  int j;  // flat token-major index; INT_MAX = none
};

__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
  if (b.j == INT_MAX) return a.j != INT_MAX;
  if (a.j == INT_MAX) return false;
  return a.s > b.s || (a.s == b.s && a.j < b.j);
}

__device__ __forceinline__ Cand warp_best(Cand c) {
  for (int off = 16; off; off >>= 1) {
    Cand o;
    o.s = __shfl_xor_sync(0xffffffffu, c.s, off);
    o.j = __shfl_xor_sync(0xffffffffu, c.j, off);
    if (better(o, c)) c = o;
  }
  return c;
}

// ---- block-wide exact top-K for large candidate sets ---------------------------
// The first K of (key desc, id asc) among the finite keys -- what K rounds of
// block argmax produce -- without K passes over the keys:
//  1. bucket = order-preserving bits of the key rounded DOWN to fp32 (monotone,
//     so the K best keys lie in the K best buckets);
//  2. radix select (4 x 8-bit digits) of the K-th largest bucket T;
//  3. compact every key with bucket >= T (K plus fp32-bucket ties);
//  4. exact rank of each survivor among the survivors (C^2 compares, C small).
// More than cmax survivors (massive exact ties) falls back to argmax rounds.
#ifndef FB_RADIX_MIN
#define FB_RADIX_MIN 256
#endif
constexpr int kRadixMin = FB_RADIX_MIN;  // candidate count from which the radix path pays

__host__ __device__ inline int topk_cmax(int K) { return 4 * K + 64; }

__device__ __forceinline__ uint32_t key_bucket(double x) {
  if (x == -INFINITY) return 0u;                     // never selected
  const uint32_t u = __float_as_uint(__double2float_rd(x));
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // >= 0x007FFFFF for finite x
}

__device__ void block_topk(const double* key, const int* id, int n, int K, int* out,
                           int* n_out, uint32_t* bkt, int* cl, int cmax, unsigned char* taken) {
  __shared__ int hist[256];
  __shared__ int s_cnt, s_need, s_elig;
  __shared__ uint32_t s_prefix, s_mask;
  __shared__ Cand wb[kSelThreads / 32];
  __shared__ int s_stop, s_n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) { s_elig = 0; s_prefix = 0u; s_mask = 0u; s_need = K; s_cnt = 0; }
  __syncthreads();
  int el = 0;
  for (int j = tid; j < n; j += kSelThreads) {
    const uint32_t b = key_bucket(key[j]);
    bkt[j] = b;
    el += b != 0u;
  }
  for (int off = 16; off; off >>= 1) el += __shfl_xor_sync(0xffffffffu, el, off);
  if (lane == 0) atomicAdd(&s_elig, el);
  __syncthreads();
  uint32_t T = 1u;                                   // every finite key
  if (s_elig > K) {
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = tid; i < 256; i += kSelThreads) hist[i] = 0;
      __syncthreads();
      const uint32_t pre = s_prefix, msk = s_mask;
      for (int j = tid; j < n; j += kSelThreads) {
        const uint32_t b = bkt[j];
        if (b != 0u && (b & msk) == pre) atomicAdd(&hist[(b >> shift) & 255u], 1);
      }
      __syncthreads();
      if (warp == 0) {
        // lane l owns digits 255-8l .. 248-8l (descending)
        int c8[8], cs = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) { c8[q] = hist[255 - 8 * lane - q]; cs += c8[q]; }
        int incl = cs;
        for (int off = 1; off < 32; off <<= 1) {
          const int o = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += o;
        }
        const int need = s_need, excl = incl - cs;
        if (excl < need && need <= incl) {
          int run = excl;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (run + c8[q] >= need) {
              const uint32_t d = 255u - 8u * lane - q;
              s_prefix = pre | (d << shift);
              s_mask = msk | (255u << shift);
              s_need = need - run;
              break;
            }
            run += c8[q];
          }
        }
      }
      __syncthreads();
    }
    T = s_prefix;
  }
  for (int j = tid; j < n; j += kSelThreads) {
    if (bkt[j] >= T) {
      const int pos = atomicAdd(&s_cnt, 1);
      if (pos < cmax) cl[pos] = j;
    }
  }
  __syncthreads();
  const int C = s_cnt;
  if (C <= cmax) {
    for (int i = tid; i < C; i += kSelThreads) {
      const int ci = cl[i];
      const Cand a{key[ci], id ? id[ci] : ci};
      int rank = 0;
      for (int q = 0; q < C; ++q) {
        const int cq = cl[q];
        rank += better(Cand{key[cq], id ? id[cq] : cq}, a);
      }
      if (rank < K) out[rank] = a.j;
    }
    if (tid == 0) *n_out = C < K ? C : K;
    __syncthreads();
    return;
  }
  // fallback: K rounds of block argmax over the survivors' superset (all keys)
  for (int j = tid; j < n; j += kSelThreads) taken[j] = 0;
  if (tid == 0) { s_n = 0; s_stop = 0; }
  __syncthreads();
  for (int k = 0; k < K; ++k) {
    Cand b{-INFINITY, INT_MAX};
    for (int j = tid; j < n; j += kSelThreads)
      if (!taken[j] && bkt[j] >= T) {
        const Cand x{key[j], id ? id[j] : j};
        if (better(x, b)) b = x;
      }
    b = warp_best(b);
    if (lane == 0) wb[warp] = b;
    __syncthreads();
    if (tid == 0) {
      Cand w = wb[0];
      for (int q = 1; q < kSelThreads / 32; ++q)
        if (better(wb[q], w)) w = wb[q];
      if (w.j == INT_MAX || w.s == -INFINITY) s_stop = 1;
      else out[s_n++] = w.j;
    }
    __syncthreads();
    if (s_stop) break;
    const int won = out[s_n - 1];
    for (int j = tid; j < n; j += kSelThreads)
      if ((id ? id[j] : j) == won) taken[j] = 1;
    __syncthreads();
  }
  if (tid == 0) *n_out = s_n;
  __syncthreads();
}

// Lexicographic compare of two token rows of equal length L: -1, 0, 1.
__device__ __forceinline__ int lex_cmp(const int32_t* a, const int32_t* b, int L) {
  for (int i = 0; i < L; ++i) {
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  }
  return 0;
}

// (-total, len, tokens) ordering of decoder.py:322-323: true if a sorts first.
__device__ __forceinline__ bool key_less(double ta, int la, const int32_t* ka, double tb, int lb,
                                         const int32_t* kb) {
  if (ta != tb) return ta > tb;
  if (la != lb) return la < lb;
  return lex_cmp(ka, kb, la) < 0;
}

template <typename AM>
__device__ __forceinline__ double step_score(const fb_search_cfg_t& c, const AM* am,
                                             int64_t am_stride, const double* fus,
                                             int64_t f_stride, int slot, int t, bool gated,
                                             const double* norm = nullptr, double floor_ = 0.0) {
  if (t == c.pad_id) return -INFINITY;
  if (t == c.eos_id && gated) return -INFINITY;
  double s = (double)am[(int64_t)slot * am_stride + t];
  if (c.has_fusion) {
    double f;
    if (norm) {        // fp32 logits + fp64 log-normaliser per row, floored (char_lm.py:20,93)
      f = dadd((double)reinterpret_cast<const float*>(fus)[(int64_t)slot * f_stride + t],
               -norm[slot]);
      f = f < floor_ ? floor_ : f;
    } else {
      f = fus[(int64_t)slot * f_stride + t];
    }
    s = dadd(s, dmul(c.lm_weight, f));
  }
  return s;
}

__host__ __device__ inline int topk_cmax(int K);

// cand (8) + bucket (4) + taken (1) per candidate (+ flat index (4) in list mode)
__host__ __device__ inline size_t sel_smem_bytes(int beam, int vocab, bool list_mode = false) {
  const size_t nv = (size_t)beam * (list_mode ? (beam < vocab ? beam : vocab) : vocab);
  return 8 * (nv + 2 * (size_t)beam) + 4 * 6 * (size_t)beam + (list_mode ? 4 * nv : 0) +
         4 * nv + 4 * (size_t)topk_cmax(beam) + nv + 16;
}

// Stage 1 of the large-vocabulary selection: one CTA per live row keeps the
// row's top-beam candidates by (score desc, token asc).
template <typename AM>
__global__ void __launch_bounds__(kSelThreads)
row_topk_kernel(fb_search_cfg_t c, fb_search_state_t st, const AM* __restrict__ am,
                int64_t am_stride, const double* __restrict__ fus, int64_t f_stride) {
  pdl_entry();
  extern __shared__ unsigned char sm_raw[];
  const int slot = blockIdx.x;
  const int K = c.beam, V = c.vocab;
  const int u = slot / K, p = slot % K;
  if (!st.active[u] || p >= st.n_live[u]) return;
  const int n = st.n_live[u];
  const int Kc = K < V ? K : V;           // a row never has more than V candidates
  const int cmax = topk_cmax(K);
  double* sc = reinterpret_cast<double*>(sm_raw);                      // [V]
  uint32_t* bkt = reinterpret_cast<uint32_t*>(sc + V);                 // [V]
  int* cl = reinterpret_cast<int*>(bkt + V);                           // [cmax]
  int* win = cl + cmax;                                                // [K]
  unsigned char* taken = reinterpret_cast<unsigned char*>(win + K);    // [V]
  __shared__ int s_gated, s_nwin;
  __shared__ AM wmax[kSelThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const AM* row = am + (int64_t)slot * am_stride;
  if (c.gate_on) {
    AM mx = row[0];
    for (int t = tid; t < V; t += kSelThreads) mx = row[t] > mx ? row[t] : mx;
    for (int off = 16; off; off >>= 1) {
      const AM o = __shfl_xor_sync(0xffffffffu, mx, off);
      mx = o > mx ? o : mx;
    }
    if (lane == 0) wmax[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      AM m = wmax[0];
      for (int w = 1; w < kSelThreads / 32; ++w) m = wmax[w] > m ? wmax[w] : m;
      s_gated = row[c.eos_id] <= (AM)c.gamma * m;
    }
  } else if (tid == 0) {
    s_gated = 0;
  }
  __syncthreads();
  const double tot = st.total_in[slot];
  for (int t = tid; t < V; t += kSelThreads)
    sc[t] = dadd(tot, step_score(c, am, am_stride, fus, f_stride, slot, t, s_gated,
                                  st.fus_norm, st.fus_floor));
  __syncthreads();
  block_topk(sc, nullptr, V, Kc, win, &s_nwin, bkt, cl, cmax, taken);
  double* os = st.cand_score_ws + (int64_t)slot * K;
  int32_t* of = st.cand_flat_ws + (int64_t)slot * K;
  for (int k = tid; k < Kc; k += kSelThreads) {
    if (k < s_nwin) {
      const int t = win[k];
      os[k] = sc[t];
      of[k] = t * n + p;                 // token-major flat index of decoder.py:404
    } else {
      os[k] = -INFINITY;
      of[k] = INT_MAX;
    }
  }
}

template <typename AM>
__device__ __forceinline__ void
search_step_body(const fb_search_cfg_t& c, const fb_search_state_t& st, const AM* __restrict__ am,
                 int64_t am_stride, const double* __restrict__ fus, int64_t f_stride,
                 int list_mode) {
  extern __shared__ unsigned char sm_raw[];
  const int u = blockIdx.x;
  if (!st.active[u]) return;
  const int K = c.beam, V = c.vocab;
  const int n = st.n_live[u];
  const int base = u * K;
  const int steps = st.steps[u];
  const int MT = c.max_tokens;
  const int Kc = K < V ? K : V;
  const int NV = list_mode ? n * Kc : n * V;    // list mode: n rows x their top-min(K, V)

  // dynamic layout: doubles | ints | bytes (any beam; see sel_smem_bytes)
  double* cand = reinterpret_cast<double*>(sm_raw);                    // [NV]
  double* new_base = cand + NV;                                        // [K]
  double* new_total = new_base + K;                                    // [K]
  int* gated = reinterpret_cast<int*>(new_total + K);                  // [K]
  int* sel = gated + K;                                                // [K]
  int* new_par = sel + K;                                              // [K]
  int* new_tok = new_par + K;                                          // [K]
  int* fin_slot = new_tok + K;                                         // [K]
  int* fin_par = fin_slot + K;                                         // [K]
  int* cflat = fin_par + K;                                            // [NV] list mode
  uint32_t* bkt = reinterpret_cast<uint32_t*>(cflat + (list_mode ? NV : 0));  // [NV]
  const int cmax = topk_cmax(K);
  int* cl = reinterpret_cast<int*>(bkt + NV);                          // [cmax]
  unsigned char* taken = reinterpret_cast<unsigned char*>(cl + cmax);  // [NV]
  __shared__ Cand wbest[kSelThreads / 32];
  __shared__ int s_nsel, s_stop;
  __shared__ int n_new, n_fin_new;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  STRACE(0);

  // EOS gate per parent (decoder.py:396-398), compared in the AM row dtype.
  if (c.gate_on) {
    for (int p = warp; p < n; p += kSelThreads / 32) {
      const AM* row = am + (int64_t)(base + p) * am_stride;
      AM mx = row[0];
      for (int t = lane; t < V; t += 32) mx = row[t] > mx ? row[t] : mx;
      for (int off = 16; off; off >>= 1) {
        const AM o = __shfl_xor_sync(0xffffffffu, mx, off);
        mx = o > mx ? o : mx;
      }
      if (lane == 0) gated[p] = row[c.eos_id] <= (AM)c.gamma * mx;
    }
  } else {
    for (int p = tid; p < n; p += kSelThreads) gated[p] = 0;
  }
  __syncthreads();

  // candidates, token-major flat index j = t * n + p (decoder.py:404)
  if (list_mode) {
    for (int j = tid; j < NV; j += kSelThreads) {
      const int64_t src = (int64_t)(base + j / Kc) * K + j % Kc;
      cand[j] = st.cand_score_ws[src];
      cflat[j] = st.cand_flat_ws[src];
      taken[j] = 0;
    }
  } else {
    for (int j = tid; j < NV; j += kSelThreads) {
      const int t = j / n, p = j % n;
      const double s = step_score(c, am, am_stride, fus, f_stride, base + p, t, gated[p],
                                  st.fus_norm, st.fus_floor);
      cand[j] = dadd(st.total_in[base + p], s);
      taken[j] = 0;
    }
  }
  if (tid == 0) s_nsel = 0, s_stop = 0;
  __syncthreads();
  STRACE(1);

  if (NV >= kRadixMin || (st.force_two_stage & 2)) {
    block_topk(cand, list_mode ? cflat : nullptr, NV, K, sel, &s_nsel, bkt, cl, cmax, taken);
  } else
  // K rounds of block argmax == the first K entries of argsort(-flat, stable)
  for (int k = 0; k < K; ++k) {
    Cand b{-INFINITY, INT_MAX};
    for (int j = tid; j < NV; j += kSelThreads) {
      if (!taken[j]) {
        Cand x{cand[j], list_mode ? cflat[j] : j};
        if (better(x, b)) b = x;
      }
    }
    b = warp_best(b);
    if (lane == 0) wbest[warp] = b;
    __syncthreads();
    if (tid == 0) {
      Cand w = wbest[0];
      for (int q = 1; q < kSelThreads / 32; ++q)
        if (better(wbest[q], w)) w = wbest[q];
      if (w.j == INT_MAX || w.s == -INFINITY) {
        s_stop = 1;
      } else {
        sel[s_nsel++] = w.j;
        if (!list_mode) taken[w.j] = 1;
      }
    }
    __syncthreads();
    if (s_stop) break;
    if (list_mode) {                       // flat -> position (unique flat indices)
      const int fj = sel[s_nsel - 1];
      for (int j = tid; j < NV; j += kSelThreads)
        if (cflat[j] == fj) taken[j] = 1;
      __syncthreads();
    }
  }

  STRACE(2);
  // plan children in selection order (decoder.py:410-432); the selected
  // candidates' scores are computed in parallel first (one thread each), so
  // the sequential slot assignment below touches shared memory only
  {
    const bool cov_on = c.cov_mode != 0;
    for (int k = tid; k < s_nsel; k += kSelThreads) {
      const int j = sel[k];
      const int t = j / n, p = j % n;
      const int ps = base + p;
      const double s = step_score(c, am, am_stride, fus, f_stride, ps, t, gated[p],
                                  st.fus_norm, st.fus_floor);
      const double nb = dadd(st.base_in[ps], s);
      new_base[k] = nb;                      // staged by selection rank k
      new_total[k] = cov_on ? dadd(nb, dmul(c.cov_weight, st.cov_post[ps])) : nb;
    }
  }
  __syncthreads();
  if (tid == 0) {
    int nn = 0, nf = 0;
    const int cap = 2 * K;
    int free_slot = 0;
    for (int k = 0; k < s_nsel; ++k) {
      const int j = sel[k];
      const int t = j / n, p = j % n;
      const int ps = base + p;
      const double nb = new_base[k];         // nn <= k: compaction in place
      const double tt = new_total[k];
      if (t == c.eos_id) {
        while (free_slot < cap && st.fin_valid[u * cap + free_slot]) ++free_slot;
        const int f = free_slot++;
        st.fin_valid[u * cap + f] = 1;
        st.fin_total[u * cap + f] = tt;
        st.fin_len[u * cap + f] = steps + 1;
        fin_slot[nf] = f;
        fin_par[nf] = ps;
        ++nf;
      } else {
        new_par[nn] = ps;
        new_tok[nn] = t;
        new_base[nn] = nb;
        new_total[nn] = tt;
        ++nn;
      }
    }
    n_new = nn;
    n_fin_new = nf;
  }
  __syncthreads();

  STRACE(3);
  // token rows and accumulators: one flat parallel copy per array (all rows'
  // loads in flight together)
  if (steps > 0) {
    for (int x = tid; x < n_new * steps; x += kSelThreads) {
      const int i = x / steps, q = x - i * steps;
      st.tok_out[(int64_t)(base + i) * MT + q] = st.tok_in[(int64_t)new_par[i] * MT + q];
    }
    for (int x = tid; x < n_fin_new * steps; x += kSelThreads) {
      const int i = x / steps, q = x - i * steps;
      st.fin_tokens[((int64_t)u * 2 * K + fin_slot[i]) * MT + q] =
          st.tok_in[(int64_t)fin_par[i] * MT + q];
    }
  }
  for (int i = tid; i < n_new; i += kSelThreads) {
    st.tok_out[(int64_t)(base + i) * MT + steps] = new_tok[i];
    st.base_out[base + i] = new_base[i];
    st.total_out[base + i] = new_total[i];
    st.parent[base + i] = new_par[i];
    st.last_tok[base + i] = new_tok[i];
  }
  for (int i = tid; i < n_fin_new; i += kSelThreads)
    st.fin_tokens[((int64_t)u * 2 * K + fin_slot[i]) * MT + steps] = c.eos_id;
  const int T = st.t_enc[u];
  if (T > 0) {
    for (int x = tid; x < n_fin_new * T; x += kSelThreads) {
      const int i = x / T, q = x - i * T;
      st.fin_acc[((int64_t)u * 2 * K + fin_slot[i]) * c.t_max + q] =
          st.acc_post[(int64_t)fin_par[i] * c.t_max + q];
    }
  }
  __syncthreads();

  STRACE(4);
  // finished-set cap, stop tests, result pick (decoder.py:433-450, :464-480)
  __shared__ int res_src, res_is_fin, res_L;
  if (tid == 0) {
    const int cap = 2 * K;
    int* fv = st.fin_valid + u * cap;
    const double* ft = st.fin_total + u * cap;
    const int* fl = st.fin_len + u * cap;
    const int32_t* fk = st.fin_tokens + (int64_t)u * cap * MT;
    int cnt = 0;
    for (int f = 0; f < cap; ++f) cnt += fv[f];
    while (cnt > K) {  // drop the entry that sorts last
      int worst = -1;
      for (int f = 0; f < cap; ++f) {
        if (!fv[f]) continue;
        if (worst < 0 || key_less(ft[worst], fl[worst], fk + (int64_t)worst * MT, ft[f], fl[f],
                                  fk + (int64_t)f * MT))
          worst = f;
      }
      fv[worst] = 0;
      --cnt;
    }
    const int steps1 = steps + 1;
    st.steps[u] = steps1;
    st.n_live[u] = n_new;
    bool on = true;
    if (n_new == 0 || steps1 >= st.max_len[u]) {
      on = false;
    } else if (cnt > 0 && c.early_stop) {
      const double slack = c.cov_mode != 0 ? dmul(c.cov_weight, (double)T) : 0.0;
      double best = new_base[0];
      for (int i = 1; i < n_new; ++i) best = fmax(best, new_base[i]);
      best = dadd(best, slack);
      double worst = INFINITY;
      for (int f = 0; f < cap; ++f)
        if (fv[f]) worst = fmin(worst, ft[f]);
      if (best < worst) on = false;
    }
    st.active[u] = on ? 1 : 0;
    res_src = -1;
    if (!on) {
      if (cnt > 0) {
        int b = -1;
        for (int f = 0; f < cap; ++f) {
          if (!fv[f]) continue;
          if (b < 0 || key_less(ft[f], fl[f], fk + (int64_t)f * MT, ft[b], fl[b],
                                fk + (int64_t)b * MT))
            b = f;
        }
        res_src = b;
        res_is_fin = 1;
        res_L = fl[b];
        st.res_score[u] = ft[b];
      } else if (n_new > 0) {
        int b = 0;
        for (int i = 1; i < n_new; ++i) {
          if (key_less(new_total[i], steps1, st.tok_out + (int64_t)(base + i) * MT,
                       new_total[b], steps1, st.tok_out + (int64_t)(base + b) * MT))
            b = i;
        }
        res_src = b;
        res_is_fin = 0;
        res_L = steps1;
        st.res_score[u] = new_total[b];
      }
      st.res_finished[u] = cnt > 0;
      st.res_steps[u] = steps1;
      st.res_len[u] = -1;  // "no hypotheses survived" unless set below
    }
  }
  __syncthreads();
  if (res_src >= 0) {
    const int32_t* src;
    const double* asrc;
    if (res_is_fin) {
      const int64_t fe = (int64_t)u * 2 * K + res_src;
      src = st.fin_tokens + fe * MT;
      asrc = st.fin_acc + fe * c.t_max;
    } else {
      src = st.tok_out + (int64_t)(base + res_src) * MT;
      asrc = st.acc_post + (int64_t)new_par[res_src] * c.t_max;
    }
    int L = res_L;
    if (L > 0 && src[L - 1] == c.eos_id) --L;   // strip trailing <eos>
    int32_t* dst = st.res_tokens + (int64_t)u * MT;
    for (int q = tid; q < L; q += kSelThreads) dst[q] = src[q];
    double* ad = st.res_acc + (int64_t)u * c.t_max;
    for (int q = tid; q < T; q += kSelThreads) ad[q] = asrc[q];
    if (tid == 0) st.res_len[u] = L;
  }
  STRACE(5);
}

// Deterministic compact list of the rows that enter the next step (active
// utterances' live rows in utterance order) and each slot's position in it.
__device__ __forceinline__ void compact_rows_block(int B, int K, const int32_t* active,
                                                   const int32_t* n_live, int32_t* rows,
                                                   int32_t* count, int32_t* row_pos) {
  __shared__ int wsum[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int b0 = 0; b0 < B; b0 += blockDim.x) {
    const int u = b0 + threadIdx.x;
    const int cnt = (u < B && active[u]) ? n_live[u] : 0;
    int x = cnt;
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, off);
        if (lane >= off) w += y;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    const int pos = carry + (warp ? wsum[warp - 1] : 0) + x - cnt;
    for (int i = 0; i < cnt; ++i) rows[pos + i] = u * K + i;
    if (row_pos != nullptr)
      for (int i = 0; i < cnt; ++i) row_pos[u * K + i] = pos + i;
    __syncthreads();
    if (threadIdx.x == 0) carry += wsum[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = carry;
}

// One CTA per utterance; with st.select_arrive the last CTA to finish also
// builds the next step's compact row list (no separate launch on the chain).
template <typename AM>
__global__ void __launch_bounds__(kSelThreads)
search_step_kernel(fb_search_cfg_t c, fb_search_state_t st, const AM* __restrict__ am,
                   int64_t am_stride, const double* __restrict__ fus, int64_t f_stride,
                   int list_mode) {
  pdl_entry();
  search_step_body<AM>(c, st, am, am_stride, fus, f_stride, list_mode);
  if (st.select_arrive == nullptr) return;
  __shared__ int s_last;
  __threadfence();                                   // this utterance's state, visible
  __syncthreads();
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(st.select_arrive, 1);
    s_last = prev == (int)gridDim.x - 1;
    if (s_last) *st.select_arrive = 0;               // zero again for the next step
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  compact_rows_block(gridDim.x, c.beam, st.active, st.n_live, st.next_rows, st.next_count,
                     st.next_row_pos);
}

// Exact pruning of speculative <eos> LM events (see fb_spec_select in the
// header).  One CTA per active utterance; candidates as in search_step.
template <typename AM>
__global__ void __launch_bounds__(kSelThreads)
spec_select_kernel(fb_search_cfg_t c, fb_search_state_t st, fb_trie_t trie,
                   const int32_t* __restrict__ tstate, const int32_t* __restrict__ hslot,
                   const AM* __restrict__ am, int64_t am_stride, double* __restrict__ fus,
                   int64_t f_stride, int32_t* ev_row, int32_t* ev_rank, int32_t* ev_slot,
                   int32_t* ev_count, int32_t* row_ev) {
  pdl_entry();
  extern __shared__ unsigned char sm_raw[];
  const int u = blockIdx.x;
  if (!st.active[u]) return;
  const int K = c.beam, V = c.vocab;
  const int n = st.n_live[u];
  const int base = u * K;
  const int NV = n * V;
  double* cand = reinterpret_cast<double*>(sm_raw);                    // [NV]
  int* gated = reinterpret_cast<int*>(cand + NV);                      // [K]
  int* fin = gated + K;                                                // [K]
  int* rank_of = fin + K;                                              // [K]
  unsigned char* taken = reinterpret_cast<unsigned char*>(rank_of + K); // [NV]
  // radix-path scratch (NV >= kRadixMin): keys with the unsure entries at
  // -inf, buckets, candidate list, picks
  double* key2 = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(taken + NV) + 7) & ~uintptr_t(7));   // [NV]
  uint32_t* bkt = reinterpret_cast<uint32_t*>(key2 + NV);              // [NV]
  const int cmax = topk_cmax(K);
  int* cl = reinterpret_cast<int*>(bkt + NV);                          // [cmax]
  int* pick = cl + cmax;                                               // [K]
  __shared__ Cand wbest[kSelThreads / 32];
  __shared__ double s_thr;
  __shared__ int s_found, s_npick;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int p = warp; p < n; p += kSelThreads / 32) {
    const AM* row = am + (int64_t)(base + p) * am_stride;
    int g = 0;
    if (c.gate_on) {
      AM mx = row[0];
      for (int t = lane; t < V; t += 32) mx = row[t] > mx ? row[t] : mx;
      for (int off = 16; off; off >>= 1) {
        const AM o = __shfl_xor_sync(0xffffffffu, mx, off);
        mx = o > mx ? o : mx;
      }
      g = row[c.eos_id] <= (AM)c.gamma * mx;
    }
    if (lane == 0) {
      const int s = tstate[base + p];
      const int rk = s > 0 ? trie.info[4 * s + 2] : -1;
      gated[p] = g;
      fin[p] = rk >= 0;
      rank_of[p] = rk;
    }
  }
  __syncthreads();
  // exactly known candidates; uncertain eos-at-final entries are excluded
  for (int j = tid; j < NV; j += kSelThreads) {
    const int t = j / n, p = j % n;
    const bool unsure = (t == c.eos_id) && fin[p] && !gated[p];
    cand[j] = dadd(st.total_in[base + p],
                   step_score(c, am, am_stride, fus, f_stride, base + p, t, gated[p]));
    taken[j] = unsure ? 1 : 0;
  }
  __syncthreads();
  // beam-th best of the known candidates
  if (tid == 0) { s_thr = -INFINITY; s_found = 0; }
  __syncthreads();
  if (NV >= kRadixMin) {
    for (int j = tid; j < NV; j += kSelThreads) key2[j] = taken[j] ? -INFINITY : cand[j];
    __syncthreads();
    block_topk(key2, nullptr, NV, K, pick, &s_npick, bkt, cl, cmax, taken);
    __syncthreads();
    if (tid == 0) {
      s_found = s_npick;
      if (s_npick > 0) s_thr = key2[pick[s_npick - 1]];
    }
    __syncthreads();
  } else
  for (int k = 0; k < K; ++k) {
    Cand b{-INFINITY, INT_MAX};
    for (int j = tid; j < NV; j += kSelThreads)
      if (!taken[j]) {
        Cand x{cand[j], j};
        if (better(x, b)) b = x;
      }
    b = warp_best(b);
    if (lane == 0) wbest[warp] = b;
    __syncthreads();
    if (tid == 0) {
      Cand w = wbest[0];
      for (int q = 1; q < kSelThreads / 32; ++q)
        if (better(wbest[q], w)) w = wbest[q];
      if (w.j != INT_MAX && w.s != -INFINITY) {
        taken[w.j] = 1;
        ++s_found;
        s_thr = w.s;
      }
    }
    __syncthreads();
  }
  const bool prune_ok = s_found == K;   // else every uncertain row must be resolved
  for (int p = tid; p < n; p += kSelThreads) {
    const int r = base + p;
    int e = -1;
    if (fin[p]) {
      bool need = true;
      if (gated[p]) {
        need = false;                     // -inf either way: no LM step
      } else if (prune_ok) {
        const double ub = cand[c.eos_id * n + p];   // total + am + lm_weight * word_end
        need = !(ub < s_thr);
      }
      if (need) {
        e = atomicAdd(ev_count, 1);
        ev_row[e] = r;
        ev_rank[e] = rank_of[p];
        ev_slot[e] = hslot[r];
      } else {
        fus[(int64_t)r * f_stride + c.eos_id] = -INFINITY;
      }
    }
    row_ev[r] = e;
  }
}

__global__ void eos_fixup_kernel(int n_max, const int32_t* __restrict__ cnt,
                                 const int32_t* __restrict__ ev_row,
                                 const double* __restrict__ eos_lp, double* __restrict__ fus,
                                 int64_t f_stride, int eos_id) {
  pdl_entry();
  const int n = row_count(n_max, cnt);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int r = ev_row[e];
    double* f = fus + (int64_t)r * f_stride + eos_id;
    *f = dadd(*f, eos_lp[r]);
  }
}

// Deterministic compact list of rows that enter the next step.
__global__ void compact_rows_kernel(int B, int K, const int32_t* active, const int32_t* n_live,
                                    int32_t* rows, int32_t* count, int32_t* row_pos) {
  pdl_entry();
  compact_rows_block(B, K, active, n_live, rows, count, row_pos);
}

__global__ void search_init_kernel(fb_search_cfg_t c, fb_search_state_t st, int B) {
  const int K = c.beam;
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < B; u += gridDim.x * blockDim.x) {
    st.active[u] = 1;
    st.n_live[u] = 1;
    st.steps[u] = 0;
    st.res_len[u] = -1;
    for (int f = 0; f < 2 * K; ++f) st.fin_valid[u * 2 * K + f] = 0;
    // entering-step row of the first step (decoder.py:358)
    const_cast<double*>(st.base_in)[u * K] = 0.0;
    const_cast<double*>(st.total_in)[u * K] = 0.0;
    st.parent[u * K] = u * K;
    st.last_tok[u * K] = -1;
    st.next_rows[u] = u * K;
    if (st.next_row_pos != nullptr) st.next_row_pos[u * K] = u;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *st.next_count = B;
}

}  // namespace fb

using namespace fb;

extern "C" int fb_search_init(const fb_search_cfg_t* cfg, const fb_search_state_t* st,
                              int32_t num_utts, void* stream) {
  FB_CHECK_ARG(cfg && st && num_utts >= 0, "null search state");
  if (num_utts == 0) return FB_OK;
  search_init_kernel<<<std::min((num_utts + 255) / 256, kNumSMs), 256, 0,
                       (cudaStream_t)stream>>>(*cfg, *st, num_utts);
  count_launch();
  return check_launch("search_init");
}

extern "C" int fb_attend_coverage(const fb_search_cfg_t* cfg, int32_t n_max, const int32_t* n_dev,
                                  const int32_t* rows, const int32_t* parent,
                                  const int32_t* t_enc, const double* acc_in, const void* attn,
                                  int32_t attn_f32, int64_t attn_stride, double* acc_out,
                                  double* cov_out, void* stream) {
  FB_CHECK_ARG(cfg && acc_in && attn && acc_out, "null accumulator buffers");
  FB_CHECK_ARG(cfg->cov_mode == 0 || cov_out, "coverage output required");
  if (n_max <= 0) return FB_OK;
  const int threads = 256;
  const int blocks = std::min((n_max + 7) / 8, kNumSMs * 8);
  if (attn_f32)
    attend_coverage_kernel<float><<<blocks, threads, 0, (cudaStream_t)stream>>>(
        *cfg, n_max, n_dev, rows, parent, t_enc, acc_in, (const float*)attn, attn_stride,
        acc_out, cov_out);
  else
    attend_coverage_kernel<double><<<blocks, threads, 0, (cudaStream_t)stream>>>(
        *cfg, n_max, n_dev, rows, parent, t_enc, acc_in, (const double*)attn, attn_stride,
        acc_out, cov_out);
  count_launch();
  return check_launch("attend_coverage");
}

extern "C" int fb_search_step(const fb_search_cfg_t* cfg, const fb_search_state_t* st,
                              int32_t num_utts, const void* am, int64_t am_stride,
                              const double* fusion, int64_t fusion_stride, void* stream) {
  FB_CHECK_ARG(cfg && st && am, "null search arguments");
  FB_CHECK_ARG(cfg->beam >= 1, "beam must be positive");
  FB_CHECK_ARG(!cfg->has_fusion || fusion, "fusion rows required");
  constexpr size_t kBudget = 220 * 1024;
  bool list_mode = false;
  size_t smem = sel_smem_bytes(cfg->beam, cfg->vocab);
  if (smem > kBudget || (st->force_two_stage & 1)) {
    if (!st->cand_score_ws || !st->cand_flat_ws)
      return fail(FB_ERR_CONFIG, "beam x vocabulary too large: pass the two-stage workspace");
    list_mode = true;
    smem = sel_smem_bytes(cfg->beam, cfg->vocab, true);
    const size_t row_smem = (size_t)cfg->vocab * 13 + 4 * (size_t)(topk_cmax(cfg->beam) + cfg->beam) + 16;
    if (smem > kBudget || row_smem > kBudget)
      return fail(FB_ERR_CONFIG, "beam or vocabulary too large for the selection kernels");
  }
  if (num_utts <= 0) return FB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int N = num_utts * cfg->beam;
  const size_t row_smem = (size_t)cfg->vocab * 13 + 4 * (size_t)(topk_cmax(cfg->beam) + cfg->beam) + 16;
#define FB_SEL(AMT)                                                                           \
  {                                                                                           \
    auto k = search_step_kernel<AMT>;                                                         \
    auto kr = row_topk_kernel<AMT>;                                                           \
    static bool set = false;                                                                  \
    if (!set) {                                                                               \
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBudget);      \
      cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBudget);     \
      set = true;                                                                             \
    }                                                                                         \
    if (list_mode) {                                                                          \
      launch_pdl(kr, dim3(N), dim3(kSelThreads), row_smem, s, *cfg, *st, (const AMT*)am,      \
                 am_stride, fusion, fusion_stride);                                           \
      count_launch();                                                                         \
    }                                                                                         \
    launch_pdl(k, dim3(num_utts), dim3(kSelThreads), smem, s, *cfg, *st, (const AMT*)am,      \
               am_stride, fusion, fusion_stride, list_mode ? 1 : 0);                          \
  }
  if (cfg->am_f32) FB_SEL(float) else FB_SEL(double)
#undef FB_SEL
  count_launch();
  int rc = check_launch("search_step");
  if (rc) return rc;
  if (st->select_arrive != nullptr) return FB_OK;     // compacted by the last selection CTA
  launch_pdl(compact_rows_kernel, dim3(1), dim3(1024), 0, s, num_utts, cfg->beam, st->active,
             st->n_live, st->next_rows, st->next_count, st->next_row_pos);
  count_launch();
  return check_launch("compact_rows");
}

extern "C" int fb_spec_select(const fb_search_cfg_t* cfg, const fb_search_state_t* st,
                              int32_t num_utts, const fb_trie_t* trie, const int32_t* trie_state,
                              const int32_t* hist_slot, const void* am, int64_t am_stride,
                              double* fusion, int64_t fusion_stride, int32_t* ev_row,
                              int32_t* ev_rank, int32_t* ev_slot, int32_t* ev_count,
                              int32_t* row_ev, const int32_t* ev_start, void* stream) {
  FB_CHECK_ARG(cfg && st && trie && am && fusion && ev_count && row_ev, "null spec-select args");
  const size_t nv = (size_t)cfg->beam * cfg->vocab;
  const size_t smem = nv * 9 + 12 * (size_t)cfg->beam + 8 +                     // cand, taken
                      (nv >= (size_t)kRadixMin                                     // radix
                           ? nv * 12 + 4 * ((size_t)topk_cmax(cfg->beam) + cfg->beam) + 16
                           : 0);
  if (smem > 220 * 1024) return fail(FB_ERR_CONFIG, "beam x vocabulary too large");
  cudaStream_t s = (cudaStream_t)stream;
  if (ev_start)   // events appended after the late events queued by the last step
    cudaMemcpyAsync(ev_count, ev_start, sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
  else
    cudaMemsetAsync(ev_count, 0, sizeof(int32_t), s);
  if (num_utts <= 0) return check_launch("spec_select");
  if (cfg->am_f32) {
    auto k = spec_select_kernel<float>;
    static bool set = false;
    if (!set) { cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024); set = true; }
    launch_pdl(k, dim3(num_utts), dim3(kSelThreads), smem, s, *cfg, *st, *trie, trie_state,
               hist_slot, (const float*)am, am_stride, fusion, fusion_stride, ev_row, ev_rank,
               ev_slot, ev_count, row_ev);
  } else {
    auto k = spec_select_kernel<double>;
    static bool set = false;
    if (!set) { cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024); set = true; }
    launch_pdl(k, dim3(num_utts), dim3(kSelThreads), smem, s, *cfg, *st, *trie, trie_state,
               hist_slot, (const double*)am, am_stride, fusion, fusion_stride, ev_row, ev_rank,
               ev_slot, ev_count, row_ev);
  }
  count_launch();
  return check_launch("spec_select");
}

extern "C" int fb_eos_fixup(int32_t n_max, const int32_t* ev_count, const int32_t* ev_row,
                            const double* eos_lp, double* fusion, int64_t fusion_stride,
                            int32_t eos_id, void* stream) {
  FB_CHECK_ARG(ev_row && eos_lp && fusion, "null eos-fixup args");
  if (n_max <= 0) return FB_OK;
  launch_pdl(eos_fixup_kernel, dim3(std::min((n_max + 255) / 256, kNumSMs)), dim3(256), 0,
      (cudaStream_t)stream, n_max, ev_count, ev_row, eos_lp, fusion, fusion_stride, eos_id);
  count_launch();
  return check_launch("eos_fixup");
}

#ifdef FB_SEARCH_TRACE
extern "C" int fb_search_trace_read(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, fb::g_strace, sizeof(fb::g_strace)) == cudaSuccess ? 0 : 3;
}
#endif
