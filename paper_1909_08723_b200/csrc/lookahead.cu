// Look-ahead word-LM fusion kernels: CSR trie gather (Eq. 4), trie advance,
// fp64 prefix sums of word distributions.
//
// Reference semantics: fusion.py:118-185 (char_scores), :187-224 (advance),
// :40-42 / :223 (cumsum_distribution).  HBM-bound integer/byte gathers; no
// tensor-core work here.
#include "common.cuh"

namespace fb {

__device__ __forceinline__ double mass(const double* __restrict__ g, int hi, int lo) {
  // g[hi] - g[lo] with g[-1] := 0   (fusion.py:135-146)
  double up = __ldg(g + hi);
  double low = lo >= 0 ? __ldg(g + lo) : 0.0;
  return dsub(up, low);
}

// One warp per hypothesis row; the row's scores are staged in shared memory
// (penalty fill -> edge columns -> <space>/<eos>) and written out coalesced.
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
lookahead_scores_kernel(fb_trie_t trie, int n_max, const int32_t* __restrict__ n_dev,
                        const int32_t* __restrict__ rows, const int32_t* __restrict__ tstate,
                        const int32_t* __restrict__ hslot, const double* __restrict__ g_pool,
                        int64_t g_stride, const double* __restrict__ hist_eos,
                        const double* __restrict__ ext_eos, int space_id, int eos_id,
                        double pen, double floor_v, double* __restrict__ out,
                        int64_t out_stride, unsigned long long* floored) {
  pdl_entry();
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int V = trie.alphabet;
  double* srow = smem + warp * V;
  const int n = row_count(n_max, n_dev);
  unsigned nfloor = 0;
  for (int i = blockIdx.x * WARPS + warp; i < n; i += gridDim.x * WARPS) {
    const int r = row_at(rows, i);
    const int s = tstate[r];
    for (int c = lane; c < V; c += 32) srow[c] = pen;
    __syncwarp();
    if (s >= 0) {
      const double* g = g_pool + (int64_t)hslot[r] * g_stride;
      const int4 inf = reinterpret_cast<const int4*>(trie.info)[s];
      const double denom = mass(g, inf.x, inf.y);
      const double ldenom = log(denom);
      const int e0 = trie.row_ptr[s], e1 = trie.row_ptr[s + 1];
      for (int e = e0 + lane; e < e1; e += 32) {
        const int c = trie.edge_label[e];
        const int4 ci = reinterpret_cast<const int4*>(trie.info)[trie.edge_child[e]];
        const double numer = mass(g, ci.x, ci.y);
        double v;
        if (numer > 0.0 && denom > 0.0) {
          v = dsub(log(numer), ldenom);
        } else {
          v = floor_v;
          ++nfloor;
        }
        srow[c] = v;
      }
      if (lane == 0) {
        double wend = pen;
        const bool fin = inf.z >= 0;
        if (fin) {
          const int rk = inf.z;
          const double wm = mass(g, rk, rk - 1);
          if (wm > 0.0 && denom > 0.0) {
            wend = dsub(log(wm), ldenom);
          } else {
            wend = floor_v;
            ++nfloor;
          }
        }
        srow[space_id] = fin ? wend : pen;
        double ecol = pen;
        if (s == 0) {
          ecol = hist_eos ? hist_eos[hslot[r]] : ext_eos[r];
        } else if (fin) {
          ecol = dadd(wend, ext_eos[r]);
        }
        srow[eos_id] = ecol;
      }
    }
    __syncwarp();
    double* o = out + (int64_t)r * out_stride;
    for (int c = lane; c < V; c += 32) o[c] = srow[c];
    __syncwarp();
  }
  if (floored) {
    for (int off = 16; off; off >>= 1) nfloor += __shfl_xor_sync(0xffffffffu, nfloor, off);
    if (lane == 0 && nfloor) atomicAdd(floored, (unsigned long long)nfloor);
  }
}

__device__ __forceinline__ int find_child(const fb_trie_t& t, int s, int c) {
  int lo = t.row_ptr[s], hi = t.row_ptr[s + 1] - 1;
  while (lo <= hi) {  // labels ascend within a state
    const int mid = (lo + hi) >> 1;
    const int l = t.edge_label[mid];
    if (l == c) return t.edge_child[mid];
    if (l < c) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

__global__ void trie_advance_kernel(fb_trie_t trie, int n_max, const int32_t* __restrict__ n_dev,
                                    const int32_t* __restrict__ rows,
                                    const int32_t* __restrict__ parent,
                                    const int32_t* __restrict__ sin,
                                    const int32_t* __restrict__ hin,
                                    const int32_t* __restrict__ tokens, int space_id,
                                    int eos_id, int pad_id, int32_t* __restrict__ sout,
                                    int32_t* __restrict__ hout, int32_t* __restrict__ brank) {
  pdl_entry();
  const int n = row_count(n_max, n_dev);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int r = row_at(rows, i);
    const int p = parent ? parent[r] : r;
    const int s = sin[p];
    const int tok = tokens[r];
    int ns = s;
    int rk = -2;
    if (tok == space_id) {
      ns = 0;
      rk = -1;                                  // <unk> unless s is final
      if (s >= 0) {
        const int wr = trie.info[4 * s + 2];
        if (wr >= 0) rk = wr;
      }
    } else if (tok != eos_id && tok != pad_id) {
      int c = -1;
      if (s >= 0) {
        const int tc = min(max(tok, 0), trie.alphabet - 1);
        c = find_child(trie, s, tc);
      }
      ns = c >= 0 ? c : -2;                     // OOV_STATE
    }
    sout[r] = ns;
    if (brank) brank[r] = rk;
    if (hout && hin) hout[r] = hin[p];
  }
}

// ---- multilevel fusion (reference fusion.py:268-380) ---------------------
// Row adjustment of the boundary columns (fusion.py:321-339): rows[b] holds the
// char-LM row; <space> and <eos> get += adj with
//   adj = 0                                 empty word (state 0, accum 0)
//   adj = log P_W(w | h) - accum            known word (final state; P from the
//                                           history's distribution row dist_pool[slot])
//   adj = oov_factor                        otherwise (OOV / partial word)
__global__ void multilevel_rows_kernel(fb_trie_t trie, int n, const int32_t* __restrict__ states,
                                       const int32_t* __restrict__ slots,
                                       const double* __restrict__ dist_pool, int64_t d_stride,
                                       const double* __restrict__ accum, int space_id,
                                       int eos_id, double oov_factor, double score_floor,
                                       double* __restrict__ rows, int64_t r_stride) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < n; b += gridDim.x * blockDim.x) {
    const int st = states[b];
    const double acc = accum[b];
    double adj;
    if (st == 0 && acc == 0.0) {
      adj = 0.0;
    } else if (st >= 0 && trie.info[4 * st + 2] >= 0) {
      const double p = dist_pool[(int64_t)slots[b] * d_stride + trie.info[4 * st + 2]];
      adj = dsub(p > 0.0 ? log(p) : score_floor, acc);
    } else {
      adj = oov_factor;
    }
    double* r = rows + (int64_t)b * r_stride;
    r[space_id] = dadd(r[space_id], adj);
    r[eos_id] = dadd(r[eos_id], adj);
  }
}

// State update (fusion.py:341-371): pad keeps the row; <space>/<eos> close the
// word (brank = its rank or -1 for <unk>, state 0, accum 0, counting empty
// words); a character adds the unadjusted char-LM log-prob of the token at the
// previous state (char_rows) to accum and walks the trie (OOV_STATE = -2).
__global__ void multilevel_advance_kernel(fb_trie_t trie, int n, const int32_t* __restrict__ sin,
                                          const double* __restrict__ ain,
                                          const int32_t* __restrict__ tokens,
                                          const double* __restrict__ char_rows, int64_t c_stride,
                                          int space_id, int eos_id, int pad_id,
                                          int32_t* __restrict__ sout, double* __restrict__ aout,
                                          int32_t* __restrict__ brank,
                                          unsigned long long* __restrict__ empty_words) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < n; b += gridDim.x * blockDim.x) {
    const int s = sin[b];
    const double acc = ain[b];
    const int tok = tokens[b];
    int ns = s, rk = -2;
    double na = acc;
    if (tok == pad_id) {
      // unchanged
    } else if (tok == space_id || tok == eos_id) {
      if (s == 0 && acc == 0.0) atomicAdd(empty_words, 1ull);
      rk = (s >= 0 && trie.info[4 * s + 2] >= 0) ? trie.info[4 * s + 2] : -1;
      ns = 0;
      na = 0.0;
    } else {
      na = dadd(acc, char_rows[(int64_t)b * c_stride + tok]);
      int c = -1;
      if (s >= 0 && tok >= 0 && tok < trie.alphabet) c = find_child(trie, s, tok);
      ns = c >= 0 ? c : -2;
    }
    sout[b] = ns;
    aout[b] = na;
    brank[b] = rk;
  }
}

// ---- fp64 running sums over word-distribution rows ----------------------
// One CTA per row, tiles of TILE elements staged in shared memory; each thread
// scans ITEMS consecutive values, the block scans the thread totals, and the
// carry crosses tiles.  Bandwidth-bound: 8 B read (or 4 B logits) + 8 B write
// per word.
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ double block_exclusive_scan(double v, double* wsum, double& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double x = v;
  for (int off = 1; off < 32; off <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    double w = lane < nw ? wsum[lane] : 0.0;
    for (int off = 1; off < 32; off <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w += y;
    }
    if (lane < nw) wsum[lane] = w;
  }
  __syncthreads();
  total = wsum[(blockDim.x >> 5) - 1];
  const double before = warp ? wsum[warp - 1] : 0.0;
  double excl = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane == 0) excl = 0.0;
  __syncthreads();
  return before + excl;
}


// Scan of one kScanTile-element tile held in registers: thread t owns elements
// [8t, 8t+8) (consecutive -> vectorised, coalesced global access, no shared-
// memory bank conflicts).  Returns the exclusive prefix of this thread's first
// element and the tile total.
__device__ __forceinline__ double tile_scan8(const double (&x)[kScanItems], double (&loc)[kScanItems],
                                            double* wsum, double& total) {
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    acc += x[k];
    loc[k] = acc;
  }
  return block_exclusive_scan(acc, wsum, total);
}

__device__ __forceinline__ void load8_exp(const float* __restrict__ src, int base, int cnt, float m,
                                          double (&x)[kScanItems]) {
  const int j0 = threadIdx.x * kScanItems;
  const float* p = src + base + j0;
  if (j0 + kScanItems <= cnt && ((reinterpret_cast<uintptr_t>(p) & 31) == 0)) {
    // one 256-bit load (sm_100): a warp's request covers 1 KB in 8 full lines
    float a[8];
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(a[0]), "=f"(a[1]), "=f"(a[2]), "=f"(a[3]), "=f"(a[4]), "=f"(a[5]),
                   "=f"(a[6]), "=f"(a[7])
                 : "l"(p));
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = expf(a[k] - m);
  } else if (j0 + kScanItems <= cnt && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *reinterpret_cast<const float4*>(p + 4);
    x[0] = expf(a.x - m); x[1] = expf(a.y - m); x[2] = expf(a.z - m); x[3] = expf(a.w - m);
    x[4] = expf(b.x - m); x[5] = expf(b.y - m); x[6] = expf(b.z - m); x[7] = expf(b.w - m);
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
      x[k] = (j0 + k < cnt) ? (double)expf(src[base + j0 + k] - m) : 0.0;
  }
}

__device__ __forceinline__ void store8(double* __restrict__ dst, int base, int cnt,
                                       const double (&v)[kScanItems]) {
  const int j0 = threadIdx.x * kScanItems;
  if (j0 + kScanItems <= cnt && ((reinterpret_cast<uintptr_t>(dst + base + j0) & 15) == 0)) {
#pragma unroll
    for (int k = 0; k < kScanItems; k += 2)
      *reinterpret_cast<double2*>(dst + base + j0 + k) = make_double2(v[k], v[k + 1]);
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
      if (j0 + k < cnt) dst[base + j0 + k] = v[k];
  }
}

template <bool FROM_LOGITS>
__global__ void __launch_bounds__(kScanThreads)
row_scan_kernel(int m_max, const int32_t* __restrict__ m_dev, const void* __restrict__ src,
                int64_t s_stride, const int32_t* __restrict__ src_rows, int vw, int v_out,
                const int32_t* __restrict__ slots, double* __restrict__ g_pool, int64_t g_stride,
                double* __restrict__ eos_out) {
  __shared__ double wsum[32];
  __shared__ float red_f[32];
  __shared__ float red_g[32];
  __shared__ double red_d[32];
  const int m = row_count(m_max, m_dev);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int row = blockIdx.x; row < m; row += gridDim.x) {
    const int dst = slots ? slots[row] : row;
    const int64_t srow = src_rows ? src_rows[row] : row;
    double* g = g_pool ? g_pool + (int64_t)dst * g_stride : nullptr;
    float mw = 0.f;
    double sw = 1.0;
    const float* lg = nullptr;
    if constexpr (FROM_LOGITS) {
      lg = reinterpret_cast<const float*>(src) + srow * s_stride;
      // pass A: max over the words and over all outputs (for </s>)
      float mx = -INFINITY, mall = -INFINITY;
      for (int j = threadIdx.x; j < v_out; j += blockDim.x) {
        const float z = lg[j];
        if (j < vw) mx = fmaxf(mx, z);
        mall = fmaxf(mall, z);
      }
      for (int off = 16; off; off >>= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        mall = fmaxf(mall, __shfl_xor_sync(0xffffffffu, mall, off));
      }
      if (lane == 0) { red_f[warp] = mx; red_g[warp] = mall; }
      __syncthreads();
      mx = -INFINITY; mall = -INFINITY;
      for (int w = 0; w < nw; ++w) { mx = fmaxf(mx, red_f[w]); mall = fmaxf(mall, red_g[w]); }
      mw = mx;
      // pass B: word mass relative to the word max (fp64 accumulation)
      double part = 0.0;
      for (int j = threadIdx.x; j < vw; j += blockDim.x) part += (double)expf(lg[j] - mw);
      for (int off = 16; off; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
      if (lane == 0) red_d[warp] = part;
      __syncthreads();
      sw = 0.0;
      for (int w = 0; w < nw; ++w) sw += red_d[w];
      if (threadIdx.x == 0 && eos_out) {
        // log-softmax of </s> over all outputs: words rescaled + the specials
        double sall = sw * exp((double)mw - (double)mall);
        for (int j = vw; j < v_out; ++j) sall += exp((double)lg[j] - (double)mall);
        eos_out[dst] = (double)lg[vw] - ((double)mall + log(sall));
      }
      __syncthreads();
    }
    if (!g) continue;
    // pass: running sums tile by tile (register-resident, see tile_scan8)
    double carry = 0.0;
    for (int base = 0; base < vw; base += kScanTile) {
      const int cnt = min(kScanTile, vw - base);
      double x[kScanItems], loc[kScanItems];
      if constexpr (FROM_LOGITS) {
        load8_exp(lg, base, cnt, mw, x);
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) x[k] /= sw;
      } else {
        const double* pr = reinterpret_cast<const double*>(src) + srow * s_stride;
        const int j0 = threadIdx.x * kScanItems;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) x[k] = (j0 + k < cnt) ? pr[base + j0 + k] : 0.0;
      }
      double total;
      const double pre = tile_scan8(x, loc, wsum, total) + carry;
#pragma unroll
      for (int k = 0; k < kScanItems; ++k) loc[k] += pre;
      store8(g, base, cnt, loc);
      carry += total;
    }
  }
}

// ---- softmax statistics from the LM-output GEMM epilogue -------------------
constexpr int kSegCols = kScanTile;          // 4096 columns per segment CTA
constexpr int kRnThreads = kScanThreads;     // row normaliser CTA (a thread per 8 columns)
constexpr int kRnMaxSeg = 32;                // segments the fused sums handle (131k words)

// Row-wide word max (exact) and all-output log-sum-exp from the tile stats.

// Per event row, once: M_w = max over the word logits (tile statistics),
// lse = log-sum-exp over all outputs (fp64), log P(</s>) = z[vw] - lse.
// One warp per row; norm_out[i] = M_w for the segment passes.
__global__ void __launch_bounds__(kRnThreads)
row_norm_kernel(int m_max, const int32_t* __restrict__ m_dev, const float* __restrict__ logits,
                int64_t ld, const float4* __restrict__ stats, int ntiles,
                const int32_t* __restrict__ src_rows, int vw, const int32_t* __restrict__ slots,
                double* __restrict__ eos_out, double* __restrict__ norm_out,
                double* __restrict__ stat_out, double* __restrict__ seg_out, int nseg,
                double* __restrict__ fus, int64_t fus_stride, int fus_eos) {
  // one CTA per row (grid-strided): the row's ~1,000 tile statistics are read
  // once, 4 per thread in flight, and reduced across the block (a warp per
  // row walked them 32 at a time, a latency chain of 64 loads)
  pdl_entry();
  __shared__ float red_f[2][kRnThreads / 32];
  __shared__ double red_d[kRnThreads / 32];
  __shared__ double seg_part[kRnMaxSeg][kRnThreads / 32];
  __shared__ float s_mw;
  const int m = row_count(m_max, m_dev);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kPer = 4;
  for (int i = blockIdx.x; i < m; i += gridDim.x) {
    const int64_t srow = src_rows ? src_rows[i] : i;
    const float4* st = stats + srow * ntiles;
    float ma = -INFINITY, mw = -INFINITY;
    for (int t0 = 0; t0 < ntiles; t0 += kPer * blockDim.x) {
      float4 v[kPer];
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int t = t0 + q * blockDim.x + tid;
        v[q] = t < ntiles ? st[t] : make_float4(-INFINITY, 0.f, -INFINITY, 0.f);
      }
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        ma = fmaxf(ma, v[q].x);
        mw = fmaxf(mw, v[q].z);
      }
    }
    for (int off = 16; off; off >>= 1) {
      ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, off));
      mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, off));
    }
    if (lane == 0) { red_f[0][warp] = ma; red_f[1][warp] = mw; }
    __syncthreads();
    ma = red_f[0][0];
    mw = red_f[1][0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      ma = fmaxf(ma, red_f[0][w]);
      mw = fmaxf(mw, red_f[1][w]);
    }
    double sa = 0.0;
    for (int t = tid; t < ntiles; t += blockDim.x) {     // L1-resident second pass
      const float4 v = st[t];
      if (v.x > -INFINITY) sa += (double)v.y * exp((double)v.x - (double)ma);
    }
    for (int off = 16; off; off >>= 1) sa += __shfl_xor_sync(0xffffffffu, sa, off);
    if (lane == 0) red_d[warp] = sa;
    __syncthreads();
    if (seg_out != nullptr) {
      // the g-row segment sums of exp(z - M_w) (fp64, the segment-sum pass
      // folded in): thread t owns columns [8t, 8t+8) of each 4096-column
      // segment, four segments' 256-bit loads in flight at a time
      const float* lg = logits + srow * ld;
      const int j0 = tid * kScanItems;
      for (int k0 = 0; k0 < nseg; k0 += 4) {
        float zs[4][kScanItems];                       // raw logits, -inf past the words
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c0 = (k0 + q) * kSegCols;
          const int cnt = k0 + q < nseg ? min(vw, c0 + kSegCols) - c0 : 0;
          const float* p = lg + c0 + j0;
          if (j0 + kScanItems <= cnt) {                // 32-byte aligned: ld % 8 == 0
            asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=f"(zs[q][0]), "=f"(zs[q][1]), "=f"(zs[q][2]), "=f"(zs[q][3]),
                           "=f"(zs[q][4]), "=f"(zs[q][5]), "=f"(zs[q][6]), "=f"(zs[q][7])
                         : "l"(p));
          } else {
#pragma unroll
            for (int e = 0; e < kScanItems; ++e) zs[q][e] = j0 + e < cnt ? p[e] : -INFINITY;
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double x = 0.0;
#pragma unroll
          for (int e = 0; e < kScanItems; ++e) x += (double)expf(zs[q][e] - mw);
          for (int off = 16; off; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
          if (lane == 0 && k0 + q < nseg) seg_part[k0 + q][warp] = x;
        }
      }
    }
    __syncthreads();
    if (seg_out != nullptr && tid < nseg) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += seg_part[tid][w];
      seg_out[(int64_t)i * nseg + tid] = t;
    }
    if (tid == 0) {
      double tot = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red_d[w];
      const double lse = (double)ma + log(tot);
      const double eos = (double)logits[srow * ld + vw] - lse;
      const int d = slots ? slots[i] : i;
      if (eos_out) eos_out[d] = eos;
      // fused fb_eos_fixup: the row's fusion <eos> column += log P(</s>)
      if (fus) fus[(int64_t)d * fus_stride + fus_eos] = dadd(fus[(int64_t)d * fus_stride + fus_eos], eos);
      if (norm_out) norm_out[i] = (double)mw;          // M_w per row (segment passes)
      if (stat_out) {
        stat_out[2 * i] = (double)mw;
        stat_out[2 * i + 1] = lse;
      }
    }
    __syncthreads();
  }
}

// pass 1 (g_pool): exact fp64 sum of exp(z - M_w) per 4096-column segment;
// CTA (row, 0) also writes log P(</s>).
__global__ void __launch_bounds__(kScanThreads)
seg_sum_kernel(int m_max, const int32_t* __restrict__ m_dev, const float* __restrict__ logits,
               int64_t ld, const int32_t* __restrict__ src_rows, int vw,
               double* __restrict__ seg_ws, int nseg, const double* __restrict__ norm,
               const double* __restrict__ stat_in, const int32_t* __restrict__ slots,
               double* __restrict__ eos_out) {
  pdl_entry();
  __shared__ double red_d[32];
  const int m = row_count(m_max, m_dev);
  for (int i = blockIdx.x; i < m; i += gridDim.x) {
    const int64_t srow = src_rows ? src_rows[i] : i;
    const float mw = (float)(stat_in ? stat_in[2 * srow] : norm[i]);
    if (stat_in && eos_out && blockIdx.y == 0 && threadIdx.x == 0)   // == row_norm_kernel
      eos_out[slots ? slots[i] : i] = (double)logits[srow * ld + vw] - stat_in[2 * srow + 1];
    const float* lg = logits + srow * ld;
    const int c0 = blockIdx.y * kSegCols, c1 = min(vw, c0 + kSegCols);
    double s = 0.0;
    {
      // thread t: columns [8t, 8t+8) of the segment, one 256-bit load when aligned
      double x[kScanItems];
      load8_exp(lg, c0, c1 - c0, mw, x);
#pragma unroll
      for (int k = 0; k < kScanItems; ++k) s += x[k];
    }
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if ((threadIdx.x & 31) == 0) red_d[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red_d[w];
      seg_ws[(int64_t)i * nseg + blockIdx.y] = t;
    }
    __syncthreads();
  }
}

// pass 2: scan each segment with its exact fp64 offset; g = prefix / S_w.
__global__ void __launch_bounds__(kScanThreads)
seg_scan_kernel(int m_max, const int32_t* __restrict__ m_dev, const float* __restrict__ logits,
                int64_t ld, const int32_t* __restrict__ src_rows, int vw,
                const int32_t* __restrict__ slots, const double* __restrict__ seg_ws, int nseg,
                const double* __restrict__ norm, double* __restrict__ g_pool, int64_t g_stride,
                const double* __restrict__ stat_in) {
  pdl_entry();
  __shared__ double wsum[32];
  const int m = row_count(m_max, m_dev);
  for (int i = blockIdx.x; i < m; i += gridDim.x) {
  const int64_t srow = src_rows ? src_rows[i] : i;
  const float mw = (float)(stat_in ? stat_in[2 * srow] : norm[i]);
  const double* sw = seg_ws + (int64_t)i * nseg;
  double off = 0.0, tot = 0.0;
  for (int k = 0; k < nseg; ++k) {          // same order in every CTA: deterministic
    if (k < (int)blockIdx.y) off += sw[k];
    tot += sw[k];
  }
  const float* lg = logits + srow * ld;
  double* g = g_pool + (int64_t)(slots ? slots[i] : i) * g_stride;
  const int c0 = blockIdx.y * kSegCols;
  const int cnt = min(kSegCols, vw - c0);
  double x[kScanItems], loc[kScanItems];
  load8_exp(lg, c0, cnt, mw, x);
  double total;
  const double pre = tile_scan8(x, loc, wsum, total) + off;
  const double inv = 1.0 / tot;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) loc[k] = (pre + loc[k]) * inv;
  store8(g, c0, cnt, loc);
  __syncthreads();
  }
}

__global__ void gather_rows_kernel(int n, const int32_t* __restrict__ idx, const char* __restrict__ src,
                                   char* __restrict__ dst, int64_t row_bytes) {
  const bool vec = (row_bytes % 16 == 0) && ((uintptr_t)src % 16 == 0) && ((uintptr_t)dst % 16 == 0);
  for (int r = blockIdx.x; r < n; r += gridDim.x) {
    const char* s = src + (int64_t)idx[r] * row_bytes;
    char* d = dst + (int64_t)r * row_bytes;
    if (vec) {
      const int64_t nv = row_bytes / 16;
      for (int64_t j = threadIdx.x; j < nv; j += blockDim.x)
        reinterpret_cast<int4*>(d)[j] = reinterpret_cast<const int4*>(s)[j];
    } else {
      for (int64_t j = threadIdx.x; j < row_bytes; j += blockDim.x) d[j] = s[j];
    }
  }
}

}  // namespace fb

using namespace fb;

extern "C" int fb_lookahead_scores(const fb_trie_t* trie, int32_t n_max, const int32_t* n_dev,
                                   const int32_t* rows, const int32_t* trie_state,
                                   const int32_t* hist_slot, const double* g_pool,
                                   int64_t g_stride, const double* hist_eos,
                                   const double* ext_eos, int32_t space_id, int32_t eos_id,
                                   double oov_penalty, double score_floor, double* out,
                                   int64_t out_stride, unsigned long long* floored,
                                   void* stream) {
  FB_CHECK_ARG(trie && trie->row_ptr && trie->info, "trie is null");
  FB_CHECK_ARG(n_max >= 0, "negative row count");
  FB_CHECK_ARG(out_stride >= trie->alphabet, "out stride smaller than the alphabet");
  FB_CHECK_ARG(hist_eos || ext_eos, "need hist_eos or ext_eos");
  if (n_max == 0) return FB_OK;
  constexpr int W = 8;
  const int blocks = std::min((n_max + W - 1) / W, kNumSMs * 16);
  const size_t sm = sizeof(double) * W * trie->alphabet;
  launch_pdl(lookahead_scores_kernel<W>, dim3(blocks), dim3(W * 32), sm, (cudaStream_t)stream,
      *trie, n_max, n_dev, rows, trie_state, hist_slot, g_pool, g_stride, hist_eos, ext_eos,
      space_id, eos_id, oov_penalty, score_floor, out, out_stride, floored);
  count_launch();
  return check_launch("lookahead_scores");
}

extern "C" int fb_multilevel_rows(const fb_trie_t* trie, int32_t n, const int32_t* states,
                                  const int32_t* slots, const double* dist_pool,
                                  int64_t d_stride, const double* accum, int32_t space_id,
                                  int32_t eos_id, double oov_factor, double score_floor,
                                  double* rows, int64_t r_stride, void* stream) {
  FB_CHECK_ARG(trie && trie->info && states && slots && dist_pool && accum && rows,
               "null multilevel arguments");
  if (n <= 0) return FB_OK;
  multilevel_rows_kernel<<<std::min((n + 255) / 256, kNumSMs * 8), 256, 0, (cudaStream_t)stream>>>(
      *trie, n, states, slots, dist_pool, d_stride, accum, space_id, eos_id, oov_factor,
      score_floor, rows, r_stride);
  count_launch();
  return check_launch("multilevel_rows");
}

extern "C" int fb_multilevel_advance(const fb_trie_t* trie, int32_t n, const int32_t* states_in,
                                     const double* accum_in, const int32_t* tokens,
                                     const double* char_rows, int64_t c_stride, int32_t space_id,
                                     int32_t eos_id, int32_t pad_id, int32_t* states_out,
                                     double* accum_out, int32_t* boundary_rank,
                                     unsigned long long* empty_words, void* stream) {
  FB_CHECK_ARG(trie && trie->row_ptr && states_in && accum_in && tokens && char_rows &&
                   states_out && accum_out && boundary_rank && empty_words,
               "null multilevel arguments");
  if (n <= 0) return FB_OK;
  multilevel_advance_kernel<<<std::min((n + 255) / 256, kNumSMs * 8), 256, 0,
                              (cudaStream_t)stream>>>(
      *trie, n, states_in, accum_in, tokens, char_rows, c_stride, space_id, eos_id, pad_id,
      states_out, accum_out, boundary_rank, empty_words);
  count_launch();
  return check_launch("multilevel_advance");
}

extern "C" int fb_trie_advance(const fb_trie_t* trie, int32_t n_max, const int32_t* n_dev,
                               const int32_t* rows, const int32_t* parent,
                               const int32_t* state_in, const int32_t* hist_in,
                               const int32_t* tokens, int32_t space_id, int32_t eos_id,
                               int32_t pad_id, int32_t* state_out, int32_t* hist_out,
                               int32_t* boundary_rank, void* stream) {
  FB_CHECK_ARG(trie && trie->row_ptr, "trie is null");
  if (n_max <= 0) return FB_OK;
  const int threads = 256;
  const int blocks = std::min((n_max + threads - 1) / threads, kNumSMs * 8);
  launch_pdl(trie_advance_kernel, dim3(blocks), dim3(threads), 0, (cudaStream_t)stream,
      *trie, n_max, n_dev, rows, parent, state_in, hist_in, tokens, space_id, eos_id, pad_id,
      state_out, hist_out, boundary_rank);
  count_launch();
  return check_launch("trie_advance");
}

extern "C" int fb_cumsum_rows(int32_t m, const double* probs, int64_t p_stride, int32_t vw,
                              const int32_t* slots, double* g_pool, int64_t g_stride,
                              void* stream) {
  FB_CHECK_ARG(vw > 0 && p_stride >= vw && g_stride >= vw, "bad cumsum sizes");
  if (m <= 0) return FB_OK;
  const int blocks = std::min(m, kNumSMs * 4);
  row_scan_kernel<false><<<blocks, kScanThreads, 0, (cudaStream_t)stream>>>(
      m, nullptr, probs, p_stride, nullptr, vw, vw, slots, g_pool, g_stride, nullptr);
  count_launch();
  return check_launch("cumsum_rows");
}

extern "C" int fb_logits_to_g(int32_t m_max, const int32_t* m_dev, const float* logits,
                              int64_t l_stride, const int32_t* src_rows, int32_t vw,
                              int32_t v_out, const int32_t* slots, double* g_pool,
                              int64_t g_stride, double* eos_out, void* stream) {
  FB_CHECK_ARG(vw > 0 && v_out > vw && l_stride >= v_out, "bad logits sizes");
  FB_CHECK_ARG(!g_pool || g_stride >= vw, "bad g stride");
  if (m_max <= 0) return FB_OK;
  const int blocks = std::min(m_max, kNumSMs * 4);
  row_scan_kernel<true><<<blocks, kScanThreads, 0, (cudaStream_t)stream>>>(
      m_max, m_dev, logits, l_stride, src_rows, vw, v_out, slots, g_pool, g_stride, eos_out);
  count_launch();
  return check_launch("logits_to_g");
}

extern "C" int fb_gather_rows(int32_t n, const int32_t* idx, const void* src, void* dst,
                              int64_t row_bytes, void* stream) {
  FB_CHECK_ARG(row_bytes > 0, "bad row size");
  if (n <= 0) return FB_OK;
  const int blocks = std::min(n, kNumSMs * 8);
  gather_rows_kernel<<<blocks, 128, 0, (cudaStream_t)stream>>>(
      n, idx, (const char*)src, (char*)dst, row_bytes);
  count_launch();
  return check_launch("gather_rows");
}

extern "C" int fb_stats_to_g(int32_t m_max, const int32_t* m_dev, const float* logits,
                             int64_t l_stride, const float* row_stats, int32_t n_out,
                             const int32_t* src_rows, int32_t vw, const int32_t* slots,
                             double* g_pool, int64_t g_stride, double* eos_out, double* seg_ws,
                             double* stat_out, const double* stat_in, double* fus,
                             int64_t fus_stride, int32_t fus_eos, void* stream) {
  FB_CHECK_ARG(logits && row_stats && vw > 0 && n_out > vw, "bad stats_to_g arguments");
  FB_CHECK_ARG(!fus || (!stat_in && fus_eos >= 0 && fus_stride > fus_eos),
               "fusion <eos> update needs the statistics pass and a valid column");
  FB_CHECK_ARG(!g_pool || (seg_ws && g_stride >= vw), "g rows need seg_ws and g_stride");
  FB_CHECK_ARG(!stat_in || g_pool, "stat_in only feeds the g-row passes");
  if (m_max <= 0) return FB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int ntiles = (n_out + 63) / 64;       // GEMM epilogue statistics granule
  const int nseg = (vw + kSegCols - 1) / kSegCols;
  const float4* st = reinterpret_cast<const float4*>(row_stats);
  // seg_ws layout: [m_max][nseg] segment sums, then [m_max] M_w
  double* norm = g_pool ? seg_ws + (int64_t)m_max * nseg : nullptr;
  int rc = 0;
  // the segment sums come with the row normaliser (one CTA per row) unless
  // the statistics are reused from an earlier pass (stat_in)
  const bool fused = g_pool && !stat_in && nseg <= kRnMaxSeg &&
                     (l_stride % 8) == 0 && ((uintptr_t)logits % 32) == 0;
  if (!stat_in) {
#ifndef FB_ROWS_GRID
#define FB_ROWS_GRID (kNumSMs * 2)
#endif
    launch_pdl(row_norm_kernel, dim3(std::min(m_max, FB_ROWS_GRID)), dim3(kRnThreads), 0, s,
        m_max, m_dev, logits, l_stride, st, ntiles, src_rows, vw, slots, eos_out, norm, stat_out,
        fused ? seg_ws : nullptr, nseg, fus, fus_stride, fus_eos);
    count_launch();
    rc = check_launch("row_norm");
  }
  if (rc || !g_pool) return rc;
#ifndef FB_SEG_ROWS_GRID
#define FB_SEG_ROWS_GRID 64
#endif
  // row CTAs per segment column (rows are grid-strided): few enough that the
  // usually-empty late-event launch is cheap
  const int gx = std::min(m_max, FB_SEG_ROWS_GRID);
  if (!fused) {
    launch_pdl(seg_sum_kernel, dim3(gx, nseg), dim3(kScanThreads), 0, s, m_max, m_dev, logits,
               l_stride, src_rows, vw, seg_ws, nseg, norm, stat_in, slots, eos_out);
    count_launch();
    rc = check_launch("seg_sum");
    if (rc) return rc;
  }
  launch_pdl(seg_scan_kernel, dim3(gx, nseg), dim3(kScanThreads), 0, s,
      m_max, m_dev, logits, l_stride, src_rows, vw, slots, seg_ws, nseg, norm, g_pool, g_stride,
      stat_in);
  count_launch();
  return check_launch("seg_scan");
}
