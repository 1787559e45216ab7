// TEST-ONLY fp32 SIMT GEMM (not part of the product library): the tcgen05
// GEMM's epilogues (bias / LSTM cell / residual / row scatter) over exact fp32
// products, used by tests/test_gpu_gemm.py and scripts/gemm_accuracy.py as an
// independent device cross-check.  Built into tests/libfb_testkit.so.
// 128x128x16 tile, 8x8 per thread.
#include <string>

#include "common.cuh"

namespace fbt {

using fb::row_count;
static thread_local std::string g_err;

constexpr int BM = 128, BN = 128, BK = 16, TPB = 256;

__device__ __forceinline__ float sigm(float x) { return 1.0f / (1.0f + expf(-x)); }

struct CellCtx {
  int hidden;
  const int32_t* rows;
  const int32_t* parent;
  const float* c_in; int64_t ld_cin;
  float* c_out; int64_t ld_cout;
  float* h_out; int64_t ld_h;
  const float* h_res; int64_t ld_res;
};

// Apply the LSTM cell to one (row, unit) with its 4 interleaved gate values.
__device__ __forceinline__ void lstm_cell(const fb_gemm_t& g, int m, int unit, float gi, float gf,
                                          float gg, float go) {
  const int slot = g.rows ? g.rows[m] : m;
  const int p = g.parent ? g.parent[slot] : slot;
  const float cp = g.c_in ? g.c_in[(int64_t)p * g.ld_cin + unit] : 0.0f;
  const float c = sigm(gf) * cp + sigm(gi) * tanhf(gg);
  float h = sigm(go) * tanhf(c);
  if (g.h_res) h += g.h_res[(int64_t)slot * g.ld_res + unit];
  g.c_out[(int64_t)slot * g.ld_cout + unit] = c;
  g.h_out[(int64_t)slot * g.ld_h + unit] = h;
}

__global__ void __launch_bounds__(TPB)
gemm_simt_kernel(fb_gemm_t g) {
  const int M = row_count(g.m_max, g.m_dev);
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= M) return;
  __shared__ float As[BK][BM + 4];
  __shared__ float Ws[BK][BN + 4];
  const float* A = reinterpret_cast<const float*>(g.a);
  const float* W = reinterpret_cast<const float*>(g.w);
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  // loader mapping: 128 rows x 16 k = 2048 floats = 512 float4; 2 per thread
  const int lr = tid >> 2;          // 0..63
  const int lk = (tid & 3) * 4;     // 0,4,8,12
  for (int k0 = 0; k0 < g.k; k0 += BK) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = lr + h * 64;
      const int am = min(m0 + r, M - 1);
      const float4 av = *reinterpret_cast<const float4*>(A + (int64_t)am * g.lda + k0 + lk);
      As[lk + 0][r] = av.x; As[lk + 1][r] = av.y; As[lk + 2][r] = av.z; As[lk + 3][r] = av.w;
      const int wn = min(n0 + r, g.n - 1);
      const float4 wv = *reinterpret_cast<const float4*>(W + (int64_t)wn * g.ldw + k0 + lk);
      Ws[lk + 0][r] = wv.x; Ws[lk + 1][r] = wv.y; Ws[lk + 2][r] = wv.z; Ws[lk + 3][r] = wv.w;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[8], b[8];
      const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][ty * 4 + 64]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Ws[kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Ws[kk][tx * 4 + 64]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
      b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + ty * 4 + (i & 3) + (i >> 2) * 64;
    if (m >= M) continue;
#pragma unroll
    for (int hj = 0; hj < 2; ++hj) {
      const int nb = n0 + tx * 4 + hj * 64;
      if (nb >= g.n) continue;
      float v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        v[q] = acc[i][hj * 4 + q];
        if (g.bias && nb + q < g.n) v[q] += g.bias[nb + q];
        if (g.addend && nb + q < g.n) v[q] += g.addend[(int64_t)m * g.ld_add + nb + q];
      }
      if (g.mode == 1) {
        lstm_cell(g, m, nb >> 2, v[0], v[1], v[2], v[3]);
      } else {
        const int orow = g.rows ? g.rows[m] : m;
        float* c = g.c + (int64_t)orow * g.ldc;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (nb + q < g.n) c[nb + q] = v[q];
      }
    }
  }
}

}  // namespace fbt

using namespace fbt;

#undef FB_CHECK_ARG
#define FB_CHECK_ARG(cond, msg)   \
  do {                             \
    if (!(cond)) {                 \
      g_err = msg;                 \
      return FB_ERR_VALUE;         \
    }                              \
  } while (0)

extern "C" const char* fbt_last_error(void) { return g_err.c_str(); }

extern "C" int fbt_gemm_simt(const fb_gemm_t* g, void* stream) {
  FB_CHECK_ARG(g && g->a && g->w, "null GEMM operands");
  FB_CHECK_ARG(g->k % BK == 0, "GEMM k must be a multiple of 16 (pad the operands)");
  FB_CHECK_ARG(g->lda % 4 == 0 && g->ldw % 4 == 0, "GEMM leading dims must be multiples of 4");
  FB_CHECK_ARG(g->mode == 0 || g->mode == 1, "unknown GEMM epilogue");
  FB_CHECK_ARG(g->mode != 1 || (g->n == 4 * g->hidden && g->h_out && g->c_out),
               "LSTM epilogue needs n == 4*hidden and state outputs");
  FB_CHECK_ARG(g->mode != 0 || g->c, "GEMM output is null");
  if (g->m_max <= 0) return FB_OK;
  dim3 grid((g->n + BN - 1) / BN, (g->m_max + BM - 1) / BM);
  gemm_simt_kernel<<<grid, TPB, 0, (cudaStream_t)stream>>>(*g);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_err = std::string("gemm_simt: ") + cudaGetErrorString(e);
    return FB_ERR_CUDA;
  }
  return FB_OK;
}
