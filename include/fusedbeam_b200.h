/*
 * fusedbeam_b200 -- C ABI of the B200 (sm_100a) kernels behind the
 * reference's decoder / look-ahead-fusion plugin API.
 *
 * Conventions
 *  - Every entry point returns an int status (FB_OK = 0) and never throws;
 *    fb_last_error() gives a thread-local message for the last failure.
 *  - All array arguments are DEVICE pointers owned by the caller (the Python
 *    host allocates them with torch); sizes are plain integers.  `stream` is a
 *    cudaStream_t passed as void*.  No entry point allocates or synchronises.
 *  - Optional "device count" arguments (`*_dev`) let a CUDA graph replay a
 *    launch whose row count is only known on the device: the grid is sized
 *    for the host maximum and blocks past the device count exit at once.
 *
 * Reference interfaces each group replaces are cited per function
 * (paths relative to /root/reference/pkg/src/fusedbeam/).
 */
#ifndef FUSEDBEAM_B200_H
#define FUSEDBEAM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  FB_OK = 0,
  FB_ERR_VALUE = 1,   /* bad argument / shape      -> ValueError       */
  FB_ERR_CONFIG = 2,  /* unusable configuration    -> ConfigError      */
  FB_ERR_CUDA = 3,    /* CUDA launch/runtime error -> RuntimeError     */
  FB_ERR_FORMAT = 4,  /* malformed file / input    -> FormatError      */
  FB_ERR_IO = 5       /* open / truncated read     -> OSError          */
};

const char* fb_last_error(void);
int fb_abi_version(void);
/* Number of kernel launches issued through this library by the calling
 * process (for bench.py's gpu_launches claim); reset with fb_launch_reset. */
unsigned long long fb_launch_count(void);
void fb_launch_reset(void);

/* ---- prefix-tree automaton, CSR packed (lexicon_trie.py:47-129) ---------- */
typedef struct {
  const int32_t* row_ptr;    /* [S+1] edge offsets per state                 */
  const int32_t* edge_label; /* [E]   token id, ascending within a state     */
  const int32_t* edge_child; /* [E]   child state                            */
  const int32_t* info;       /* [S*4] {ub, lb, rank (-1 if not final), 0}   */
  int32_t num_states;
  int32_t num_words;
  int32_t alphabet;          /* == len(token_dict)                          */
} fb_trie_t;

/* LookaheadFusion.char_scores (fusion.py:118-185), Eq. 4 of PAPER.md.
 * Row r = rows ? rows[i] : i for i < (n_dev ? *n_dev : n_max).
 *   trie_state[r] >= 0 (OOV_STATE = -2 scores the penalty everywhere),
 *   g row = g_pool + hist_slot[r]*g_stride (cumulative word mass, fp64),
 *   LM eos term: state 0 -> hist_eos[hist_slot[r]] (or ext_eos[r] when
 *   hist_eos is NULL); final state -> word_end + ext_eos[r].
 * Writes out[r*out_stride + c] for all c < alphabet (fp64, natural log) and
 * adds the number of floored scores to *floored (may be NULL). */
int fb_lookahead_scores(const fb_trie_t* trie, int32_t n_max, const int32_t* n_dev,
                        const int32_t* rows, const int32_t* trie_state,
                        const int32_t* hist_slot, const double* g_pool, int64_t g_stride,
                        const double* hist_eos, const double* ext_eos,
                        int32_t space_id, int32_t eos_id, double oov_penalty,
                        double score_floor, double* out, int64_t out_stride,
                        unsigned long long* floored, void* stream);

/* Trie half of LookaheadFusion.advance (fusion.py:187-207): for row r with
 * parent p = parent ? parent[r] : r:
 *   state_out[r] = child(state_in[p], tok) for in-word tokens (OOV_STATE when
 *   missing), 0 for <space>, state_in[p] for <eos>/<pad>;
 *   boundary_rank[r] = rank of the closed word (final state), -1 (<unk>) or
 *   -2 (no boundary).  hist_out[r] = hist_in[p] when both are non-NULL. */
int fb_trie_advance(const fb_trie_t* trie, int32_t n_max, const int32_t* n_dev,
                    const int32_t* rows, const int32_t* parent, const int32_t* state_in,
                    const int32_t* hist_in, const int32_t* tokens, int32_t space_id,
                    int32_t eos_id, int32_t pad_id, int32_t* state_out, int32_t* hist_out,
                    int32_t* boundary_rank, void* stream);

/* cumsum_distribution (fusion.py:40-42, :223): g_pool[slots[m]] = running
 * fp64 sum of probs[m, :vw]. */
int fb_cumsum_rows(int32_t m, const double* probs, int64_t p_stride, int32_t vw,
                   const int32_t* slots, double* g_pool, int64_t g_stride, void* stream);

/* Word-LM logits -> look-ahead mass (word_lm.py:169-179 for an LSTM LM).
 * For row i < m: logits row src_rows ? src_rows[i] : i, destination
 * d = slots ? slots[i] : i.  If g_pool: g_pool[d] = cumsum(softmax(logits[:vw]))
 * in fp64; if eos_out: eos_out[d] = logits[vw] - logsumexp(logits[:v_out]). */
int fb_logits_to_g(int32_t m_max, const int32_t* m_dev, const float* logits,
                   int64_t l_stride, const int32_t* src_rows, int32_t vw, int32_t v_out,
                   const int32_t* slots, double* g_pool, int64_t g_stride, double* eos_out,
                   void* stream);

/* Same quantities using the LM-output GEMM's per-tile statistics
 * (fb_gemm_t.row_stats): eos_out[d] = logits[vw] - logsumexp(all outputs)
 * without another pass over the logits; if g_pool, g_pool[d] =
 * cumsum(softmax over the vw words) in fp64, segment-parallel over
 * (rows x 4096-column segments) with exact fp64 segment offsets (two passes;
 * seg_ws: scratch of m_max * (ceil(vw/4096) + 2) doubles).  Row i < *m_dev reads
 * logits/stats row src_rows[i]; d = slots ? slots[i] : i.
 * stat_out (optional): {M_w, logsumexp} of row i at stat_out[2i], [2i+1].
 * stat_in (optional): those pairs from an earlier call, indexed by the source
 * row -- the statistics pass is skipped (the word-boundary rows reuse what the
 * speculative-event pass computed).
 * fus (optional, with the statistics pass): fus[d * fus_stride + fus_eos] +=
 * log P(</s>) of row i, as fb_eos_fixup does (fused into the same launch). */
int fb_stats_to_g(int32_t m_max, const int32_t* m_dev, const float* logits, int64_t l_stride,
                  const float* row_stats, int32_t n_out, const int32_t* src_rows, int32_t vw,
                  const int32_t* slots, double* g_pool, int64_t g_stride, double* eos_out,
                  double* seg_ws, double* stat_out, const double* stat_in, double* fus,
                  int64_t fus_stride, int32_t fus_eos, void* stream);

/* norm_out[d] = log(sum_{j != skip_col} exp(logits[row][j])) in fp64 for the
 * first *m_dev (or m_max) rows; row = d = rows ? rows[i] : i.  skip_col < 0:
 * every column.  (The log-normaliser of a token LM row, <pad> excluded.) */
int fb_row_logsumexp(int32_t m_max, const int32_t* m_dev, const int32_t* rows,
                     const float* logits, int64_t l_stride, int32_t n_cols, int32_t skip_col,
                     double* norm_out, void* stream);

/* ---- beam search step (decoder.py:339-480) ------------------------------ */
typedef struct {
  int32_t beam, vocab, pad_id, eos_id;
  int32_t cov_mode;            /* 0 off, 1 original (Eq.5), 2 improved (Eq.6) */
  int32_t gate_on;             /* EOS threshold (Eq.7) on/off               */
  int32_t early_stop;          /* fusion is None or nonpositive_scores       */
  int32_t has_fusion;
  int32_t am_f32;              /* am rows are fp32 (else fp64)               */
  int32_t max_tokens;          /* token row capacity (>= max_len + 1)        */
  int32_t t_max;               /* attention accumulator row capacity         */
  int32_t pad0;
  double lm_weight, cov_weight, tau1, tau2, cov_margin, gamma;
} fb_search_cfg_t;

typedef struct {
  /* per utterance [B] */
  int32_t* active;
  int32_t* n_live;
  int32_t* steps;
  const int32_t* max_len;
  const int32_t* t_enc;
  /* per slot [B*beam]: entering-step values, ping-pong pairs (in -> out) */
  const double* base_in;  double* base_out;
  const double* total_in; double* total_out;
  const int32_t* tok_in;  int32_t* tok_out;      /* [B*beam][max_tokens] */
  int32_t* parent;        /* [B*beam] out: parent slot of the new row      */
  int32_t* last_tok;      /* [B*beam] out: chosen token of the new row     */
  /* per row accumulated attention AFTER this step (accum + attn), and its
   * coverage -- produced by fb_attend_coverage or the attention kernel   */
  const double* acc_post; /* [B*beam][t_max] */
  const double* cov_post; /* [B*beam]        */
  /* finished pool [B][2*beam] */
  int32_t* fin_valid; double* fin_total; int32_t* fin_len;
  int32_t* fin_tokens;    /* [B][2*beam][max_tokens] */
  double* fin_acc;        /* [B][2*beam][t_max]      */
  /* results [B] (written when an utterance terminates) */
  int32_t* res_len; double* res_score; int32_t* res_finished; int32_t* res_steps;
  int32_t* res_tokens;    /* [B][max_tokens] */
  double* res_acc;        /* [B][t_max]      */
  /* compact list of the rows that enter the NEXT step (active utterances) */
  int32_t* next_rows; int32_t* next_count;
  /* large vocabularies (beam*vocab too big for one CTA): workspace [B*beam][beam]
   * for the exact two-stage selection (per-row top-beam, then the beam cut
   * over the survivors); NULL = single-stage only */
  double* cand_score_ws; int32_t* cand_flat_ws;
  int32_t force_two_stage;     /* test knobs: bit 0 two-stage selection even when one
                                  CTA fits, bit 1 radix top-K at any candidate count */
  int32_t pad1;
  /* token-level LM fusion from raw logits (char_lm.py:23-33 rows computed on
   * the fly): when non-NULL, the fusion argument of fb_search_step is fp32
   * logits and the fused score is max(logit - fus_norm[slot], fus_floor) */
  const double* fus_norm; double fus_floor;
  /* optional [B*beam]: position of each slot in next_rows (written with it;
   * the attention context kernel stores the output GEMM's A there) */
  int32_t* next_row_pos;
  /* optional int32 arrival counter, zero (left zero): the last selection CTA
   * builds next_rows / next_count / next_row_pos itself (no separate launch) */
  int32_t* select_arrive;
} fb_search_state_t;

/* One lock-step selection over every active utterance: combine am + lm_weight
 * * fusion, pad -> -inf, EOS gate, token-major stable top-beam with the
 * reference tie-break, coverage bonus, finished-set cap, early stop and
 * result pick.  am/fusion rows are indexed by slot.  When beam*vocab exceeds
 * the one-CTA shared-memory budget and st->cand_*_ws are given, each live row
 * first keeps its own top-beam candidates (ordered score desc, token asc --
 * consistent with the token-major flat order), which provably contains the
 * utterance's top-beam. */
int fb_search_step(const fb_search_cfg_t* cfg, const fb_search_state_t* st,
                   int32_t num_utts, const void* am, int64_t am_stride,
                   const double* fusion, int64_t fusion_stride, void* stream);

/* accum_post[r] = accum_in[parent(r)] + attn[r] (fp64) and its coverage
 * (decoder.py:36-48 and :421-425); attn is fp32 or fp64 (attn_f32).  Rows with
 * t >= t_enc[row/beam] are left untouched. */
int fb_attend_coverage(const fb_search_cfg_t* cfg, int32_t n_max, const int32_t* n_dev,
                       const int32_t* rows, const int32_t* parent, const int32_t* t_enc,
                       const double* acc_in, const void* attn, int32_t attn_f32,
                       int64_t attn_stride, double* acc_out, double* cov_out, void* stream);

/* Initialise the per-utterance search state for a new batch (one live row per
 * utterance, decoder.py:350-359). */
int fb_search_init(const fb_search_cfg_t* cfg, const fb_search_state_t* st,
                   int32_t num_utts, void* stream);


/* ---- dense contractions (attention-LSTM decoder step, word-LM step) ------ */
/* C = A . W^T (+ bias) with a fused epilogue, on the tensor cores
 * (fb_gemm_tc below).  A = operand planes of the fp32 activations [m, k]
 * (compact rows, fb_operand_format), W [n, k] row-major in the operand format.
 *   mode 0: out row = rows ? rows[i] : i ;  c[out*ldc + j] = acc + bias[j]
 *   mode 1: LSTM cell.  n == 4*hidden with gate columns interleaved
 *           (column 4u+q, q = i,f,g,o); slot = rows ? rows[i] : i,
 *           p = parent ? parent[slot] : slot;
 *           gates += addend[i*ld_add + ..] (if addend);
 *           c = sig(f)*c_in[p] + sig(i)*tanh(g); h = sig(o)*tanh(c)
 *           (+ h_res[slot] if h_res);  c_out[slot], h_out[slot]. */
typedef struct {
  int32_t m_max;
  const int32_t* m_dev;
  int32_t n, k;
  const void* a; int64_t lda;
  const void* w; int64_t ldw;
  const float* bias;
  float* c; int64_t ldc;
  int32_t mode;
  int32_t hidden;
  const int32_t* rows;
  const int32_t* parent;
  const float* c_in; int64_t ld_cin;
  float* c_out; int64_t ld_cout;
  float* h_out; int64_t ld_h;
  const float* h_res; int64_t ld_res;
  const float* addend; int64_t ld_add;
  /* mode 1, optional: h also written as operand planes (fb_operand_format) at
   * [p*hs_plane_rows + slot][unit] -- the A operand of a following GEMM */
  void* h_split; int64_t hs_plane_rows; int64_t ld_hs;
  /* mode 0, optional: per (output row, 64-column block) softmax statistics
   * {max, sum exp(x-max)} over all columns and over columns < stats_vw,
   * float4 at row_stats[orow * ceil(n/64) + block] (forces 128-wide tiles) */
  float* row_stats; int32_t stats_vw;
  /* fb_gemm_tc: K blocks (64) per TMEM accumulation chunk, 0 = default (4).
   * 1 = most accurate: the tensor core's in-TMEM accumulation truncates, so
   * score-producing projections drain every 64-K chunk into fp32 registers. */
  int32_t kcb;
  /* h_split row: 0 = the output slot (rows[i]), 1 = the GEMM row i (the next
   * GEMM's A operand in the same row order) */
  int32_t hs_row_mode;
  /* fb_gemm_tc, optional stream-K: when the (device-side) tile count is
   * below the SM count, every SM takes an equal share of the tile x K-block
   * space; a tile split over several CTAs is summed in K order by its last
   * arriving CTA (deterministic) before the epilogue.  splitk_ws: fp32
   * [2 * 148 * 128 * 128] partial tiles, splitk_cnt: uint32 [148] zeroed
   * arrival counters (left zeroed).  One workspace per stream: concurrent
   * GEMMs must not share it. */
  float* splitk_ws;
  uint32_t* splitk_cnt;
  /* mode 0: store exp(2 x) instead of x (the attention query, see
   * fb_attention_step q_is_exp) */
  int32_t out_exp2;
  /* mode 0, n <= 64: store the row log-softmax over the n columns instead of
   * the logits (same arithmetic as fb_log_softmax_rows) */
  int32_t out_logsoftmax;
  /* accumulator scale applied in the epilogue: 1 / (activation scale x
   * weight scale) of the operand format (fb_operand_format); 0 means
   * 1 / activation scale (weights stored unscaled) */
  float acc_scale;
  int32_t pad_fmt;
} fb_gemm_t;

/* Tensor-core operand format of this build: planes per fp32 activation
 * (2: fp16 hi/lo of x * act_scale; 3: bf16 hi/mid/lo), is_fp16, act_scale.
 * Weight operands are fp16 times a power of two per matrix (fp16 builds) or
 * bf16.  Writers of A planes (fb_pack_rows out_mode 1, the LSTM epilogues'
 * h_split) use this format. */
int fb_operand_format(int32_t* planes, int32_t* is_fp16, float* act_scale);

/* 5th-gen tensor cores (tcgen05 + TMEM + TMA): A is
 * a_planes operand planes of [a_plane_rows, lda] (the fp32 activation split
 * by fb_pack_rows out_mode 1), W [n, ldw] in the operand format; fp32
 * accumulation in TMEM.  k % 64 == 0, lda/ldw % 8 == 0. */
int fb_gemm_tc(const fb_gemm_t* g, int32_t a_planes, int64_t a_plane_rows, void* stream);

/* Encoder LSTM recurrence for one direction: for t < steps,
 * gates = xp[:, t] + acc_scale h_{t-1} W_hh^T (tensor cores, W_hh [4H, k] in
 * the operand format), cell epilogue, h_t -> y[:, t] and, split into operand
 * planes, into rec[(t+1)%2] ([2][planes][batch][k], rec[0] zero on entry); the cell state
 * lives in registers (zero at t = 0).
 * Row b of step t: xp + t*step_xp + b*ld_xp, y + t*step_y + b*ld_y (time-major
 * layouts -- step_* = batch * row width -- keep each step's rows contiguous).
 * Persistent cooperative launches: one per block of rows whose grid fits the
 * device (SM count and occupancy read at run time; rows never interact, so a
 * batch too large for one co-resident grid runs as several): the CTAs of each
 * 128-row tile loop over t behind a barrier on their own counter in sync_ws
 * (32 * ceil(batch/128) uint32: one 128-byte line per tile, reset here).
 * W_hh stays in shared memory.
 * t_rev (optional, [batch] int32): the backward direction -- step t of row b
 * reads xp and writes y at frame t_rev[b] - 1 - t (t < t_rev[b]), so a
 * length-padded batch needs no reversed copies of its inputs or outputs. */
int fb_lstm_recurrence(int32_t steps, int32_t batch, int32_t hidden, const void* w_hh,
                       int32_t k, const float* xp, int64_t ld_xp, int64_t step_xp, float* y,
                       int64_t ld_y, int64_t step_y, void* rec, uint32_t* sync_ws,
                       float acc_scale, const int32_t* t_rev, void* stream);

/* Row gather-concatenate into a GEMM A operand:
 *   out[i, :] = [seg0 | seg1 | ... | zero pad up to k_pad], i < m.
 * Segment source row: mode 0 -> i, 1 -> slot = rows[i], 2 -> parent[slot],
 * 3 -> token id tokens[slot] (negative -> tok_default) for embeddings,
 * 4 -> rank from ranks[i] (negative -> tok_default), 5 -> skip: the
 * segment's columns are left untouched (another kernel writes them, e.g. a
 * GEMM epilogue's h_split). */
typedef struct {
  const float* src; int64_t ld; int32_t width; int32_t mode;
} fb_seg_t;
typedef struct {
  fb_seg_t seg[4];
  int32_t nseg;
  int32_t k_pad;
  int32_t tok_default;
  int32_t out_mode;      /* 0: fp32 rows; 1: operand planes (fb_operand_format) */
  int64_t plane_rows;    /* out_mode 1: rows per plane ([3][plane_rows][ld])  */
} fb_pack_t;

int fb_pack_rows(const fb_pack_t* p, int32_t m_max, const int32_t* m_dev, const int32_t* rows,
                 const int32_t* parent, const int32_t* tokens, const int32_t* ranks,
                 float* out, int64_t ld_out, void* stream);

/* Row log-softmax of x[slot, :n] into out[slot, :n] (slot = rows[i]). */
int fb_log_softmax_rows(int32_t m_max, const int32_t* m_dev, const int32_t* rows,
                        const float* x, int64_t ldx, int32_t n, float* out, int64_t ldo,
                        void* stream);

/* Bahdanau attention step for every active utterance:
 * e[r,t] = v . tanh(K[u,t] + q[r]); a = softmax_t(e) over t < t_enc[u];
 * `keys` holds E_K^T = exp(2 K) per utterance as [num_utts][att_dim][t_max]
 * (fb_keys_exp2t), so tanh(k+q) = 1 - 2/(1 + E_k E_q);
 * ctx[r] = sum_t a[r,t] enc[u,t]; acc_out[r] = acc_in[parent[r]] + a[r]
 * (fp64) and its coverage (cfg->cov_mode).  Rows r = u*beam + i, i < n_live[u].
 * q is consumed in place: its live rows are overwritten with E_q = exp(2 q)
 * (q_is_exp != 0: q already holds E_q, e.g. from fb_gemm_t.out_exp2).
 * energy_ws: scratch [2][num_utts*beam][t_max] fp32 (the energies of the two
 * halves of the attention dims, summed in that order); plane 0 holds the
 * attention weights a[r, t] on return.  sync_ws: num_utts*ceil(beam/2) int32, zero on the
 * first call (the kernels leave it zeroed).  ctx_planes (optional): the context
 * is also stored in the operand format (fb_operand_format) at
 * ctx_planes + p*ctx_plane_stride + ctx_row_pos[r]*ctx_plane_ld, p < planes
 * (16-bit elements; the output GEMM's A from its column H on, see
 * fb_search_state_t.next_row_pos). */
/* Tiling of the following fb_attention_step launches (0 = default): frame
 * warps per energy CTA (2/4/8), rows per energy CTA (even, <= 16), encoder
 * column quads per context CTA.  Finer tiles pay off when few utterances are
 * live (the lock-step tail of a batch). */
int fb_set_attention_tiling(int32_t frames_warps, int32_t rows, int32_t quads);

int fb_attention_step(const fb_search_cfg_t* cfg, int32_t num_utts, const int32_t* active,
                      const int32_t* n_live, const int32_t* t_enc, const float* keys,
                      const float* enc, int32_t att_dim, int32_t ctx_dim, const float* v,
                      float* q, int64_t ldq, const int32_t* parent, const double* acc_in,
                      double* acc_out, double* cov_out, float* ctx_out, int64_t ld_ctx,
                      float* attn_out, int64_t ld_attn, float* energy_ws, int32_t* sync_ws,
                      int32_t q_is_exp, void* ctx_planes, int64_t ctx_plane_stride,
                      int64_t ctx_plane_ld, const int32_t* ctx_row_pos, void* stream);

/* y[i] = exp(2 x[i]) (attention keys -> E_K, once per batch). */
int fb_exp2x(int64_t n, const float* x, float* y, void* stream);

/* ekt[u][a][t] = exp(2 keys[u][t][a]) for u < num_utts, t < t_max, a < att_dim:
 * the attention keys in the layout fb_attention_step reads (out of place). */
int fb_keys_exp2t(int32_t num_utts, int32_t t_max, int32_t att_dim, const float* keys,
                  float* ekt, void* stream);

/* ---- word-LM bookkeeping for the fused engine ---------------------------- */
/* Speculative <eos> events (fusion.py:181-183): for every listed row whose
 * trie state is final: e = next event index; ev_row[e] = row, ev_rank[e] =
 * word rank, ev_slot[e] = hist_slot[row] (LM state to extend), row_ev[row] = e;
 * other rows get row_ev = -1.  *ev_count is reset first. */
int fb_spec_events(const fb_trie_t* trie, int32_t n_max, const int32_t* n_dev,
                   const int32_t* rows, const int32_t* trie_state, const int32_t* hist_slot,
                   int32_t* ev_row, int32_t* ev_rank, int32_t* ev_slot, int32_t* ev_count,
                   int32_t* row_ev, void* stream);

/* Pruned speculative <eos> events (exact): per active utterance, the eos
 * candidate of a row at a final trie state is bounded above by
 * total + am[eos] + lm_weight * word_end (log P(</s>) <= 0).  With T_K the
 * beam-th best of all other (exactly known) candidates, a row whose bound is
 * < T_K cannot be selected: its fusion eos entry is set to -inf and no LM
 * event is made.  Other final rows become events as in fb_spec_events.
 * `fusion` must hold word_end (not yet + log P(</s>)) in the eos column of
 * final rows (fb_lookahead_scores with ext_eos = 0).  Event numbering starts
 * at *ev_start (late events already queued) when ev_start is non-NULL. */
int fb_spec_select(const fb_search_cfg_t* cfg, const fb_search_state_t* st, int32_t num_utts,
                   const fb_trie_t* trie, const int32_t* trie_state, const int32_t* hist_slot,
                   const void* am, int64_t am_stride, double* fusion, int64_t fusion_stride,
                   int32_t* ev_row, int32_t* ev_rank, int32_t* ev_slot, int32_t* ev_count,
                   int32_t* row_ev, const int32_t* ev_start, void* stream);

/* fusion[ev_row[e], eos_id] += eos_lp[ev_row[e]] for e < *ev_count. */
int fb_eos_fixup(int32_t n_max, const int32_t* ev_count, const int32_t* ev_row,
                 const double* eos_lp, double* fusion, int64_t fusion_stride, int32_t eos_id,
                 void* stream);

/* Word-boundary plan after selection (fusion.py:206-223).  New rows
 * rows[i] (i < *n_dev) whose boundary_rank >= -1 closed a word: each gets a
 * fresh history slot (slots referenced by the rows that entered this step,
 * cur_rows/hist_cur, stay live), in row order; hist_next[row] = slot.
 * Rows whose parent ran a speculative LM event (row_ev[parent] >= 0) reuse it:
 * bnd_slot/bnd_src (event row) list, *bnd_count.  The others become late
 * events for the next step's LM batch: late_slot[k] = hist_cur[parent] (LM
 * input state), late_tok[k] = rank or -1 (<unk>), late_row[k] = late_sink_row,
 * late_dst[k] = slot, *late_count.  slot_mark: scratch of 2*num_slots int32. */
int fb_boundary_plan(int32_t n_max, const int32_t* n_dev, const int32_t* rows,
                     const int32_t* parent, const int32_t* boundary_rank,
                     const int32_t* row_ev, const int32_t* cur_rows, const int32_t* cur_count,
                     const int32_t* hist_cur, int32_t* hist_next, int32_t num_slots,
                     int32_t* slot_mark, int32_t* bnd_slot, int32_t* bnd_src,
                     int32_t* bnd_count, int32_t* late_slot, int32_t* late_tok,
                     int32_t* late_row, int32_t* late_dst, int32_t* late_count,
                     int32_t late_sink_row, void* stream);

/* Copy n rows of row_bytes: dst[dst_idx[i]] = src[src_idx[i]] (NULL = i). */
int fb_copy_rows(int32_t n_max, const int32_t* n_dev, const int32_t* src_idx,
                 const int32_t* dst_idx, const void* src, void* dst, int64_t row_bytes,
                 void* stream);

/* Row gather (the reorder of fusion.py:226-233 / an AcousticScorer): for r <
 * n: dst[r*row_bytes..] = src[idx[r]*row_bytes..]. */
int fb_gather_rows(int32_t n, const int32_t* idx, const void* src, void* dst,
                   int64_t row_bytes, void* stream);

/* ---- multilevel fusion (reference fusion.py:268-380) -------------------- */
/* rows[b][space_id], rows[b][eos_id] += the word-boundary adjustment of row b:
 * 0 for an empty word, log dist_pool[slots[b]][rank(state)] - accum[b] at a
 * final trie state (score_floor for zero probability), oov_factor otherwise. */
int fb_multilevel_rows(const fb_trie_t* trie, int32_t n, const int32_t* states,
                       const int32_t* slots, const double* dist_pool, int64_t d_stride,
                       const double* accum, int32_t space_id, int32_t eos_id,
                       double oov_factor, double score_floor, double* rows, int64_t r_stride,
                       void* stream);
/* Per-row state update for chosen tokens; char_rows = the unadjusted char-LM
 * rows of the previous states; boundary_rank[b] = word rank, -1 (<unk>) or -2
 * (no boundary); empty_words counts boundaries that close an empty word. */
int fb_multilevel_advance(const fb_trie_t* trie, int32_t n, const int32_t* states_in,
                          const double* accum_in, const int32_t* tokens,
                          const double* char_rows, int64_t c_stride, int32_t space_id,
                          int32_t eos_id, int32_t pad_id, int32_t* states_out,
                          double* accum_out, int32_t* boundary_rank,
                          unsigned long long* empty_words, void* stream);

/* ---- host-side data formats (no GPU; csrc/host_io.cu) -------------------- */
/* Kaldi binary ARK float32 matrix at `offset` (reference kaldi_io.py:82-130):
 * rows/cols out; the payload goes to dst when dst != NULL (dst_capacity floats,
 * e.g. pinned staging memory).  Reference messages: bad marker / token /
 * size byte / shape / non-finite -> FB_ERR_FORMAT, truncation -> FB_ERR_IO. */
int fb_ark_read_matrix(const char* ark_path, int64_t offset, float* dst, int64_t dst_capacity,
                       int32_t* rows, int32_t* cols);
/* n records on a host thread pool; record i -> dst + dst_offsets[i] (floats,
 * capacities[i]); dst == NULL queries every record's rows/cols.  On failure
 * the first failing record (input order) is reported. */
int fb_ark_read_batch(int32_t n, const char* const* ark_paths, const int64_t* offsets,
                      float* dst, const int64_t* dst_offsets, const int64_t* capacities,
                      int32_t* rows, int32_t* cols, int32_t threads);
/* Kaldi SCP index (reference kaldi_io.py:46-77; replaces read_scp's line
 * loop) over the file's bytes: per entry "utt_id\0ark_path\0" into out and
 * its offset into offsets.  Lines split like Python's text mode, fields like
 * str.strip/split(None, 1)/rpartition(':')/int().  FB_ERR_FORMAT: err[0] =
 * 1 field count | 2 missing ':offset' | 3 offset not an integer | 4 negative
 * offset | 5 duplicate id, err[1] = line, err[2] = first line of the
 * duplicate; out holds the offending text (out_len bytes). */
int fb_scp_parse(const char* text, int64_t len, char* out, int64_t out_cap, int64_t* out_len,
                 int64_t* offsets, int32_t* n_entries, int32_t* err);
/* Append one binary float32 record and its SCP line (reference
 * kaldi_io.py:129-150; replaces write_ark_matrix's writes); *offset = the
 * record's position after "utt_id ". */
int fb_ark_append_matrix(const char* ark_path, const char* scp_path, const char* utt_id,
                         const float* data, int32_t rows, int32_t cols, int64_t* offset);
/* n host memcpys (dsts[i] <- srcs[i], bytes[i]) on a thread pool: staging a
 * batch of feature matrices into one pinned buffer. */
int fb_host_copy_batch(int32_t n, const void* const* srcs, void* const* dsts,
                       const int64_t* bytes, int32_t threads);
/* PTA1 prefix-tree files (lexicon_trie.py:178-224): header, arrays, write. */
int fb_pta1_read_header(const char* path, int32_t* num_states, int32_t* num_words,
                        int32_t* max_out, int32_t* alphabet);
int fb_pta1_read(const char* path, int32_t* transitions, int32_t* edge_labels,
                 uint8_t* is_final, int32_t* word_index, int32_t* ub_index,
                 int32_t* lb_index);
int fb_pta1_write(const char* path, int32_t num_states, int32_t num_words, int32_t max_out,
                  int32_t alphabet, const int32_t* transitions, const int32_t* edge_labels,
                  const uint8_t* is_final, const int32_t* word_index, const int32_t* ub_index,
                  const int32_t* lb_index);
/* build_trie (lexicon_trie.py:227-276) over char-id sequences
 * chars[word_offsets[i] .. word_offsets[i+1]): sizes first, then the arrays in
 * the reference layout (transitions/edge_labels [S][max_out], -1 padded). */
int fb_trie_build_sizes(int32_t n_words, const int32_t* chars, const int64_t* word_offsets,
                        int32_t alphabet, int32_t* num_states, int32_t* max_out);
int fb_trie_build(int32_t n_words, const int32_t* chars, const int64_t* word_offsets,
                  int32_t alphabet, int32_t num_states, int32_t max_out, int32_t* transitions,
                  int32_t* edge_labels, uint8_t* is_final, int32_t* word_index,
                  int32_t* ub_index, int32_t* lb_index);

#ifdef __cplusplus
}
#endif
#endif /* FUSEDBEAM_B200_H */
