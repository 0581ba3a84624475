/*
 * tetris_oracle.c — CPU restatement of the TETRIS hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load this library,
 * and only as the checker (or the timed CPU baseline) — never as the product path.
 *
 * Every function restates the reference algorithm (paths relative to /root/reference/pkg/src/tetris_sched/):
 *   oracle_select            cumulative_products (selector.py:95-110) + select_tetris (selector.py:133-176):
 *                            a literal port of the heapq schedule (CPython heapify/_siftup/_siftdown) with the
 *                            _HeapItem key (-cum,row,depth) (selector.py:113-130), counting comparisons.
 *                            It is deliberately a different algorithm from the GPU's radix select.
 *   oracle_verify_matrix     apply_verification (sim_engine.py:374-404).
 *   oracle_sample            the sampling contract of include/tetris_b200.h (fixed fp64 hierarchy) that replaces
 *                            numpy's Generator.choice (accept_model.py:364,368); checked statistically and
 *                            per-draw against the numpy path by tests/test_oracle.py.
 *   oracle_verify_stochastic verify_token (accept_model.py:291-313) per position + first-rejection cascade
 *                            (sim_engine.py:388-403) + residual_distribution (accept_model.py:316-327) / bonus.
 *   oracle_verify_greedy     verify_token on one-hot distributions (accept_model.py:309-313) = argmax match.
 *   oracle_compact           credit min(acc+1, remaining) (sim_engine.py:467-471) + token gather.
 *   oracle_expected_accepted expected_accepted (selector.py:286-306).
 *   oracle_probs_from_logits_bf16  the logits contract of include/tetris_b200.h (bf16 logits + row lse -> fp32
 *                            probabilities with C fmaf()); no reference counterpart: the logits
 *                            steps are checked as the fp32 oracle applied to these probabilities.
 * Pinned against golden vectors produced by the reference itself: tests/golden/ (tests/golden/make_golden.py).
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off: every fp64 operation is one IEEE round-to-nearest op).
 */
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/tetris_b200.h"

#define LANE TETRIS_LANE_ELEMS
#define SEG TETRIS_SEG_ELEMS
#define WSEGS TETRIS_WARP_SEGS
#define CWARPS TETRIS_CHUNK_WARPS
#define CHUNK TETRIS_CHUNK_ELEMS
#define WELEMS (SEG * WSEGS)

/* ------------------------------------------------------------------------------------------------------------ */
/* selection: heapq port                                                                                          */
/* ------------------------------------------------------------------------------------------------------------ */
typedef struct {
  double cum;
  int32_t row, depth;
} item_t;

static int item_lt(const item_t* a, const item_t* b, int64_t* cmp) {
  ++*cmp;
  double na = -a->cum, nb = -b->cum;
  if (na != nb) return na < nb;
  if (a->row != b->row) return a->row < b->row;
  return a->depth < b->depth;
}

static void siftdown(item_t* h, int start, int pos, int64_t* cmp) {
  item_t nw = h[pos];
  while (pos > start) {
    int pp = (pos - 1) >> 1;
    item_t parent = h[pp];
    if (item_lt(&nw, &parent, cmp)) {
      h[pos] = parent;
      pos = pp;
      continue;
    }
    break;
  }
  h[pos] = nw;
}

static void siftup(item_t* h, int n, int pos, int64_t* cmp) {
  int start = pos;
  item_t nw = h[pos];
  int child = 2 * pos + 1;
  while (child < n) {
    int right = child + 1;
    if (right < n && !item_lt(&h[child], &h[right], cmp)) child = right;
    h[pos] = h[child];
    pos = child;
    child = 2 * pos + 1;
  }
  h[pos] = nw;
  siftdown(h, start, pos, cmp);
}

/* vals [B][k]; len may be NULL.  vals_are_cum=0: alpha rates -> cum by sequential product.  Returns 0, or 1 on a
 * bad argument (negative capacity, selector.py:145-146).  stats4 = extracts, inserts, peak_queue, comparisons. */
int oracle_select(const double* vals, const int32_t* len, int B, int k, int64_t C, int vals_are_cum,
                  int32_t* windows, double* cum_out, int64_t* stats4) {
  if (C < 0) return 1;
  double* cum = (double*)malloc(sizeof(double) * (size_t)(B > 0 ? B : 1) * (size_t)(k > 0 ? k : 1));
  for (int r = 0; r < B; ++r) {
    int L = len ? len[r] : k;
    double c = 1.0;
    for (int j = 0; j < L; ++j) {
      double v = vals[(int64_t)r * k + j];
      c = vals_are_cum ? v : c * v; /* selector.py:107 cum *= alpha */
      cum[(int64_t)r * k + j] = c;
      if (cum_out) cum_out[(int64_t)r * k + j] = c;
    }
    windows[r] = 0;
  }
  int64_t cmp = 0, extracts = 0, inserts = 0, peak = 0;
  if (C > 0) {
    item_t* heap = (item_t*)malloc(sizeof(item_t) * (size_t)(B > 0 ? B : 1));
    int n = 0;
    for (int r = 0; r < B; ++r) {
      int L = len ? len[r] : k;
      if (L > 0) {
        heap[n].cum = cum[(int64_t)r * k];
        heap[n].row = r;
        heap[n].depth = 1;
        ++n;
      }
    }
    for (int i = n / 2 - 1; i >= 0; --i) siftup(heap, n, i, &cmp);
    inserts = n;
    peak = n;
    while (n > 0 && extracts < C) {
      item_t last = heap[--n], item = last;
      if (n > 0) {
        item = heap[0];
        heap[0] = last;
        siftup(heap, n, 0, &cmp);
      }
      ++extracts;
      int r = item.row, j = item.depth;
      windows[r] = j;
      int L = len ? len[r] : k;
      if (j < L) {
        heap[n].cum = cum[(int64_t)r * k + j];
        heap[n].row = r;
        heap[n].depth = j + 1;
        ++n;
        siftdown(heap, 0, n - 1, &cmp);
        ++inserts;
        if (n > peak) peak = n;
      }
    }
    free(heap);
  }
  if (stats4) {
    stats4[0] = extracts;
    stats4[1] = inserts;
    stats4[2] = peak;
    stats4[3] = cmp;
  }
  free(cum);
  return 0;
}

double oracle_expected_accepted(const double* alpha, const int32_t* len, const int32_t* windows, int B, int k) {
  double value = 0.0;
  for (int r = 0; r < B; ++r) {
    double c = 1.0;
    for (int j = 0; j < windows[r]; ++j) {
      c *= alpha[(int64_t)r * k + j];
      value += c;
    }
  }
  (void)len;
  return value;
}

/* verify_token's rule (accept_model.py:309-313) on the two gathered masses. */
int oracle_verify_token(double s, double m, double u) { return (s <= m) || (u < m / s); }

void oracle_verify_matrix(const double* alpha, const int32_t* windows, const int32_t* win_off, const double* u,
                          int B, int k, int32_t* accepted) {
  for (int r = 0; r < B; ++r) {
    int count = 0;
    for (int j = 0; j < windows[r]; ++j) {
      if (u[win_off[r] + j] < alpha[(int64_t)r * k + j])
        ++count;
      else
        break;
    }
    accepted[r] = count;
  }
}

/* ------------------------------------------------------------------------------------------------------------ */
/* the sampling contract                                                                                          */
/* ------------------------------------------------------------------------------------------------------------ */
static int seq_find(const double* v, int n, double* T) {
  double P = 0.0;
  for (int i = 0; i < n; ++i) {
    double Pn = P + v[i];
    if (Pn > *T) {
      *T = *T - P;
      return i;
    }
    P = Pn;
  }
  int last = -1;
  for (int i = 0; i < n; ++i)
    if (v[i] > 0.0) last = i;
  *T = INFINITY;
  return last;
}

static double lane_sum(const double* w, int64_t e) {
  double o = 0.0;
  for (int i = 0; i < LANE; ++i) o = o + w[e + i];
  return o;
}

/* balanced binary tree over lanes [g, g+n) of the segment starting at element eb */
static double tree_sum(const double* w, int64_t eb, int g, int n) {
  if (n == 1) return lane_sum(w, eb + (int64_t)g * LANE);
  return tree_sum(w, eb, g, n / 2) + tree_sum(w, eb, g + n / 2, n / 2);
}

static double warp_sum(const double* w, int64_t e0, double* G) {
  double W = 0.0;
  for (int s = 0; s < WSEGS; ++s) {
    G[s] = tree_sum(w, e0 + (int64_t)s * SEG, 0, 32);
    W = W + G[s];
  }
  return W;
}

/* w: weights padded with zeros to nch*CHUNK.  Returns the sampled index (or -1 when mass == 0). */
static int sample_padded(const double* w, int V, double u, double* mass_out) {
  int nch = (V + CHUNK - 1) / CHUNK;
  double S[64], Wsum[64][CWARPS], G[WSEGS];
  double mass = 0.0;
  for (int c = 0; c < nch; ++c) {
    double Sc = 0.0;
    for (int ww = 0; ww < CWARPS; ++ww) {
      Wsum[c][ww] = warp_sum(w, (int64_t)c * CHUNK + (int64_t)ww * WELEMS, G);
      Sc = Sc + Wsum[c][ww];
    }
    S[c] = Sc;
    mass = mass + Sc;
  }
  if (mass_out) *mass_out = mass;
  if (!(mass > 0.0)) return -1;
  double T = u * mass;
  int c = seq_find(S, nch, &T);
  int ww = seq_find(Wsum[c], CWARPS, &T);
  int64_t e0 = (int64_t)c * CHUNK + (int64_t)ww * WELEMS;
  warp_sum(w, e0, G);
  int s = seq_find(G, WSEGS, &T);
  if (s < 0) return -1;
  int64_t eb = e0 + (int64_t)s * SEG;
  int g = 0;
  for (int t = 4; t >= 0; --t) {
    int n = 1 << t;
    double L = tree_sum(w, eb, g, n), R = tree_sum(w, eb, g + n, n);
    if (!(L > T || R == 0.0)) {
      T = T - L;
      g += n;
    }
  }
  int li = seq_find(w + eb + (int64_t)g * LANE, LANE, &T);
  if (li < 0) return -1;
  return (int)(eb + (int64_t)g * LANE + li);
}

static double* padded_buffer(int V) {
  int nch = (V + CHUNK - 1) / CHUNK;
  return (double*)calloc((size_t)nch * CHUNK, sizeof(double));
}

/* weights = max(0, p - q) (q != NULL) or max(0, p); fp64 inputs. */
int oracle_sample_f64(const double* p, const double* q, int V, double u, double* mass_out) {
  double* w = padded_buffer(V);
  for (int v = 0; v < V; ++v) {
    double x = q ? p[v] - q[v] : p[v];
    w[v] = x > 0.0 ? x : 0.0;
  }
  int r = sample_padded(w, V, u, mass_out);
  free(w);
  return r;
}

int oracle_sample_f32(const float* p, const float* q, int V, double u, double* mass_out) {
  double* w = padded_buffer(V);
  for (int v = 0; v < V; ++v) {
    double x = q ? (double)p[v] - (double)q[v] : (double)p[v];
    w[v] = x > 0.0 ? x : 0.0;
  }
  int r = sample_padded(w, V, u, mass_out);
  free(w);
  return r;
}

/* residual_distribution: out = max(0, pt - ps) / mass (hierarchical mass); returns 0 or 2 (degenerate). */
int oracle_residual_f64(const double* ps, const double* pt, int V, double* out, double* mass_out) {
  double mass;
  oracle_sample_f64(pt, ps, V, 0.0, &mass);
  if (mass_out) *mass_out = mass;
  if (!(mass > 0.0)) return 2;
  for (int v = 0; v < V; ++v) {
    double x = pt[v] - ps[v];
    out[v] = (x > 0.0 ? x : 0.0) / mass;
  }
  return 0;
}

/* ------------------------------------------------------------------------------------------------------------ */
/* a minimal parallel-for over requests (pthreads; dynamic schedule, one request per grab)                        */
/* ------------------------------------------------------------------------------------------------------------ */
typedef struct {
  void (*fn)(void*, int);
  void* ctx;
  int n;
  atomic_int next;
} pfor_t;

static void* pfor_worker(void* arg) {
  pfor_t* pf = (pfor_t*)arg;
  for (;;) {
    int i = atomic_fetch_add(&pf->next, 1);
    if (i >= pf->n) break;
    pf->fn(pf->ctx, i);
  }
  return NULL;
}

static void parallel_for(int n, int nthreads, void (*fn)(void*, int), void* ctx) {
  pfor_t pf;
  pf.fn = fn;
  pf.ctx = ctx;
  pf.n = n;
  atomic_init(&pf.next, 0);
  if (nthreads <= 1 || n <= 1) {
    pfor_worker(&pf);
    return;
  }
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  int started = 0;
  for (int t = 1; t < nthreads; ++t)
    if (pthread_create(&th[started], NULL, pfor_worker, &pf) == 0) ++started;
  pfor_worker(&pf);
  for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------------------------------------------------------------ */
/* batched verification                                                                                           */
/* ------------------------------------------------------------------------------------------------------------ */
static int verify_one_stochastic(const float* p, const float* q, const int32_t* d, int w, const double* u_acc,
                                 double u_res, int b, int k, int V, int32_t* out_tok, double* mass) {
  int a = w;
  for (int j = 0; j < w; ++j) {
    int t = d[(int64_t)b * k + j];
    int rej;
    if (t < 0 || t >= V) {
      rej = 1;
    } else {
      double s = (double)q[((int64_t)b * k + j) * V + t];
      double m = (double)p[((int64_t)b * (k + 1) + j) * V + t];
      rej = !(s <= m) && !(u_acc[j] < m / s); /* accept_model.py:311-313 */
    }
    if (rej) {
      a = j;
      break;
    }
  }
  if (a < w)
    *out_tok = oracle_sample_f32(p + ((int64_t)b * (k + 1) + a) * V, q + ((int64_t)b * k + a) * V, V, u_res, mass);
  else
    *out_tok = oracle_sample_f32(p + ((int64_t)b * (k + 1) + w) * V, NULL, V, u_res, mass);
  return a;
}

typedef struct {
  const float *p, *q;
  const int32_t *d, *windows, *win_off;
  const double *u_acc, *u_res;
  int k, V;
  int32_t *accepted, *out_tok;
  double* mass_out;
} stoch_ctx_t;

static void stoch_one(void* vctx, int b) {
  stoch_ctx_t* c = (stoch_ctx_t*)vctx;
  const double* ub = c->u_acc + (c->win_off ? (int64_t)c->win_off[b] : (int64_t)b * c->k);
  double mass = 0.0;
  c->accepted[b] =
      verify_one_stochastic(c->p, c->q, c->d, c->windows[b], ub, c->u_res[b], b, c->k, c->V, &c->out_tok[b], &mass);
  if (c->mass_out) c->mass_out[b] = mass;
}

/* win_off == NULL -> dense u_acc[b*k + j]; else packed u_acc[win_off[b] + j].  nthreads > 1: pthreads. */
void oracle_verify_stochastic_f32(const float* p, const float* q, const int32_t* d, const int32_t* windows,
                                  const int32_t* win_off, const double* u_acc, const double* u_res, int B, int k,
                                  int V, int32_t* accepted, int32_t* out_tok, double* mass_out, int nthreads) {
  stoch_ctx_t c = {p, q, d, windows, win_off, u_acc, u_res, k, V, accepted, out_tok, mass_out};
  parallel_for(B, nthreads, stoch_one, &c);
}

static int argmax_f32(const float* row, int V) {
  /* numpy.argmax: first NaN if any, else first maximal element */
  int bi = 0;
  float bv = row[0];
  if (isnan(bv)) return 0;
  for (int v = 1; v < V; ++v) {
    float x = row[v];
    if (isnan(x)) return v;
    if (x > bv) {
      bv = x;
      bi = v;
    }
  }
  return bi;
}

typedef struct {
  const float* p;
  const int32_t *d, *windows;
  int k, V;
  int32_t *accepted, *out_tok;
} greedy_ctx_t;

static void greedy_one(void* vctx, int b) {
  greedy_ctx_t* c = (greedy_ctx_t*)vctx;
  int w = c->windows[b], a = w, x = -1;
  for (int j = 0; j <= w; ++j) {
    int am = argmax_f32(c->p + ((int64_t)b * (c->k + 1) + j) * c->V, c->V);
    if (j == w || am != c->d[(int64_t)b * c->k + j]) {
      a = j;
      x = am;
      break;
    }
  }
  c->accepted[b] = a;
  c->out_tok[b] = x;
}

void oracle_verify_greedy_f32(const float* p, const int32_t* d, const int32_t* windows, int B, int k, int V,
                              int32_t* accepted, int32_t* out_tok, int nthreads) {
  greedy_ctx_t c = {p, d, windows, k, V, accepted, out_tok};
  parallel_for(B, nthreads, greedy_one, &c);
}

void oracle_compact(const int32_t* accepted, const int32_t* out_tok, const int32_t* d, const int32_t* cap, int B,
                    int k, int32_t* offsets, int32_t* tokens) {
  int64_t off = 0;
  for (int b = 0; b < B; ++b) {
    int a = accepted[b], n = a + 1;
    if (cap) n = n < (cap[b] > 0 ? cap[b] : 0) ? n : (cap[b] > 0 ? cap[b] : 0);
    offsets[b] = (int32_t)off;
    for (int i = 0; i < n; ++i) tokens[off + i] = i < a ? d[(int64_t)b * k + i] : out_tok[b];
    off += n;
  }
  offsets[B] = (int32_t)off;
}

/* ---- the logits contract (tetris_b200.h): prob(z, lse) with C99 fmaf (correctly rounded), fp32 RN ------------ */
typedef union {
  uint32_t u;
  float f;
} fbits;

static uint32_t bf16_round_up(uint32_t b) { return ((b & 0xffffu) && !(b >> 31)) ? (b >> 16) + 1u : b >> 16; }
static uint32_t bf16_round_down(uint32_t b) { return ((b & 0xffffu) && (b >> 31)) ? (b >> 16) + 1u : b >> 16; }

static float prob_from_logit(uint16_t z16, float lse) {
  fbits z, lo, hi, a, b, t, e, o;
  a.f = lse + TETRIS_EXP_LO;
  b.f = lse + TETRIS_EXP_HI;
  lo.u = bf16_round_up(a.u) << 16;
  hi.u = bf16_round_down(b.u) << 16;
  z.u = (uint32_t)z16 << 16;
  float zc = fminf(fmaxf(z.f, lo.f), hi.f); /* maxNum / minNum: a NaN logit takes the lower bound */
  const float x = zc + (-lse);
  t.f = fmaf(x, TETRIS_EXP_L2E, TETRIS_EXP_MAGIC);
  const float j = t.f + (-TETRIS_EXP_MAGIC);
  const float r = fmaf(j, -TETRIS_EXP_LN2, x);
  float p = fmaf(TETRIS_EXP_C5, r, TETRIS_EXP_C4);
  p = fmaf(p, r, TETRIS_EXP_C3);
  p = fmaf(p, r, TETRIS_EXP_C2);
  p = fmaf(p, r, TETRIS_EXP_C1);
  e.f = fmaf(p, r, TETRIS_EXP_C0);
  o.u = (t.u << 23) + e.u;
  return o.f;
}

void oracle_probs_from_logits_bf16(const uint16_t* z, const float* lse, int64_t R, int V, float* out) {
  for (int64_t r = 0; r < R; ++r)
    for (int v = 0; v < V; ++v) out[r * V + v] = prob_from_logit(z[r * V + v], lse[r]);
}
