/*
 * adpsgd_oracle.c -- plain, slow, obviously-correct CPU ORACLE for AD-PSGD
 * (Lian, Zhang, Zhang, Liu: "Asynchronous Decentralized Parallel Stochastic
 * Gradient Descent", arXiv 1710.06952).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1710_06952_b200/) never links, imports or calls it, and this file shares
 * no code, header, table or constant generator with the CUDA path.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared
 *        (no FMA contraction, no FTZ/DAZ: IEEE-754 binary32 round-to-nearest-even
 *        for every fp32 operation written below, reading R6).
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n.
 *
 * What it follows, step by step:
 *   Alg. 1, logical view, in the matrix form of Sec. 4:
 *       X_{k+1} = X_k W_k - gamma * dg(Xhat_k; xi_k, i_k),  Xhat_k = X_{k - tau_k}
 *   with W_k the pairwise average of P:411-414 (x^i, x^j <- x^i/2 + x^j/2).
 *
 * Parity pins (tests/test_oracle_*.py): Philox known-answer tests, fp32 golden
 * vectors, the S:254-256 worked example, n=1 == serial SGD
 * (P:699-705), column-sum invariant, brute-force enumeration of all
 * schedules vs. the fp64 linear recursion, finite-difference gradients, the
 * consensus-decay lemma, M_k worked example.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* Coordinates are independent in every per-coordinate loop below (each c is
 * written once from its own inputs), so the optional OpenMP build
 * (liboracle_omp.so, bench.py's all-cores CPU baseline)
 * is bit-identical to the serial one (tests/test_oracle.py checks it).  The
 * default build ignores the pragmas.                                          */
#ifdef _OPENMP
#define ORC_OMP_FOR _Pragma("omp parallel for schedule(static)")
#define ORC_OMP_FOR_BAD _Pragma("omp parallel for schedule(static) reduction(|:bad)")
#else
#define ORC_OMP_FOR
#define ORC_OMP_FOR_BAD
#endif

int oracle_consensus_mean(int32_t n, int64_t d, const float* X, const double* p, float* out,
                          double* mk);

/* ---------------------------------------------------------------- status -- */
enum {
  ORC_OK = 0, ORC_E_INVALID = 1, ORC_E_NOT_BIPARTITE = 2, ORC_E_DISCONNECTED = 3,
  ORC_E_NOT_NEIGHBOURS = 4, ORC_E_STALENESS = 5, ORC_E_DIVERGED = 6, ORC_E_OOM = 10
};

/* ---------------------------------------------------- Philox4x32-10 -------- *
 * Salmon et al. (SC'11) counter-based RNG, written from its definition:
 * 10 rounds; round: (hi0,lo0)=mul(M0,c0), (hi1,lo1)=mul(M1,c2),
 * c = (hi1^c1^k0, lo1, hi0^c3^k1, lo0); key += (W0,W1) between rounds.        */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* 32-bit integer finaliser ("lowbias32", C. Wellons) used by the synthetic
 * quadratic workload definition.           */
uint32_t oracle_lowbias32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

/* ------------------------------------------------------------- graph ----- *
 * Undirected graph (V,E).  Deadlock-free pairing requires a
 * bipartite split V = A u P with every edge joining A and P.
 * role: 0 = active, 1 = passive.  role_in == NULL -> BFS 2-colouring from
 * node 0 coloured active.  A graph with n >= 2 must be connected (rho < 1,
 * S:36).                                                               */
int oracle_check_graph(int32_t n, int32_t n_edges, const int32_t* edges,
                       const int8_t* role_in, int8_t* role_out) {
  if (n < 1 || n_edges < 0 || (n_edges > 0 && !edges)) return ORC_E_INVALID;
  for (int32_t e = 0; e < n_edges; ++e) {
    int32_t a = edges[2 * e], b = edges[2 * e + 1];
    if (a < 0 || a >= n || b < 0 || b >= n || a == b) return ORC_E_INVALID;
    for (int32_t f = 0; f < e; ++f) {           /* duplicates */
      int32_t c = edges[2 * f], d = edges[2 * f + 1];
      if ((a == c && b == d) || (a == d && b == c)) return ORC_E_INVALID;
    }
  }
  int8_t* col = (int8_t*)malloc((size_t)n);
  int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  if (!col || !queue) { free(col); free(queue); return ORC_E_OOM; }
  for (int32_t v = 0; v < n; ++v) col[v] = -1;
  /* connectivity + colouring by BFS from node 0 */
  int32_t head = 0, tail = 0, seen = 1;
  col[0] = 0; queue[tail++] = 0;
  int bip = 1;
  while (head < tail) {
    int32_t u = queue[head++];
    for (int32_t e = 0; e < n_edges; ++e) {
      int32_t a = edges[2 * e], b = edges[2 * e + 1], w;
      if (a == u) w = b; else if (b == u) w = a; else continue;
      if (col[w] < 0) { col[w] = (int8_t)(1 - col[u]); queue[tail++] = w; ++seen; }
      else if (col[w] == col[u]) bip = 0;
    }
  }
  int st = ORC_OK;
  if (seen != n) st = ORC_E_DISCONNECTED;
  else if (role_in) {
    for (int32_t e = 0; e < n_edges; ++e)
      if (role_in[edges[2 * e]] == role_in[edges[2 * e + 1]]) st = ORC_E_NOT_BIPARTITE;
    for (int32_t v = 0; v < n && st == ORC_OK; ++v)
      if (role_in[v] != 0 && role_in[v] != 1) st = ORC_E_INVALID;
    if (st == ORC_OK && role_out) memcpy(role_out, role_in, (size_t)n);
  } else if (!bip) st = ORC_E_NOT_BIPARTITE;
  else if (role_out) memcpy(role_out, col, (size_t)n);
  free(col); free(queue);
  return st;
}

static int is_edge(int32_t n_edges, const int32_t* edges, int32_t a, int32_t b) {
  for (int32_t e = 0; e < n_edges; ++e)
    if ((edges[2 * e] == a && edges[2 * e + 1] == b) || (edges[2 * e] == b && edges[2 * e + 1] == a))
      return 1;
  return 0;
}

/* -------------------------------------------------------------- problems -- */
enum { ORC_MODEL_NONE = 0, ORC_MODEL_QUADRATIC = 2, ORC_MODEL_LSQ = 3, ORC_MODEL_LOGREG = 4,
       ORC_MODEL_MLP = 5 };

typedef struct {
  int32_t kind;          /* ORC_MODEL_*                                         */
  int32_t M;             /* batch size                              */
  float   gamma;         /* learning rate                                       */
  /* quadratic: */
  uint32_t data_key;     /* Ds, host-derived key of the data landscape          */
  uint32_t noise_key;    /* Ns, host-derived key of the gradient noise          */
  float   noise_s;       /* s = sigma*sqrt(3M) (fp32, host computed)            */
  const float* h_explicit;     /* optional d curvatures (tests); NULL -> hashed */
  const float* xstar_explicit; /* optional d minimiser  (tests); NULL -> hashed  */
  /* lsq / logreg / mlp datasets (Strategy-1: every worker sees all data) */
  int32_t S;             /* number of samples                                   */
  const float* A;        /* S x feat, row major                                 */
  const float* b;        /* lsq targets / logreg labels (+-1) ; S               */
  const int32_t* y;      /* mlp labels in [0, n_out)                            */
  int32_t n_in, n_hid, n_out;  /* mlp dims; lsq/logreg use n_in = d             */
  uint32_t batch_key[2]; /* Philox key for device-mode batch sampling           */
} oracle_problem;

/* Synthetic quadratic f(x) = 1/2 sum_c h_c (x_c - x*_c)^2.  The
 * stochastic batch-sum gradient (a SUM over the M samples) is
 *   g_c = fl( fl(M*h_c) * fl(xhat_c - x*_c) ) + fl( s * v_c )
 * with v_c = (u>>9) * 2^-22 - 1 (23-bit uniform grid on [-1,1)) and
 * u = mix(c ^ K_k); the single draw s*v_c has the variance M*sigma^2 of the sum
 * of M per-sample uniform noises.  The landscape word is the Weyl sequence
 * w_c = (c * 0x9E3779B1) ^ data_key: h_c from its high 16 bits, x*_c from its
 * low 16 bits (definition v3).  Every op is
 * one rounded fp32 op (no FMA): this is the workload's definition, so the
 * oracle evaluates it exactly.                                               */
uint32_t oracle_quad_noise_mix(uint32_t x) {
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  return x;
}

static void quad_data(const oracle_problem* p, int64_t c, float* h, float* xs) {
  if (p->h_explicit) { *h = p->h_explicit[c]; *xs = p->xstar_explicit[c]; return; }
  uint32_t w = ((uint32_t)c * 0x9E3779B1u) ^ p->data_key;
  float u_h = (float)(w >> 16) * (1.0f / 65536.0f);     /* exact */
  float t = 0.99f * u_h;
  *h = 0.01f + t;
  float u_x = (float)(w & 0xffffu) * (1.0f / 32768.0f);  /* exact, in [0,2) */
  *xs = u_x - 1.0f;
}

uint32_t oracle_quad_event_key(uint32_t noise_key, uint64_t k) {
  return oracle_lowbias32(oracle_lowbias32((uint32_t)k ^ noise_key) ^ (uint32_t)(k >> 32));
}

int oracle_quadratic_grad(const oracle_problem* p, int64_t d, const float* xhat, uint64_t k,
                          float* g) {
  uint32_t kk = oracle_quad_event_key(p->noise_key, k);
  float Mf = (float)p->M;
  ORC_OMP_FOR
  for (int64_t c = 0; c < d; ++c) {
    float h, xs;
    quad_data(p, c, &h, &xs);
    uint32_t u = oracle_quad_noise_mix((uint32_t)c ^ kk);
    float m = (float)(u >> 9) * (1.0f / 4194304.0f);    /* exact: (u>>9) * 2^-22, in [0,2) */
    float v = m - 1.0f;                                  /* exact, uniform grid in [-1,1) */
    float noise = p->noise_s * v;
    float mh = Mf * h;
    float diff = xhat[c] - xs;
    float det = mh * diff;
    g[c] = det + noise;
  }
  return ORC_OK;
}

/* quadratic loss at x (fp64): f(x) = 1/2 sum_c h_c (x_c - x*_c)^2 */
double oracle_quadratic_loss(const oracle_problem* p, int64_t d, const float* x) {
  double f = 0.0;
  for (int64_t c = 0; c < d; ++c) {
    float h, xs; quad_data(p, c, &h, &xs);
    double e = (double)x[c] - (double)xs;
    f += 0.5 * (double)h * e * e;
  }
  return f;
}

/* device-mode batch index: idx = (u32 * S) >> 32, u32 = Philox(key, (lo32(k), m, BATCH,
 * hi32(k))).out0 (sampling with replacement).  hi32(k) = 0 for every event index
 * k < 2^32; it separates the keys of App. A reads (R20) and super-learners (R22). */
#define ORC_STREAM_BATCH 0x42415443u
static int32_t batch_index(const oracle_problem* p, uint64_t k, uint32_t m) {
  uint32_t ctr[4] = {(uint32_t)k, m, ORC_STREAM_BATCH, (uint32_t)(k >> 32)}, out[4];
  oracle_philox4x32_10(ctr, p->batch_key, out);
  return (int32_t)(((uint64_t)out[0] * (uint64_t)(uint32_t)p->S) >> 32);
}

/* least squares F(x;(a,b)) = 1/2 (a.x - b)^2, grad = a (a.x - b); batch SUM,
 * accumulated in fp64, rounded once to fp32.             */
static int lsq_grad(const oracle_problem* p, int64_t d, const float* xhat, const int32_t* idx,
                    float* g) {
  double* acc = (double*)calloc((size_t)d, sizeof(double));
  if (!acc) return ORC_E_OOM;
  for (int32_t m = 0; m < p->M; ++m) {
    const float* a = p->A + (int64_t)idx[m] * d;
    double r = 0.0;
    for (int64_t c = 0; c < d; ++c) r += (double)a[c] * (double)xhat[c];
    r -= (double)p->b[idx[m]];
    for (int64_t c = 0; c < d; ++c) acc[c] += (double)a[c] * r;
  }
  for (int64_t c = 0; c < d; ++c) g[c] = (float)acc[c];
  free(acc);
  return ORC_OK;
}

/* logistic F(x;(a,y)) = log(1 + exp(-y a.x)), grad = -y sigma(-y a.x) a */
static int logreg_grad(const oracle_problem* p, int64_t d, const float* xhat, const int32_t* idx,
                       float* g) {
  double* acc = (double*)calloc((size_t)d, sizeof(double));
  if (!acc) return ORC_E_OOM;
  for (int32_t m = 0; m < p->M; ++m) {
    const float* a = p->A + (int64_t)idx[m] * d;
    double y = (double)p->b[idx[m]];
    double z = 0.0;
    for (int64_t c = 0; c < d; ++c) z += (double)a[c] * (double)xhat[c];
    double sig = 1.0 / (1.0 + exp(y * z));     /* sigma(-y z) */
    double coef = -y * sig;
    for (int64_t c = 0; c < d; ++c) acc[c] += coef * (double)a[c];
  }
  for (int64_t c = 0; c < d; ++c) g[c] = (float)acc[c];
  free(acc);
  return ORC_OK;
}

/* 2-layer MLP n_in -> n_hid (tanh) -> n_out, softmax cross-entropy summed over
 * the batch (reading R18; tanh as in SPEC's small-mlp: a smooth
 * activation has no floating-point-decided mask).  Flat parameter layout
 * [W1 (n_hid x n_in, out x in) | b1 | W2 (n_out x n_hid) | b2].  Plain fp64
 * loops, rounded once to fp32.  Returns the batch loss (fp64) via loss_out. */
static int mlp_grad(const oracle_problem* p, const float* xhat, const int32_t* idx, float* g,
                    double* loss_out) {
  const int64_t I = p->n_in, H = p->n_hid, O = p->n_out;
  const float* W1 = xhat; const float* b1 = W1 + H * I;
  const float* W2 = b1 + H; const float* b2 = W2 + O * H;
  const int64_t d = H * I + H + O * H + O;
  double* acc = (double*)calloc((size_t)d, sizeof(double));
  double* z1 = (double*)malloc(sizeof(double) * (size_t)H);
  double* h1 = (double*)malloc(sizeof(double) * (size_t)H);
  double* dz1 = (double*)malloc(sizeof(double) * (size_t)H);
  double* z2 = (double*)malloc(sizeof(double) * (size_t)O);
  double* dz2 = (double*)malloc(sizeof(double) * (size_t)O);
  if (!acc || !z1 || !h1 || !dz1 || !z2 || !dz2) {
    free(acc); free(z1); free(h1); free(dz1); free(z2); free(dz2); return ORC_E_OOM;
  }
  double* gW1 = acc; double* gb1 = gW1 + H * I; double* gW2 = gb1 + H; double* gb2 = gW2 + O * H;
  double loss = 0.0;
  for (int32_t m = 0; m < p->M; ++m) {
    const float* a = p->A + (int64_t)idx[m] * I;
    int32_t y = p->y[idx[m]];
    for (int64_t u = 0; u < H; ++u) {
      double s = (double)b1[u];
      for (int64_t c = 0; c < I; ++c) s += (double)W1[u * I + c] * (double)a[c];
      z1[u] = s; h1[u] = tanh(s);
    }
    double zmax = -INFINITY;
    for (int64_t o = 0; o < O; ++o) {
      double s = (double)b2[o];
      for (int64_t u = 0; u < H; ++u) s += (double)W2[o * H + u] * h1[u];
      z2[o] = s; if (s > zmax) zmax = s;
    }
    double se = 0.0;
    for (int64_t o = 0; o < O; ++o) se += exp(z2[o] - zmax);
    loss += log(se) + zmax - z2[y];
    for (int64_t o = 0; o < O; ++o) dz2[o] = exp(z2[o] - zmax) / se - (o == y ? 1.0 : 0.0);
    for (int64_t o = 0; o < O; ++o) {
      gb2[o] += dz2[o];
      for (int64_t u = 0; u < H; ++u) gW2[o * H + u] += dz2[o] * h1[u];
    }
    for (int64_t u = 0; u < H; ++u) {
      double s = 0.0;
      for (int64_t o = 0; o < O; ++o) s += (double)W2[o * H + u] * dz2[o];
      dz1[u] = s * (1.0 - h1[u] * h1[u]);
    }
    for (int64_t u = 0; u < H; ++u) {
      gb1[u] += dz1[u];
      if (dz1[u] != 0.0)
        for (int64_t c = 0; c < I; ++c) gW1[u * I + c] += dz1[u] * (double)a[c];
    }
  }
  for (int64_t c = 0; c < d; ++c) g[c] = (float)acc[c];
  if (loss_out) *loss_out = loss;
  free(acc); free(z1); free(h1); free(dz1); free(z2); free(dz2);
  return ORC_OK;
}

int64_t oracle_mlp_dim(int32_t n_in, int32_t n_hid, int32_t n_out) {
  return (int64_t)n_hid * n_in + n_hid + (int64_t)n_out * n_hid + n_out;
}

/* One minibatch gradient g = sum_m grad F(xhat; xi_m) (Alg. 1 step 4).
 * idx: M sample indices, or NULL -> device-mode Philox sampling for event k.  */
int oracle_gradient(const oracle_problem* p, int64_t d, const float* xhat, uint64_t k,
                    const int32_t* idx_in, float* g, double* loss_out) {
  if (!p || !xhat || !g) return ORC_E_INVALID;
  if (p->kind == ORC_MODEL_QUADRATIC) return oracle_quadratic_grad(p, d, xhat, k, g);
  if (p->kind != ORC_MODEL_LSQ && p->kind != ORC_MODEL_LOGREG && p->kind != ORC_MODEL_MLP)
    return ORC_E_INVALID;
  int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)p->M);
  if (!idx) return ORC_E_OOM;
  for (int32_t m = 0; m < p->M; ++m)
    idx[m] = idx_in ? idx_in[m] : batch_index(p, k, (uint32_t)m);
  int st;
  if (p->kind == ORC_MODEL_LSQ) st = lsq_grad(p, d, xhat, idx, g);
  else if (p->kind == ORC_MODEL_LOGREG) st = logreg_grad(p, d, xhat, idx, g);
  else st = mlp_grad(p, xhat, idx, g, loss_out);
  free(idx);
  return st;
}

/* Full-data objective f at x (fp64), used for loss thresholds. */
double oracle_full_loss(const oracle_problem* p, int64_t d, const float* x) {
  if (p->kind == ORC_MODEL_QUADRATIC) return oracle_quadratic_loss(p, d, x);
  double f = 0.0;
  if (p->kind == ORC_MODEL_LSQ || p->kind == ORC_MODEL_LOGREG) {
    for (int32_t s = 0; s < p->S; ++s) {
      const float* a = p->A + (int64_t)s * d;
      double z = 0.0;
      for (int64_t c = 0; c < d; ++c) z += (double)a[c] * (double)x[c];
      if (p->kind == ORC_MODEL_LSQ) { double r = z - (double)p->b[s]; f += 0.5 * r * r; }
      else { double m = -(double)p->b[s] * z; f += m > 0 ? m + log1p(exp(-m)) : log1p(exp(m)); }
    }
    return f / (double)p->S;
  }
  if (p->kind == ORC_MODEL_MLP) {
    oracle_problem q = *p;
    int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)p->S);
    float* gtmp = (float*)malloc(sizeof(float) * (size_t)d);
    double loss = 0.0;
    if (!idx || !gtmp) { free(idx); free(gtmp); return NAN; }
    for (int32_t s = 0; s < p->S; ++s) idx[s] = s;
    q.M = p->S;
    mlp_grad(&q, x, idx, gtmp, &loss);
    free(idx); free(gtmp);
    return loss / (double)p->S;
  }
  return NAN;
}

/* ------------------------------------------------------------ replay ----- *
 * Event k = (i, j, tau, flags), reading R5: i is the
 * worker making gradient update k (the virtual counter of P:429-432); j is its
 * averaging partner (W_k = pair average of P:411-414) or -1 (W_k = I, still
 * doubly stochastic); tau is the staleness of the read, Xhat_k = X_{k-tau}
 * (P:561), 0 <= tau <= min(k, T).  flags bit0 = NO_GRAD (pure
 * averaging, W_k only).
 * Per event, in Alg. 1 order (reading R1 "average, then update"):
 *   xhat = column i of X_{k - tau}                        (stale read)
 *   g    = sum_m grad F(xhat; xi_{k,m})                   (step 4)
 *   X_{k+1/2} = X_k W_k :  m = fl(fl(x_i + x_j) * 0.5f); x_i = x_j = m   (step 5)
 *   x_i <- fl(x_i - fl(gamma * g))                       (step 6)
 * X is row-major n x d (worker-major: the transpose of the paper's N x n).
 * mk_trace (nullable, K+1 entries): M_k with p_i = 1/n after each event
 * (P:1389-1391).  loss_trace unused (NULL).
 *
 * App. A events (the wait-free runtime; reading R20):
 *   flags bit1 FLUSH_FIRST: Alg. 2's order -- "if g != 0:
 *     x^i <- x^i - gamma g", then "x^i <- (x^i + x^j)/2" (the passive takes the
 *     same average, Alg. 3):  x_i <- fl(x_i - fl(gamma g)); m = fl(fl(x_i + x_j)
 *     * 0.5f); x_i = x_j = m.  The gradient's random draws are keyed by its read
 *     point, key = 2^62 | (k0 + k - tau) << 20 | i, since it exists before its
 *     flush event.
 *   flags bit2 COMPENSATE: Alg. 1's footnote -- the computation
 *     thread pulls x^i and applies "x^i <- x^i - gamma g" with the gradient g
 *     still in the buffer, i.e. worker i's previous gradient event k_p when
 *     k_p >= k - tau (not yet part of X_{k-tau}):  xhat <- fl(xhat - fl(gamma
 *     g_p)).  One gradient at a time per worker (Alg. 1 blocks until g = 0):
 *     k_p - tau_p > k - tau is ORC_E_STALENESS.                                */
#define ORC_EV_NO_GRAD 1u
#define ORC_EV_FLUSH_FIRST 2u
#define ORC_EV_COMPENSATE 4u

uint64_t oracle_read_key(uint64_t t_read, int32_t i) {
  return (1ull << 62) | (t_read << 20) | (uint64_t)(uint32_t)i;
}

int oracle_replay(const oracle_problem* p, int32_t n, int64_t d, float* X,
                  int32_t n_edges, const int32_t* edges, const int8_t* role,
                  const int32_t* events, int64_t K, const int32_t* batch_idx,
                  int32_t T, int32_t clamp_tau, uint64_t k0, double* mk_trace) {
  if (!p || n < 1 || d < 1 || !X || K < 0 || (K > 0 && !events) || T < 0) return ORC_E_INVALID;
  int8_t* r = (int8_t*)malloc((size_t)n);
  if (!r) return ORC_E_OOM;
  int st = oracle_check_graph(n, n_edges, edges, role, r);
  if (n == 1 && n_edges == 0) st = ORC_OK, r[0] = 0;
  if (st != ORC_OK) { free(r); return st; }
  const int64_t nd = (int64_t)n * d;
  /* history ring: hist[q] holds X_q for q in [k-T, k] at slot q mod (T+1) */
  float* hist = (float*)malloc(sizeof(float) * (size_t)(nd * (T + 1)));
  float* xhat = (float*)malloc(sizeof(float) * (size_t)d);
  float* g = (float*)malloc(sizeof(float) * (size_t)d);
  /* App. A state: each worker's previous gradient event, its read point and value */
  int64_t* kp = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* rp = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int any_comp = 0;
  for (int64_t k = 0; k < K; ++k) any_comp |= (events[4 * k + 3] & (int32_t)ORC_EV_COMPENSATE) != 0;
  float* gp = any_comp ? (float*)malloc(sizeof(float) * (size_t)nd) : NULL;
  if (!hist || !xhat || !g || !kp || !rp || (any_comp && !gp)) {
    free(r); free(hist); free(xhat); free(g); free(kp); free(rp); free(gp);
    return ORC_E_OOM;
  }
  for (int32_t w = 0; w < n; ++w) kp[w] = -1, rp[w] = -1;
  memcpy(hist, X, sizeof(float) * (size_t)nd);      /* X_0 at slot 0 */
  if (mk_trace) {
    double dummy;
    oracle_consensus_mean(n, d, X, NULL, NULL, &dummy); mk_trace[0] = dummy;
  }
  for (int64_t k = 0; k < K; ++k) {
    int32_t i = events[4 * k], j = events[4 * k + 1], tau = events[4 * k + 2];
    uint32_t flags = (uint32_t)events[4 * k + 3];
    if (i < 0 || i >= n || j < -1 || j >= n || j == i) { st = ORC_E_INVALID; break; }
    if (j >= 0) {
      if (!is_edge(n_edges, edges, i, j)) { st = ORC_E_NOT_NEIGHBOURS; break; }
      if (r[i] == r[j]) { st = ORC_E_NOT_BIPARTITE; break; }
    }
    if (tau < 0) { st = ORC_E_STALENESS; break; }
    if (tau > T || tau > k) {
      if (!clamp_tau) { st = ORC_E_STALENESS; break; }
      if (tau > T) tau = T;
      if (tau > k) tau = (int32_t)k;
    }
    float* Xk = hist + nd * (k % (T + 1));
    /* stale read: Xhat_k = X_{k - tau} */
    const float* Xs = hist + nd * ((k - tau) % (T + 1));
    memcpy(xhat, Xs + (int64_t)i * d, sizeof(float) * (size_t)d);
    int do_grad = !(flags & ORC_EV_NO_GRAD) && p->kind != ORC_MODEL_NONE;
    const int flush_first = (flags & ORC_EV_FLUSH_FIRST) != 0;
    if (do_grad) {
      const int32_t* idx = batch_idx ? batch_idx + k * p->M : NULL;
      uint64_t key = k0 + (uint64_t)k;
      if (flush_first) key = oracle_read_key(k0 + (uint64_t)(k - tau), i);
      if ((flags & ORC_EV_COMPENSATE) && kp[i] >= k - tau) {
        /* pulled while g_p was still in the buffer: local update */
        if (rp[i] > k - tau) { st = ORC_E_STALENESS; break; }
        const float* gpi = gp + (int64_t)i * d;
        for (int64_t c = 0; c < d; ++c) {
          float step = p->gamma * gpi[c];
          xhat[c] = xhat[c] - step;
        }
      }
      st = oracle_gradient(p, d, xhat, key, idx, g, NULL);
      if (st != ORC_OK) break;
      kp[i] = k; rp[i] = k - tau;
      if (gp) memcpy(gp + (int64_t)i * d, g, sizeof(float) * (size_t)d);
    }
    /* X_{k+1} starts as a copy of X_k in the next history slot */
    float* Xn = hist + nd * ((k + 1) % (T + 1));
    if (Xn != Xk) memcpy(Xn, Xk, sizeof(float) * (size_t)nd);
    float* xi = Xn + (int64_t)i * d;
    if (do_grad && flush_first) {       /* Alg. 2: flush g first */
      int bad = 0;
      ORC_OMP_FOR_BAD
      for (int64_t c = 0; c < d; ++c) {
        float step = p->gamma * g[c];
        xi[c] = xi[c] - step;
        if (!isfinite(xi[c])) bad = 1;
      }
      if (bad) st = ORC_E_DIVERGED;
      if (st != ORC_OK) break;
      do_grad = 0;
    }
    if (j >= 0) {                       /* X_{k+1/2} = X_k W_k */
      float* xj = Xn + (int64_t)j * d;
      ORC_OMP_FOR
      for (int64_t c = 0; c < d; ++c) {
        float s = xi[c] + xj[c];
        float m = s * 0.5f;
        xi[c] = m; xj[c] = m;
      }
    }
    if (do_grad) {                      /* x_{k+1}^{i_k} = x_{k+1/2}^{i_k} - gamma g */
      int bad = 0;
      ORC_OMP_FOR_BAD
      for (int64_t c = 0; c < d; ++c) {
        float step = p->gamma * g[c];
        xi[c] = xi[c] - step;
        if (!isfinite(xi[c])) bad = 1;
      }
      if (bad) st = ORC_E_DIVERGED;
      if (st != ORC_OK) break;
    }
    if (mk_trace) {
      double mk;
      oracle_consensus_mean(n, d, Xn, NULL, NULL, &mk); mk_trace[k + 1] = mk;
    }
  }
  if (st == ORC_OK) memcpy(X, hist + nd * (K % (T + 1)), sizeof(float) * (size_t)nd);
  free(r); free(hist); free(xhat); free(g); free(kp); free(rp); free(gp);
  return st;
}

/* ------------------------------------------------------ consensus output --
 * "Output the average of the models on all workers":
 *   xbar_c = fl32( (sum_i x_{i,c}) / n )  with the sum in fp64.
 * M_k = sum_i p_i || X 1/n - X e_i ||^2 with the exact (fp64)
 * column mean; p = NULL -> p_i = 1/n.                                       */
int oracle_consensus_mean(int32_t n, int64_t d, const float* X, const double* p, float* out,
                          double* mk) {
  if (n < 1 || d < 1 || !X) return ORC_E_INVALID;
  double M = 0.0;
  for (int64_t c = 0; c < d; ++c) {
    double s = 0.0;
    for (int32_t i = 0; i < n; ++i) s += (double)X[(int64_t)i * d + c];
    double mean = s / (double)n;
    if (out) out[c] = (float)mean;
    if (mk)
      for (int32_t i = 0; i < n; ++i) {
        double e = mean - (double)X[(int64_t)i * d + c];
        M += (p ? p[i] : 1.0 / (double)n) * e * e;
      }
  }
  if (mk) *mk = M;
  return ORC_OK;
}

/* ------------------------------------------------------ AllReduce-SGD -----
 * every worker computes a minibatch gradient at the (common) model,
 * AllReduce averages them, every replica applies the average.  Reading R12:
 *   x <- fl( x - fl( gamma * fl( (sum_i g_i)/n ) ) ), sum in fp64.
 * grads: n x d fp32 (worker-major).                                         */
int oracle_allreduce_update(int32_t n, int64_t d, float gamma, const float* grads, float* x) {
  if (n < 1 || d < 1 || !grads || !x) return ORC_E_INVALID;
  for (int64_t c = 0; c < d; ++c) {
    double s = 0.0;
    for (int32_t i = 0; i < n; ++i) s += (double)grads[(int64_t)i * d + c];
    float mean = (float)(s / (double)n);
    float step = gamma * mean;
    x[c] = x[c] - step;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------- D-PSGD -----
 * in every synchronous round all workers compute a minibatch
 * gradient at their own model and average with their neighbours; the gradients
 * are then applied.  Reading R19: X <- X W - gamma G with
 * W = I - L/(deg_max + 1) (L the graph Laplacian), gradients at the pre-mix
 * models.  fp32 op order (the definition both sides follow):
 *   acc = fl(w_self_i * x_i); for j in N(i) ascending: acc = fl(acc + fl(w_nb * x_j));
 *   x_i' = fl(acc - fl(gamma * g_i)),   w_nb = fl32(1/(deg_max+1)),
 *   w_self_i = fl32(1 - deg_i/(deg_max+1)),  g_i = gradient at x_i for event k_base + i.
 * X: n x d worker-major, updated in place (all reads see the pre-round X).    */
int oracle_dpsgd_round(const oracle_problem* p, int32_t n, int64_t d, float* X, int32_t n_edges,
                       const int32_t* edges, uint64_t k_base) {
  if (!p || n < 1 || d < 1 || !X) return ORC_E_INVALID;
  int32_t* deg = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  float* Xn = (float*)malloc(sizeof(float) * (size_t)n * (size_t)d);
  float* g = (float*)malloc(sizeof(float) * (size_t)d);
  if (!deg || !Xn || !g) { free(deg); free(Xn); free(g); return ORC_E_OOM; }
  int32_t dmax = 0;
  for (int32_t e = 0; e < n_edges; ++e) { deg[edges[2 * e]]++; deg[edges[2 * e + 1]]++; }
  for (int32_t i = 0; i < n; ++i) if (deg[i] > dmax) dmax = deg[i];
  const float w_nb = (float)(1.0 / (double)(dmax + 1));
  int st = ORC_OK;
  for (int32_t i = 0; i < n && st == ORC_OK; ++i) {
    const float w_self = (float)(1.0 - (double)deg[i] / (double)(dmax + 1));
    const float* xi = X + (int64_t)i * d;
    if (p->kind != ORC_MODEL_NONE) st = oracle_gradient(p, d, xi, k_base + (uint64_t)i, NULL, g, NULL);
    int32_t nb[64], nn = 0;                             /* neighbours in ascending order */
    for (int32_t j = 0; j < n && nn < 64; ++j)
      if (j != i && is_edge(n_edges, edges, i, j)) nb[nn++] = j;
    for (int64_t c = 0; c < d; ++c) {
      float acc = w_self * xi[c];
      for (int32_t t = 0; t < nn; ++t) {
        float v = w_nb * X[(int64_t)nb[t] * d + c];
        acc = acc + v;
      }
      if (p->kind != ORC_MODEL_NONE) {
        float step = p->gamma * g[c];
        acc = acc - step;
      }
      Xn[(int64_t)i * d + c] = acc;
    }
  }
  if (st == ORC_OK) memcpy(X, Xn, sizeof(float) * (size_t)n * (size_t)d);
  free(deg); free(Xn); free(g);
  return st;
}

/* ------------------------------------------------------- super-learner ----
 * "combining learners on the same computing node as a super-learner
 * (via Nvidia NCCL AllReduce collectives)".  DESIGN.md reading R22: a
 * super-learner s is one AD-PSGD worker made of R learners; its gradient is the
 * all-reduce SUM of the learners' minibatch gradients (batch R*M), each learner r
 * drawing its noise with key(s, c, r) = 2^61 | s<<44 | c<<8 | r, c = the number
 * of earlier gradient events of s.  The sum is taken in fp64 and rounded once to
 * fp32 (for R = 2 this is exactly the fp32 sum an all-reduce computes).        */
uint64_t oracle_super_key(int32_t s, int64_t c, int32_t r) {
  return (1ull << 61) | ((uint64_t)(uint32_t)s << 44) | ((uint64_t)c << 8) | (uint64_t)(uint32_t)r;
}

int oracle_super_gradient(const oracle_problem* p, int64_t d, const float* x, int32_t s, int64_t c, int32_t R,
                          float* g) {
  if (!p || !x || !g || R < 1 || p->kind == ORC_MODEL_NONE) return ORC_E_INVALID;
  double* acc = (double*)calloc((size_t)d, sizeof(double));
  float* gr = (float*)malloc(sizeof(float) * (size_t)d);
  if (!acc || !gr) { free(acc); free(gr); return ORC_E_OOM; }
  int st = ORC_OK;
  /* any built-in model: learner r's minibatch (Philox indices for lsq / logreg /
     mlp, noise for the quadratic) is drawn with key(s, c, r) */
  for (int32_t r = 0; r < R && st == ORC_OK; ++r) {
    st = oracle_gradient(p, d, x, oracle_super_key(s, c, r), NULL, gr, NULL);
    for (int64_t e = 0; e < d; ++e) acc[e] += (double)gr[e];
  }
  for (int64_t e = 0; e < d; ++e) g[e] = (float)acc[e];
  free(acc); free(gr);
  return st;
}

/* Replay of super-learner events (i, j, 0, flags) over S super-learners in
 * Alg. 1 order (average, then x_i <- m - gamma g), tau = 0, X: S x d (one
 * model per super-learner: its R replicas are identical by construction).   */
int oracle_super_replay(const oracle_problem* p, int32_t S, int64_t d, float* X, int32_t n_edges,
                        const int32_t* edges, const int8_t* role, const int32_t* events, int64_t K, int32_t R) {
  if (!p || S < 1 || d < 1 || !X || K < 0 || (K > 0 && !events) || R < 1) return ORC_E_INVALID;
  int8_t* rl = (int8_t*)malloc((size_t)S);
  int64_t* cnt = (int64_t*)calloc((size_t)S, sizeof(int64_t));
  float* g = (float*)malloc(sizeof(float) * (size_t)d);
  if (!rl || !cnt || !g) { free(rl); free(cnt); free(g); return ORC_E_OOM; }
  int st = oracle_check_graph(S, n_edges, edges, role, rl);
  if (S == 1 && n_edges == 0) st = ORC_OK;
  for (int64_t k = 0; k < K && st == ORC_OK; ++k) {
    const int32_t i = events[4 * k], j = events[4 * k + 1];
    const uint32_t flags = (uint32_t)events[4 * k + 3];
    if (i < 0 || i >= S || j < -1 || j >= S || j == i) { st = ORC_E_INVALID; break; }
    if (j >= 0 && (!is_edge(n_edges, edges, i, j) || rl[i] == rl[j])) { st = ORC_E_NOT_NEIGHBOURS; break; }
    float* xi = X + (int64_t)i * d;
    const int grad = !(flags & ORC_EV_NO_GRAD) && p->kind != ORC_MODEL_NONE;
    if (grad) {
      st = oracle_super_gradient(p, d, xi, i, cnt[i], R, g);
      cnt[i] += 1;
      if (st != ORC_OK) break;
    }
    if (j >= 0) {
      float* xj = X + (int64_t)j * d;
      for (int64_t c = 0; c < d; ++c) {
        float s2 = xi[c] + xj[c];
        float m = s2 * 0.5f;
        xi[c] = m; xj[c] = m;
      }
    }
    if (grad)
      for (int64_t c = 0; c < d; ++c) {
        float step = p->gamma * g[c];
        xi[c] = xi[c] - step;
      }
  }
  free(rl); free(cnt); free(g);
  return st;
}
