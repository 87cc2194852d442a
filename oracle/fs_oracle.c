/*
 * fs_oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, single-threaded CPU oracle
 * for the Founsure 1.0 encode hot path (arXiv 1702.07409).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product path (paper_1702_07409_b200/) never links,
 * imports or executes anything under oracle/.  This file shares no code, header,
 * table or constant generator with the CUDA path: it re-derives everything from the
 * paper and from the readings recorded in DESIGN.md §3.
 *
 * What it computes (§2.2, Fig. 1 steps (1) and (2)):
 *   checks   C_i = XOR_{m in P(i)} D_m                      i < p    (precode, "Check #1")
 *   coded    Y_j = XOR_{m in N(j)} I_m,  I = D ++ C          j < n    (LT / LDGM stage)
 * with the bipartite graph drawn from a seeded PRNG (§2.2) and the
 * coded-symbol degree drawn from Omega(x) or the Robust Soliton
 * distribution (§1).  The decoder follows Algorithm 1 (BP)
 * "at most twice (once for the outer graph code and ... the inner precode)"
 * and then finishes with GF(2) elimination on the residual system (
 * not in the paper, used only to certify the encoder's output).
 *
 * Readings of silent / ambiguous points (R2..R15):
 *   R2  PRNG = splitmix64 (Steele, Lea, Flood 2014); state += 0x9E3779B97F4A7C15, then mix.
 *   R5  one stream: all precode checks first (d_p draws each), then LT rows
 *       (one degree draw, then neighbour draws per row).
 *   R6  neighbour index = x mod range; redraw on duplicate.
 *   R7  u = (x >> 11) * 2^-53; degree = smallest support degree with u < CDF[d];
 *       CDF built ascending: total = sum of weights (ascending), CDF[d] = CDF[d-1] + w_d/total,
 *       last entry forced to 1.0.
 *   R9  Omega's coefficients are normalised by their sum.
 *   R10 RSD over K = k+p: R = c ln(K/delta) sqrt(K), m = floor(K/R), rho(1) = 1/K,
 *       rho(i) = 1/(i(i-1)), tau(i) = R/(iK) for i < m, tau(m) = R ln(R/delta)/K.
 *   R11 precode neighbours drawn from [0,k), distinct within a check.
 *   R12 LT neighbours drawn from [0,K), index k+i = check i.
 *   R14 neighbours stored sorted ascending within a row.
 *   R15 degrees > K are merged into degree K.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ PRNG (R2) */
uint64_t or_splitmix64_next(uint64_t *state) {
  uint64_t z;
  *state += 0x9E3779B97F4A7C15ULL;
  z = *state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

void or_splitmix64_fill(uint64_t seed, uint64_t count, uint64_t *out) {
  uint64_t s = seed, i;
  for (i = 0; i < count; ++i) out[i] = or_splitmix64_next(&s);
}

/* ------------------------------------------------------- degree law (R7-R10) */
/* kind 1 = RSD, kind 2 = finite max-degree Omega.
 * Writes the support degrees and the CDF (double) into out_deg / out_cdf, whose
 * capacity must be >= K (RSD) or >= fin_len (finite).  Returns the support length,
 * or -1 on an invalid distribution. */
int or_build_cdf(int kind, uint32_t K, double rsd_c, double rsd_delta,
                 const uint32_t *fin_deg, const double *fin_prob, uint32_t fin_len,
                 uint32_t *out_deg, double *out_cdf) {
  uint32_t len = 0, i;
  double *w;
  double total = 0.0, acc = 0.0;
  if (K == 0) return -1;
  w = (double *)malloc(sizeof(double) * (K > fin_len ? K : fin_len) + 8);
  if (!w) return -1;
  if (kind == 1) {
    double R, tau;
    uint32_t m;
    if (!(rsd_c > 0.0) || !(rsd_delta > 0.0 && rsd_delta < 1.0)) { free(w); return -1; }
    R = rsd_c * log((double)K / rsd_delta) * sqrt((double)K);
    if (!(R / rsd_delta > 1.0)) { free(w); return -1; }
    m = (uint32_t)floor((double)K / R);
    if (m < 1) { free(w); return -1; }
    for (i = 1; i <= K; ++i) {
      double rho = (i == 1) ? 1.0 / (double)K : 1.0 / ((double)i * (double)(i - 1));
      if (i < m) tau = R / ((double)i * (double)K);
      else if (i == m) tau = R * log(R / rsd_delta) / (double)K;
      else tau = 0.0;
      out_deg[len] = i;
      w[len] = rho + tau;
      ++len;
    }
  } else if (kind == 2) {
    /* degrees strictly increasing, positive; degrees > K merged into K (R15) */
    for (i = 0; i < fin_len; ++i) {
      uint32_t d = fin_deg[i];
      if (d == 0 || fin_prob[i] < 0.0) { free(w); return -1; }
      if (i > 0 && d <= fin_deg[i - 1]) { free(w); return -1; }
      if (d > K) d = K;
      if (len > 0 && out_deg[len - 1] == d) {
        w[len - 1] += fin_prob[i];
      } else {
        out_deg[len] = d;
        w[len] = fin_prob[i];
        ++len;
      }
    }
    if (len == 0) { free(w); return -1; }
  } else {
    free(w);
    return -1;
  }
  for (i = 0; i < len; ++i) total += w[i];
  if (!(total > 0.0)) { free(w); return -1; }
  for (i = 0; i < len; ++i) {
    acc = acc + w[i] / total;
    out_cdf[i] = acc;
  }
  out_cdf[len - 1] = 1.0;
  free(w);
  return (int)len;
}

static uint32_t draw_degree(uint64_t *st, const uint32_t *deg, const double *cdf, uint32_t len) {
  uint64_t x = or_splitmix64_next(st);
  double u = (double)(x >> 11) * (1.0 / 9007199254740992.0); /* 2^-53 */
  uint32_t i;
  for (i = 0; i < len; ++i)
    if (u < cdf[i]) return deg[i];
  return deg[len - 1];
}

/* d distinct indices in [0, range): modulo with duplicate rejection (R6), sorted (R14). */
static void draw_neighbours(uint64_t *st, uint32_t d, uint32_t range, int32_t *out) {
  uint32_t got = 0, i, j;
  while (got < d) {
    uint32_t idx = (uint32_t)(or_splitmix64_next(st) % (uint64_t)range);
    int dup = 0;
    for (i = 0; i < got; ++i)
      if ((uint32_t)out[i] == idx) { dup = 1; break; }
    if (!dup) out[got++] = (int32_t)idx;
  }
  for (i = 1; i < d; ++i) { /* insertion sort */
    int32_t v = out[i];
    j = i;
    while (j > 0 && out[j - 1] > v) { out[j] = out[j - 1]; --j; }
    out[j] = v;
  }
}

/* ------------------------------------------------------------ graph (a1) */
/* Generates the precode and LT neighbour lists.  lt_col capacity must be >= n * max_degree.
 * Returns the LT nnz, or -1 on error. */
/* ------------------------------------------- array LDPC precode (Alg 2, NEXT-2) */
static uint32_t largest_prime_factor(uint32_t x) {
  uint32_t best = 1, d;
  for (d = 2; (uint64_t)d * d <= x; ++d)
    while (x % d == 0) { best = d; x /= d; }
  return x > 1 ? x : best;
}

/* Algorithm 2 for the paper's (b, k) = (our k data symbols, our K = k+p):
 *   P = largest_prime_factor(K), k' = K/P, j' = k' - b/P,
 *   for j < j', i < P, m = 1..k'-j':  l[i+jP][m-1] = k'P - (j'-j+m-1)P - ((m(j'-j-1) - i - 1 + P) mod P) - 1
 * with the mod taken as the non-negative residue (reading R18).  Row r lists the k'-j' members of
 * check r (symbol indices in [0,K): data m < k, check m-k otherwise); the check symbol itself is
 * index k+r, so the group {members, k+r} XORs to zero.  Realizable (Alg 3's conditions): P | b,
 * j' >= 1, k' - j' >= 1, k' <= P.  Returns the members per check, or -1. */
int32_t or_array_precode(uint32_t k, uint32_t K, int32_t *pre_row_ptr, int32_t *pre_col) {
  uint32_t P, kp, jp, j, i, m, d, r = 0;
  if (K <= k || k == 0) return -1;
  P = largest_prime_factor(K);
  if (P < 2 || k % P != 0) return -1;
  kp = K / P;
  jp = kp - k / P;
  if (jp < 1 || kp <= jp || kp > P) return -1;
  d = kp - jp;
  pre_row_ptr[0] = 0;
  for (j = 0; j < jp; ++j)
    for (i = 0; i < P; ++i, ++r) {
      for (m = 1; m <= d; ++m) {
        int64_t inner = (int64_t)m * ((int64_t)jp - j - 1) - i - 1 + P;
        int64_t res = ((inner % P) + P) % P;
        int64_t v = (int64_t)kp * P - ((int64_t)jp - j + m - 1) * P - res - 1;
        pre_col[(size_t)r * d + (m - 1)] = (int32_t)v;
      }
      pre_row_ptr[r + 1] = (int32_t)((r + 1) * d);
    }
  return (int32_t)d;
}

int64_t or_generate_graph_ex(uint32_t k, uint32_t p, uint32_t d_p, uint32_t n, uint64_t seed,
                             int kind, double rsd_c, double rsd_delta,
                             const uint32_t *fin_deg, const double *fin_prob, uint32_t fin_len,
                             int precode_kind, uint32_t files,
                             int32_t *pre_row_ptr, int32_t *pre_col,
                             int32_t *lt_row_ptr, int32_t *lt_col);

int64_t or_generate_graph(uint32_t k, uint32_t p, uint32_t d_p, uint32_t n, uint64_t seed,
                          int kind, double rsd_c, double rsd_delta,
                          const uint32_t *fin_deg, const double *fin_prob, uint32_t fin_len,
                          int32_t *pre_row_ptr, int32_t *pre_col,
                          int32_t *lt_row_ptr, int32_t *lt_col) {
  return or_generate_graph_ex(k, p, d_p, n, seed, kind, rsd_c, rsd_delta, fin_deg, fin_prob, fin_len, 0, 1,
                              pre_row_ptr, pre_col, lt_row_ptr, lt_col);
}

/* precode_kind 0: p random checks of d_p distinct data symbols drawn from the stream (R5, R11);
 * 1: Alg 2 array LDPC checks (deterministic, no stream draws; d_p is implied).
 * files = s output files: "the seed of the i-th output file" -- with
 * s > 1 the n/s rows of file i >= 1 come from a fresh stream seeded seed + i, file 0 continues the
 * base stream (reading R17); s <= 1 is the single stream.  s must divide n.               */
int64_t or_generate_graph_ex(uint32_t k, uint32_t p, uint32_t d_p, uint32_t n, uint64_t seed,
                             int kind, double rsd_c, double rsd_delta,
                             const uint32_t *fin_deg, const double *fin_prob, uint32_t fin_len,
                             int precode_kind, uint32_t files,
                             int32_t *pre_row_ptr, int32_t *pre_col,
                             int32_t *lt_row_ptr, int32_t *lt_col) {
  uint32_t K = k + p, i, j, len;
  uint64_t st = seed;
  int64_t nnz = 0;
  uint32_t *deg;
  double *cdf;
  int r;
  if (k == 0 || n == 0) return -1;
  if (files > 1 && n % files != 0) return -1;
  if (precode_kind == 0 && p > 0 && (d_p == 0 || d_p > k)) return -1;
  if (precode_kind == 1 && (p == 0 || or_array_precode(k, K, pre_row_ptr, pre_col) < 0)) return -1;
  deg = (uint32_t *)malloc(sizeof(uint32_t) * (K + fin_len + 1));
  cdf = (double *)malloc(sizeof(double) * (K + fin_len + 1));
  r = or_build_cdf(kind, K, rsd_c, rsd_delta, fin_deg, fin_prob, fin_len, deg, cdf);
  if (r < 0) { free(deg); free(cdf); return -1; }
  len = (uint32_t)r;
  /* step (1): precode checks first (R5, R11); the array precode draws nothing */
  if (precode_kind == 0) {
    pre_row_ptr[0] = 0;
    for (i = 0; i < p; ++i) {
      draw_neighbours(&st, d_p, k, pre_col + (size_t)i * d_p);
      pre_row_ptr[i + 1] = (int32_t)((i + 1) * d_p);
    }
  }
  /* step (2): LT rows: one degree draw, then the neighbour draws (R5, R12) */
  lt_row_ptr[0] = 0;
  for (j = 0; j < n; ++j) {
    uint32_t d;
    if (files > 1 && j > 0 && j % (n / files) == 0) st = seed + j / (n / files);  /* file i's stream */
    d = draw_degree(&st, deg, cdf, len);
    if (d > K) d = K;
    draw_neighbours(&st, d, K, lt_col + nnz);
    nnz += d;
    lt_row_ptr[j + 1] = (int32_t)nnz;
  }
  free(deg);
  free(cdf);
  return nnz;
}

/* ----------------------------------------------------------- encode (a3, a4) */
static void xor_into(uint8_t *dst, const uint8_t *src, uint64_t t) {
  uint64_t w;
  uint64_t a, b;
  for (w = 0; w + 8 <= t; w += 8) {
    memcpy(&a, dst + w, 8);
    memcpy(&b, src + w, 8);
    a ^= b;
    memcpy(dst + w, &a, 8);
  }
  for (; w < t; ++w) dst[w] ^= src[w];
}

/* One stripe: data k*t -> checks p*t, coded n*t.  Plain definition. */
void or_encode_stripe(uint32_t k, uint32_t p, uint32_t n, uint64_t t,
                      const int32_t *pre_row_ptr, const int32_t *pre_col,
                      const int32_t *lt_row_ptr, const int32_t *lt_col,
                      const uint8_t *data, uint8_t *checks, uint8_t *coded) {
  uint32_t i, j;
  int32_t e;
  /* checks in row order: a member m >= k is an earlier check (array precode, Alg 2) */
  for (i = 0; i < p; ++i) {
    uint8_t *c = checks + (uint64_t)i * t;
    memset(c, 0, t);
    for (e = pre_row_ptr[i]; e < pre_row_ptr[i + 1]; ++e) {
      uint32_t m = (uint32_t)pre_col[e];
      xor_into(c, m < k ? data + (uint64_t)m * t : checks + (uint64_t)(m - k) * t, t);
    }
  }
  for (j = 0; j < n; ++j) {
    uint8_t *y = coded + (uint64_t)j * t;
    memset(y, 0, t);
    for (e = lt_row_ptr[j]; e < lt_row_ptr[j + 1]; ++e) {
      uint32_t m = (uint32_t)lt_col[e];
      const uint8_t *src = (m < k) ? data + (uint64_t)m * t : checks + (uint64_t)(m - k) * t;
      xor_into(y, src, t);
    }
  }
}

/* Stripe loop: the same graph for every stripe, stripes independent. */
void or_encode_stripes(uint32_t S, uint32_t k, uint32_t p, uint32_t n, uint64_t t,
                       const int32_t *pre_row_ptr, const int32_t *pre_col,
                       const int32_t *lt_row_ptr, const int32_t *lt_col,
                       const uint8_t *data, uint64_t data_stride,
                       uint8_t *checks, uint64_t checks_stride,
                       uint8_t *coded, uint64_t coded_stride) {
  uint32_t s;
  for (s = 0; s < S; ++s)
    or_encode_stripe(k, p, n, t, pre_row_ptr, pre_col, lt_row_ptr, lt_col,
                     data + (uint64_t)s * data_stride,
                     p ? checks + (uint64_t)s * checks_stride : checks,
                     coded + (uint64_t)s * coded_stride);
}

/* ---------------------------------------------------------------- decode */
/* Unknowns: the K intermediate symbols I (k data, then p checks).
 * Equations: every received coded symbol j (recv[j] != 0): XOR_{m in N(j)} I_m = Y_j;
 *            every check i: I_{k+i} XOR XOR_{m in P(i)} I_m = 0.
 * Pass A = Algorithm 1 on the LT survivors: sweep the surviving coded
 * symbols g = 0..; after zeroing the rows of recovered symbols, a column of weight 1
 * recovers its remaining neighbour.  Pass B = the same rule on the precode checks
 * ("BP ... at most twice").  Reading (R22): A and B alternate until
 * neither recovers anything.  Then, if use_elim, GF(2) Gauss-Jordan elimination on the
 * residual system recovers every symbol the received equations determine.
 * out_I: K*t bytes.  state[m]: 0 unrecovered, 1 recovered by BP, 2 recovered by elimination.
 * Returns the number of recovered intermediate symbols, -1 on allocation failure. */
static int eq_unknowns(int32_t nmem, const int32_t *mem, const uint8_t *state, int32_t *last) {
  int32_t e, cnt = 0;
  for (e = 0; e < nmem; ++e)
    if (!state[mem[e]]) { ++cnt; *last = mem[e]; }
  return cnt;
}

int64_t or_decode(uint32_t k, uint32_t p, uint32_t n, uint64_t t,
                  const int32_t *pre_row_ptr, const int32_t *pre_col,
                  const int32_t *lt_row_ptr, const int32_t *lt_col,
                  const uint8_t *recv, const uint8_t *coded,
                  int use_elim, uint8_t *out_I, uint8_t *state) {
  uint32_t K = k + p, i, j;
  int progress = 1;
  int64_t recovered = 0;
  int32_t e, *chk = NULL;
  memset(state, 0, K);
  memset(out_I, 0, (size_t)K * t);
  /* precode equation i as a member list: P(i) ++ {k+i} */
  if (p) {
    chk = (int32_t *)malloc(sizeof(int32_t) * ((size_t)pre_row_ptr[p] + p));
    if (!chk) return -1;
  }
  while (progress) {
    progress = 0;
    /* pass A: Algorithm 1 over surviving LT columns */
    for (j = 0; j < n; ++j) {
      int32_t last = -1, cnt;
      if (!recv[j]) continue;
      cnt = eq_unknowns(lt_row_ptr[j + 1] - lt_row_ptr[j], lt_col + lt_row_ptr[j], state, &last);
      if (cnt == 1) {
        uint8_t *dst = out_I + (uint64_t)last * t;
        memcpy(dst, coded + (uint64_t)j * t, t);
        for (e = lt_row_ptr[j]; e < lt_row_ptr[j + 1]; ++e)
          if (lt_col[e] != last) xor_into(dst, out_I + (uint64_t)lt_col[e] * t, t);
        state[last] = 1;
        ++recovered;
        progress = 1;
      }
    }
    /* pass B: the same rule on the precode checks */
    for (i = 0; i < p; ++i) {
      int32_t last = -1, cnt, nm = 0;
      for (e = pre_row_ptr[i]; e < pre_row_ptr[i + 1]; ++e) chk[nm++] = pre_col[e];
      chk[nm++] = (int32_t)(k + i);
      cnt = eq_unknowns(nm, chk, state, &last);
      if (cnt == 1) {
        uint8_t *dst = out_I + (uint64_t)last * t;
        memset(dst, 0, t);
        for (e = 0; e < nm; ++e)
          if (chk[e] != last) xor_into(dst, out_I + (uint64_t)chk[e] * t, t);
        state[last] = 1;
        ++recovered;
        progress = 1;
      }
    }
  }
  if (use_elim && recovered < (int64_t)K) {
    /* residual system over the unrecovered unknowns */
    uint32_t nu = 0, neq = 0, W, r, c, piv_row = 0;
    int32_t *col_of = (int32_t *)malloc(sizeof(int32_t) * K);
    int32_t *unk = (int32_t *)malloc(sizeof(int32_t) * K);
    uint32_t maxeq = 0;
    uint64_t *bits;
    uint8_t *rhs;
    int32_t *pivcol;
    for (i = 0; i < K; ++i) col_of[i] = -1;
    for (i = 0; i < K; ++i)
      if (!state[i]) { col_of[i] = (int32_t)nu; unk[nu++] = (int32_t)i; }
    W = (nu + 63) / 64;
    for (j = 0; j < n; ++j) maxeq += recv[j] ? 1 : 0;
    maxeq += p;
    bits = (uint64_t *)calloc((size_t)maxeq * W, sizeof(uint64_t));
    rhs = (uint8_t *)calloc((size_t)maxeq * t + 1, 1);
    pivcol = (int32_t *)malloc(sizeof(int32_t) * (maxeq + 1));
    if (!col_of || !unk || !bits || !rhs || !pivcol) return -1;
    for (j = 0; j < n; ++j) {
      int any = 0;
      if (!recv[j]) continue;
      memcpy(rhs + (uint64_t)neq * t, coded + (uint64_t)j * t, t);
      for (e = lt_row_ptr[j]; e < lt_row_ptr[j + 1]; ++e) {
        int32_t m = lt_col[e];
        if (state[m]) xor_into(rhs + (uint64_t)neq * t, out_I + (uint64_t)m * t, t);
        else { bits[(size_t)neq * W + col_of[m] / 64] ^= 1ULL << (col_of[m] % 64); any = 1; }
      }
      if (any) ++neq;
    }
    for (i = 0; i < p; ++i) {
      int any = 0;
      int32_t nm = 0;
      for (e = pre_row_ptr[i]; e < pre_row_ptr[i + 1]; ++e) chk[nm++] = pre_col[e];
      chk[nm++] = (int32_t)(k + i);
      memset(rhs + (uint64_t)neq * t, 0, t);
      for (e = 0; e < nm; ++e) {
        int32_t m = chk[e];
        if (state[m]) xor_into(rhs + (uint64_t)neq * t, out_I + (uint64_t)m * t, t);
        else { bits[(size_t)neq * W + col_of[m] / 64] ^= 1ULL << (col_of[m] % 64); any = 1; }
      }
      if (any) ++neq;
    }
    /* Gauss-Jordan over GF(2), payload rows follow the same row operations */
    for (c = 0; c < nu && piv_row < neq; ++c) {
      uint32_t wc = c / 64;
      uint64_t bc = 1ULL << (c % 64);
      uint32_t sel = neq;
      for (r = piv_row; r < neq; ++r)
        if (bits[(size_t)r * W + wc] & bc) { sel = r; break; }
      if (sel == neq) continue;
      if (sel != piv_row) {
        uint32_t w2;
        for (w2 = 0; w2 < W; ++w2) {
          uint64_t tmp = bits[(size_t)sel * W + w2];
          bits[(size_t)sel * W + w2] = bits[(size_t)piv_row * W + w2];
          bits[(size_t)piv_row * W + w2] = tmp;
        }
        {
          uint64_t b;
          for (b = 0; b < t; ++b) {
            uint8_t tmp = rhs[(uint64_t)sel * t + b];
            rhs[(uint64_t)sel * t + b] = rhs[(uint64_t)piv_row * t + b];
            rhs[(uint64_t)piv_row * t + b] = tmp;
          }
        }
      }
      for (r = 0; r < neq; ++r) {
        if (r != piv_row && (bits[(size_t)r * W + wc] & bc)) {
          uint32_t w2;
          for (w2 = 0; w2 < W; ++w2) bits[(size_t)r * W + w2] ^= bits[(size_t)piv_row * W + w2];
          xor_into(rhs + (uint64_t)r * t, rhs + (uint64_t)piv_row * t, t);
        }
      }
      pivcol[piv_row] = (int32_t)c;
      ++piv_row;
    }
    /* a pivot row that is exactly e_c determines unknown c */
    for (r = 0; r < piv_row; ++r) {
      uint32_t w2, pop = 0;
      for (w2 = 0; w2 < W; ++w2) pop += (uint32_t)__builtin_popcountll(bits[(size_t)r * W + w2]);
      if (pop == 1) {
        int32_t m = unk[pivcol[r]];
        memcpy(out_I + (uint64_t)m * t, rhs + (uint64_t)r * t, t);
        state[m] = 2;
        ++recovered;
      }
    }
    free(col_of); free(unk); free(bits); free(rhs); free(pivcol);
  }
  free(chk);
  return recovered;
}

/* ------------------------------------------------- CGA, Algorithm 4 (NEXT-3, repair/update)
 * Check Generation Algorithm, written out step by step on dense 0/1
 * matrices.  B in F2^{K x n}: column j = the neighbours of coded symbol j (the generator matrix
 * of the base code; the paper's k = our K = k+p intermediate symbols,
 * reading R19).  L^{(2,3)} starts as I_n.  Column-major storage:
 * B[j*K + x], L[j*n + s].
 *   while zero_columns(B) < n - K:              (R19: the test counts ZERO columns)
 *     temp = 0
 *     for j in 0..n-1: for i in 0..n-1:
 *       if j != i and 2 w(b_j) > w(b_i):
 *         if w(b_j XOR b_i) < w(b_j): b_j ^= b_i; l_j ^= l_i; temp = 1
 *     if temp == 0: break
 * Returns the number of executed sweeps (passes of the while body).                        */
static uint32_t col_weight(const uint8_t *c, uint32_t len) {
  uint32_t x, w = 0;
  for (x = 0; x < len; ++x) w += c[x];
  return w;
}

int32_t or_cga(uint32_t K, uint32_t n, const int32_t *lt_row_ptr, const int32_t *lt_col,
               uint8_t *B, uint8_t *L) {
  uint32_t i, j, x;
  int32_t e, sweeps = 0;
  memset(B, 0, (size_t)K * n);
  memset(L, 0, (size_t)n * n);
  for (j = 0; j < n; ++j) {
    for (e = lt_row_ptr[j]; e < lt_row_ptr[j + 1]; ++e) B[(size_t)j * K + (uint32_t)lt_col[e]] = 1;
    L[(size_t)j * n + j] = 1;
  }
  for (;;) {
    uint32_t zero = 0;
    int temp = 0;
    for (j = 0; j < n; ++j) zero += col_weight(B + (size_t)j * K, K) == 0;
    if (!((int64_t)zero < (int64_t)n - (int64_t)K)) break;
    ++sweeps;
    for (j = 0; j < n; ++j) {
      uint8_t *bj = B + (size_t)j * K;
      for (i = 0; i < n; ++i) {
        const uint8_t *bi = B + (size_t)i * K;
        uint32_t wj, wx = 0;
        if (i == j) continue;
        wj = col_weight(bj, K);
        if (!(2 * wj > col_weight(bi, K))) continue;
        for (x = 0; x < K; ++x) wx += bj[x] ^ bi[x];
        if (wx < wj) {
          uint8_t *lj = L + (size_t)j * n;
          const uint8_t *li = L + (size_t)i * n;
          for (x = 0; x < K; ++x) bj[x] ^= bi[x];
          for (x = 0; x < n; ++x) lj[x] ^= li[x];
          temp = 1;
        }
      }
    }
    if (!temp) break;
  }
  return sweeps;
}
