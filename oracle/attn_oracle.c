/*
 * oracle/attn_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU attention forward and backward.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this file's shared object.  The product
 * path (paper_2601_21824_b200/, libdash.so) never calls it and shares no
 * code, header, helper or constant with it.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *   Algorithm 1, read per SURVEY.md §8(c) / DESIGN.md "Readings":
 *     S_rc  = scale * sum_k q[r,k] k[c,k]          (causal: key c > query r masked)
 *     L_r   = m_r + log sum_c exp(S_rc - m_r)      natural-log logsumexp (AMB-15)
 *     P_rc  = exp(S_rc - L_r)                      (Alg.1 line 24, AMB-3)
 *     O_r   = sum_c P_rc v_c
 *     D_r   = sum_k dO[r,k] O[r,k]                 (Alg.1 line 1, D in R^N: AMB-2)
 *     dP_rc = sum_k dO[r,k] v[c,k]                 (Alg.1 line 22)
 *     dS_rc = P_rc (dP_rc - D_r)                   (Alg.1 line 24, AMB-3)
 *     dV_c  = sum_r P_rc dO_r                      (Alg.1 line 25)
 *     dK_c  = scale sum_r dS_rc q_r                (Alg.1 line 26; scale: AMB-1)
 *     dQ_r  = scale sum_c dS_rc k_c                (Alg.1 line 28 + the global
 *                                                   reduction over KV, §2.1)
 *   The method reaches exactly this gradient (it only reorders the fp32
 *   reduction of dQ), so the oracle is the plain definition in fp64, row by
 *   row, with no tiling, fusion or reordering.
 *
 * Layout: q, k, v, dout, o, dq, dk, dv are [B][N][H][d] row-major doubles;
 * lse and Dvec are [B][H][N].  Parallelism: OpenMP over (b, h) only; each
 * (b, h) writes disjoint elements, so the result does not depend on the
 * thread count.
 *
 * Pins (tests/test_oracle_attention.py): central finite differences of
 * sum(dO * O), torch float64 scaled_dot_product_attention autograd, the
 * invariants sum_c dK_c = 0, sum_c dV_c = sum_r dO_r, <Q,dQ> = <K,dK>,
 * causal dQ_0 = 0, and the special cases N = 1, causal row 0, equal keys.
 */
#include <math.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static size_t at(int b, int r, int h, int c, int N, int H, int d) {
  return (((size_t)b * N + r) * H + h) * (size_t)d + c;
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Row r of one head: fills s[0..ncols) with scale*q_r.k_c and returns L_r. */
static double row_scores(int b, int h, int r, int N, int H, int d, double scale, int causal,
                         const double* q, const double* k, double* s, int* ncols_out) {
  int ncols = causal ? r + 1 : N;
  double m = -INFINITY;
  for (int c = 0; c < ncols; ++c) {
    double acc = 0.0;
    for (int t = 0; t < d; ++t) acc += q[at(b, r, h, t, N, H, d)] * k[at(b, c, h, t, N, H, d)];
    s[c] = scale * acc;
    if (s[c] > m) m = s[c];
  }
  double sum = 0.0;
  for (int c = 0; c < ncols; ++c) sum += exp(s[c] - m);
  *ncols_out = ncols;
  return m + log(sum);
}

/* Forward: O and natural-log L (Alg.1 "Require" inputs). */
void oracle_attn_fwd(int B, int N, int H, int d, double scale, int causal,
                     const double* q, const double* k, const double* v,
                     double* o, double* lse) {
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int b = 0; b < B; ++b) {
    for (int h = 0; h < H; ++h) {
      double* s = (double*)malloc(sizeof(double) * (size_t)N);
      for (int r = 0; r < N; ++r) {
        int ncols;
        double L = row_scores(b, h, r, N, H, d, scale, causal, q, k, s, &ncols);
        for (int t = 0; t < d; ++t) {
          double acc = 0.0;
          for (int c = 0; c < ncols; ++c) acc += exp(s[c] - L) * v[at(b, c, h, t, N, H, d)];
          o[at(b, r, h, t, N, H, d)] = acc;
        }
        lse[((size_t)b * H + h) * N + r] = L;
      }
      free(s);
    }
  }
}

/* Backward: dQ, dK, dV of loss sum(dO * O).  o_out / lse_out / D_out may be
 * NULL; when given they receive the oracle's own O, L and D. */
void oracle_attn_bwd(int B, int N, int H, int d, double scale, int causal,
                     const double* q, const double* k, const double* v, const double* dout,
                     double* dq, double* dk, double* dv,
                     double* o_out, double* lse_out, double* D_out) {
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int b = 0; b < B; ++b) {
    for (int h = 0; h < H; ++h) {
      double* s = (double*)malloc(sizeof(double) * (size_t)N);
      double* orow = (double*)malloc(sizeof(double) * (size_t)d);
      for (int c = 0; c < N; ++c)
        for (int t = 0; t < d; ++t) {
          dk[at(b, c, h, t, N, H, d)] = 0.0;
          dv[at(b, c, h, t, N, H, d)] = 0.0;
        }
      for (int r = 0; r < N; ++r) {
        int ncols;
        double L = row_scores(b, h, r, N, H, d, scale, causal, q, k, s, &ncols);
        /* P_rc = exp(S_rc - L_r); O_r = sum_c P_rc v_c */
        for (int c = 0; c < ncols; ++c) s[c] = exp(s[c] - L);
        for (int t = 0; t < d; ++t) {
          double acc = 0.0;
          for (int c = 0; c < ncols; ++c) acc += s[c] * v[at(b, c, h, t, N, H, d)];
          orow[t] = acc;
        }
        /* D_r = rowsum(dO o O) */
        double D = 0.0;
        for (int t = 0; t < d; ++t) D += dout[at(b, r, h, t, N, H, d)] * orow[t];
        for (int t = 0; t < d; ++t) dq[at(b, r, h, t, N, H, d)] = 0.0;
        for (int c = 0; c < ncols; ++c) {
          double P = s[c];
          double dP = 0.0;
          for (int t = 0; t < d; ++t) dP += dout[at(b, r, h, t, N, H, d)] * v[at(b, c, h, t, N, H, d)];
          double dS = P * (dP - D);
          for (int t = 0; t < d; ++t) {
            dq[at(b, r, h, t, N, H, d)] += scale * dS * k[at(b, c, h, t, N, H, d)];
            dk[at(b, c, h, t, N, H, d)] += scale * dS * q[at(b, r, h, t, N, H, d)];
            dv[at(b, c, h, t, N, H, d)] += P * dout[at(b, r, h, t, N, H, d)];
          }
        }
        if (o_out)
          for (int t = 0; t < d; ++t) o_out[at(b, r, h, t, N, H, d)] = orow[t];
        if (lse_out) lse_out[((size_t)b * H + h) * N + r] = L;
        if (D_out) D_out[((size_t)b * H + h) * N + r] = D;
      }
      free(orow);
      free(s);
    }
  }
}

/* dQ rows only, for sampled checks at full size: rows[] lists the query
 * rows (per head, same for every (b, h) listed in heads[] as b*H+h).
 * dq_rows is [nheads][nrows][d]. */
void oracle_attn_bwd_dq_rows(int B, int N, int H, int d, double scale, int causal,
                             const double* q, const double* k, const double* v, const double* dout,
                             int nheads, const int* heads, int nrows, const int* rows,
                             double* dq_rows) {
  (void)B;
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int hh = 0; hh < nheads; ++hh) {
    for (int rr = 0; rr < nrows; ++rr) {
      int b = heads[hh] / H, h = heads[hh] % H, r = rows[rr];
      double* s = (double*)malloc(sizeof(double) * (size_t)N);
      double* orow = (double*)malloc(sizeof(double) * (size_t)d);
      int ncols;
      double L = row_scores(b, h, r, N, H, d, scale, causal, q, k, s, &ncols);
      for (int c = 0; c < ncols; ++c) s[c] = exp(s[c] - L);
      for (int t = 0; t < d; ++t) {
        double acc = 0.0;
        for (int c = 0; c < ncols; ++c) acc += s[c] * v[at(b, c, h, t, N, H, d)];
        orow[t] = acc;
      }
      double D = 0.0;
      for (int t = 0; t < d; ++t) D += dout[at(b, r, h, t, N, H, d)] * orow[t];
      double* out = dq_rows + ((size_t)hh * nrows + rr) * d;
      for (int t = 0; t < d; ++t) out[t] = 0.0;
      for (int c = 0; c < ncols; ++c) {
        double dP = 0.0;
        for (int t = 0; t < d; ++t) dP += dout[at(b, r, h, t, N, H, d)] * v[at(b, c, h, t, N, H, d)];
        double dS = s[c] * (dP - D);
        for (int t = 0; t < d; ++t) out[t] += scale * dS * k[at(b, c, h, t, N, H, d)];
      }
      free(orow);
      free(s);
    }
  }
}

/* dK and dV rows only (key rows cols[] of the heads listed in heads[]), for
 * sampled checks at full size.  Needs L_r of every query row first, which
 * this computes by the same row definition.  dk_rows, dv_rows: [nheads][ncols][d]. */
void oracle_attn_bwd_kv_rows(int B, int N, int H, int d, double scale, int causal,
                             const double* q, const double* k, const double* v, const double* dout,
                             int nheads, const int* heads, int ncols_sel, const int* cols,
                             double* dk_rows, double* dv_rows) {
  (void)B;
  double* Lall = (double*)malloc(sizeof(double) * (size_t)nheads * N);
  double* Dall = (double*)malloc(sizeof(double) * (size_t)nheads * N);
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int hh = 0; hh < nheads; ++hh) {
    for (int r = 0; r < N; ++r) {
      int b = heads[hh] / H, h = heads[hh] % H;
      double* s = (double*)malloc(sizeof(double) * (size_t)N);
      int ncols;
      double L = row_scores(b, h, r, N, H, d, scale, causal, q, k, s, &ncols);
      double D = 0.0;
      for (int t = 0; t < d; ++t) {
        double acc = 0.0;
        for (int c = 0; c < ncols; ++c) acc += exp(s[c] - L) * v[at(b, c, h, t, N, H, d)];
        D += dout[at(b, r, h, t, N, H, d)] * acc;
      }
      Lall[(size_t)hh * N + r] = L;
      Dall[(size_t)hh * N + r] = D;
      free(s);
    }
  }
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int hh = 0; hh < nheads; ++hh) {
    for (int cc = 0; cc < ncols_sel; ++cc) {
      int b = heads[hh] / H, h = heads[hh] % H, c = cols[cc];
      double* dko = dk_rows + ((size_t)hh * ncols_sel + cc) * d;
      double* dvo = dv_rows + ((size_t)hh * ncols_sel + cc) * d;
      for (int t = 0; t < d; ++t) { dko[t] = 0.0; dvo[t] = 0.0; }
      for (int r = causal ? c : 0; r < N; ++r) {
        double acc = 0.0;
        for (int t = 0; t < d; ++t) acc += q[at(b, r, h, t, N, H, d)] * k[at(b, c, h, t, N, H, d)];
        double P = exp(scale * acc - Lall[(size_t)hh * N + r]);
        double dP = 0.0;
        for (int t = 0; t < d; ++t) dP += dout[at(b, r, h, t, N, H, d)] * v[at(b, c, h, t, N, H, d)];
        double dS = P * (dP - Dall[(size_t)hh * N + r]);
        for (int t = 0; t < d; ++t) {
          dko[t] += scale * dS * q[at(b, r, h, t, N, H, d)];
          dvo[t] += P * dout[at(b, r, h, t, N, H, d)];
        }
      }
    }
  }
  free(Dall);
  free(Lall);
}
