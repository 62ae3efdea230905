/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the condensed-KKT hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_2405_14236_b200/); neither
 * includes or links the other.
 *
 * Every function follows a plain definition from PAPER.md (arXiv 2405.14236) or the
 * readings recorded in DESIGN.md §3 (numbered R1..R17; they restate SURVEY.md §8(c)):
 *
 *   oracle_condense      K = W + D_x + delta_w I + J^T D J
 *                        D_r = gamma (r < m_eq) else (Ss+dw)/(1+dc(Ss+dw))
 *                        every sum accumulated in __float128, rounded once (R1)
 *   oracle_md_order      MD-exact-v1 minimum degree by literal elimination graph (R11)
 *   oracle_symbolic      etree parent(j) = min{i>j : L_ij != 0}, column counts   (R3 / Liu)
 *   oracle_cholesky      left-looking column Cholesky of P K P^T, no pivoting
 *   oracle_trisolve      L y = P b, L^T z = y, x = P^T z
 *   oracle_solve_refined Richardson refinement with the residual of the
 *                        UNASSEMBLED operator evaluated in __float128 and x carried in
 *                        __float128 (R8/R9): the exact-input solution x_ref.
 *   oracle_hykkt         HyKKT steps 1-3 + __float128 outer refinement on the
 *                        saddle system [K G^T; G 0] -> (dx_ref, dy_ref)
 *   oracle_cg            Hestenes-Stiefel CG (stopping rule R10)
 *   oracle_cr            Hestenes-Stiefel conjugate residuals (same stop rule)
 *   oracle_ldlt          pivot-free LDL^T of P K P^T with inertia counts (P:424-429,
 *                        P:1345-1346; zero-pivot rule R6)    + oracle_ldlt_solve
 *
 * Parity pins for each function live in tests/test_oracle_*.py (-m "not gpu").
 */
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef __float128 q128;

typedef struct {
  int n, m, m_eq;
  const int *Wp, *Wc;      /* W lower CSR (col <= row), n x n                       */
  const double *Wv;
  const int *Jp, *Jc;      /* J CSR, m x n; rows [0, m_eq) are G (weight gamma)      */
  const double *Jv;
  const double *Sx;        /* Sigma_x = D_x [n]                                       */
  const double *Ss;        /* Sigma_s = D_s [m - m_eq]                                */
  const double *D;         /* optional override [m]; NULL -> formula                  */
  double dw, dc, gamma;
} osys;

/* ---------------------------------------------------------------- D_r */
static q128 oracle_Dr(const osys *s, int r) {
  if (s->D) return (q128)s->D[r];
  if (r < s->m_eq) return (q128)s->gamma;
  q128 t = (q128)s->Ss[r - s->m_eq] + (q128)s->dw;      /* D_s + delta_w                 */
  return t / ((q128)1 + (q128)s->dc * t);               /* (D_s + dw) C, C=(1+dc(D_s+dw))^-1 */
}

/* ------------------------------------------------------- sorted-int helpers */
static int cmp_int(const void *a, const void *b) {
  int x = *(const int *)a, y = *(const int *)b;
  return (x > y) - (x < y);
}

/* =====================================================================================
 * Condensation.  Output: lower CSC of K in ORIGINAL indices, rows sorted.
 * Kv == NULL -> pattern only (Kp filled, Ki filled if non-NULL).  Returns nnz(K).
 * ===================================================================================*/
long oracle_condense(const osys *s, int *Kp, int *Ki, double *Kv) {
  const int n = s->n, m = s->m;
  /* column access to W (entries (i,j), i >= j, stored in W row i) */
  int *wtp = calloc(n + 1, sizeof(int));
  int nnzW = s->Wp[n];
  int *wti = malloc(sizeof(int) * (nnzW + 1)), *wtk = malloc(sizeof(int) * (nnzW + 1));
  for (int i = 0; i < n; i++)
    for (int p = s->Wp[i]; p < s->Wp[i + 1]; p++) wtp[s->Wc[p] + 1]++;
  for (int j = 0; j < n; j++) wtp[j + 1] += wtp[j];
  int *fill = malloc(sizeof(int) * (n + 1));
  memcpy(fill, wtp, sizeof(int) * (n + 1));
  for (int i = 0; i < n; i++)
    for (int p = s->Wp[i]; p < s->Wp[i + 1]; p++) {
      int j = s->Wc[p];
      wti[fill[j]] = i; wtk[fill[j]] = p; fill[j]++;
    }
  /* column access to J: for column j the (row, position) pairs */
  int nnzJ = m ? s->Jp[m] : 0;
  int *jtp = calloc(n + 1, sizeof(int));
  int *jtr = malloc(sizeof(int) * (nnzJ + 1)), *jtk = malloc(sizeof(int) * (nnzJ + 1));
  for (int p = 0; p < nnzJ; p++) jtp[s->Jc[p] + 1]++;
  for (int j = 0; j < n; j++) jtp[j + 1] += jtp[j];
  memcpy(fill, jtp, sizeof(int) * (n + 1));
  for (int r = 0; r < m; r++)
    for (int p = s->Jp[r]; p < s->Jp[r + 1]; p++) {
      int j = s->Jc[p];
      jtr[fill[j]] = r; jtk[fill[j]] = p; fill[j]++;
    }
  q128 *acc = malloc(sizeof(q128) * (n > 0 ? n : 1));
  int *mark = malloc(sizeof(int) * (n > 0 ? n : 1));
  int *list = malloc(sizeof(int) * (n > 0 ? n : 1));
  for (int i = 0; i < n; i++) mark[i] = -1;
  long nz = 0;
  if (Kp) Kp[0] = 0;
  for (int j = 0; j < n; j++) {
    int cnt = 0;
#define TOUCH(i) do { if (mark[i] != j) { mark[i] = j; acc[i] = 0; list[cnt++] = (i); } } while (0)
    TOUCH(j);                                                 /* diagonal always present */
    acc[j] += (q128)s->Sx[j] + (q128)s->dw;                   /* D_x + delta_w I           */
    for (int t = wtp[j]; t < wtp[j + 1]; t++) {               /* W_ij, i >= j              */
      int i = wti[t];
      TOUCH(i);
      acc[i] += (q128)s->Wv[wtk[t]];
    }
    for (int t = jtp[j]; t < jtp[j + 1]; t++) {               /* sum_r D_r J_ri J_rj       */
      int r = jtr[t];
      q128 d = oracle_Dr(s, r) * (q128)s->Jv[jtk[t]];
      for (int p = s->Jp[r]; p < s->Jp[r + 1]; p++) {
        int i = s->Jc[p];
        if (i < j) continue;
        TOUCH(i);
        acc[i] += d * (q128)s->Jv[p];
      }
    }
#undef TOUCH
    qsort(list, cnt, sizeof(int), cmp_int);
    for (int t = 0; t < cnt; t++) {
      if (Ki) Ki[nz + t] = list[t];
      if (Kv) Kv[nz + t] = (double)acc[list[t]];              /* one rounding               */
    }
    nz += cnt;
    if (Kp) Kp[j + 1] = (int)nz;
  }
  free(wtp); free(wti); free(wtk); free(fill); free(jtp); free(jtr); free(jtk);
  free(acc); free(mark); free(list);
  return nz;
}

/* =====================================================================================
 * MD-exact-v1 (R11): on the off-diagonal graph of K, repeatedly eliminate
 *   v* = argmin over uneliminated v of (deg(v), v),
 * where deg(v) is v's degree in the CURRENT ELIMINATION GRAPH (= |Reach(v)| through
 * eliminated vertices).  Eliminating v makes its neighbours a clique and deletes v.
 * Literal elimination graph, one vertex at a time, no approximations.
 * perm[k] = original index of the k-th eliminated vertex (new -> old).
 * ===================================================================================*/
typedef struct { int *a; int len, cap; } ivec;

static void iv_reserve(ivec *v, int c) {
  if (c > v->cap) { v->cap = c + c / 2 + 4; v->a = realloc(v->a, sizeof(int) * v->cap); }
}

/* binary min-heap on (deg, vertex) with lazy deletion */
typedef struct { long long *k; int len, cap; } heap;
static void hpush(heap *h, long long key) {
  if (h->len == h->cap) { h->cap = h->cap * 2 + 16; h->k = realloc(h->k, sizeof(long long) * h->cap); }
  int i = h->len++;
  h->k[i] = key;
  while (i > 0) {
    int p = (i - 1) / 2;
    if (h->k[p] <= h->k[i]) break;
    long long t = h->k[p]; h->k[p] = h->k[i]; h->k[i] = t; i = p;
  }
}
static long long hpop(heap *h) {
  long long top = h->k[0];
  h->k[0] = h->k[--h->len];
  int i = 0;
  for (;;) {
    int l = 2 * i + 1, r = l + 1, b = i;
    if (l < h->len && h->k[l] < h->k[b]) b = l;
    if (r < h->len && h->k[r] < h->k[b]) b = r;
    if (b == i) break;
    long long t = h->k[b]; h->k[b] = h->k[i]; h->k[i] = t; i = b;
  }
  return top;
}

int oracle_md_order(int n, const int *Kp, const int *Ki, int *perm) {
  ivec *adj = calloc(n > 0 ? n : 1, sizeof(ivec));
  /* adjacency from the lower CSC pattern (both directions, no diagonal) */
  int *deg0 = calloc(n > 0 ? n : 1, sizeof(int));
  for (int j = 0; j < n; j++)
    for (int p = Kp[j]; p < Kp[j + 1]; p++)
      if (Ki[p] != j) { deg0[j]++; deg0[Ki[p]]++; }
  for (int v = 0; v < n; v++) iv_reserve(&adj[v], deg0[v]);
  for (int j = 0; j < n; j++)
    for (int p = Kp[j]; p < Kp[j + 1]; p++) {
      int i = Ki[p];
      if (i == j) continue;
      adj[j].a[adj[j].len++] = i;
      adj[i].a[adj[i].len++] = j;
    }
  for (int v = 0; v < n; v++) qsort(adj[v].a, adj[v].len, sizeof(int), cmp_int);
  char *elim = calloc(n > 0 ? n : 1, 1);
  heap h = {0};
  for (int v = 0; v < n; v++) hpush(&h, ((long long)adj[v].len << 32) | v);
  int *nb = NULL, nbcap = 0, *tmp = NULL, tmpcap = 0;
  for (int k = 0; k < n; k++) {
    int v;
    for (;;) {                                   /* pop the current argmin (deg, v)   */
      long long key = hpop(&h);
      v = (int)(key & 0xffffffff);
      int d = (int)(key >> 32);
      if (!elim[v] && adj[v].len == d) break;  /* skip stale heap entries           */
    }
    perm[k] = v;
    elim[v] = 1;
    int L = adj[v].len;
    if (L > nbcap) { nbcap = L; nb = realloc(nb, sizeof(int) * nbcap); }
    memcpy(nb, adj[v].a, sizeof(int) * L);      /* N = neighbours of v (sorted)       */
    free(adj[v].a); adj[v].a = NULL; adj[v].len = adj[v].cap = 0;
    for (int t = 0; t < L; t++) {                /* adj(u) <- (adj(u) U N) \ {u, v}    */
      int u = nb[t];
      ivec *A = &adj[u];
      int need = A->len + L;
      if (need > tmpcap) { tmpcap = need; tmp = realloc(tmp, sizeof(int) * tmpcap); }
      int a = 0, b = 0, c = 0;
      while (a < A->len || b < L) {
        int x;
        if (b >= L || (a < A->len && A->a[a] < nb[b])) x = A->a[a++];
        else if (a >= A->len || nb[b] < A->a[a]) x = nb[b++];
        else { x = A->a[a]; a++; b++; }
        if (x == u || x == v) continue;
        tmp[c++] = x;
      }
      iv_reserve(A, c);
      memcpy(A->a, tmp, sizeof(int) * c);
      A->len = c;
      hpush(&h, ((long long)c << 32) | u);
    }
  }
  for (int v = 0; v < n; v++) free(adj[v].a);
  free(adj); free(deg0); free(elim); free(h.k); free(nb); free(tmp);
  return 0;
}

/* =====================================================================================
 * Symbolic factorisation of A = P K P^T by definition:
 *   struct(L_j) = {j} U struct(A_{>j, j}) U  U_{c : parent(c)=j} struct(L_c) \ {c}
 *   parent(j)   = min (struct(L_j) \ {j})   (-1 for a root)
 * Outputs parent[n], colcount[n] (incl. diagonal); optionally the L pattern (Lp, Li)
 * when Lp != NULL (Li sized by sum(colcount)).  Returns nnz(L).
 * ===================================================================================*/
static int *oracle_permuted_lower(int n, const int *Kp, const int *Ki, const int *perm,
                                  int **ApOut) {
  int *iperm = malloc(sizeof(int) * (n > 0 ? n : 1));
  for (int k = 0; k < n; k++) iperm[perm[k]] = k;
  int *Ap = calloc(n + 1, sizeof(int));
  for (int j = 0; j < n; j++)
    for (int p = Kp[j]; p < Kp[j + 1]; p++) {
      int a = iperm[Ki[p]], b = iperm[j];
      int col = a < b ? a : b;
      Ap[col + 1]++;
    }
  for (int j = 0; j < n; j++) Ap[j + 1] += Ap[j];
  int *fill = malloc(sizeof(int) * (n + 1));
  memcpy(fill, Ap, sizeof(int) * (n + 1));
  int *Ai = malloc(sizeof(int) * (Ap[n] + 1));
  for (int j = 0; j < n; j++)
    for (int p = Kp[j]; p < Kp[j + 1]; p++) {
      int a = iperm[Ki[p]], b = iperm[j];
      int col = a < b ? a : b, row = a < b ? b : a;
      Ai[fill[col]++] = row;
    }
  for (int j = 0; j < n; j++) qsort(Ai + Ap[j], Ap[j + 1] - Ap[j], sizeof(int), cmp_int);
  free(iperm); free(fill);
  *ApOut = Ap;
  return Ai;
}

long oracle_symbolic(int n, const int *Kp, const int *Ki, const int *perm, int *parent,
                     int *colcount, int *Lp, int *Li) {
  int *Ap; int *Ai = oracle_permuted_lower(n, Kp, Ki, perm, &Ap);
  ivec *col = calloc(n > 0 ? n : 1, sizeof(ivec));
  int *head = malloc(sizeof(int) * (n > 0 ? n : 1)), *next = malloc(sizeof(int) * (n > 0 ? n : 1));
  for (int j = 0; j < n; j++) head[j] = -1;
  int *mark = malloc(sizeof(int) * (n > 0 ? n : 1));
  for (int j = 0; j < n; j++) mark[j] = -1;
  long nnz = 0;
  int *buf = malloc(sizeof(int) * (n > 0 ? n : 1));
  for (int j = 0; j < n; j++) {
    int c = 0;
    mark[j] = j; buf[c++] = j;
    for (int p = Ap[j]; p < Ap[j + 1]; p++) {
      int i = Ai[p];
      if (mark[i] != j) { mark[i] = j; buf[c++] = i; }
    }
    for (int ch = head[j]; ch != -1; ch = next[ch])
      for (int t = 0; t < col[ch].len; t++) {
        int i = col[ch].a[t];
        if (i > j && mark[i] != j) { mark[i] = j; buf[c++] = i; }
      }
    qsort(buf, c, sizeof(int), cmp_int);
    col[j].a = malloc(sizeof(int) * c); col[j].len = c; col[j].cap = c;
    memcpy(col[j].a, buf, sizeof(int) * c);
    parent[j] = c > 1 ? buf[1] : -1;
    colcount[j] = c;
    nnz += c;
    if (parent[j] >= 0) { next[j] = head[parent[j]]; head[parent[j]] = j; }
  }
  if (Lp) {
    Lp[0] = 0;
    for (int j = 0; j < n; j++) {
      Lp[j + 1] = Lp[j] + col[j].len;
      if (Li) memcpy(Li + Lp[j], col[j].a, sizeof(int) * col[j].len);
    }
  }
  for (int j = 0; j < n; j++) free(col[j].a);
  free(col); free(head); free(next); free(mark); free(buf); free(Ap); free(Ai);
  return nnz;
}

/* =====================================================================================
 * Left-looking column Cholesky of A = P K P^T on the symbolic pattern (Lp, Li), no
 * pivoting.  Returns -1 on success, else the first (permuted) column whose
 * pivot is <= 0 or non-finite (R6).
 * ===================================================================================*/
int oracle_cholesky(int n, const int *Kp, const int *Ki, const double *Kv, const int *perm,
                    const int *Lp, const int *Li, double *Lx) {
  int *iperm = malloc(sizeof(int) * (n > 0 ? n : 1));
  for (int k = 0; k < n; k++) iperm[perm[k]] = k;
  /* A columns with values */
  int *Ap = calloc(n + 1, sizeof(int));
  for (int j = 0; j < n; j++)
    for (int p = Kp[j]; p < Kp[j + 1]; p++) {
      int a = iperm[Ki[p]], b = iperm[j];
      Ap[(a < b ? a : b) + 1]++;
    }
  for (int j = 0; j < n; j++) Ap[j + 1] += Ap[j];
  int *fill = malloc(sizeof(int) * (n + 1)); memcpy(fill, Ap, sizeof(int) * (n + 1));
  int *Ai = malloc(sizeof(int) * (Ap[n] + 1)); double *Ax = malloc(sizeof(double) * (Ap[n] + 1));
  for (int j = 0; j < n; j++)
    for (int p = Kp[j]; p < Kp[j + 1]; p++) {
      int a = iperm[Ki[p]], b = iperm[j];
      int c = a < b ? a : b, r = a < b ? b : a;
      Ai[fill[c]] = r; Ax[fill[c]] = Kv[p]; fill[c]++;
    }
  /* row lists of L: for row i, the (column k, position p) with Li[p] == i, k < i */
  int nnzL = Lp[n];
  int *rp = calloc(n + 1, sizeof(int));
  for (int k = 0; k < n; k++)
    for (int p = Lp[k] + 1; p < Lp[k + 1]; p++) rp[Li[p] + 1]++;
  for (int i = 0; i < n; i++) rp[i + 1] += rp[i];
  int *rk = malloc(sizeof(int) * (nnzL + 1)), *rpos = malloc(sizeof(int) * (nnzL + 1));
  memcpy(fill, rp, sizeof(int) * (n + 1));
  for (int k = 0; k < n; k++)
    for (int p = Lp[k] + 1; p < Lp[k + 1]; p++) {
      int i = Li[p];
      rk[fill[i]] = k; rpos[fill[i]] = p; fill[i]++;
    }
  double *x = calloc(n > 0 ? n : 1, sizeof(double));
  int fail = -1;
  for (int j = 0; j < n && fail < 0; j++) {
    for (int p = Lp[j]; p < Lp[j + 1]; p++) x[Li[p]] = 0.0;
    for (int p = Ap[j]; p < Ap[j + 1]; p++) x[Ai[p]] += Ax[p];
    for (int t = rp[j]; t < rp[j + 1]; t++) {                /* columns k with L_jk != 0 */
      int k = rk[t], p0 = rpos[t];
      double ljk = Lx[p0];
      for (int p = p0; p < Lp[k + 1]; p++) x[Li[p]] -= Lx[p] * ljk;
    }
    double d = x[j];
    if (!(d > 0.0) || !isfinite(d)) { fail = j; break; }
    double ljj = sqrt(d);
    Lx[Lp[j]] = ljj;
    for (int p = Lp[j] + 1; p < Lp[j + 1]; p++) Lx[p] = x[Li[p]] / ljj;
  }
  free(iperm); free(Ap); free(fill); free(Ai); free(Ax); free(rp); free(rk); free(rpos); free(x);
  return fail;
}

/* Pivot-free LDL^T (NEXT-2; P:424-429 inertia, P:1345-1346 the paper's GPU LDL^T) of P K P^T on
 * the symbolic pattern (Lp, Li): left-looking columns, unit-lower L stored below the diagonal slot,
 * d_j in the diagonal slot.  d_j = a_jj - sum_k l_jk^2 d_k ; l_ij = (a_ij - sum_k l_ik d_k l_jk) / d_j.
 * Zero-pivot rule (R6): |d_j| <= 1e-14 |K_jj| counts as zero and d_j is replaced by
 * sign(d_j) max(1e-14 |K_jj|, 1e-300) (sign(0) = +).  inertia[3] = (positive, negative, zero).
 * Returns the first non-finite pivot column or -1. */
int oracle_ldlt(int n, const int *Kp, const int *Ki, const double *Kv, const int *perm,
                const int *Lp, const int *Li, double *Lx, int *inertia) {
  int *iperm = malloc(sizeof(int) * (n > 0 ? n : 1));
  for (int k = 0; k < n; k++) iperm[perm[k]] = k;
  int *Ap = calloc(n + 1, sizeof(int));
  for (int j = 0; j < n; j++)
    for (int p = Kp[j]; p < Kp[j + 1]; p++) {
      int a = iperm[Ki[p]], b = iperm[j];
      Ap[(a < b ? a : b) + 1]++;
    }
  for (int j = 0; j < n; j++) Ap[j + 1] += Ap[j];
  int *fill = malloc(sizeof(int) * (n + 1)); memcpy(fill, Ap, sizeof(int) * (n + 1));
  int *Ai = malloc(sizeof(int) * (Ap[n] + 1)); double *Ax = malloc(sizeof(double) * (Ap[n] + 1));
  double *Kd = calloc(n > 0 ? n : 1, sizeof(double));   /* K_jj in the permuted order */
  for (int j = 0; j < n; j++)
    for (int p = Kp[j]; p < Kp[j + 1]; p++) {
      int a = iperm[Ki[p]], b = iperm[j];
      int c = a < b ? a : b, r = a < b ? b : a;
      Ai[fill[c]] = r; Ax[fill[c]] = Kv[p]; fill[c]++;
      if (a == b) Kd[a] = Kv[p];
    }
  int nnzL = Lp[n];
  int *rp = calloc(n + 1, sizeof(int));
  for (int k = 0; k < n; k++)
    for (int p = Lp[k] + 1; p < Lp[k + 1]; p++) rp[Li[p] + 1]++;
  for (int i = 0; i < n; i++) rp[i + 1] += rp[i];
  int *rk = malloc(sizeof(int) * (nnzL + 1)), *rpos = malloc(sizeof(int) * (nnzL + 1));
  memcpy(fill, rp, sizeof(int) * (n + 1));
  for (int k = 0; k < n; k++)
    for (int p = Lp[k] + 1; p < Lp[k + 1]; p++) {
      int i = Li[p];
      rk[fill[i]] = k; rpos[fill[i]] = p; fill[i]++;
    }
  double *x = calloc(n > 0 ? n : 1, sizeof(double));
  int fail = -1;
  inertia[0] = inertia[1] = inertia[2] = 0;
  for (int j = 0; j < n; j++) {
    for (int p = Lp[j]; p < Lp[j + 1]; p++) x[Li[p]] = 0.0;
    for (int p = Ap[j]; p < Ap[j + 1]; p++) x[Ai[p]] += Ax[p];
    for (int t = rp[j]; t < rp[j + 1]; t++) {                /* columns k with L_jk != 0 */
      int k = rk[t], p0 = rpos[t];
      double w = Lx[p0] * Lx[Lp[k]];                          /* l_jk d_k */
      for (int p = p0; p < Lp[k + 1]; p++) x[Li[p]] -= Lx[p] * w;
    }
    double d = x[j];
    if (!isfinite(d)) { if (fail < 0) fail = j; }
    double thr = 1e-14 * fabs(Kd[j]);
    if (!(fabs(d) > thr)) {
      inertia[2]++;
      double mag = thr > 1e-300 ? thr : 1e-300;
      d = (d < 0) ? -mag : mag;
    } else if (d > 0) inertia[0]++;
    else inertia[1]++;
    Lx[Lp[j]] = d;
    for (int p = Lp[j] + 1; p < Lp[j + 1]; p++) Lx[p] = x[Li[p]] / d;
  }
  free(iperm); free(Ap); free(fill); free(Ai); free(Ax); free(Kd); free(rp); free(rk); free(rpos); free(x);
  return fail;
}

/* L D L^T x = P b with the factor of oracle_ldlt (fp64) */
void oracle_ldlt_solve(int n, const int *Lp, const int *Li, const double *Lx, const int *perm,
                       const double *b, double *x) {
  double *y = malloc(sizeof(double) * (n > 0 ? n : 1));
  for (int k = 0; k < n; k++) y[k] = b[perm[k]];
  for (int j = 0; j < n; j++)
    for (int p = Lp[j] + 1; p < Lp[j + 1]; p++) y[Li[p]] -= Lx[p] * y[j];
  for (int j = 0; j < n; j++) y[j] /= Lx[Lp[j]];
  for (int j = n - 1; j >= 0; j--)
    for (int p = Lp[j] + 1; p < Lp[j + 1]; p++) y[j] -= Lx[p] * y[Li[p]];
  for (int k = 0; k < n; k++) x[perm[k]] = y[k];
  free(y);
}

/* L y = P b ; L^T z = y ; x = P^T z   (fp64) */
void oracle_trisolve(int n, const int *Lp, const int *Li, const double *Lx, const int *perm,
                     const double *b, double *x) {
  double *y = malloc(sizeof(double) * (n > 0 ? n : 1));
  for (int k = 0; k < n; k++) y[k] = b[perm[k]];
  for (int j = 0; j < n; j++) {
    y[j] /= Lx[Lp[j]];
    for (int p = Lp[j] + 1; p < Lp[j + 1]; p++) y[Li[p]] -= Lx[p] * y[j];
  }
  for (int j = n - 1; j >= 0; j--) {
    double s = y[j];
    for (int p = Lp[j] + 1; p < Lp[j + 1]; p++) s -= Lx[p] * y[Li[p]];
    y[j] = s / Lx[Lp[j]];
  }
  for (int k = 0; k < n; k++) x[perm[k]] = y[k];
  free(y);
}

/* =====================================================================================
 * Unassembled operator in __float128 (P:415 written out; R8):
 *   y = W x + (Sx + dw) o x + sum_{r >= r0} J_r^T D_r (J_r x)
 * r0 = 0 for K / K_gamma;  r0 = m_eq excludes the gamma rows (the K of the saddle system).
 * ===================================================================================*/
static void oracle_apply_q(const osys *s, int r0, const q128 *x, q128 *y) {
  int n = s->n;
  for (int i = 0; i < n; i++) y[i] = ((q128)s->Sx[i] + (q128)s->dw) * x[i];
  for (int i = 0; i < n; i++)
    for (int p = s->Wp[i]; p < s->Wp[i + 1]; p++) {
      int j = s->Wc[p];
      q128 w = (q128)s->Wv[p];
      y[i] += w * x[j];
      if (j != i) y[j] += w * x[i];
    }
  for (int r = r0; r < s->m; r++) {
    q128 t = 0;
    for (int p = s->Jp[r]; p < s->Jp[r + 1]; p++) t += (q128)s->Jv[p] * x[s->Jc[p]];
    t *= oracle_Dr(s, r);
    for (int p = s->Jp[r]; p < s->Jp[r + 1]; p++) y[s->Jc[p]] += (q128)s->Jv[p] * t;
  }
}

/* y (double, rounded once) = unassembled operator applied to double x */
void oracle_apply(const osys *s, int exclude_eq, const double *x, double *y) {
  int n = s->n;
  q128 *xq = malloc(sizeof(q128) * (n > 0 ? n : 1)), *yq = malloc(sizeof(q128) * (n > 0 ? n : 1));
  for (int i = 0; i < n; i++) xq[i] = x[i];
  oracle_apply_q(s, exclude_eq ? s->m_eq : 0, xq, yq);
  for (int i = 0; i < n; i++) y[i] = (double)yq[i];
  free(xq); free(yq);
}

/* Richardson refinement, residual and iterate in __float128 (R8/R9).
 * x_hi = rounded solution; x_lo (optional) = (x - x_hi) rounded.  Returns sweeps. */
int oracle_solve_refined(const osys *s, const int *Lp, const int *Li, const double *Lx,
                         const int *perm, const double *b, double *x_hi, double *x_lo,
                         int max_sweeps, double stop_rel) {
  int n = s->n;
  q128 *x = calloc(n > 0 ? n : 1, sizeof(q128)), *y = malloc(sizeof(q128) * (n > 0 ? n : 1));
  double *r = malloc(sizeof(double) * (n > 0 ? n : 1)), *dx = malloc(sizeof(double) * (n > 0 ? n : 1));
  oracle_trisolve(n, Lp, Li, Lx, perm, b, dx);
  for (int i = 0; i < n; i++) x[i] = dx[i];
  int it = 0;
  for (it = 0; it < max_sweeps; it++) {
    oracle_apply_q(s, 0, x, y);
    for (int i = 0; i < n; i++) r[i] = (double)((q128)b[i] - y[i]);
    oracle_trisolve(n, Lp, Li, Lx, perm, r, dx);
    q128 nd = 0, nx = 0;
    for (int i = 0; i < n; i++) {
      x[i] += dx[i];
      q128 a = dx[i] < 0 ? -(q128)dx[i] : (q128)dx[i];
      q128 c = x[i] < 0 ? -x[i] : x[i];
      if (a > nd) nd = a;
      if (c > nx) nx = c;
    }
    if (nd <= (q128)stop_rel * nx) { it++; break; }
  }
  for (int i = 0; i < n; i++) {
    x_hi[i] = (double)x[i];
    if (x_lo) x_lo[i] = (double)(x[i] - (q128)x_hi[i]);
  }
  free(x); free(y); free(r); free(dx);
  return it;
}

/* Backward errors of a candidate x (R7): residual in __float128.
 *   eta   = ||b - K x||_inf / (||K||_inf ||x||_inf + ||b||_inf), ||K||_inf from assembled K
 *   omega = max_i |b - K x|_i / (|W||x| + |Sx+dw||x| + |J|^T|D||J||x| + |b|)_i           */
double oracle_backward_error(const osys *s, const int *Kp, const int *Ki, const double *Kv,
                             const double *b, const double *xd, double *omega_out) {
  int n = s->n;
  q128 *x = malloc(sizeof(q128) * (n > 0 ? n : 1)), *y = malloc(sizeof(q128) * (n > 0 ? n : 1));
  for (int i = 0; i < n; i++) x[i] = xd[i];
  oracle_apply_q(s, 0, x, y);
  /* ||K||_inf: row abs sums over both triangles of the lower CSC */
  q128 *rs = calloc(n > 0 ? n : 1, sizeof(q128));
  for (int j = 0; j < n; j++)
    for (int p = Kp[j]; p < Kp[j + 1]; p++) {
      q128 a = fabsq((q128)Kv[p]);
      rs[Ki[p]] += a;
      if (Ki[p] != j) rs[j] += a;
    }
  q128 nK = 0, nx = 0, nb = 0, nr = 0;
  for (int i = 0; i < n; i++) {
    if (rs[i] > nK) nK = rs[i];
    if (fabsq(x[i]) > nx) nx = fabsq(x[i]);
    if (fabsq((q128)b[i]) > nb) nb = fabsq((q128)b[i]);
    q128 r = fabsq((q128)b[i] - y[i]);
    if (r > nr) nr = r;
  }
  /* componentwise denominators */
  q128 *ax = malloc(sizeof(q128) * (n > 0 ? n : 1)), *den = calloc(n > 0 ? n : 1, sizeof(q128));
  for (int i = 0; i < n; i++) ax[i] = fabsq(x[i]);
  for (int i = 0; i < n; i++) den[i] = fabsq((q128)s->Sx[i] + (q128)s->dw) * ax[i] + fabsq((q128)b[i]);
  for (int i = 0; i < n; i++)
    for (int p = s->Wp[i]; p < s->Wp[i + 1]; p++) {
      int j = s->Wc[p];
      q128 w = fabsq((q128)s->Wv[p]);
      den[i] += w * ax[j];
      if (j != i) den[j] += w * ax[i];
    }
  for (int r = 0; r < s->m; r++) {
    q128 t = 0;
    for (int p = s->Jp[r]; p < s->Jp[r + 1]; p++) t += fabsq((q128)s->Jv[p]) * ax[s->Jc[p]];
    t *= fabsq(oracle_Dr(s, r));
    for (int p = s->Jp[r]; p < s->Jp[r + 1]; p++) den[s->Jc[p]] += fabsq((q128)s->Jv[p]) * t;
  }
  q128 om = 0;
  for (int i = 0; i < n; i++) {
    q128 r = fabsq((q128)b[i] - y[i]);
    q128 w = den[i] > 0 ? r / den[i] : (r > 0 ? (q128)INFINITY : 0);
    if (w > om) om = w;
  }
  if (omega_out) *omega_out = (double)om;
  double eta = (double)(nr / (nK * nx + nb));
  free(x); free(y); free(rs); free(ax); free(den);
  return eta;
}

/* =====================================================================================
 * Conjugate gradient, Hestenes-Stiefel, x0 = 0, stop ||r_k||_2 <= rtol ||r_0||_2
 * (R10).  Returns 0 converged, 1 not converged, 2 breakdown (non-finite).
 * ===================================================================================*/
typedef void (*oracle_op)(void *ctx, const double *x, double *y);

int oracle_cg(int n, oracle_op A, void *ctx, const double *b, double *x, double rtol, int maxit,
              int *iters) {
  double *r = malloc(sizeof(double) * (n > 0 ? n : 1)), *p = malloc(sizeof(double) * (n > 0 ? n : 1));
  double *q = malloc(sizeof(double) * (n > 0 ? n : 1));
  double rr = 0;
  for (int i = 0; i < n; i++) { x[i] = 0; r[i] = b[i]; p[i] = b[i]; rr += b[i] * b[i]; }
  double r0 = sqrt(rr);
  int k = 0, status = 1;
  if (r0 == 0.0) { status = 0; goto done; }
  for (k = 0; k < maxit;) {
    A(ctx, p, q);
    double pq = 0;
    for (int i = 0; i < n; i++) pq += p[i] * q[i];
    double alpha = rr / pq;
    if (!isfinite(alpha)) { status = 2; break; }
    double rr2 = 0;
    for (int i = 0; i < n; i++) { x[i] += alpha * p[i]; r[i] -= alpha * q[i]; rr2 += r[i] * r[i]; }
    k++;
    if (!isfinite(rr2)) { status = 2; break; }
    if (sqrt(rr2) <= rtol * r0) { status = 0; break; }
    double beta = rr2 / rr;
    rr = rr2;
    for (int i = 0; i < n; i++) p[i] = r[i] + beta * p[i];
  }
done:
  if (iters) *iters = k;
  free(r); free(p); free(q);
  return status;
}

/* Conjugate residuals (Hestenes & Stiefel 1952; P:534-535 names CR as the alternative to CG
 * for S_gamma): for SPD A, x0 = 0, r0 = b, p0 = r0, s0 = q0 = A r0;
 *   alpha = (r, s) / (q, q);  x += alpha p;  r -= alpha q;  s' = A r;
 *   beta = (r, s') / (r_old, s_old);  p = r + beta p;  q = s' + beta q.
 * Same stop rule as oracle_cg (R10).  hist (optional, maxit + 1): ||r_k||_2 for k = 0.. */
int oracle_cr(int n, oracle_op A, void *ctx, const double *b, double *x, double rtol, int maxit,
              int *iters, double *hist) {
  size_t sz = sizeof(double) * (n > 0 ? n : 1);
  double *r = malloc(sz), *p = malloc(sz), *q = malloc(sz), *sv = malloc(sz);
  double rr = 0;
  for (int i = 0; i < n; i++) { x[i] = 0; r[i] = b[i]; p[i] = b[i]; rr += b[i] * b[i]; }
  double r0 = sqrt(rr);
  if (hist) hist[0] = r0;
  int k = 0, status = 1;
  if (r0 == 0.0) { status = 0; goto done; }
  A(ctx, r, sv);
  double rs = 0;
  for (int i = 0; i < n; i++) { q[i] = sv[i]; rs += r[i] * sv[i]; }
  for (k = 0; k < maxit;) {
    double qq = 0;
    for (int i = 0; i < n; i++) qq += q[i] * q[i];
    double alpha = rs / qq;
    if (!isfinite(alpha)) { status = 2; break; }
    double rr2 = 0;
    for (int i = 0; i < n; i++) { x[i] += alpha * p[i]; r[i] -= alpha * q[i]; rr2 += r[i] * r[i]; }
    k++;
    if (hist) hist[k] = sqrt(rr2);
    if (!isfinite(rr2)) { status = 2; break; }
    if (sqrt(rr2) <= rtol * r0) { status = 0; break; }
    A(ctx, r, sv);
    double rs2 = 0;
    for (int i = 0; i < n; i++) rs2 += r[i] * sv[i];
    double beta = rs2 / rs;
    rs = rs2;
    for (int i = 0; i < n; i++) { p[i] = r[i] + beta * p[i]; q[i] = sv[i] + beta * q[i]; }
  }
done:
  if (iters) *iters = k;
  free(r); free(p); free(q); free(sv);
  return status;
}

typedef struct { int n; const double *A; } dense_ctx;
static void dense_op(void *c, const double *x, double *y) {
  dense_ctx *d = c;
  for (int i = 0; i < d->n; i++) {
    double s = 0;
    for (int j = 0; j < d->n; j++) s += d->A[(long)i * d->n + j] * x[j];
    y[i] = s;
  }
}
int oracle_cg_dense(int n, const double *A, const double *b, double *x, double rtol, int maxit,
                    int *iters) {
  dense_ctx c = {n, A};
  return oracle_cg(n, dense_op, &c, b, x, rtol, maxit, iters);
}
int oracle_cr_dense(int n, const double *A, const double *b, double *x, double rtol, int maxit,
                    int *iters, double *hist) {
  dense_ctx c = {n, A};
  return oracle_cr(n, dense_op, &c, b, x, rtol, maxit, iters, hist);
}

/* =====================================================================================
 * HyKKT with the factor (Lp,Li,Lx,perm) of K_gamma = K + gamma G^T G, and
 * outer refinement on the saddle system [K G^T; G 0][dx;dy] = [rbar1; rbar2]
 * with residuals in __float128 (R5 of SURVEY §8(c) item 5).
 * ===================================================================================*/
typedef struct {
  const osys *s; const int *Lp, *Li; const double *Lx; const int *perm;
  double *t1, *t2;
} schur_ctx;

static void G_apply(const osys *s, const double *x, double *y) {     /* y = G x  [m_eq] */
  for (int r = 0; r < s->m_eq; r++) {
    double t = 0;
    for (int p = s->Jp[r]; p < s->Jp[r + 1]; p++) t += s->Jv[p] * x[s->Jc[p]];
    y[r] = t;
  }
}
static void GT_apply(const osys *s, const double *y, double *x) {    /* x = G^T y [n]  */
  for (int i = 0; i < s->n; i++) x[i] = 0;
  for (int r = 0; r < s->m_eq; r++)
    for (int p = s->Jp[r]; p < s->Jp[r + 1]; p++) x[s->Jc[p]] += s->Jv[p] * y[r];
}
static void schur_op(void *c, const double *v, double *out) {        /* S_gamma v (eq 14) */
  schur_ctx *S = c;
  GT_apply(S->s, v, S->t1);
  oracle_trisolve(S->s->n, S->Lp, S->Li, S->Lx, S->perm, S->t1, S->t2);
  G_apply(S->s, S->t2, out);
}

/* one pass of HyKKT steps 2-3 for RHS (r1, r2): returns CG status; dx, dy out */
static int oracle_hykkt_pass(const osys *s, schur_ctx *S, const double *r1, const double *r2,
                             double *dx, double *dy, double rtol, int maxit, int *iters) {
  int n = s->n, me = s->m_eq;
  double *sg = malloc(sizeof(double) * (n > 0 ? n : 1)), *t = malloc(sizeof(double) * (n > 0 ? n : 1));
  double *rhs = malloc(sizeof(double) * (me > 0 ? me : 1));
  GT_apply(s, r2, t);
  for (int i = 0; i < n; i++) sg[i] = r1[i] + s->gamma * t[i];      /* rbar1 + gamma G^T rbar2 */
  oracle_trisolve(n, S->Lp, S->Li, S->Lx, S->perm, sg, t);
  G_apply(s, t, rhs);
  for (int r = 0; r < me; r++) rhs[r] -= r2[r];                     /* G K_g^-1 s - rbar2     */
  int st = oracle_cg(me, schur_op, S, rhs, dy, rtol, maxit, iters);
  GT_apply(s, dy, t);
  for (int i = 0; i < n; i++) t[i] = sg[i] - t[i];                  /* s - G^T dy             */
  oracle_trisolve(n, S->Lp, S->Li, S->Lx, S->perm, t, dx);
  free(sg); free(t); free(rhs);
  return st;
}

int oracle_hykkt(const osys *s, const int *Lp, const int *Li, const double *Lx, const int *perm,
                 const double *rbar1, const double *rbar2, double *dx_out, double *dy_out,
                 double cg_rtol, int cg_maxit, int max_outer, int *cg_iters_first, int *outer_out) {
  int n = s->n, me = s->m_eq;
  schur_ctx S = {s, Lp, Li, Lx, perm, malloc(sizeof(double) * (n > 0 ? n : 1)),
                 malloc(sizeof(double) * (n > 0 ? n : 1))};
  double *dx = malloc(sizeof(double) * (n > 0 ? n : 1)), *dy = malloc(sizeof(double) * (me > 0 ? me : 1));
  int it0 = 0;
  int st = oracle_hykkt_pass(s, &S, rbar1, rbar2, dx, dy, cg_rtol, cg_maxit, &it0);
  if (cg_iters_first) *cg_iters_first = it0;
  q128 *X = malloc(sizeof(q128) * (n > 0 ? n : 1)), *Y = malloc(sizeof(q128) * (me > 0 ? me : 1));
  q128 *KX = malloc(sizeof(q128) * (n > 0 ? n : 1));
  double *r1 = malloc(sizeof(double) * (n > 0 ? n : 1)), *r2 = malloc(sizeof(double) * (me > 0 ? me : 1));
  for (int i = 0; i < n; i++) X[i] = dx[i];
  for (int r = 0; r < me; r++) Y[r] = dy[r];
  int k;
  for (k = 0; k < max_outer; k++) {
    /* rho1 = rbar1 - K X - G^T Y ; rho2 = rbar2 - G X  (K excludes the gamma rows) */
    oracle_apply_q(s, s->m_eq, X, KX);
    for (int r = 0; r < me; r++)
      for (int p = s->Jp[r]; p < s->Jp[r + 1]; p++) KX[s->Jc[p]] += (q128)s->Jv[p] * Y[r];
    for (int i = 0; i < n; i++) r1[i] = (double)((q128)rbar1[i] - KX[i]);
    for (int r = 0; r < me; r++) {
      q128 t = 0;
      for (int p = s->Jp[r]; p < s->Jp[r + 1]; p++) t += (q128)s->Jv[p] * X[s->Jc[p]];
      r2[r] = (double)((q128)rbar2[r] - t);
    }
    int itk = 0;
    oracle_hykkt_pass(s, &S, r1, r2, dx, dy, cg_rtol, cg_maxit, &itk);
    q128 nd = 0, nx = 0;
    for (int i = 0; i < n; i++) {
      X[i] += dx[i];
      if (fabsq((q128)dx[i]) > nd) nd = fabsq((q128)dx[i]);
      if (fabsq(X[i]) > nx) nx = fabsq(X[i]);
    }
    for (int r = 0; r < me; r++) {
      Y[r] += dy[r];
      if (fabsq((q128)dy[r]) > nd) nd = fabsq((q128)dy[r]);
      if (fabsq(Y[r]) > nx) nx = fabsq(Y[r]);
    }
    if (nd <= (q128)1e-25 * nx) { k++; break; }
  }
  if (outer_out) *outer_out = k;
  for (int i = 0; i < n; i++) dx_out[i] = (double)X[i];
  for (int r = 0; r < me; r++) dy_out[r] = (double)Y[r];
  free(S.t1); free(S.t2); free(dx); free(dy); free(X); free(Y); free(KX); free(r1); free(r2);
  return st;
}
