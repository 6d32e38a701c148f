/* oracle/oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain C99, double precision, no SIMD, no blocking or fusion, built with
 * -O2 and without -ffast-math. Every function cites the passage it follows.
 *
 * Why naive recursion is the right oracle: properties P.1-P.3 (PAPER.md
 * P:753-771) make any children-before-parent order produce the values of the
 * plain recursive definition; dynamic batching only
 * reorders independent work. So the forward oracle is the recursive
 * definition itself, and the linearization oracle is the definition of the
 * numbering written out with naive loops.
 *
 * MUT(k): the mutation check (tests/test_oracle_mutations.py) rebuilds this
 * file with -DCX_ORACLE_MUTATION=k, each k one plausible bug (a dropped term,
 * a swapped operand, a wrong index), and asserts that some pin fails. The
 * default build has CX_ORACLE_MUTATION = 0: every MUT(k) is false.
 */
#include "oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef CX_ORACLE_MUTATION
#define CX_ORACLE_MUTATION 0
#endif
#define MUT(k) (CX_ORACLE_MUTATION == (k))

/* ------------------------------------------------------------------------ */
/* error latch: lowest (code, node) wins (SURVEY §8(c) "Error reporting")    */
/* ------------------------------------------------------------------------ */
static void latch(int *code, int32_t *node, int c, int32_t n) {
  if (*code == OR_OK || c < *code || (c == *code && n < *node)) {
    *code = c;
    *node = n;
  }
}

/* number of present children of input node v (children form a prefix) */
static int child_count(const int32_t *ch, int32_t n, int32_t maxc, int32_t v) {
  int k = 0;
  while (k < maxc && ch[(int64_t)k * n + v] != -1) k++;
  return k;
}

/* ------------------------------------------------------------------------ */
/* a1: validation ("maximum number of children per node, and the  */
/* kind ... can be easily verified at runtime"; readings Q7, Q20)            */
/* ------------------------------------------------------------------------ */
static void validate(const int32_t *ch, int32_t n, int32_t maxc, int32_t kind,
                     int32_t *indeg, int *code, int32_t *bad) {
  for (int32_t v = 0; v < n; v++) indeg[v] = 0;
  for (int32_t v = 0; v < n; v++) {
    for (int k = 0; k < maxc; k++) {
      int32_t c = ch[(int64_t)k * n + v];
      if (c != -1 && (c < 0 || c >= n)) latch(code, bad, OR_E_CHILD_RANGE, v);
      if (c == -1) {
        for (int k2 = k + 1; k2 < maxc; k2++)
          if (ch[(int64_t)k2 * n + v] != -1) latch(code, bad, OR_E_CHILD_LAYOUT, v);
      }
      if (c >= 0 && c < n) {
        indeg[c]++;
        for (int k2 = k + 1; k2 < maxc; k2++)
          if (ch[(int64_t)k2 * n + v] == c) latch(code, bad, OR_E_KIND, v); /* duplicate */
      }
    }
  }
  if (kind != OR_DAG)
    for (int32_t v = 0; v < n; v++)
      if (indeg[v] > 1) latch(code, bad, OR_E_KIND, v); /* two parents in a tree/sequence */
}

/* ------------------------------------------------------------------------ */
/* a2: heights (pseudocode P:1069-1085 batches nodes by node.height; Q6:     */
/* height(leaf) = 0, height(v) = 1 + max over children). Memoized recursion  */
/* with three colours, written with an explicit stack so 10^5-long chains    */
/* do not overflow the C stack. Returns the lowest node whose height is      */
/* undefined (on or reaching a cycle), or -1.                                */
/* ------------------------------------------------------------------------ */
enum { WHITE = 0, GREY = 1, DONE = 2, UNDEF = 3 };

static int32_t heights(const int32_t *ch, int32_t n, int32_t maxc, int32_t *height) {
  unsigned char *col = calloc((size_t)n + 1, 1);
  int32_t *stk = malloc(sizeof(int32_t) * ((size_t)n + 1));
  int *slot = malloc(sizeof(int) * ((size_t)n + 1));
  for (int32_t root = 0; root < n; root++) {
    if (col[root] != WHITE) continue;
    int32_t sp = 0;
    stk[sp] = root; slot[sp] = 0; col[root] = GREY; height[root] = 0;
    while (sp >= 0) {
      int32_t v = stk[sp];
      int k = slot[sp];
      if (k < maxc && ch[(int64_t)k * n + v] != -1) {
        int32_t c = ch[(int64_t)k * n + v];
        slot[sp] = k + 1;
        if (col[c] == WHITE) {          /* recurse into the child */
          sp++; stk[sp] = c; slot[sp] = 0; col[c] = GREY; height[c] = 0;
        } else if (col[c] == GREY || col[c] == UNDEF) {
          col[v] = UNDEF;               /* back edge or reaches a cycle */
        } else if (col[v] != UNDEF && height[c] + 1 > height[v]) {
          height[v] = height[c] + 1;
        }
        continue;
      }
      /* all children visited: v is finished */
      if (col[v] != UNDEF) col[v] = DONE;
      sp--;
      if (sp >= 0) {
        int32_t p = stk[sp];
        if (col[v] == UNDEF) col[p] = UNDEF;
        else if (col[p] != UNDEF && height[v] + 1 > height[p]) height[p] = height[v] + 1;
      }
    }
  }
  int32_t bad = -1;
  for (int32_t v = 0; v < n; v++)
    if (col[v] == UNDEF) { bad = v; break; }
  free(col); free(stk); free(slot);
  return bad;
}

/* ------------------------------------------------------------------------ */
/* a3-a5: numbering (nodes of a batch numbered consecutively    */
/* and higher than their parents, leaves higher than all internal nodes;     */
/* P:2061-2065 batch_begin/batch_length). Q4: ascending input id inside a    */
/* level. Q5: root-most level first. Deliberately naive O(N*L) loops.        */
/* ------------------------------------------------------------------------ */
int oracle_linearize(const int32_t *children, int32_t n, int32_t maxc, int32_t kind,
                     oracle_lin_header *hdr, int32_t *perm, int32_t *inv,
                     int32_t *children_new, int32_t *height_new, int32_t *level_begin,
                     int32_t *level_size, int32_t *roots, int32_t *structure) {
  memset(hdr, 0, sizeof *hdr);
  hdr->bad_node = -1;
  hdr->num_nodes = n;
  if (n < 0 || maxc < 1 || kind < 0 || kind > 2 || (kind == OR_SEQUENCE && maxc != 1)) {
    hdr->status = OR_E_ARG;
    return hdr->status;
  }
  if (n == 0) return OR_OK;

  int code = OR_OK;
  int32_t bad = -1;
  int32_t *indeg = malloc(sizeof(int32_t) * (size_t)n);
  validate(children, n, maxc, kind, indeg, &code, &bad);
  if (code != OR_OK) {
    hdr->status = code; hdr->bad_node = bad;
    free(indeg);
    return code;
  }
  int32_t *h = malloc(sizeof(int32_t) * (size_t)n);
  int32_t cyc = heights(children, n, maxc, h);
  if (cyc >= 0) {
    hdr->status = OR_E_CYCLE; hdr->bad_node = cyc;
    free(indeg); free(h);
    return OR_E_CYCLE;
  }

  int32_t L = 0;
  for (int32_t v = 0; v < n; v++) if (h[v] + 1 > L) L = h[v] + 1;
  for (int32_t l = 0; l < L; l++) level_size[l] = 0;
  for (int32_t v = 0; v < n; v++) level_size[h[v]]++;
  int32_t acc = 0, maxsz = 0;
  for (int32_t l = L - 1; l >= 0; l--) {
    if (MUT(10)) { level_begin[L - 1 - l] = acc; acc += level_size[L - 1 - l]; continue; }
    level_begin[l] = acc;
    acc += level_size[l];
    if (level_size[l] > maxsz) maxsz = level_size[l];
  }
  int32_t next = 0;
  for (int32_t l = L - 1; l >= 0; l--)
    for (int32_t v = 0; v < n; v++) {
      const int32_t u = MUT(9) ? n - 1 - v : v;
      if (h[u] == l) perm[next++] = u;
    }
  for (int32_t i = 0; i < n; i++) inv[perm[i]] = i;
  for (int k = 0; k < maxc; k++)
    for (int32_t i = 0; i < n; i++) {
      int32_t c = children[(int64_t)k * n + perm[i]];
      children_new[(int64_t)k * n + i] = (c == -1) ? -1 : inv[c];
    }
  for (int32_t i = 0; i < n; i++) height_new[i] = h[perm[i]];
  int32_t r = 0;
  for (int32_t v = 0; v < n; v++)
    if (indeg[v] == 0) roots[r++] = inv[v];
  /* structures (P.3 P:759-761: independent structures): roots in ascending
     index r each claim every not-yet-claimed node they reach (explicit-stack
     DFS), so a node belongs to the smallest r whose root reaches it. */
  {
    int32_t *own = malloc(sizeof(int32_t) * (size_t)n);
    int32_t *stk = malloc(sizeof(int32_t) * (size_t)n);
    for (int32_t v = 0; v < n; v++) own[v] = -1;
    for (int32_t q = 0; q < r; q++) {
      int32_t sp = 0, root = perm[roots[q]];
      if (own[root] >= 0) continue;
      own[root] = q;
      stk[sp++] = root;
      while (sp > 0) {
        int32_t v = stk[--sp];
        for (int k = 0; k < maxc; k++) {
          int32_t c = children[(int64_t)k * n + v];
          if (c == -1) break;
          if (own[c] < 0) { own[c] = q; stk[sp++] = c; }
        }
      }
    }
    for (int32_t i = 0; i < n; i++) structure[i] = own[perm[i]];
    free(own); free(stk);
  }

  hdr->status = OR_OK;
  hdr->num_levels = L;
  hdr->num_leaves = level_size[0];
  hdr->first_leaf = n - level_size[0];
  hdr->max_level_size = maxsz;
  hdr->num_roots = r;
  free(indeg); free(h);
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Forward cells (SURVEY §8(c) cell table). sigma(x) = 1/(1+e^-x); dot        */
/* products run sequentially over the input index; child sums in position    */
/* order.                                                                    */
/* ------------------------------------------------------------------------ */
static double sigm(double x) { return 1.0 / (1.0 + exp(-x)); }

/* y[r] = sum_k W[(row0 + r) * ld + col0 + k] * x[k] for r < rows, k < K */
static void matvec(const float *W, int64_t ld, int64_t row0, int64_t col0, int rows, int K,
                   const double *x, double *y) {
  for (int r = 0; r < rows; r++) {
    double s = 0.0;
    for (int k = 0; k < K; k++) s += (double)W[(row0 + r) * ld + col0 + k] * x[k];
    y[r] = s;
  }
}

typedef struct {
  int32_t cell, H, V, n, maxc;
  const float *const *w;
  const float *emb;
  const int32_t *words;
  const int32_t *ch;
  double *h;    /* [n][H] */
  double *c;    /* TreeLSTM memory cell [n][H] */
  double *A;    /* MV-RNN matrices [n][H][H] */
  double *tmp;  /* scratch, 8*H + 4*H*H */
  int code;
  int32_t bad;
} fwd_ctx;

/* x_v = Emb[word[v]] or NULL after latching CX_E_WORD_RANGE (Q16) */
static int load_x(fwd_ctx *F, int32_t v, double *x) {
  int32_t w = F->words[v];
  if (w < 0 || w >= F->V) { latch(&F->code, &F->bad, OR_E_WORD_RANGE, v); return 0; }
  for (int i = 0; i < F->H; i++) x[i] = (double)F->emb[(int64_t)w * F->H + i];
  return 1;
}

/* Evaluate node v; all its children are already evaluated. */
static void eval_node(fwd_ctx *F, int32_t v) {
  const int H = F->H;
  const int nc = child_count(F->ch, F->n, F->maxc, v);
  double *hv = F->h + (int64_t)v * H;
  double *x = F->tmp, *ht = F->tmp + H, *g = F->tmp + 2 * H; /* g: up to 4H */
  const float *const *W = F->w;
  int binary = (F->cell == OR_TREERNN || F->cell == OR_TREEFC || F->cell == OR_MVRNN);
  if (binary && nc != 0 && nc != 2) {
    latch(&F->code, &F->bad, OR_E_ARITY, v);
    for (int i = 0; i < H; i++) hv[i] = 0.0;
    return;
  }
  /* child-sum h~ = sum_k h_k (empty sum = 0) */
  for (int i = 0; i < H; i++) ht[i] = 0.0;
  for (int k = 0; k < nc; k++) {
    const double *hk = F->h + (int64_t)F->ch[(int64_t)k * F->n + v] * H;
    for (int i = 0; i < H; i++) ht[i] += hk[i];
  }

  switch (F->cell) {
  case OR_TREERNN: /* Listing 1: leaf Emb[words[n]], internal tanh(lh + rh) */
    if (nc == 0) {
      if (!load_x(F, v, x)) { for (int i = 0; i < H; i++) hv[i] = 0.0; return; }
      for (int i = 0; i < H; i++) hv[i] = x[i];
    } else {
      const double *hl = F->h + (int64_t)F->ch[v] * H;
      const double *hr = F->h + (int64_t)F->ch[(int64_t)F->n + v] * H;
      for (int i = 0; i < H; i++) hv[i] = tanh(hl[i] + hr[i]);
    }
    break;

  case OR_TREEFC: /* Q2: h = tanh(W [h_l; h_r] + b), W in R^{H x 2H}; leaf = Emb */
    if (nc == 0) {
      if (!load_x(F, v, x)) { for (int i = 0; i < H; i++) hv[i] = 0.0; return; }
      for (int i = 0; i < H; i++) hv[i] = x[i];
    } else {
      const double *hl = F->h + (int64_t)F->ch[v] * H;
      const double *hr = F->h + (int64_t)F->ch[(int64_t)F->n + v] * H;
      for (int r = 0; r < H; r++) {
        double s = 0.0;
        const double *h0 = MUT(6) ? hr : hl, *h1 = MUT(6) ? hl : hr;
        for (int k = 0; k < H; k++) s += (double)W[0][(int64_t)r * 2 * H + k] * h0[k];
        for (int k = 0; k < H; k++) s += (double)W[0][(int64_t)r * 2 * H + H + k] * h1[k];
        hv[r] = tanh(s + (double)W[1][r]);
      }
    }
    break;

  case OR_TREELSTM: { /* Q1: child-sum TreeLSTM [Tai et al.] */
    double *cv = F->c + (int64_t)v * H;
    if (nc == 0) { /* [i;o;u] = W_iou x + b_iou */
      if (!load_x(F, v, x)) { for (int i = 0; i < H; i++) hv[i] = cv[i] = 0.0; return; }
      matvec(W[0], H, 0, 0, 3 * H, H, x, g);
    } else {       /* [i;o;u] = U_iou h~ + b_iou */
      matvec(W[1], H, 0, 0, 3 * H, H, ht, g);
    }
    for (int r = 0; r < 3 * H; r++) g[r] += (double)W[2][r];
    for (int i = 0; i < H; i++)
      cv[i] = sigm(g[i]) * (MUT(8) && nc == 0 ? sigm(g[2 * H + i]) : tanh(g[2 * H + i]));
    for (int k = 0; k < nc; k++) { /* f_k = sigma(U_f h_k + b_f); c += f_k * c_k */
      int32_t ck = F->ch[(int64_t)k * F->n + v];
      double *f = g + 3 * H; /* reuse the tail of the 4H scratch */
      matvec(W[3], H, 0, 0, H, H, MUT(1) ? ht : F->h + (int64_t)ck * H, f);
      if (MUT(13)) ck = F->ch[(int64_t)((k + 1) % nc) * F->n + v];
      for (int i = 0; i < H; i++)
        cv[i] += sigm(f[i] + (double)W[4][i]) * F->c[(int64_t)ck * H + i];
    }
    for (int i = 0; i < H; i++) hv[i] = sigm(g[H + i]) * tanh(cv[i]);
    break;
  }

  case OR_TREEGRU:         /* Q3: child-sum TreeGRU, reset gate per child before U_h */
  case OR_SIMPLETREEGRU: { /* Q24 (footnote P:1638-1640): h = (1 - z) h' at internal nodes */
    double *z = g, *s = g + H, *t = g + 2 * H, *r = g + 3 * H;
    if (nc == 0) { /* z = sigma(W_z x + b_z); g = tanh(W_h x + b_h); h = (1-z) g */
      if (!load_x(F, v, x)) { for (int i = 0; i < H; i++) hv[i] = 0.0; return; }
      matvec(W[0], H, 0, 0, H, H, x, z);
      matvec(W[0], H, H, 0, H, H, x, t);
      for (int i = 0; i < H; i++) {
        double zz = sigm(z[i] + (double)W[4][i]);
        double gg = tanh(t[i] + (double)W[6][i]);
        hv[i] = MUT(14) ? zz * gg : (1.0 - zz) * gg;
      }
    } else {
      matvec(W[1], H, 0, 0, H, H, ht, z);               /* U_z h~ */
      for (int i = 0; i < H; i++) s[i] = 0.0;
      for (int k = 0; k < nc; k++) {                    /* s = sum_k r_k * h_k */
        const double *hk = F->h + (int64_t)F->ch[(int64_t)k * F->n + v] * H;
        const double *rk = MUT(5) ? ht : hk;             /* (mutation: reset on h~) */
        matvec(W[2], H, 0, 0, H, H, rk, r);             /* U_r h_k */
        for (int i = 0; i < H; i++) s[i] += sigm(r[i] + (double)W[5][i]) * rk[i];
        if (MUT(5)) break;
      }
      matvec(W[3], H, 0, 0, H, H, s, t);                /* U_h s */
      for (int i = 0; i < H; i++) {
        double zz = sigm(z[i] + (double)W[4][i]);
        double gg = tanh(t[i] + (double)W[6][i]);
        if (F->cell == OR_SIMPLETREEGRU && !MUT(11)) hv[i] = (1.0 - zz) * gg;
        else if (MUT(3)) hv[i] = (1.0 - zz) * ht[i] + zz * gg;
        else hv[i] = zz * ht[i] + (1.0 - zz) * gg;
      }
    }
    break;
  }

  case OR_MVRNN: { /* Q9: [Socher et al. 2012] a = tanh(W [B a; A b] + beta), A = W_M [A; B] */
    double *Av = F->A + (int64_t)v * H * H;
    if (nc == 0) {
      int32_t w = F->words[v];
      if (!load_x(F, v, x)) {
        for (int i = 0; i < H; i++) hv[i] = 0.0;
        for (int64_t i = 0; i < (int64_t)H * H; i++) Av[i] = 0.0;
        return;
      }
      for (int i = 0; i < H; i++) hv[i] = x[i];
      for (int64_t i = 0; i < (int64_t)H * H; i++) Av[i] = (double)W[0][(int64_t)w * H * H + i];
    } else {
      int32_t l = F->ch[v], rr = F->ch[(int64_t)F->n + v];
      const double *a = F->h + (int64_t)l * H, *b = F->h + (int64_t)rr * H;
      const double *Al = F->A + (int64_t)l * H * H, *Br = F->A + (int64_t)rr * H * H;
      double *p = g; /* [B a; A b], 2H */
      for (int i = 0; i < H; i++) {
        double s1 = 0.0, s2 = 0.0;
        const double *m1 = MUT(2) ? Al : Br, *m2 = MUT(2) ? Br : Al;
        for (int k = 0; k < H; k++)
          s1 += (MUT(12) ? m1[(int64_t)k * H + i] : m1[(int64_t)i * H + k]) * a[k];
        for (int k = 0; k < H; k++) s2 += m2[(int64_t)i * H + k] * b[k];
        p[i] = s1; p[H + i] = s2;
      }
      for (int i = 0; i < H; i++) {
        double s = 0.0;
        for (int k = 0; k < 2 * H; k++) s += (double)W[1][(int64_t)i * 2 * H + k] * p[k];
        hv[i] = tanh(s + (double)W[2][i]);
      }
      for (int i = 0; i < H; i++)
        for (int j = 0; j < H; j++) {
          double s = 0.0;
          for (int k = 0; k < H; k++)
            s += (double)W[3][(int64_t)i * 2 * H + k] * (MUT(4) ? Al[(int64_t)j * H + k] : Al[(int64_t)k * H + j]);
          for (int k = 0; k < H; k++)
            s += (double)W[3][(int64_t)i * 2 * H + H + k] * (MUT(4) ? Br[(int64_t)j * H + k] : Br[(int64_t)k * H + j]);
          Av[(int64_t)i * H + j] = s;
        }
    }
    break;
  }

  case OR_DAGRNN: { /* Q8: h = tanh(W_x x + U h~ + b), every node has an input */
    if (!load_x(F, v, x)) { for (int i = 0; i < H; i++) hv[i] = 0.0; return; }
    matvec(W[0], H, 0, 0, H, H, x, g);
    if (MUT(7) && nc > 0) for (int i = 0; i < H; i++) g[i] = 0.0;
    matvec(W[1], H, 0, 0, H, H, ht, g + H);
    for (int i = 0; i < H; i++) hv[i] = tanh(g[i] + g[H + i] + (double)W[2][i]);
    break;
  }
  }
}

/* Memoized recursion eval(v) (each node evaluated once, so it
 * is DAG-safe), written with an explicit stack: v is evaluated after all of
 * its children have been. */
static int forward_impl(int32_t cell, int32_t H, int32_t V, const float *const *weights,
                        const float *emb, const int32_t *words, const int32_t *children,
                        int32_t n, int32_t maxc, const int32_t *targets, int32_t n_targets,
                        double *h_out, double *aux_out, int32_t *bad_node) {
  fwd_ctx F;
  memset(&F, 0, sizeof F);
  F.cell = cell; F.H = H; F.V = V; F.n = n; F.maxc = maxc;
  F.w = weights; F.emb = emb; F.words = words; F.ch = children;
  F.h = h_out; F.code = OR_OK; F.bad = -1;
  int own_aux = 0;
  if (cell == OR_TREELSTM) {
    F.c = aux_out ? aux_out : malloc(sizeof(double) * (size_t)n * H);
    own_aux = aux_out == NULL;
  } else if (cell == OR_MVRNN) {
    F.A = aux_out ? aux_out : malloc(sizeof(double) * (size_t)n * H * H);
    own_aux = aux_out == NULL;
  }
  F.tmp = malloc(sizeof(double) * (8 * (size_t)H + 8));
  unsigned char *done = calloc((size_t)n + 1, 1);
  int32_t *stk = malloc(sizeof(int32_t) * ((size_t)n + 1));
  int *slot = malloc(sizeof(int) * ((size_t)n + 1));

  int32_t count = targets ? n_targets : n;
  for (int32_t t = 0; t < count; t++) {
    int32_t root = targets ? targets[t] : t;
    if (done[root]) continue;
    int32_t sp = 0;
    stk[0] = root; slot[0] = 0;
    while (sp >= 0) {
      int32_t v = stk[sp];
      int k = slot[sp];
      if (k < maxc && children[(int64_t)k * n + v] != -1) {
        int32_t c = children[(int64_t)k * n + v];
        slot[sp] = k + 1;
        if (!done[c]) { sp++; stk[sp] = c; slot[sp] = 0; }
        continue;
      }
      if (!done[v]) { eval_node(&F, v); done[v] = 1; }
      sp--;
    }
  }
  free(done); free(stk); free(slot); free(F.tmp);
  if (own_aux) { free(F.c); free(F.A); }
  if (bad_node) *bad_node = F.bad;
  return F.code;
}

int oracle_forward(int32_t cell, int32_t H, int32_t V, const float *const *weights,
                   const float *emb, const int32_t *words, const int32_t *children,
                   int32_t n, int32_t maxc, double *h_out, double *aux_out,
                   int32_t *bad_node) {
  return forward_impl(cell, H, V, weights, emb, words, children, n, maxc, NULL, 0,
                      h_out, aux_out, bad_node);
}

int oracle_forward_subset(int32_t cell, int32_t H, int32_t V, const float *const *weights,
                          const float *emb, const int32_t *words, const int32_t *children,
                          int32_t n, int32_t maxc, const int32_t *targets, int32_t n_targets,
                          double *h_out, double *aux_out, int32_t *bad_node) {
  return forward_impl(cell, H, V, weights, emb, words, children, n, maxc, targets,
                      n_targets, h_out, aux_out, bad_node);
}
