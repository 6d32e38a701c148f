/* oracle/oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the Cortex hot
 * path computes (PAPER.md = arXiv 2011.01383): data-structure linearization
 * (§4.2, App. B) and the recursive cell evaluation
 * it accelerates (Listing 1 P:853-871 and the readings Q1-Q23 of SURVEY.md
 * §8(c)). Double precision throughout ("oracle comparisons use
 * float64 exact mode").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library. It shares no code, header, table or
 * constant with the product (paper_2011_01383_b200/, include/); the status
 * codes below are restated from SURVEY §8(b), not included.
 */
#ifndef CX_ORACLE_H
#define CX_ORACLE_H
#include <stdint.h>

enum {
  OR_OK = 0, OR_E_ARG = 1, OR_E_CHILD_RANGE = 2, OR_E_CHILD_LAYOUT = 3,
  OR_E_KIND = 4, OR_E_CYCLE = 5, OR_E_ARITY = 6, OR_E_WORD_RANGE = 7
};
enum { OR_SEQUENCE = 0, OR_TREE = 1, OR_DAG = 2 };
enum { OR_TREERNN = 0, OR_TREEFC = 1, OR_TREELSTM = 2, OR_TREEGRU = 3,
       OR_MVRNN = 4, OR_DAGRNN = 5, OR_SIMPLETREEGRU = 6 };

typedef struct {
  int32_t status, bad_node;
  int32_t num_nodes, num_levels, num_leaves, first_leaf, max_level_size, num_roots;
} oracle_lin_header;

/* Linearize: children is SoA [maxc][n] of input ids (-1 = absent).
 * Outputs (all caller-allocated, n or maxc*n entries): perm (new -> input),
 * inv (input -> new), children_new [maxc][n] (new ids), height_new [n],
 * level_begin [n], level_size [n], roots [n], structure [n] (per new id: the
 * index r in roots[] of the first root, in ascending r, whose descendants
 * include the node). Returns hdr->status. */
int oracle_linearize(const int32_t *children, int32_t n, int32_t maxc, int32_t kind,
                     oracle_lin_header *hdr, int32_t *perm, int32_t *inv,
                     int32_t *children_new, int32_t *height_new, int32_t *level_begin,
                     int32_t *level_size, int32_t *roots, int32_t *structure);

/* Forward: naive memoized recursion in INPUT numbering. weights[] are the
 * fp32 tensors in cx_weights order. h_out [n][H] double;
 * aux_out (TreeLSTM c [n][H], MV-RNN A [n][H][H]) may be NULL. The structure
 * must already be valid (acyclic) -- run oracle_linearize first. Returns the
 * lowest (code, node) forward error, OR_OK if none; *bad_node receives the id. */
int oracle_forward(int32_t cell, int32_t H, int32_t V, const float *const *weights,
                   const float *emb, const int32_t *words, const int32_t *children,
                   int32_t n, int32_t maxc, double *h_out, double *aux_out,
                   int32_t *bad_node);

/* Same as oracle_forward but evaluates only the nodes reachable from the
 * listed nodes (used to sample a few outputs of a huge batch). Rows of
 * unreached nodes in h_out are left untouched. */
int oracle_forward_subset(int32_t cell, int32_t H, int32_t V, const float *const *weights,
                          const float *emb, const int32_t *words, const int32_t *children,
                          int32_t n, int32_t maxc, const int32_t *targets, int32_t n_targets,
                          double *h_out, double *aux_out, int32_t *bad_node);
#endif
