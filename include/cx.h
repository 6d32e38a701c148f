/* include/cx.h -- C ABI of the B200-native Cortex hot path.
 *
 * What it computes (PAPER.md = arXiv 2011.01383, "Cortex: A Compiler for
 * Recursive Deep Learning Models"):
 *   cx_linearize  the data-structure linearizer of §4.2 with
 *                 dynamic batching by node height and the node
 *                 numbering of §6 / App. B: nodes of
 *                 a batch (level) are numbered consecutively and higher than
 *                 their parents, all leaves higher than all internal nodes,
 *                 batches described by batch_begin/batch_length arrays.
 *                 The caller declares max children and the structure kind
 *                 (sequence/tree/DAG), "verified at runtime".
 *   cx_forward    the lowered recursive computation of Listing 2:
 *                 a specialised leaf phase followed by one batch
 *                 per level with a barrier in the batch loop (App. A.4,
 *                 P:2010-2040), fused into one persistent kernel (P:1441
 *                 "#Kernel calls 1") with the weights kept on chip
 *                 (model persistence). Cells: TreeRNN
 *                 (Listing 1) and TreeFC, TreeLSTM, TreeGRU,
 *                 MV-RNN, DAG-RNN (Table 2) under the readings
 *                 Q1-Q23 of SURVEY.md §8(c), restated in DESIGN.md.
 *
 * Conventions (all calls):
 *   - Every pointer is a DEVICE pointer unless marked (host).
 *   - Every call is asynchronous and ordered on `stream` (a cudaStream_t
 *     passed as void* so that this header needs no CUDA headers).
 *   - The library never allocates or frees device memory and keeps no
 *     per-call global state; the only static state is a mutex-guarded cache
 *     of device attributes. Functions are thread-safe. No C++ exception
 *     crosses the ABI.
 *   - Argument errors are returned synchronously before any launch.
 *     Data-dependent errors are latched on the device in the linearization
 *     header: the lowest (code, input node id) wins, so error reporting is
 *     deterministic. cx_status_sync() reads them back.
 */
#ifndef CX_H
#define CX_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { CX_SEQUENCE = 0, CX_TREE = 1, CX_DAG = 2 } cx_kind;
typedef enum {
  CX_TREERNN = 0, CX_TREEFC = 1, CX_TREELSTM = 2, CX_TREEGRU = 3, CX_MVRNN = 4, CX_DAGRNN = 5,
  CX_SIMPLETREEGRU = 6  /* footnote P:1638-1640: h = (1 - z) h' at internal nodes; TreeGRU's weights */
} cx_cell;
/* compute precision; inputs, weights and outputs are always fp32 */
typedef enum { CX_F32 = 0, CX_BF16 = 1 } cx_dtype;
/* order matters: data errors are ranked by code, then by node id */
typedef enum {
  CX_OK = 0,
  CX_E_ARG = 1,          /* sync: null pointer, n < 0, max_children < 1, bad enum,
                            sequence with max_children != 1                         */
  CX_E_CHILD_RANGE = 2,  /* data: a child id outside [0, n) and != -1               */
  CX_E_CHILD_LAYOUT = 3, /* data: a -1 before a present child (children must be a prefix) */
  CX_E_KIND = 4,         /* data: two parents in a tree/sequence; a duplicate child */
  CX_E_CYCLE = 5,        /* data: a cycle; bad_node = lowest id on/reaching it      */
  CX_E_ARITY = 6,        /* data (forward): binary cell, internal node without 2 children */
  CX_E_WORD_RANGE = 7,   /* data (forward): a word id outside [0, V) where one is used */
  CX_E_UNSUPPORTED = 8,  /* sync: no instantiation for (cell, H, dtype, max_children) */
  CX_E_WORKSPACE = 9,    /* sync: workspace smaller than the *_workspace_bytes query */
  CX_E_CUDA = 10         /* sync: a CUDA launch/runtime failure                    */
} cx_status;

/* Device-resident header written by cx_linearize and updated by cx_forward. */
typedef struct {
  int32_t status;          /* cx_status of the latched data error, CX_OK if none   */
  int32_t bad_node;        /* input id of the offending node, -1 if none           */
  int32_t num_nodes;       /* n                                                    */
  int32_t num_levels;      /* L = 1 + max height (0 when n == 0)                   */
  int32_t num_leaves;      /* size of level 0 (the leaf batch)                     */
  int32_t first_leaf;      /* n - num_leaves: new id i is a leaf iff i >= first_leaf */
  int32_t max_level_size;  /* max over levels of level_size                        */
  int32_t num_roots;       /* nodes of in-degree 0                                 */
  uint64_t err_key;        /* internal latch (code << 32 | id); UINT64_MAX = none  */
} cx_lin_header;

/* Caller-allocated device buffers written by cx_linearize (element counts).
 * New ids number nodes level by level, root-most level first (level L-1 gets
 * ids [0, level_size[L-1])), ascending input id inside a level (reading Q4). */
typedef struct {
  cx_lin_header *header;   /* 1                                                    */
  int32_t *perm;           /* n        new id -> input id                          */
  int32_t *inv;            /* n        input id -> new id                          */
  int32_t *children;       /* maxc*n   SoA [k][new]: child new ids, -1 = absent    */
  int32_t *height;         /* n        level of each new id (0 = leaf)             */
  int32_t *level_begin;    /* n        first new id of level l (l < num_levels)    */
  int32_t *level_size;     /* n        nodes in level l (l < num_levels)           */
  int32_t *roots;          /* n        new ids of roots, ascending input id        */
  int32_t *structure;      /* n        structure of each new id: index r in roots[]
                                       of the root that owns it (trees/sequences: its
                                       unique root; DAGs: the smallest r whose root
                                       reaches it). Independent structures (P.3,
                                       P:759-761) are the unit of sharding.            */
  int32_t n;               /* (host) number of nodes                               */
  int32_t max_children;    /* (host) declared maximum children per node            */
  int32_t kind;            /* (host) cx_kind                                       */
} cx_linearization;

/* Bytes of device workspace cx_linearize needs for (n, max_children). The
 * workspace must be zero-filled before its first use; every call leaves its
 * synchronisation words zero again, so it can be reused without clearing by
 * calls with the same shape arguments (n, max_children and, for the forward
 * calls, the model). The words' offsets depend on those arguments: a workspace
 * reused for another shape must be zero-filled again first. */
size_t cx_linearize_workspace_bytes(int32_t n, int32_t max_children);

/* Linearize a batch (forest) of structures.
 *   children  [max_children][n] int32 input ids, -1 = absent; present children
 *             of a node form a prefix (position k = the k-th child, e.g. left=0).
 *   n         nodes (0 allowed: num_levels = 0), max_children >= 1, kind.
 *   out       buffers above; out->n/max_children/kind are written (host).
 * Validation: range, prefix layout, no duplicate child, in-degree
 * <= 1 unless kind == CX_DAG, acyclic. Heights: h = 0 for a leaf, else
 * 1 + max child height (P:1080 internal_batches[node.height]). */
cx_status cx_linearize(const int32_t *children, int32_t n, int32_t max_children, cx_kind kind,
                       void *workspace, size_t workspace_bytes, cx_linearization *out,
                       void *stream);

typedef struct {
  int32_t cell;    /* cx_cell                                                      */
  int32_t hidden;  /* H: 8, 16 or a multiple of 32 up to 1024 (MV-RNN: H <= 128)   */
  int32_t vocab;   /* V: rows of the embedding table (and of MV-RNN's Mw)          */
  int32_t dtype;   /* cx_dtype                                                     */
} cx_model;

/* Weights, fp32 row-major [out][in], in this order:
 *   TREERNN  -
 *   TREEFC   W [H][2H], b [H]
 *   TREELSTM W_iou [3H][H], U_iou [3H][H], b_iou [3H], U_f [H][H], b_f [H]  (gate rows i, o, u)
 *   TREEGRU  W_zh [2H][H] (rows z then h), U_z [H][H], U_r [H][H], U_h [H][H], b_z, b_r, b_h [H]
 *   MVRNN    Mw [V][H][H], W [H][2H], beta [H], W_M [H][2H]
 *   DAGRNN   W_x [H][H], U [H][H], b [H]                                        */
typedef struct { const float *p[8]; } cx_weights;

/* Bytes of device workspace cx_forward needs (same zero-fill contract as
 * cx_linearize_workspace_bytes). */
size_t cx_forward_workspace_bytes(const cx_model *model, int32_t n);

/* Evaluate every node of a linearized batch (a cx_linearize output on the
 * same stream; the level structure is read from the device header, so there
 * is no host synchronisation between the two calls).
 *   model, weights  (host structs) holding device pointers.
 *   emb        [V][H] fp32.
 *   word_ids   [n] input numbering; read for leaves (every node for DAG-RNN),
 *              ignored elsewhere.
 *   lin        the linearization (host struct of device pointers).
 *   h_out      [n][H] fp32, INPUT numbering (reading Q15). Required.
 *   aux_out    TreeLSTM memory cell c [n][H] | MV-RNN matrices A [n][H][H] | NULL.
 *   root_out   [num_roots][H] packed root states, ascending input id | NULL.
 * If the header already holds an error the kernel exits without touching the
 * outputs. Forward errors (CX_E_ARITY, CX_E_WORD_RANGE) are latched inline;
 * outputs are unspecified whenever the final status != CX_OK. */
cx_status cx_forward(const cx_model *model, const cx_weights *weights, const float *emb,
                     const int32_t *word_ids, const cx_linearization *lin, float *h_out,
                     float *aux_out, float *root_out, void *workspace, size_t workspace_bytes,
                     void *stream);

/* Bytes of device workspace cx_linearize_forward needs (same zero-fill
 * contract as the other workspaces). */
size_t cx_linearize_forward_workspace_bytes(const cx_model *model, int32_t n, int32_t max_children);

/* cx_linearize followed by cx_forward in ONE launch where the batch allows it
 * (the paper's single fused kernel, T6 "#Kernel calls 1"
 * P:1441, with the linearizer of §4.2 P:1060-1085 moved from the host into the
 * kernel's prologue). Results are exactly those of the two calls in sequence
 * on `stream`: every output of cx_linearize in `out` (header included) and
 * every output of cx_forward.
 *   children, n, max_children, kind   as cx_linearize.
 *   model, weights, emb, word_ids, h_out, aux_out, root_out   as cx_forward.
 *   workspace  >= cx_linearize_forward_workspace_bytes(model, n, max_children),
 *              zero-filled before first use, reusable.
 * One launch: fp32 TreeLSTM / DAG-RNN with H in {64, 128, 256}, max_children
 * <= 4 and a batch small enough for the latency (cluster) kernel (n <= ~600 at
 * H = 256): every CTA linearizes the batch in its shared memory (CTA 0 also
 * writes `out`) while it loads its register weights and prefetches the
 * batch's embedding rows into L2. Otherwise the two kernels are launched back
 * to back (no host synchronisation either way). Argument errors return
 * synchronously; data errors are latched in out->header exactly as by the
 * two calls (CX_E_CHILD_* / KIND / CYCLE from the linearization take
 * precedence: the forward part does not run). CX_FUSED=0 in the environment
 * forces the two-launch path (for measurement). */
cx_status cx_linearize_forward(const int32_t *children, int32_t n, int32_t max_children,
                               cx_kind kind, const cx_model *model, const cx_weights *weights,
                               const float *emb, const int32_t *word_ids, cx_linearization *out,
                               float *h_out, float *aux_out, float *root_out, void *workspace,
                               size_t workspace_bytes, void *stream);

/* Synchronise `stream` and return the latched status of lin->header;
 * *bad_node (host, may be NULL) receives the offending input id or -1. */
cx_status cx_status_sync(const cx_linearization *lin, int32_t *bad_node, void *stream);

/* Static description of a status code. */
const char *cx_status_str(cx_status s);

/* Number of CTAs / threads / dynamic shared memory the forward kernel would
 * use for this model on the current device (host, for reporting). Returns
 * CX_E_UNSUPPORTED for models without an instantiation. */
cx_status cx_forward_launch_info(const cx_model *model, int32_t *ctas, int32_t *threads,
                                 int32_t *smem_bytes);

/* The launch cx_linearize_forward would make for a batch of n nodes (host,
 * for reporting): *fused = 1 for the single fused launch, then the shape of
 * that kernel (CTAs, threads per CTA, dynamic shared memory per CTA, cluster
 * size); *fused = 0 for the two-launch path, then the shape of cx_forward's
 * kernel. Any output pointer may be NULL. */
cx_status cx_linearize_forward_launch_info(const cx_model *model, int32_t n, int32_t max_children,
                                           int32_t *fused, int32_t *ctas, int32_t *threads,
                                           int32_t *smem_bytes, int32_t *cluster);

/* ---- Diagnostics (measurement; not part of the hot path) -------------------
 * cx_diag_sync_cycles: SM cycles per level of one synchronisation or
 * dependent-arithmetic step of the critical-path bound of SURVEY.md §8(d),
 * T_cp = t_launch + (L - 1) t_sync + L t_chain, measured on the current
 * device (see csrc/diag.cu): kind 0 = the cluster kernel's push hand-off
 * (st.async + mbarrier, 16-CTA cluster), 1 = barrier.cluster, 2 = grid
 * barrier (release/acquire counter, one CTA per SM; `workspace` = 128 zeroed
 * bytes, left zeroed), 3 = the dependent arithmetic of one level (H = 256,
 * one warp). out (device, >= 2 entries): out[0] = cycles per level, out[1] =
 * levels. Asynchronous on `stream`. */
cx_status cx_diag_sync_cycles(int32_t kind, int32_t levels, unsigned long long *out,
                              void *workspace, void *stream);

/* Debug hooks (tools/trace_*.py, tests): %globaltimer / clock64 timelines of
 * the trace build (libcx_trace.so) and reporting helpers. buf = NULL turns a
 * trace off. */
cx_status cx_debug_set_trace(unsigned long long *buf, int32_t slots);
cx_status cx_debug_set_lin_trace(unsigned long long *buf);
int32_t cx_debug_fused_applies(const cx_model *model, int32_t n, int32_t max_children);
int32_t cx_debug_forward_family(const cx_model *model, int32_t n, int32_t max_children);
cx_status cx_debug_empty(int32_t ctas, int32_t threads, int32_t coop, unsigned long long *t,
                         void *stream);

#ifdef __cplusplus
}
#endif
#endif /* CX_H */
