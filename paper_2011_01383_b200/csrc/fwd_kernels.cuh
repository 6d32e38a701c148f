// fwd_kernels.cuh -- internal interface between api.cu and forward.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "common.cuh"
#include "lin_kernels.cuh"

namespace cx {

constexpr int kFwdThreads = 256;  // 8 warps; warps split the contraction (K) dim
constexpr int kUG = 32;           // hidden units per CTA (lane = unit)

struct FwdArgs {
  cx_lin_header *hdr;
  const int32_t *perm, *chn, *lbeg, *lsize, *hnew, *roots, *sid;
  int n, maxc, H, V;
  int kind;  // cx_kind of the linearization
  const float *emb;
  const int32_t *words;
  const float *w[8];
  float *h_out, *aux_out, *root_out;
  float *cbuf;  // TreeLSTM memory cells [n][H] (aux_out or workspace)
  float *zbuf;  // TreeGRU update gates [n][H]
  float *sbuf;  // TreeGRU sum_k r_k * h_k [n][H]
  float *pbuf;  // DAG-RNN input projections W_x x + b [n][H]
  float *Abuf;  // MV-RNN matrices [n][H][H] (aux_out or workspace)
  // bf16 tensor-core path (forward_tc.cu), workspace:
  unsigned short *hb;  // [n][H] bf16 hidden states, new numbering (MMA operand)
  float *cs;           // [n][H] fp32 TreeLSTM memory cells, new numbering
  unsigned short *xb;  // bf16 input rows: [V][H] (xmode 0) or [n - xlo][H] node order (xmode 1)
  int xmode;
  int cell_has_x;      // the cell gathers input rows (TreeLSTM, DAG-RNN)
  int hoist;           // TreeLSTM leaf cell evaluated per vocabulary word (tc_hoist)
  float *hf;           // [V][H] fp32 h of every word (hoist)
  int *crow;           // [n] state row of node i: its word if a leaf, else V + i (hoist)
  unsigned short *pb;  // TreeLSTM: [J*n][H] bf16 h of node i stored in its parent's child
                       // slot row k*n + parent (a level tile's k-th children are contiguous)
  int *pslot;          // [n] that row for every non-root node
  int *pslot1;         // [n] split-fp32 DAG-RNN: a second parent's slot row (-1: none)
  int *pcnt;           // [n] split-fp32 DAG-RNN: parents counted in the prologue
  GridBar *bar;
  int Gn, Gu;   // node groups x unit groups = CTAs
  unsigned long long *trace;  // debug: %globaltimer per CTA and phase (cx_debug_set_trace)
  int trace_slots;
  int push_off;  // measurement/test: CX_PUSH=0 forces the cluster kernel's barrier + pull mode
  int tc_fma_off;  // measurement/test: CX_TC_FMA=0 -- tensor-core kernel runs every level on UMMA tiles
  int bf16ops;   // dtype CX_BF16 on the FMA cluster path: operands rounded to bf16 (reading Q18)
  int discard_off;  // measurement: CX_DISCARD=0 keeps the tc kernel's dead workspace lines in L2
  LinArgs lin;  // fused linearize + forward (cx_linearize_forward): the linearizer's arguments
};

// thread 0 of each CTA records %globaltimer into slot `s`. Compiled in only in
// the separate trace build (libcx_trace.so, -DCX_TRACE: SURVEY §8(d)
// "per-level breakdown from a separate CX_TRACE_LEVELS build"); the product
// library carries no trace checks on the hot path.
// Marks record clock64() (a few cycles; %globaltimer reads cost ~0.2 us each
// and distorted per-level timings); slot 0 (entry) and the last slot (exit)
// also record %globaltimer into trace[gridDim.x * slots + 2 * cta + {0, 1}]
// so the host can align CTAs on different SMs.
__device__ __forceinline__ void trace_mark(const FwdArgs &a, int s) {
#ifdef CX_TRACE
  if (a.trace && threadIdx.x == 0 && s < a.trace_slots) {
    a.trace[(size_t)blockIdx.x * a.trace_slots + s] = clock64();
    if (s == 0 || s == a.trace_slots - 1) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[(size_t)gridDim.x * a.trace_slots + 2 * blockIdx.x + (s ? 1 : 0)] = t;
    }
  }
#else
  (void)a;
  (void)s;
#endif
}

struct FwdPlan {
  int ctas, threads;
  size_t smem;
  const void *kernel;
  int cluster = 1;  // > 1: thread-block clusters of this size (no cooperative launch)
  bool big = false; // large-batch pipelined kernel: workspace holds hs, st [n][H] + words [n]
  bool tc = false;  // bf16 tensor-core kernel (forward_tc.cu): launched by tc_launch
  bool fused = false;  // the kernel also linearizes (FwdArgs::lin), cx_linearize_forward
  // kernel family (reporting / tests): 1 smem weights (forward.cu), 2 register
  // weights (forward_rw.cu), 3 cluster (forward_cluster.cu), 4 large-batch
  // (forward_big.cu), 5 MV-RNN, 6 bf16 tensor cores (forward_tc.cu), 7 fused
  // single-CTA (forward_single.cu), 8 split-fp32 tensor cores (forward_tc.cu)
  int family = 0;
  bool bf16ops = false;  // dtype CX_BF16 served by an FMA kernel with bf16-rounded operands
  int tc_sp = 1;         // tensor-core kernel operands: 1 bf16, 2 split fp32 (hi + lo bf16)
  int tc_nab = 1;        // tensor-core kernel: K-atoms per TMA stage (3D tensor maps when > 1)
};

// Returns false (CX_E_UNSUPPORTED) when no instantiation covers the model.
// path: 0 = automatic (cluster kernel for small batches of TreeLSTM / DAG-RNN,
// register weights when n <= kRwMaxNodes, shared-memory weights above),
// 1 = force the register-weight kernel, 2 = force the shared-memory-weight
// kernel, 3 = force the cluster kernel, 4 = force the large-batch pipelined kernel.
constexpr int kRwMaxNodes = 32768;
bool fwd_plan(int cell, int H, int maxc, int n, int path, int num_sms, FwdPlan *plan, int *Gn,
              int *Gu);
size_t fwd_workspace_bytes(int cell, int H, int n, int V);
// bf16 tensor-core path (forward_tc.cu)
// sp = 1 bf16 operands (dtype CX_BF16); sp = 2 split fp32 operands (dtype CX_F32)
bool tc_plan(int cell, int H, int maxc, int sp, int num_sms, FwdPlan *plan, int *Gn, int *Gu);
int tc_xmode(int n, int V);
size_t tc_workspace_bytes(int cell, int H, int V, int n, int sp);
cudaError_t tc_launch(const FwdPlan &plan, const FwdArgs &args, cudaStream_t stream);
bool tc_hoist(int cell, int n, int V, int sp);
size_t tc_state_rows(int cell, int n, int V);
cudaError_t fwd_launch(const FwdPlan &plan, FwdArgs &args, cudaStream_t stream);
bool pdl_enabled();
// Fused linearize + forward (forward_cluster.cu): fp32 cluster
// path of TreeLSTM / DAG-RNN for small batches. False when not applicable.
bool fused_plan(int cell, int H, int maxc, int n, FwdPlan *plan, int *Gn, int *Gu);
// The cluster kernel without the linearizer (forward_cluster.cu); `roots` <= 0:
// unknown. False when the batch does not fit its shared memory.
bool cluster_plan(int cell, int H, int maxc, int n, int roots, FwdPlan *plan, int *Gn, int *Gu);
// Fused single-CTA-per-structure-group path (forward_single.cu, SURVEY §8(f)
// f2): TreeRNN (recursion unrolled, CX_UNROLL) and tiny TreeFC batches.
bool single_plan(int cell, int H, int maxc, int n, FwdPlan *plan, int *Gn, int *Gu);

}  // namespace cx
