// api.cu -- the C ABI of include/cx.h: argument checks, workspace carving,
// launch configuration. No C++ exception crosses the boundary; argument
// errors return before any CUDA call.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/cx.h"
#include "common.cuh"
#include "fwd_kernels.cuh"
#include "lin_kernels.cuh"

namespace {

std::mutex g_mu;  // guards the device-attribute cache and kernel attribute setup
unsigned long long *g_trace = nullptr;  // debug only (cx_debug_set_trace)
int g_trace_slots = 0;
unsigned long long *g_lin_trace = nullptr;  // debug only (cx_debug_set_lin_trace)

int num_sms_current() {
  static int cached_dev = -1, cached_sms = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (dev != cached_dev) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    cached_dev = dev;
    cached_sms = sms;
  }
  return cached_sms;
}

// Debug/test override of the forward kernel family: CX_FORWARD_PATH=rw|smem
// (read on every call; unset = automatic by batch size).
int forward_path() {
  const char *e = std::getenv("CX_FORWARD_PATH");
  if (!e) return 0;
  if (!std::strcmp(e, "rw")) return 1;
  if (!std::strcmp(e, "smem")) return 2;
  if (!std::strcmp(e, "cluster")) return 3;
  if (!std::strcmp(e, "big")) return 4;
  if (!std::strcmp(e, "tc")) return 5;  // bf16: always the tensor-core kernel
  return 0;
}

inline char *align_up(char *p, size_t a) {
  uintptr_t v = reinterpret_cast<uintptr_t>(p);
  return reinterpret_cast<char *>((v + a - 1) / a * a);
}

bool weights_ok(int cell, const cx_weights *w) {
  static const int need[7] = {0, 2, 5, 7, 4, 3, 7};
  for (int i = 0; i < need[cell]; i++)
    if (!w->p[i]) return false;
  return true;
}

}  // namespace

namespace {
void lin_args(const int32_t *children, int32_t n, int32_t max_children, cx_kind kind,
              void *workspace, cx_linearization *out, cx::LinArgs *ap) {
  cx::LinArgs &a = *ap;
  out->n = n;
  out->max_children = max_children;
  out->kind = kind;
  char *p = align_up(static_cast<char *>(workspace), 128);
  a.bar = reinterpret_cast<cx::GridBar *>(p);
  p += sizeof(cx::GridBar);
  a.misc = reinterpret_cast<int32_t *>(p);
  p += 32 * sizeof(int32_t);
  a.indeg = reinterpret_cast<int32_t *>(p);
  p += sizeof(int32_t) * (size_t)n;
  a.hgt = reinterpret_cast<int32_t *>(p);
  p += sizeof(int32_t) * (size_t)n;
  a.cnt = reinterpret_cast<int32_t *>(p);
  a.budget = (int)cx::lin_budget_entries(n);
  a.ch = children;
  a.n = n;
  a.maxc = max_children;
  a.kind = kind;
  a.hdr = out->header;
  a.perm = out->perm;
  a.inv = out->inv;
  a.chn = out->children;
  a.hnew = out->height;
  a.lbeg = out->level_begin;
  a.lsize = out->level_size;
  a.roots = out->roots;
  a.sid = out->structure;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    a.trace = g_lin_trace;
  }
  const char *hj = std::getenv("CX_LIN_JACOBI");
  a.hjacobi = hj && hj[0] == '1';  // measurement only: Jacobi rounds for trees too
}
}  // namespace

namespace {
// bf16 TreeFC batches up to this many nodes run the register-weight FMA kernel
// (b1: 255 nodes, 47 us vs 80 us on the tensor cores; b10: 2,550 nodes, tensor
// cores 96 us vs 160 us)
constexpr int kBf16FcFmaMaxN = 1024;
// fp32 batches of TreeLSTM / DAG-RNN / TreeFC with at least this many nodes run
// the split-fp32 tensor-core kernel (forward_tc.cu, SP = 2): their levels are
// dense GEMMs. Per cell, from the measured crossover against the FMA kernels
// (tools/tc32_crossover.py): TreeLSTM between 1,950 and 3,900
// nodes, DAG-RNN between 5,000 and 10,000, TreeFC (H = 512) near 600.
// CX_TC_F32_MIN_N overrides (measurement).
int tc_f32_min_n(int cell) {
  const char *e = std::getenv("CX_TC_F32_MIN_N");
  if (e) return std::atoi(e);
  return cell == CX_TREELSTM ? 3000 : cell == CX_DAGRNN ? 7000 : 1000;
}
// The one forward plan of a call (caller holds g_mu). fp32: the fused cluster /
// single-CTA kernels (cx_linearize_forward) or fwd_plan. bf16 ("per-batch
// precision dispatch", north_star: tensor cores only where the levels are
// dense GEMMs): batches small enough for the cluster kernel run it on FMA with
// bf16-rounded operands (its levels are a few nodes: 128-row UMMA tiles would
// be mostly padding), larger batches the tcgen05 kernel. CX_FORWARD_PATH (tests)
// disables the bf16 cluster route unless it asks for the cluster kernel.
// kind: the linearization's (-1 unknown: a workspace or launch-shape query)
bool plan_forward(const cx_model *m, int maxc, int n, int kind, bool fused, int sms,
                  cx::FwdPlan *plan, int *Gn, int *Gu) {
  const int path = forward_path();
  if (m->dtype == CX_BF16) {
    const bool small_ok = (path == 0 || path == 3) && m->cell != CX_TREEFC;
    if (small_ok && (fused ? cx::fused_plan(m->cell, m->hidden, maxc, n, plan, Gn, Gu)
                           : cx::cluster_plan(m->cell, m->hidden, maxc, n, 0, plan, Gn, Gu))) {
      plan->bf16ops = true;
      return true;
    }
    // TreeFC: small batches on the register-weight kernel (FMA, rounded operands)
    if (!fused && path == 0 && m->cell == CX_TREEFC && n <= kBf16FcFmaMaxN &&
        cx::fwd_plan(m->cell, m->hidden, maxc, n, 1, sms, plan, Gn, Gu)) {
      plan->bf16ops = true;
      return true;
    }
    if (fused) return false;
    return cx::tc_plan(m->cell, m->hidden, maxc, 1, sms, plan, Gn, Gu);
  }
  if (fused)
    return cx::fused_plan(m->cell, m->hidden, maxc, n, plan, Gn, Gu) ||
           cx::single_plan(m->cell, m->hidden, maxc, n, plan, Gn, Gu);
  // dense levels: the split-fp32 tensor-core kernel (a TreeLSTM DAG
  // linearization stays on FMA: that kernel hands each h to ONE parent slot)
  const bool tc_cell = m->cell == CX_TREELSTM || m->cell == CX_DAGRNN || m->cell == CX_TREEFC;
  if (tc_cell && !((m->cell == CX_TREELSTM || m->cell == CX_TREEFC) && kind == CX_DAG) &&
      (path == 5 || (path == 0 && n >= tc_f32_min_n(m->cell))) &&
      cx::tc_plan(m->cell, m->hidden, maxc, 2, sms, plan, Gn, Gu))
    return true;
  return cx::fwd_plan(m->cell, m->hidden, maxc, n, path == 5 ? 0 : path, sms, plan, Gn, Gu);
}

// cx_forward after argument checks; `fused` (non-NULL) = linearizer arguments
// for the fused launch (its plan is required to exist).
cx_status forward_impl(const cx_model *m, const cx_weights *w, const float *emb,
                       const int32_t *word_ids, const cx_linearization *lin, float *h_out,
                       float *aux_out, float *root_out, void *workspace, const cx::LinArgs *fused,
                       void *stream) {
  const int n = lin->n;

  cx::FwdPlan plan;
  int Gn = 0, Gu = 0;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    int sms = num_sms_current();
    if (sms <= 0) return CX_E_CUDA;
    const bool ok = plan_forward(m, lin->max_children, n, lin->kind, fused != nullptr, sms, &plan,
                                 &Gn, &Gu);
    if (!ok) return CX_E_UNSUPPORTED;
    // the tensor-core TreeLSTM / TreeFC store each node's h in its ONE parent's
    // child slot (forward_tc.cu): a DAG linearization (shared children) is not
    // run there (fp32 never plans it; bf16 TreeFC falls back, TreeLSTM is refused)
    if (plan.tc && (m->cell == CX_TREELSTM || m->cell == CX_TREEFC) && lin->kind == CX_DAG) {
      // a bf16 TreeFC over a DAG: the register-weight FMA kernel with rounded operands
      plan = cx::FwdPlan();
      if (m->cell == CX_TREEFC && m->dtype == CX_BF16 &&
          cx::fwd_plan(m->cell, m->hidden, lin->max_children, n, 1, sms, &plan, &Gn, &Gu)) {
        plan.bf16ops = true;
      } else {
        return CX_E_UNSUPPORTED;
      }
    }
  }
  const size_t N = (size_t)n, H = (size_t)m->hidden;
  char *p = align_up(static_cast<char *>(workspace), 128);
  cx::FwdArgs a;
  std::memset(&a, 0, sizeof a);
  a.bar = reinterpret_cast<cx::GridBar *>(p);
  p += sizeof(cx::GridBar);
  float *buf = reinterpret_cast<float *>(p);
  a.hdr = lin->header;
  a.perm = lin->perm;
  a.chn = lin->children;
  a.lbeg = lin->level_begin;
  a.lsize = lin->level_size;
  a.hnew = lin->height;
  a.roots = lin->roots;
  a.sid = lin->structure;
  a.n = n;
  a.maxc = lin->max_children;
  a.kind = lin->kind;
  a.H = m->hidden;
  a.V = m->vocab;
  a.emb = emb;
  a.words = word_ids;
  for (int i = 0; i < 8; i++) a.w[i] = w->p[i];
  a.h_out = h_out;
  a.aux_out = aux_out;
  a.root_out = root_out;
  a.bf16ops = plan.bf16ops ? 1 : 0;
  if (plan.tc) {  // hb, cs, xb [, hf, crow] [, pb, pslot] (forward_tc.cu)
    const size_t R = cx::tc_state_rows(m->cell, n, m->vocab);
    const size_t RW = H * (size_t)plan.tc_sp;  // bf16 per operand row
    char *q = reinterpret_cast<char *>(buf);
    a.hb = reinterpret_cast<unsigned short *>(q);
    q = align_up(q + 2 * R * RW, 256);
    if (m->cell == CX_TREELSTM) {
      a.cs = reinterpret_cast<float *>(q);
      q = align_up(q + 4 * R * H, 256);
    }
    a.xmode = cx::tc_xmode(n, m->vocab);
    a.cell_has_x = m->cell == CX_TREELSTM || m->cell == CX_DAGRNN;
    if (a.cell_has_x) {  // x rows (tc_workspace_bytes counts them for these cells only)
      a.xb = reinterpret_cast<unsigned short *>(q);
      q = align_up(q + 2 * (a.xmode ? N : (size_t)m->vocab) * RW, 256);
    }
    a.hoist = cx::tc_hoist(m->cell, n, m->vocab, plan.tc_sp) ? 1 : 0;
    if (a.hoist) {
      a.hf = reinterpret_cast<float *>(q);
      q = align_up(q + 4 * (size_t)m->vocab * H, 256);
      a.crow = reinterpret_cast<int *>(q);
      q = align_up(q + 4 * N, 256);
    }
    const bool dag2 = m->cell == CX_DAGRNN && plan.tc_sp == 2;
    if (m->cell == CX_TREELSTM || m->cell == CX_TREEFC || dag2) {  // parent-slot operand rows
      a.pb = reinterpret_cast<unsigned short *>(q);
      q = align_up(q + 2 * (2 * N) * RW, 256);
      a.pslot = reinterpret_cast<int *>(q);
      q = align_up(q + 4 * N, 256);
    }
    if (dag2) {  // split-fp32 DAG-RNN: a second parent's slot row, parent counts
      a.pslot1 = reinterpret_cast<int *>(q);
      q = align_up(q + 4 * N, 256);
      a.pcnt = reinterpret_cast<int *>(q);
    }
  } else if (plan.big) a.pbuf = buf;  // hs, st [n][H] + words [n] (forward_big.cu)
  else switch (m->cell) {
    case CX_TREELSTM: a.cbuf = aux_out ? aux_out : buf; break;
    case CX_TREEGRU:
    case CX_SIMPLETREEGRU: a.zbuf = buf; a.sbuf = buf + N * H; break;
    case CX_DAGRNN: a.pbuf = buf; break;
    case CX_MVRNN: a.Abuf = aux_out ? aux_out : buf; break;
    default: break;
  }
  a.Gn = Gn;
  a.Gu = Gu;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    const char *pe = std::getenv("CX_PUSH");
    a.push_off = pe && pe[0] == '0';
    const char *de = std::getenv("CX_DISCARD");
    a.discard_off = de && de[0] == '0';
    const char *fe = std::getenv("CX_TC_FMA");
    a.tc_fma_off = fe && fe[0] == '0';
    a.trace = g_trace;
    a.trace_slots = g_trace_slots;
  }
  if (fused) a.lin = *fused;
  cudaError_t e = plan.tc ? cx::tc_launch(plan, a, static_cast<cudaStream_t>(stream))
                          : cx::fwd_launch(plan, a, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? CX_OK : CX_E_CUDA;
}

}  // namespace

extern "C" {

size_t cx_linearize_workspace_bytes(int32_t n, int32_t max_children) {
  (void)max_children;
  return cx::lin_workspace_bytes(n < 0 ? 0 : n);
}

cx_status cx_linearize(const int32_t *children, int32_t n, int32_t max_children, cx_kind kind,
                       void *workspace, size_t workspace_bytes, cx_linearization *out,
                       void *stream) {
  if (!out || n < 0 || max_children < 1 || (n > 0 && !children)) return CX_E_ARG;
  if (kind != CX_SEQUENCE && kind != CX_TREE && kind != CX_DAG) return CX_E_ARG;
  if (kind == CX_SEQUENCE && max_children != 1) return CX_E_ARG;
  if (!out->header || (n > 0 && (!out->perm || !out->inv || !out->children || !out->height ||
                                 !out->level_begin || !out->level_size || !out->roots ||
                                 !out->structure)))
    return CX_E_ARG;
  if (!workspace || workspace_bytes < cx::lin_workspace_bytes(n)) return CX_E_WORKSPACE;
  cx::LinArgs a;
  lin_args(children, n, max_children, kind, workspace, out, &a);
  int sms;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    sms = num_sms_current();
  }
  if (sms <= 0) return CX_E_CUDA;
  cudaError_t e = cx::launch_linearize(a, sms, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? CX_OK : CX_E_CUDA;
}


size_t cx_forward_workspace_bytes(const cx_model *m, int32_t n) {
  if (!m) return 0;
  const size_t f32 = cx::fwd_workspace_bytes(m->cell, m->hidden, n, m->vocab) + 256;
  if (m->dtype == CX_BF16) {  // tensor-core kernel, or the FMA cluster kernel for small batches
    const size_t tc = sizeof(cx::GridBar) + cx::tc_workspace_bytes(m->cell, m->hidden, m->vocab, n, 1) + 512;
    return tc > f32 ? tc : f32;
  }
  if (m->cell == CX_TREELSTM || m->cell == CX_DAGRNN || m->cell == CX_TREEFC) {  // split-fp32 tensor cores
    const size_t tc = sizeof(cx::GridBar) + cx::tc_workspace_bytes(m->cell, m->hidden, m->vocab, n, 2) + 512;
    return tc > f32 ? tc : f32;
  }
  return f32;
}

cx_status cx_forward(const cx_model *m, const cx_weights *w, const float *emb,
                     const int32_t *word_ids, const cx_linearization *lin, float *h_out,
                     float *aux_out, float *root_out, void *workspace, size_t workspace_bytes,
                     void *stream) {
  if (!m || !w || !lin || !lin->header) return CX_E_ARG;
  if (m->cell < CX_TREERNN || m->cell > CX_SIMPLETREEGRU) return CX_E_ARG;
  if (m->dtype != CX_F32 && m->dtype != CX_BF16) return CX_E_ARG;
  if (m->hidden <= 0 || m->vocab <= 0) return CX_E_ARG;
  const int n = lin->n;
  if (n < 0) return CX_E_ARG;
  if (n > 0 && (!emb || !word_ids || !h_out || !weights_ok(m->cell, w))) return CX_E_ARG;
  if (!workspace || workspace_bytes < cx_forward_workspace_bytes(m, n)) return CX_E_WORKSPACE;
  if (n == 0) return CX_OK;
  return forward_impl(m, w, emb, word_ids, lin, h_out, aux_out, root_out, workspace, nullptr, stream);
}


static size_t lin_part_bytes(int32_t n) { return (cx::lin_workspace_bytes(n < 0 ? 0 : n) + 255) / 256 * 256; }

size_t cx_linearize_forward_workspace_bytes(const cx_model *m, int32_t n, int32_t max_children) {
  if (!m) return 0;
  (void)max_children;
  return lin_part_bytes(n) + cx_forward_workspace_bytes(m, n) + 256;
}

cx_status cx_linearize_forward(const int32_t *children, int32_t n, int32_t max_children,
                               cx_kind kind, const cx_model *m, const cx_weights *w,
                               const float *emb, const int32_t *word_ids, cx_linearization *out,
                               float *h_out, float *aux_out, float *root_out, void *workspace,
                               size_t workspace_bytes, void *stream) {
  if (!m || !w || !out) return CX_E_ARG;
  if (!workspace || workspace_bytes < cx_linearize_forward_workspace_bytes(m, n, max_children))
    return CX_E_WORKSPACE;
  char *lws = align_up(static_cast<char *>(workspace), 256);
  char *fws = lws + lin_part_bytes(n);
  const size_t fbytes = cx_forward_workspace_bytes(m, n);
  // the fused kernel: fp32 cluster path, one launch
  const char *env = std::getenv("CX_FUSED");
  const bool try_fused = !(env && env[0] == '0') && n > 0 &&
                         (forward_path() == 0 || forward_path() == 3);
  if (try_fused) {
    // the same argument checks as the two calls
    if (n < 0 || max_children < 1 || !children) return CX_E_ARG;
    if (kind != CX_SEQUENCE && kind != CX_TREE && kind != CX_DAG) return CX_E_ARG;
    if (kind == CX_SEQUENCE && max_children != 1) return CX_E_ARG;
    if (!out->header || !out->perm || !out->inv || !out->children || !out->height ||
        !out->level_begin || !out->level_size || !out->roots || !out->structure)
      return CX_E_ARG;
    if (m->cell < CX_TREERNN || m->cell > CX_SIMPLETREEGRU || m->hidden <= 0 || m->vocab <= 0)
      return CX_E_ARG;
    if (!emb || !word_ids || !h_out || !weights_ok(m->cell, w)) return CX_E_ARG;
    cx::FwdPlan plan;
    int Gn = 0, Gu = 0;
    bool ok;
    {
      std::lock_guard<std::mutex> lk(g_mu);
      ok = plan_forward(m, max_children, n, kind, true, 0, &plan, &Gn, &Gu);
    }
    if (ok) {
      cx::LinArgs la;
      lin_args(children, n, max_children, kind, lws, out, &la);
      la.trace = nullptr;
      return forward_impl(m, w, emb, word_ids, out, h_out, aux_out, root_out, fws, &la, stream);
    }
  }
  cx_status st = cx_linearize(children, n, max_children, kind, lws, lin_part_bytes(n), out, stream);
  if (st != CX_OK) return st;
  return cx_forward(m, w, emb, word_ids, out, h_out, aux_out, root_out, fws, fbytes, stream);
}

cx_status cx_status_sync(const cx_linearization *lin, int32_t *bad_node, void *stream) {
  if (!lin || !lin->header) return CX_E_ARG;
  int32_t hv[2] = {0, -1};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(hv, lin->header, sizeof hv, cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return CX_E_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return CX_E_CUDA;
  if (bad_node) *bad_node = hv[1];
  return static_cast<cx_status>(hv[0]);
}

// Debug only (not part of include/cx.h): subsequent cx_forward launches record
// %globaltimer per CTA into buf[cta * slots + s]; buf = NULL disables.
cx_status cx_debug_set_trace(unsigned long long *buf, int32_t slots) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_trace = buf;
  g_trace_slots = buf ? slots : 0;
  return CX_OK;
}

// Debug only: cx_linearize records %globaltimer per phase into buf[0..7].
cx_status cx_debug_set_lin_trace(unsigned long long *buf) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_lin_trace = buf;
  return CX_OK;
}

// Debug only (reporting): 1 if cx_linearize_forward would use the fused
// single launch for this model and batch shape, else 0.
int32_t cx_debug_fused_applies(const cx_model *m, int32_t n, int32_t max_children) {
  if (!m || n <= 0) return 0;
  const char *env = std::getenv("CX_FUSED");
  if ((env && env[0] == '0') || !(forward_path() == 0 || forward_path() == 3)) return 0;
  cx::FwdPlan plan;
  int Gn, Gu;
  std::lock_guard<std::mutex> lk(g_mu);
  return plan_forward(m, max_children, n, -1, true, 0, &plan, &Gn, &Gu) ? 1 : 0;
}

// Debug / tests: the kernel family cx_forward runs for this model and batch
// shape (FwdPlan::family: 1 smem, 2 register weights, 3 cluster, 4 large
// batch, 5 MV-RNN, 6 bf16 tensor cores, 7 fused single-CTA, 8 split-fp32 tensor
// cores), honouring CX_FORWARD_PATH; 0 if none.
int32_t cx_debug_forward_family(const cx_model *m, int32_t n, int32_t max_children) {
  if (!m || n < 1 || max_children < 1) return 0;
  cx::FwdPlan plan;
  int Gn, Gu;
  std::lock_guard<std::mutex> lk(g_mu);
  const int sms = num_sms_current();
  if (sms <= 0) return 0;
  return plan_forward(m, max_children, n, -1, false, sms, &plan, &Gn, &Gu) ? plan.family : 0;
}

// Debug only: an empty kernel launch (measures launch overhead).
cx_status cx_debug_empty(int32_t ctas, int32_t threads, int32_t coop, unsigned long long *t,
                         void *stream) {
  return cx::launch_empty(ctas, threads, coop, t, static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? CX_OK : CX_E_CUDA;
}

const char *cx_status_str(cx_status s) {
  switch (s) {
    case CX_OK: return "ok";
    case CX_E_ARG: return "invalid argument";
    case CX_E_CHILD_RANGE: return "child id out of range";
    case CX_E_CHILD_LAYOUT: return "absent child before a present child";
    case CX_E_KIND: return "structure violates its declared kind (two parents or duplicate child)";
    case CX_E_CYCLE: return "cycle in the structure";
    case CX_E_ARITY: return "binary cell applied to a node without exactly two children";
    case CX_E_WORD_RANGE: return "word id out of range";
    case CX_E_UNSUPPORTED: return "no kernel instantiation for this model";
    case CX_E_WORKSPACE: return "workspace too small";
    case CX_E_CUDA: return "CUDA error";
  }
  return "unknown status";
}

cx_status cx_linearize_forward_launch_info(const cx_model *m, int32_t n, int32_t max_children,
                                           int32_t *fused, int32_t *ctas, int32_t *threads,
                                           int32_t *smem_bytes, int32_t *cluster) {
  if (!m || n < 0 || max_children < 1) return CX_E_ARG;
  cx::FwdPlan plan;
  int Gn = 0, Gu = 0;
  std::lock_guard<std::mutex> lk(g_mu);
  const char *env = std::getenv("CX_FUSED");
  bool f = !(env && env[0] == '0') && n > 0 && (forward_path() == 0 || forward_path() == 3) &&
           plan_forward(m, max_children, n, -1, true, 0, &plan, &Gn, &Gu);
  if (!f) {
    const int sms = num_sms_current();
    if (sms <= 0) return CX_E_CUDA;
    if (!plan_forward(m, max_children, n > 0 ? n : 1, -1, false, sms, &plan, &Gn, &Gu))
      return CX_E_UNSUPPORTED;
  }
  if (fused) *fused = f ? 1 : 0;
  if (ctas) *ctas = plan.ctas;
  if (threads) *threads = plan.threads;
  if (smem_bytes) *smem_bytes = (int32_t)plan.smem;
  if (cluster) *cluster = plan.cluster;
  return CX_OK;
}

cx_status cx_forward_launch_info(const cx_model *m, int32_t *ctas, int32_t *threads,
                                 int32_t *smem_bytes) {
  if (!m) return CX_E_ARG;
  cx::FwdPlan plan;
  int Gn, Gu;
  std::lock_guard<std::mutex> lk(g_mu);
  int sms = num_sms_current();
  if (sms <= 0) return CX_E_CUDA;
  const bool ok = m->dtype == CX_BF16 ? cx::tc_plan(m->cell, m->hidden, 2, 1, sms, &plan, &Gn, &Gu)
                                      : cx::fwd_plan(m->cell, m->hidden, 2, 1, forward_path(), sms,
                                                     &plan, &Gn, &Gu);
  if (!ok) return CX_E_UNSUPPORTED;
  if (ctas) *ctas = plan.ctas;
  if (threads) *threads = plan.threads;
  if (smem_bytes) *smem_bytes = (int32_t)plan.smem;
  return CX_OK;
}

}  // extern "C"
