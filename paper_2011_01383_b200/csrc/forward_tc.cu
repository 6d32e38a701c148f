// forward_tc.cu -- the tensor-core forward: one persistent kernel per batch
// that walks the levels of the linearization (Listing 2; one
// barrier per batch, App. A.4) and runs each level's contraction as
// a dense GEMM on the 5th-generation tensor cores (tcgen05.mma, fp32
// accumulators in tensor memory), with the gates fused into the epilogue
// and the recurrent weights resident in shared memory for the
// whole batch (model persistence). Two operand precisions (TcCfg
// SP): bf16 (dtype CX_BF16) and split fp32 (dtype CX_F32, large batches: every
// operand as bf16 hi + lo, three bf16 MMAs per product).
//
// Work split. CTA (gn, gu) owns hidden units [gu*U, gu*U + U) of every gate
// and the contiguous chunk gn of each level's nodes, walked in tiles of 128
// nodes (the UMMA M dimension; rows are nodes, so a partial tile's unused rows
// never influence the valid ones). A tile's GEMM is
//     D[128 x N] (+)= A_slot[128 x K] * B_slot[N x K]^T      for each slot,
// where a slot is one operand row set: the tile's k-th children's state rows
// (zero rows for absent children) or the input rows x = Emb[word]. The child
// sums of child-sum cells use linearity (U h~ = sum_k U h_k).
//   TreeLSTM  leaf:  slot x, B = W_iou slice (i,o,u rows)      -> [i o u]
//             level: slot child k, B = [U_iou; U_f] slice     -> acc k = [i o u f]_k;
//                    epilogue: iou = sum_k acc_k, f_k from acc_k (Q1)
//   DAG-RNN   level: slot x (B = W_x slice) + child slots (B = U slice) into one
//                    accumulator, h = tanh(acc + b) (Q8); split fp32 in table
//                    mode: W_x x + b once per word (phase l = -1), levels
//                    contract the children only and add the word's row
//   TreeFC    leaf:  h = Emb[word] (copy, no GEMM)
//             level: slot left (B = W[:, :H] slice) + slot right (B = W[:, H:]) (Q2)
// Small levels (a few nodes per node group) skip the tiles and run on the
// epilogue warps' FMA pipes against the same resident B (fma_level, §6.2j).
//
// Warp roles: warps 0-7 epilogue (warp w reads TMEM lane quadrant w % 4 = tile
// rows, column half w / 4), warp 8 MMA issuer (one lane; also allocates TMEM),
// then the operand feed, then 2 bookkeeping warps that fill a 4-deep ring of
// tile metadata (node ids, children, x rows, roots, parent slots) and run ahead
// of the level barriers. Feed: TreeLSTM / TreeFC (trees) store each node's h
// in its parent's child-slot row, so a tile's operands are contiguous rows
// loaded by one lane with 3D TMA boxes of NAB K-atoms; DAG-RNN gathers rows
// with 16-byte cp.async by 4 warps. The MMA lane waits a stage's "full"
// mbarrier, issues the stage's MMAs (K = 16 each) and frees it with
// tcgen05.commit; accumulators are double-buffered in TMEM so the epilogue of
// tile t overlaps the MMAs of tile t+1.
//
// State (workspace, linearized numbering): hb state rows (DAG-RNN; hoisted
// TreeLSTM word rows), pb parent-slot rows (TreeLSTM, TreeFC), cs fp32 TreeLSTM
// memory cells, xb input rows (the embedding table converted once per call,
// or the batch's rows in node order), hf fp32 word table (hoisting); operand
// rows hold SP x H bf16 ([hi | lo] when split). h_out / aux_out / root_out are
// written by the epilogue in the caller's numbering.
#include <cuda_bf16.h>
#include <cuda.h>  // CUtensorMap types (the encoder is fetched from the driver at run time)
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "fwd_common.cuh"
#include "umma.cuh"

namespace cx {
namespace {
using namespace fwd;
using namespace umma;

// measurement knobs (tools/build_variant.sh): W_iou / [U_iou; U_f] sharing one
// region on the bf16 path too (more stages), and the stage-count cap
#ifndef CX_TC_BSHARE_ALL
#define CX_TC_BSHARE_ALL 0
#endif
#ifndef CX_TC_SKIP_LO  // timing experiment only: drop the A_hi B_lo MMAs (wrong numerics)
#define CX_TC_SKIP_LO 0
#endif
#ifndef CX_TC_TMA_MC  // measurement: the multicast TMA form even for single-CTA clusters
#define CX_TC_TMA_MC 0
#endif
#ifndef CX_TC_SMAX
#define CX_TC_SMAX 8
#endif
#ifndef CX_TC_TMA_LANES  // lanes of the TMA warp issuing stages side by side (measured: 2 or 3
#define CX_TC_TMA_LANES 1    // lanes slowed the split-fp32 TreeLSTM / TreeFC by 3-7 %, bf16 +-0)
#endif
#ifndef CX_TC_L2PF  // stages ahead whose operand tile the TMA lane prefetches into L2
#define CX_TC_L2PF 0  // (0: none; 4 or 8 measured within +-0.5 %: the operands are L2-resident)
#endif
#ifndef CX_TC_DSLOT  // split-fp32 DAG-RNN parent-slot operands (in-degree <= 2)
#define CX_TC_DSLOT 1
#endif
#ifndef CX_TC_NAB  // K-atoms per TreeLSTM TMA stage (one 3D box)
#define CX_TC_NAB 2
#endif
#ifndef CX_TC_FML_FC  // split TreeFC: nodes per node group up to which a level runs on FMA
#define CX_TC_FML_FC 10
#endif
constexpr int kTM = 128;                    // tile rows = UMMA M
// warps 0-7: epilogue (warp w reads TMEM lane quadrant w % 4 = tile rows
// 32(w%4)..+31, column half w / 4); warp 8: MMA issuer; warps 9..: operand
// feeding (TreeLSTM: 1 TMA warp; DAG-RNN / TreeFC: 4 cp.async warps); last 2
// warps: tile bookkeeping (warp m of them fills the tiles t = m mod 2, so two
// tiles' dependent index loads are in flight at once)
constexpr int kEpiWarps = 8, kMmaWarp = 8, kFeed0 = 9, kMetaWarps = 2;
constexpr int kEpiThreads = 32 * kEpiWarps;             // 256
constexpr int kMaxCluster = 8;                          // portable cluster size

// 128-byte CUtensorMap (opaque; encoded on the host by cuTensorMapEncodeTiled)
struct alignas(64) TmaDesc {
  unsigned long long d[16];
};
// kernel parameter block: tensor maps of the gathered operands + the common args
struct TcArgs {
  TmaDesc tm_x;  // TreeLSTM input rows xb, tile box 64 x 128, 128B swizzle
  TmaDesc tm_p;  // TreeLSTM parent-slot rows pb [J*n][H], same box
  FwdArgs f;
};
constexpr int kMetaRing = 4;
constexpr int kStageBytes = kTM * 128;                  // one K-atom of one slot (16 KB)
constexpr int kSmemLimit = 227 * 1024;

template <int J>
struct TcMeta {
  alignas(16) int own[kTM];    // input id (output row), -1 past cnt
  alignas(16) int xr[kTM];     // row of xb (word or node-order row), -1 = none (zeros)
  alignas(16) int root[kTM];   // index in roots[] or -1
  alignas(16) int ch[J][kTM];  // children state rows, -1 absent (zeros)
  alignas(16) int ps[kTM];     // TreeLSTM / TreeFC / DAG slots: parent-slot row of the node's h, -1 = none
  alignas(16) int ps1[kTM];    // DAG slots: a second parent's slot row, -1 = none
  int i0, cnt;
};

constexpr int pow2_cols(int c) { return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512; }

// SP = 1: bf16 operands (dtype CX_BF16). SP = 2: the fp32 path on the tensor
// cores (dtype CX_F32, large batches): every fp32 operand x is split into
// x_hi = bf16(x) and x_lo = bf16(x - x_hi) (|x - x_hi - x_lo| <= 2^-17 |x|),
// stored as one bf16 row [hi | lo] of 2H, and each product is formed as
// A_hi B_hi + A_hi B_lo + A_lo B_hi (three bf16 MMAs, fp32 accumulation in
// TMEM; the dropped A_lo B_lo term is <= 2^-16 |A B|): fp32-class accuracy on
// the bf16 tensor pipe, at 3x its MMA work.
template <int CELL, int H, int MAXC, int SP = 1>
struct TcCfg {
  static constexpr bool LSTM = CELL == CX_TREELSTM, DAG = CELL == CX_DAGRNN, FC = CELL == CX_TREEFC;
  static constexpr int J = MAXC;
  static constexpr int U = DAG ? (SP == 2 ? 64 : (H >= 128 ? 128 : H)) : 32;
  static constexpr int KA = H / 64;        // K-atoms (64 bf16) of one hi or lo half
  static constexpr int KAA = SP * KA;      // K-atoms of a gathered operand row (hi [| lo])
  static constexpr int RW = SP * H;        // bf16 elements per operand row
  // split TreeLSTM: W_iou (leaf phase) and [U_iou; U_f] (levels) take turns in
  // one shared-memory region (both at once would not fit with the stages)
  static constexpr bool BSHARE = LSTM && (SP == 2 || CX_TC_BSHARE_ALL);
  // split DAG-RNN / TreeFC: the B_hi and B_lo rows of a K-atom are adjacent
  // (one 2R-row operand), so a hi A atom meets both in ONE MMA of N = 2R (its
  // A tile is read from shared memory once, not twice) into accumulator
  // columns [0, R) (A B_hi) and [R, 2R) (A_hi B_lo), summed by the epilogue
  // (TreeLSTM's 4U = 128-column accumulators per child would not fit TMEM twice)
  static constexpr bool MERGE = SP == 2 && !LSTM && !CX_TC_SKIP_LO;
  static constexpr int MW = MERGE ? 2 : 1;  // accumulator width factor
  static constexpr int B0 = LSTM ? 3 * U : U;  // rows: LSTM W_iou | DAG W_x | FC W_left
  static constexpr int B1 = LSTM ? 4 * U : U;  // rows: LSTM [U_iou; U_f] | DAG U | FC W_right
  static constexpr int NACC = LSTM ? J : 1;    // accumulators per tile (level phase)
  static constexpr int NLVL = LSTM ? 4 * U : U;  // N of a level-phase MMA
  static constexpr int NLEAF = LSTM ? 3 * U : U;
  static constexpr int BUFC = NACC * NLVL * MW;  // TMEM columns per accumulator buffer
  static constexpr int TCOLS = pow2_cols(2 * BUFC);
  static constexpr bool XSLOT = LSTM || DAG;
  // CTAs that own different unit slices of the same node tiles form a cluster
  // of CL; each fetches 1/CL of every stage and multicasts it to all
  static constexpr int GU = H / U;
  // One CTA per cluster. Measured: cluster-multicast gathers were gated by the
  // slowest CTA and TMA gather4 is issue-bound; multicasting TreeLSTM's
  // contiguous tiles over the GU unit-group CTAs (CL = GU, stage k issued by
  // rank k mod CL, every CTA expecting the stage's bytes) was correct but
  // slower: only 15 clusters of 8 are co-resident (120 CTAs instead of 144;
  // b4096 forward 293 -> 340 us).
  static constexpr int CL = 1;
  // TreeLSTM and TreeFC (trees: one parent per node) keep each node's operand
  // row in its parent's child slot (pb), so a level tile's operands are
  // contiguous rows loaded by TMA; DAG-RNN gathers rows with cp.async
  static constexpr bool SLOTS = LSTM || FC;
  // split-fp32 DAG-RNN: when no node has more than two parents (decided on the
  // device, the prologue counts them) each h goes into both parents' slot rows
  // and the operands load by TMA as for trees; else the cp.async gathers
  static constexpr bool DSLOT = DAG && SP == 2 && CX_TC_DSLOT;
  static constexpr int FEEDW = SLOTS ? 1 : 4;            // feeding warps
  static constexpr int META0 = kFeed0 + FEEDW;           // first bookkeeping warp
  static constexpr int THREADS = 32 * (META0 + kMetaWarps);
  static constexpr int WORK = 32 * META0;                // threads of the working warps
  static constexpr size_t bbytes0 = (size_t)B0 * KAA * 128, bbytes1 = (size_t)B1 * KAA * 128;
  static constexpr size_t bregion = BSHARE ? (bbytes0 > bbytes1 ? bbytes0 : bbytes1) : bbytes0 + bbytes1;
  static constexpr size_t static_bytes = sizeof(TcMeta<J>) * kMetaRing + 4 * U * 4 + 64 * 8 + 64;
  // TreeLSTM stages hold NAB K-atoms, loaded by ONE 3D TMA instruction:
  // tools/micro/tma_rate.cu measures ~0.36 us per TMA instruction per issuing
  // thread whatever its size (16 KB: 45 GB/s/SM, 32 KB: 87, 64 KB: 137), so
  // the one-lane producer feeds twice as fast with 2-atom boxes
  static constexpr int NAB = (SLOTS || DSLOT) && KAA % CX_TC_NAB == 0 ? CX_TC_NAB : 1;
  static constexpr int STB = kStageBytes * NAB;  // bytes per stage
  static constexpr int S_fit =
      (int)((kSmemLimit - 1024 - static_bytes - bregion) / STB);
  static constexpr int S = S_fit > CX_TC_SMAX ? CX_TC_SMAX : S_fit;
  static constexpr size_t dyn_bytes = 1024 + bregion + (size_t)S * STB;
  static_assert(H % 64 == 0 && H % U == 0, "H must be a multiple of 64 and of U");
  static_assert(BUFC * 2 <= 512, "TMEM: two accumulator buffers must fit 512 columns");
  static_assert(NLVL * MW <= 256 && NLEAF * MW <= 256 && NLVL % 16 == 0, "UMMA N");

  __host__ __device__ static constexpr int nslots(bool leaf) {
    return leaf ? 1 : (LSTM ? J : DAG ? J + 1 : 2);
  }
  // slot s of a phase -> operand (-1 = x rows, k = child k), B matrix, accumulator
  __device__ static void slot(bool leaf, int s, int &src, int &bm, int &acc) {
    if (leaf) { src = -1; bm = 0; acc = 0; return; }
    if (LSTM) { src = s; bm = 1; acc = s; return; }
    if (DAG) { src = s == 0 ? -1 : s - 1; bm = s == 0 ? 0 : 1; acc = 0; return; }
    src = s; bm = s; acc = 0;  // FC
  }
};

__device__ __forceinline__ void cp16_zfill(uint32_t dst, const void *src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0) : "memory");
}
// Drop a dead 128-byte workspace line from L2 without writing it back (its
// only reader has consumed it): the TreeLSTM memory cells and parent-slot rows
// would otherwise be evicted to HBM although nobody reads them again.
__device__ __forceinline__ void discard_l2(const void *p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ uint4 f32x8_to_bf16(float4 a, float4 b) {
  return make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y),
                    pack_bf16(b.z, b.w));
}
template <int N>
__device__ __forceinline__ void store_f32(float *dst, const float (&v)[N]) {
  float4 *d = reinterpret_cast<float4 *>(dst);
#pragma unroll
  for (int q = 0; q < N / 4; q++) d[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
}
// caller outputs (never re-read by the kernel): streaming stores, so they do
// not evict the state rows and input rows the next gathers read from L2
template <int N>
__device__ __forceinline__ void store_f32_stream(float *dst, const float (&v)[N]) {
  float4 *d = reinterpret_cast<float4 *>(dst);
#pragma unroll
  for (int q = 0; q < N / 4; q++) __stcs(d + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
}
template <int N>
__device__ __forceinline__ void store_bf16(unsigned short *dst, const float (&v)[N]) {
  uint4 *d = reinterpret_cast<uint4 *>(dst);
#pragma unroll
  for (int q = 0; q < N / 8; q++)
    d[q] = make_uint4(pack_bf16(v[8 * q], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                      pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
}
// 256-bit global accesses (sm_100: LDG/STG.256): a thread's 16-unit fp32 row
// piece is 2 requests instead of 4, its bf16 piece 1 instead of 2
__device__ __forceinline__ void st256(float *p, const float *v) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]), "f"(v[1]),
               "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]) : "memory");
}
__device__ __forceinline__ void st256_cs(float *p, const float *v) {  // streaming (caller outputs)
  asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]), "f"(v[1]),
               "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]) : "memory");
}
__device__ __forceinline__ void ld256(const float *p, float *v) {  // L1-allocating
  asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
                 "=f"(v[7]) : "l"(p));
}
__device__ __forceinline__ void st256_bf16(unsigned short *p, const float *v) {  // 16 bf16
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
               "r"(pack_bf16(v[0], v[1])), "r"(pack_bf16(v[2], v[3])), "r"(pack_bf16(v[4], v[5])),
               "r"(pack_bf16(v[6], v[7])), "r"(pack_bf16(v[8], v[9])), "r"(pack_bf16(v[10], v[11])),
               "r"(pack_bf16(v[12], v[13])), "r"(pack_bf16(v[14], v[15])) : "memory");
}
template <int N>
__device__ __forceinline__ void st_row(float *p, const float (&v)[N]) {
#pragma unroll
  for (int q = 0; q < N / 8; q++) st256(p + 8 * q, v + 8 * q);
}
template <int N>
__device__ __forceinline__ void st_row_cs(float *p, const float (&v)[N]) {
#pragma unroll
  for (int q = 0; q < N / 8; q++) st256_cs(p + 8 * q, v + 8 * q);
}
template <int N>
__device__ __forceinline__ void st_row_bf16(unsigned short *p, const float (&v)[N]) {
#pragma unroll
  for (int q = 0; q < N / 16; q++) st256_bf16(p + 16 * q, v + 16 * q);
}

__device__ __forceinline__ float bf16_round(float x) {
  return __bfloat162float(__float2bfloat16_rn(x));
}
// An operand row piece: SP = 1 -> bf16(v) at row[col..]; SP = 2 (split fp32,
// see TcCfg) -> hi = bf16(v) at row[col..] and lo = bf16(v - hi) at row[H + col..]
template <int SP, int H, int N>
__device__ __forceinline__ void st_op(unsigned short *row, int col, const float (&v)[N]) {
  if constexpr (SP == 1) {
    st_row_bf16<N>(row + col, v);
  } else {
    float hi[N], lo[N];
#pragma unroll
    for (int j = 0; j < N; j++) {
      hi[j] = bf16_round(v[j]);
      lo[j] = v[j] - hi[j];  // exact in fp32
    }
    st_row_bf16<N>(row + col, hi);
    st_row_bf16<N>(row + H + col, lo);
  }
}
// 8 consecutive fp32 values -> their bf16 hi (and lo) pieces
__device__ __forceinline__ void split8(float4 a, float4 b, uint4 &hi, uint4 &lo) {
  hi = f32x8_to_bf16(a, b);
  const float4 ah = make_float4(bf16_round(a.x), bf16_round(a.y), bf16_round(a.z), bf16_round(a.w));
  const float4 bh = make_float4(bf16_round(b.x), bf16_round(b.y), bf16_round(b.z), bf16_round(b.w));
  lo = f32x8_to_bf16(make_float4(a.x - ah.x, a.y - ah.y, a.z - ah.z, a.w - ah.w),
                     make_float4(b.x - bh.x, b.y - bh.y, b.z - bh.z, b.w - bh.w));
}

// Gate nonlinearities of the bf16 path: one MUFU op each (tanh.approx.f32,
// relative error ~2^-11, far inside the bf16 path's 2e-2 budget; the fp32
// path keeps the ex2/rcp forms of common.cuh).
__device__ __forceinline__ float tanh_mufu(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sigm_mufu(float x) { return fmaf(0.5f, tanh_mufu(0.5f * x), 0.5f); }
// per path: the bf16 path's MUFU forms, the split fp32 path's those of the fp32
// kernels (common.cuh, within ~5e-6 relative)
#ifndef CX_TC_FASTACT  // timing experiment only: the bf16 MUFU forms on the split path too
#define CX_TC_FASTACT 0
#endif
template <int SP>
__device__ __forceinline__ float act_sig(float x) {
  if constexpr (SP == 1 || CX_TC_FASTACT) return sigm_mufu(x); else return sigmoidf_(x);
}
template <int SP>
__device__ __forceinline__ float act_tanh(float x) {
  if constexpr (SP == 1 || CX_TC_FASTACT) return tanh_mufu(x); else return tanhf_(x);
}


// debug timeline (cx_debug_set_trace): thread `who` of each CTA records
// %globaltimer into slot s. Slots: 0 entry, 1 prologue done, 2+4l level l
// start, 3+4l producers done, 4+4l MMA issue done, 5+4l epilogue done.
__device__ __forceinline__ void tc_mark(const FwdArgs &a, int s, int who) {
  if (a.trace && threadIdx.x == who && s >= 0 && s < a.trace_slots) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[(size_t)blockIdx.x * a.trace_slots + s] = t;
  }
}

template <int CELL, int H, int MAXC, int SP>
__global__ void __launch_bounds__(TcCfg<CELL, H, MAXC, SP>::THREADS, 1)
    tc_kernel(const __grid_constant__ TcArgs ta) {
  const FwdArgs &a = ta.f;
  using C = TcCfg<CELL, H, MAXC, SP>;
  constexpr int kMeta0 = C::META0, kWork = C::WORK;
  constexpr int J = C::J, U = C::U, KA = C::KA, KAA = C::KAA, RW = C::RW, S = C::S;
  extern __shared__ unsigned char smem_raw[];
  __shared__ TcMeta<J> meta[kMetaRing];
  __shared__ float s_bias[4 * U];
  __shared__ __align__(8) uint64_t bar_full[S], bar_empty[S], bar_tfull[2], bar_tempty[2],
      bar_mfull[kMetaRing], bar_mempty[kMetaRing];
  __shared__ uint32_t s_tmem;

  tc_mark(a, 0, 0);
  const int n = a.n;
  const int gn = blockIdx.x / a.Gu, gu = blockIdx.x % a.Gu;
  const int unit0 = gu * U;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool latch = gu == 0;
  unsigned char *sm = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char *sB0 = sm, *sB1 = C::BSHARE ? sm : sm + C::bbytes0, *sStage = sm + C::bregion;
  unsigned short *hb = a.hb;
  float *cs = a.cs;
  const unsigned short *xb = a.xb;
  unsigned epoch = 0;

  // ---- prologue: barriers, TMEM, biases, resident bf16 weights ---------------
  if (tid == 0) {
    // full: TreeLSTM 1 arrive + TMA bytes; cp.async feeding: one noinc arrival per thread
    for (int s = 0; s < S; s++) { mbar_init(&bar_full[s], C::SLOTS ? 1 : 32 * C::FEEDW); mbar_init(&bar_empty[s], C::CL); }
    for (int b = 0; b < 2; b++) { mbar_init(&bar_tfull[b], 1); mbar_init(&bar_tempty[b], kEpiThreads); }
    for (int m = 0; m < kMetaRing; m++) { mbar_init(&bar_mfull[m], 1); mbar_init(&bar_mempty[m], kEpiThreads); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) tmem_alloc<C::TCOLS>(&s_tmem);
  if constexpr (C::LSTM) {
    for (int q = tid; q < 4 * U; q += blockDim.x) {
      const int g = q / U, u = q % U;
      s_bias[q] = __ldg((g < 3 ? a.w[2] + g * H : a.w[4]) + unit0 + u);
    }
  } else {
    for (int q = tid; q < U; q += blockDim.x) s_bias[q] = __ldg(a.w[C::DAG ? 2 : 1] + unit0 + q);
  }
  // weights: B0 / B1 rows -> bf16 (SP = 2: hi atoms [0, KA), lo atoms
  // [KA, 2 KA)), K-major SW128; 8 chunks' loads in flight per thread before
  // their conversions and stores. sel: 0 both, 1 B0 only, 2 B1 only (BSHARE)
  auto load_b = [&](int sel, int nthr) {
    const int r0 = sel == 2 ? C::B0 : 0, r1 = sel == 1 ? C::B0 : C::B0 + C::B1;
    const int NCH = (r1 - r0) * KA * 8;
    auto wsrc = [&](int idx, unsigned char *&Bm, int &rows, int &q, int &ka, int &c) -> const float * {
      q = idx / (KA * 8);
      const int rem = idx - q * (KA * 8);
      ka = rem >> 3;
      c = rem & 7;
      q += r0;
      const bool second = q >= C::B0;
      if (second) q -= C::B0;
      Bm = second ? sB1 : sB0;
      rows = second ? C::B1 : C::B0;
      if constexpr (C::LSTM) {
        const int g = q / U, u = q % U;
        if (!second) return a.w[0] + (size_t)(g * H + unit0 + u) * H;                // W_iou
        return g < 3 ? a.w[1] + (size_t)(g * H + unit0 + u) * H                      // U_iou
                     : a.w[3] + (size_t)(unit0 + u) * H;                              // U_f
      } else if constexpr (C::DAG) {
        return a.w[second ? 1 : 0] + (size_t)(unit0 + q) * H;                        // U | W_x
      } else {
        return a.w[0] + (size_t)(unit0 + q) * 2 * H + (second ? H : 0);              // W [H][2H]
      }
    };
    for (int base = 0; base < NCH; base += 8 * nthr) {
      float4 lo[8], hi[8];
#pragma unroll
      for (int e = 0; e < 8; e++) {
        const int idx = base + e * nthr + tid;
        if (idx < NCH) {
          unsigned char *Bm;
          int rows, q, ka, c;
          const float *row = wsrc(idx, Bm, rows, q, ka, c);
          const float4 *sp = reinterpret_cast<const float4 *>(row + ka * 64 + c * 8);
          lo[e] = __ldg(sp);
          hi[e] = __ldg(sp + 1);
        }
      }
#pragma unroll
      for (int e = 0; e < 8; e++) {
        const int idx = base + e * nthr + tid;
        if (idx < NCH) {
          unsigned char *Bm;
          int rows, q, ka, c;
          (void)wsrc(idx, Bm, rows, q, ka, c);
          if constexpr (SP == 1) {
            *reinterpret_cast<uint4 *>(Bm + (size_t)ka * rows * 128 + sw128_off(q, c)) = f32x8_to_bf16(lo[e], hi[e]);
          } else if constexpr (C::MERGE) {  // atom ka = [hi rows; lo rows]
            uint4 ph, pl;
            split8(lo[e], hi[e], ph, pl);
            *reinterpret_cast<uint4 *>(Bm + (size_t)ka * 2 * rows * 128 + sw128_off(q, c)) = ph;
            *reinterpret_cast<uint4 *>(Bm + (size_t)ka * 2 * rows * 128 + sw128_off(rows + q, c)) = pl;
          } else {
            uint4 ph, pl;
            split8(lo[e], hi[e], ph, pl);
            *reinterpret_cast<uint4 *>(Bm + (size_t)ka * rows * 128 + sw128_off(q, c)) = ph;
            *reinterpret_cast<uint4 *>(Bm + (size_t)(ka + KA) * rows * 128 + sw128_off(q, c)) = pl;
          }
        }
      }
    }
  };
  load_b(C::BSHARE ? 1 : 0, (int)blockDim.x);

  tc_mark(a, 60, 0);
  // the linearization is read from here on (PDL: the above overlapped it)
  griddep_wait();
  const int status0 = *reinterpret_cast<volatile int *>(&a.hdr->status);
  const int L = status0 == CX_OK ? a.hdr->num_levels : 0, first_leaf = a.hdr->first_leaf;
  const int xlo = C::DAG ? 0 : first_leaf;  // node-order x rows start here
  const bool hoist = C::LSTM && a.hoist;
  // DAG-RNN computation hoisting (PAPER §4.3; the input matvecs as
  // one GEMM up front): in table mode the input projection
  // W_x x + b is computed once per vocabulary word (phase l = -1, into the fp32
  // table a.hf [V][H]); the leaves (level 0) are h = tanh(P[word]) without an
  // MMA, and a level's tiles contract only the children (U h~) and add their
  // word's P row in the epilogue.
  const bool hx = C::DAG && SP == 2 && a.hoist;
  const int l0 = hx ? -1 : 0;
  auto nsl_of = [&](int l) -> int { return hx ? (l < 0 ? 1 : l == 0 ? 0 : J) : C::nslots(l == 0); };
  auto slot_of = [&](int l, int s_, int &src, int &bm, int &acc) {
    if (hx) {
      src = l < 0 ? -1 : s_;
      bm = l < 0 ? 0 : 1;
      acc = 0;
      return;
    }
    C::slot(l == 0, s_, src, bm, acc);
  };
  const bool discard_ok = !a.discard_off;  // CX_DISCARD=0: keep dead lines (measurement)
  // Per-level precision/unit dispatch (north_star: tensor cores only where the
  // level really is a dense GEMM): a level whose node chunk has at most FMX
  // nodes per node group runs on the epilogue warps' FMA pipes (resident B from
  // shared memory, operands staged in the idle stage ring) instead of a
  // 128-row UMMA tile (whose K pipeline, MMA and epilogue latency chain would
  // cost several microseconds for a handful of rows). Same operand precision:
  // bf16 (SP = 1) or hi + lo (SP = 2), fp32 products and sums.
  // FMX: nodes per batch (staged at once); FML: nodes per node group up to
  // which a level runs on FMA, in batches (TreeFC's 2H-deep contraction of
  // split operands costs the tile path ~17 us per level: more levels qualify)
  constexpr int FMX = C::LSTM ? 4 : C::FC ? 10 : 6;
  // (bf16 TreeLSTM: its 8-stage tiles beat the FMA path, measured ~1 %: tiles only)
  constexpr int FML = C::FC ? (SP == 2 ? CX_TC_FML_FC : 10) : (C::LSTM && SP == 1) ? 0 : FMX;
  auto is_fma = [&](int l) { return l >= 1 && !a.tc_fma_off && __ldg(a.lsize + l) <= FML * a.Gn; };
  const int sbase = hoist ? a.V : 0;  // state row of internal node i = sbase + i
  if (C::DSLOT && status0 == CX_OK) {  // parent counts / slots start empty everywhere
    const size_t total_threads = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + tid; i < (size_t)n; i += total_threads) {
      a.pcnt[i] = 0;
      a.pslot[i] = -1;
      a.pslot1[i] = -1;
    }
    grid_sync(a.bar, gridDim.x, epoch);
  }
  // ---- phase 0: bf16 input rows ------------------------------------------------
  if (C::XSLOT && status0 == CX_OK) {
    const size_t total_threads = (size_t)gridDim.x * blockDim.x;
    const size_t gt = (size_t)blockIdx.x * blockDim.x + tid;
    constexpr int q8 = H / 8;
    unsigned short *xw = const_cast<unsigned short *>(xb);
    if (a.xmode == 0) {  // whole table, indexed by word
      const size_t total = (size_t)a.V * q8;
      for (size_t b0 = gt; b0 < total; b0 += 4 * total_threads) {  // 4 chunks in flight
        float4 lo[4], hi[4];
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const size_t idx = b0 + e * total_threads;
          if (idx < total) {
            const float4 *sp = reinterpret_cast<const float4 *>(a.emb + idx * 8);
            lo[e] = __ldg(sp);
            hi[e] = __ldg(sp + 1);
          }
        }
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const size_t idx = b0 + e * total_threads;
          if (idx < total) {
            if constexpr (SP == 1) {
              *reinterpret_cast<uint4 *>(xw + idx * 8) = f32x8_to_bf16(lo[e], hi[e]);
            } else {  // row idx / q8, columns 8 (idx % q8): hi, then lo at + H
              const size_t o = (idx / q8) * RW + (idx % q8) * 8;
              uint4 ph, pl;
              split8(lo[e], hi[e], ph, pl);
              *reinterpret_cast<uint4 *>(xw + o) = ph;
              *reinterpret_cast<uint4 *>(xw + o + H) = pl;
            }
          }
        }
      }
      if (hoist) {  // state row of every node: leaves -> their word's row
        for (size_t i = gt; i < (size_t)n; i += total_threads) {
          int row = a.V + (int)i;
          if ((int)i >= first_leaf) {
            const int own = __ldg(a.perm + i);
            int w = __ldg(a.words + own);
            if (w < 0 || w >= a.V) {
              latch_error(a.hdr, CX_E_WORD_RANGE, own);
              w = 0;
            }
            row = w;
          }
          a.crow[i] = row;
        }
      }
    } else {  // this batch's x rows in node order (new ids [xlo, n))
      const size_t total = (size_t)(n - xlo) * q8;
      for (size_t idx = gt; idx < total; idx += total_threads) {
        const int r = (int)(idx / q8), c = (int)(idx - (size_t)r * q8);
        const int own = __ldg(a.perm + xlo + r);
        int w = __ldg(a.words + own);
        if (w < 0 || w >= a.V) {
          if (c == 0) latch_error(a.hdr, CX_E_WORD_RANGE, own);
          w = 0;
        }
        const float4 *s = reinterpret_cast<const float4 *>(a.emb + (size_t)w * H + c * 8);
        if constexpr (SP == 1) {
          *reinterpret_cast<uint4 *>(xw + (size_t)r * H + c * 8) = f32x8_to_bf16(__ldg(s), __ldg(s + 1));
        } else {
          uint4 ph, pl;
          split8(__ldg(s), __ldg(s + 1), ph, pl);
          *reinterpret_cast<uint4 *>(xw + (size_t)r * RW + c * 8) = ph;
          *reinterpret_cast<uint4 *>(xw + (size_t)r * RW + H + c * 8) = pl;
        }
      }
    }
  }
  if (C::SLOTS && status0 == CX_OK) {  // parent-slot row of every non-root node
    const size_t total_threads = (size_t)gridDim.x * blockDim.x;
    const size_t gt = (size_t)blockIdx.x * blockDim.x + tid;
    for (size_t pn = gt; pn < (size_t)first_leaf; pn += total_threads) {
#pragma unroll
      for (int k = 0; k < J; k++) {
        const int c = __ldg(a.chn + (size_t)k * n + pn);
        if (c >= 0) a.pslot[c] = k * n + (int)pn;
      }
    }
    const int R = a.hdr->num_roots;  // roots are nobody's child: no conflict
    for (size_t r = gt; r < (size_t)R; r += total_threads) a.pslot[__ldg(a.roots + r)] = -1;
  }
  if (C::DSLOT && status0 == CX_OK) {  // up to two parents' slot rows per node
    const size_t total_threads = (size_t)gridDim.x * blockDim.x;
    const size_t gt = (size_t)blockIdx.x * blockDim.x + tid;
    for (size_t pn = gt; pn < (size_t)n; pn += total_threads) {
#pragma unroll
      for (int k = 0; k < J; k++) {
        const int c = __ldg(a.chn + (size_t)k * n + pn);
        if (c < 0) {  // an absent child's slot row is summed by the MMA: zeros (a
          // previous call of this shape may have left a child's h in it)
          uint4 *z = reinterpret_cast<uint4 *>(a.pb + ((size_t)k * n + pn) * RW);
          for (int q = 0; q < RW / 8; q++) z[q] = make_uint4(0u, 0u, 0u, 0u);
          continue;
        }
        const int idx = atomicAdd(a.pcnt + c, 1);  // which parent gets which slot: either
        if (idx == 0) a.pslot[c] = k * n + (int)pn;
        else if (idx == 1) a.pslot1[c] = k * n + (int)pn;
        else atomicOr(&a.bar->pad[2], 1u);  // a third parent: gather mode
      }
    }
  }
  tc_mark(a, 61, 0);
  fence_proxy_async();  // resident weights (generic stores) -> tensor-core reads
  fence_before();
  cluster_sync_all();   // peers' mbarriers initialised before any multicast
  grid_sync(a.bar, gridDim.x, epoch);
  fence_after();
  const uint32_t tmem = s_tmem;
  // DAG parent slots usable: no node has a third parent, and every operand row
  // set is contiguous (x rows hoisted away or in node order)
  const bool dslots = C::DSLOT && status0 == CX_OK && (hx || a.xmode == 1) &&
                      *reinterpret_cast<volatile unsigned *>(&a.bar->pad[2]) == 0u;
  if (dslots) {  // stages are filled by ONE TMA arrival (+ bytes), not per-thread cp.async arrivals
    if (tid == 0) {
      for (int s_ = 0; s_ < S; s_++) mbar_init(&bar_full[s_], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  tc_mark(a, 1, 0);

  // Hoisted leaves. slot_fill: each leaf's bf16 h copied from the word table
  // into its parent's child-slot row (needed before level 1). out_copy: the
  // leaves' caller outputs (h_out, aux_out, root_out) from the fp32 word table.
  // A warp loads the indices of 32 leaves in one coalesced round trip, then
  // copies 8 rows at a time (all loads before the stores) with 256-bit accesses.
  auto leaf_pass = [&](bool slot_fill) {
    const int nleaf = n - first_leaf;
    const int gw = (blockIdx.x * kWork + tid) >> 5, nw = (gridDim.x * kWork) >> 5;
    for (int j0 = gw * 32; j0 < nleaf; j0 += nw * 32) {
      const int jl = j0 + lane;
      int dst = -1, w = 0, r = -1;
      if (jl < nleaf) {
        const int j = first_leaf + jl;
        w = __ldcg(a.crow + j);
        if (slot_fill) {
          dst = __ldcg(a.pslot + j);
        } else {
          dst = __ldg(a.perm + j);
          if (a.root_out) {  // a one-node structure: its leaf is a root
            const int q = __ldg(a.sid + j);
            r = __ldg(a.roots + q) == j ? q : -1;
          }
        }
      }
      const int cnt = min(32, nleaf - j0);
      if (slot_fill) {  // bf16 rows: RW/16 lanes x 32 B per row, 32/(RW/16) rows per pass
        constexpr int LPR = RW / 16 > 32 ? 32 : RW / 16, RPP = 32 / LPR;  // (hoisting: TreeLSTM only)
        static_assert(!C::LSTM || RW / 16 <= 32, "one warp per operand row");
        for (int k0 = 0; k0 < cnt; k0 += 8 * RPP) {
          float v[8][8];
          int dk[8];
#pragma unroll
          for (int u = 0; u < 8; u++) {
            const int k = k0 + u * RPP + lane / LPR;
            const int kk = min(k, cnt - 1);
            dk[u] = __shfl_sync(0xffffffffu, dst, kk);
            const int wk = __shfl_sync(0xffffffffu, w, kk);
            if (k >= cnt) dk[u] = -1;
            ld256(reinterpret_cast<const float *>(hb + (size_t)wk * RW) + 8 * (lane % LPR), v[u]);
          }
#pragma unroll
          for (int u = 0; u < 8; u++)
            if (dk[u] >= 0) st256(reinterpret_cast<float *>(a.pb + (size_t)dk[u] * RW) + 8 * (lane % LPR), v[u]);
        }
      } else {  // fp32 rows: H/8 lanes x 32 B per row
        constexpr int LPR = H / 8 > 32 ? 32 : H / 8, CPL = H / 8 / LPR, RPP = 32 / LPR;
        for (int k0 = 0; k0 < cnt; k0 += 8 * RPP) {
          float v[8][CPL][8];
          int dk[8], rk[8], wk[8];
#pragma unroll
          for (int u = 0; u < 8; u++) {
            const int k = k0 + u * RPP + lane / LPR;
            const int kk = min(k, cnt - 1);
            dk[u] = __shfl_sync(0xffffffffu, dst, kk);
            rk[u] = __shfl_sync(0xffffffffu, r, kk);
            wk[u] = __shfl_sync(0xffffffffu, w, kk);
            if (k >= cnt) dk[u] = -1;
#pragma unroll
            for (int e = 0; e < CPL; e++) ld256(a.hf + (size_t)wk[u] * H + 8 * (lane % LPR + LPR * e), v[u][e]);
          }
#pragma unroll
          for (int u = 0; u < 8; u++) {
            if (dk[u] < 0) continue;
#pragma unroll
            for (int e = 0; e < CPL; e++) {
              const int col = 8 * (lane % LPR + LPR * e);
              st256_cs(a.h_out + (size_t)dk[u] * H + col, v[u][e]);
              if (rk[u] >= 0) st256(a.root_out + (size_t)rk[u] * H + col, v[u][e]);
              if (a.aux_out) {
                float cv[8];
                ld256(cs + (size_t)wk[u] * H + col, cv);
                st256_cs(a.aux_out + (size_t)dk[u] * H + col, cv);
              }
            }
          }
        }
      }
    }
  };

  // level ranges: identical in every role
  auto level_range = [&](int l, int &lo, int &hi) {
    if (l < 0 || (l == 0 && hoist)) {  // once per vocabulary word (rows [0, V))
      chunk_of(a.V, a.Gn, gn, lo, hi);
    } else {
      chunk_of(__ldg(a.lsize + l), a.Gn, gn, lo, hi);
      const int lb = __ldg(a.lbeg + l);
      lo += lb;
      hi += lb;
    }
  };
  // grid barrier between levels among the working warps (the bookkeeping warps
  // do not wait): named barrier, then thread 0's release/acquire counter
  auto level_sync = [&]() {
    named_bar(3, kWork);
    epoch += 1;
    if (tid == 0) {
      red_release_add_u32(&a.bar->count, 1u);
      const unsigned target = epoch * gridDim.x;
      unsigned long long spins = 0;
      while (ld_relaxed_u32(&a.bar->count) < target) {
        if (++spins > (1ull << 26)) __trap();
      }
      (void)ld_acquire_u32(&a.bar->count);
    }
    named_bar(3, kWork);
  };

  // ---- a small level on FMA (is_fma): the 8 epilogue warps ------------------
  // 1. node info; 2. operand rows -> fp32 in the stage ring; 3. partial dot
  // products thread = (accumulator column, K part); 4. sums + the cell's gate
  // epilogue per (node, unit), outputs as the tile epilogue writes them.
  auto fma_batch = [&](int l, int lo, int hi) {
    constexpr int NA = C::NACC, NC = C::NLVL, COLS = NA * NC;
    constexpr int KS = kEpiThreads / COLS >= 1 ? kEpiThreads / COLS : 1;
    constexpr int NSLM = C::LSTM ? J : C::DAG ? J + 1 : 2;
    static_assert(COLS <= kEpiThreads && kEpiThreads % COLS == 0 && (H / KS) % 8 == 0, "FMA split");
    constexpr size_t kAf = (size_t)NSLM * FMX * H, kDp = (size_t)KS * FMX * COLS;
    static_assert(4 * (kAf + kDp) + 4 * FMX * (9 + 2 * J) <= (size_t)S * C::STB, "FMA level fits the stage ring");
    const int cnt = hi - lo, ntid = tid;  // tid < kEpiThreads
    const int nsl = nsl_of(l);
    float *Af = reinterpret_cast<float *>(sStage), *Dp = Af + kAf;
    int *n_own = reinterpret_cast<int *>(Dp + kDp), *n_root = n_own + FMX, *n_ps = n_root + FMX,
        *n_ps1 = n_ps + FMX, *n_xr = n_ps1 + FMX, *n_ch = n_xr + FMX /* [J][FMX] operand rows */,
        *n_ck = n_ch + J * FMX;
    if (ntid < cnt) {  // 1. node info (as the bookkeeping warps compute it)
      const int i = lo + ntid, own = __ldg(a.perm + i);
      n_own[ntid] = own;
      int root = -1;
      if (a.root_out) {
        const int sv = __ldg(a.sid + i);
        root = __ldg(a.roots + sv) == i ? sv : -1;
      }
      n_root[ntid] = root;
      n_ps[ntid] = (C::SLOTS || dslots) ? __ldcg(a.pslot + i) : -1;
      n_ps1[ntid] = dslots ? __ldcg(a.pslot1 + i) : -1;
      int xr = -1;
      if (C::DAG) {
        if (a.xmode == 0) {
          int w = __ldg(a.words + own);
          if (w < 0 || w >= a.V) {
            if (latch) latch_error(a.hdr, CX_E_WORD_RANGE, own);
            w = 0;
          }
          xr = w;
        } else {
          xr = i - xlo;
        }
      }
      n_xr[ntid] = xr;
      bool absent = false;
      int nc = 0;
#pragma unroll
      for (int k = 0; k < J; k++) {
        int c = __ldg(a.chn + (size_t)k * n + i);
        absent = absent || c < 0;
        if (absent) c = -1;
        nc += c >= 0;
        const int srow = c >= 0 ? (hoist ? __ldcg(a.crow + c) : c) : -1;  // the child's state row
        n_ck[k * FMX + ntid] = srow;
        // operand row of slot k: TreeLSTM the parent-slot row, else the state row
        n_ch[k * FMX + ntid] = (C::SLOTS || dslots) ? (c >= 0 ? k * n + i : -1) : srow;
      }
      if (C::FC && nc != 2 && latch) latch_error(a.hdr, CX_E_ARITY, own);
    }
    named_bar(5, kEpiThreads);
    // 2. operands -> fp32 (hi [+ lo]); absent rows -> zeros
    constexpr int Q8 = H / 8;
    for (int idx = ntid; idx < nsl * cnt * Q8; idx += kEpiThreads) {
      const int q = idx % Q8, st = idx / Q8, t = st % cnt, sl = st / cnt;
      int src, bm, acc;
      slot_of(l, sl, src, bm, acc);
      const int row = src < 0 ? n_xr[t] : n_ch[src * FMX + t];
      const unsigned short *base = src < 0 ? xb : ((C::SLOTS || dslots) ? a.pb : hb);
      float f[8];
      if (row >= 0) {
        const uint4 hv = __ldcg(reinterpret_cast<const uint4 *>(base + (size_t)row * RW + 8 * q));
        const unsigned hw[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
        for (int e = 0; e < 4; e++) {
          f[2 * e] = __uint_as_float(hw[e] << 16);
          f[2 * e + 1] = __uint_as_float(hw[e] & 0xffff0000u);
        }
        if constexpr (SP == 2) {
          const uint4 lv = __ldcg(reinterpret_cast<const uint4 *>(base + (size_t)row * RW + H + 8 * q));
          const unsigned lw[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
          for (int e = 0; e < 4; e++) {
            f[2 * e] += __uint_as_float(lw[e] << 16);
            f[2 * e + 1] += __uint_as_float(lw[e] & 0xffff0000u);
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < 8; e++) f[e] = 0.f;
      }
      float4 *d = reinterpret_cast<float4 *>(Af + ((size_t)sl * FMX + t) * H + 8 * q);
      d[0] = make_float4(f[0], f[1], f[2], f[3]);
      d[1] = make_float4(f[4], f[5], f[6], f[7]);
    }
    named_bar(5, kEpiThreads);
    // 3. partial sums: column col of accumulator ac, K part p, every node
    {
      const int col = ntid % COLS, p = ntid / COLS;
      const int ac = col / NC, cc = col % NC;
      float part[FMX];
#pragma unroll
      for (int t = 0; t < FMX; t++) part[t] = 0.f;
      for (int sl = 0; sl < nsl; sl++) {
        int src, bm, acc;
        slot_of(l, sl, src, bm, acc);
        if (acc != ac) continue;
        const unsigned char *Bm = bm ? sB1 : sB0;
        const int rows = bm ? C::B1 : C::B0;
        for (int k = p * (H / KS); k < (p + 1) * (H / KS); k += 8) {
          const int ka = k >> 6, c8 = (k >> 3) & 7;
          float w[8];
          const unsigned char *hp, *lp = nullptr;
          if constexpr (C::MERGE) {
            hp = Bm + (size_t)ka * 2 * rows * 128 + sw128_off(cc, c8);
            lp = Bm + (size_t)ka * 2 * rows * 128 + sw128_off(rows + cc, c8);
          } else {
            hp = Bm + (size_t)ka * rows * 128 + sw128_off(cc, c8);
            if (SP == 2) lp = Bm + (size_t)(ka + KA) * rows * 128 + sw128_off(cc, c8);
          }
          const uint4 hv = *reinterpret_cast<const uint4 *>(hp);
          const unsigned hw[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
          for (int e = 0; e < 4; e++) {
            w[2 * e] = __uint_as_float(hw[e] << 16);
            w[2 * e + 1] = __uint_as_float(hw[e] & 0xffff0000u);
          }
          if (SP == 2) {
            const uint4 lv = *reinterpret_cast<const uint4 *>(lp);
            const unsigned lw[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
            for (int e = 0; e < 4; e++) {
              w[2 * e] += __uint_as_float(lw[e] << 16);
              w[2 * e + 1] += __uint_as_float(lw[e] & 0xffff0000u);
            }
          }
#pragma unroll
          for (int t = 0; t < FMX; t++) {
            if (t < cnt) {
              const float4 *ap = reinterpret_cast<const float4 *>(Af + ((size_t)sl * FMX + t) * H + k);
              const float4 x0 = ap[0], x1 = ap[1];
              float sacc = part[t];
              sacc = fmaf(x0.x, w[0], sacc); sacc = fmaf(x0.y, w[1], sacc);
              sacc = fmaf(x0.z, w[2], sacc); sacc = fmaf(x0.w, w[3], sacc);
              sacc = fmaf(x1.x, w[4], sacc); sacc = fmaf(x1.y, w[5], sacc);
              sacc = fmaf(x1.z, w[6], sacc); sacc = fmaf(x1.w, w[7], sacc);
              part[t] = sacc;
            }
          }
        }
      }
#pragma unroll
      for (int t = 0; t < FMX; t++)
        if (t < cnt) Dp[((size_t)p * FMX + t) * COLS + col] = part[t];
    }
    named_bar(5, kEpiThreads);
    auto D = [&](int t, int col) {
      float v = 0.f;
#pragma unroll
      for (int p = 0; p < KS; p++) v += Dp[((size_t)p * FMX + t) * COLS + col];
      return v;
    };
    // 4. the cell epilogue per (node, unit)
    for (int idx = ntid; idx < cnt * U; idx += kEpiThreads) {
      const int t = idx / U, u = idx % U, i = lo + t, own = n_own[t], root = n_root[t];
      const int uu = unit0 + u;
      float h;
      if constexpr (C::LSTM) {
        float c = 0.f, vi = 0.f, vo = 0.f, vu = 0.f;
#pragma unroll
        for (int k = 0; k < J; k++) {
          const int ck = n_ck[k * FMX + t];
          if (ck < 0) continue;
          c = fmaf(act_sig<SP>(D(t, k * NC + 3 * U + u) + s_bias[3 * U + u]), __ldcg(cs + (size_t)ck * H + uu), c);
          vi += D(t, k * NC + u);
          vo += D(t, k * NC + U + u);
          vu += D(t, k * NC + 2 * U + u);
        }
        c = fmaf(act_sig<SP>(vi + s_bias[u]), act_tanh<SP>(vu + s_bias[2 * U + u]), c);
        h = act_sig<SP>(vo + s_bias[U + u]) * act_tanh<SP>(c);
        cs[(size_t)(sbase + i) * H + uu] = c;
        if (a.aux_out) a.aux_out[(size_t)own * H + uu] = c;
        const int ps = n_ps[t];
        if (ps >= 0) {
          unsigned short *prow = a.pb + (size_t)ps * RW;
          const float hi_ = bf16_round(h);
          prow[uu] = (unsigned short)(__float_as_uint(hi_) >> 16);
          if (SP == 2) prow[H + uu] = (unsigned short)(__float_as_uint(bf16_round(h - hi_)) >> 16);
        }
      } else {
        float v = D(t, u);
        if (hx) v += __ldcg(a.hf + (size_t)n_xr[t] * H + uu);
        else v += s_bias[u];
        h = act_tanh<SP>(v);
        // the operand rows: TreeFC / DAG slots the parents' child slots (none for a
        // root), else the DAG-RNN state row
        const float hi_ = bf16_round(h);
        const unsigned short hb16 = (unsigned short)(__float_as_uint(hi_) >> 16);
        const unsigned short lb16 = (unsigned short)(__float_as_uint(bf16_round(h - hi_)) >> 16);
        for (int pp = 0; pp < 2; pp++) {
          const int prow = pp == 0 ? n_ps[t] : n_ps1[t];
          unsigned short *hrow = (C::SLOTS || dslots) ? (prow >= 0 ? a.pb + (size_t)prow * RW : nullptr)
                                                      : (pp == 0 ? hb + (size_t)i * RW : nullptr);
          if (hrow) {
            hrow[uu] = hb16;
            if (SP == 2) hrow[H + uu] = lb16;
          }
        }
      }
      a.h_out[(size_t)own * H + uu] = h;
      if (root >= 0) a.root_out[(size_t)root * H + uu] = h;
    }
    fence_proxy_async();  // the stage ring (generic writes) is TMA's again next level
    named_bar(5, kEpiThreads);
  };
  auto fma_level = [&](int l, int lo, int hi) {
    for (int b0 = lo; b0 < hi; b0 += FMX) fma_batch(l, b0, min(hi, b0 + FMX));
  };

  if (warp >= kMeta0) {
    // ======================== tile bookkeeping ===============================
    // It depends on the linearization only, so these warps run ahead of the
    // level barriers (bounded by the 4-slot ring the epilogue releases).
    uint32_t T0m = 0;
    for (int l = l0; l < L; l++) {
      const bool leaf = l == 0, proj = l < 0;
      if (C::FC && leaf) continue;  // TreeFC leaves: a copy, no tiles
      int lo, hi;
      level_range(l, lo, hi);
      const int ntiles = is_fma(l) ? 0 : (hi - lo + kTM - 1) / kTM;
      const uint32_t T0 = T0m;
      // lane handles rows lane + 32 q; two dependent rounds of index loads
      const int mw = warp - kMeta0;
      for (int t = mw; t < ntiles; t += kMetaWarps) {
        const uint32_t TT = T0 + t;
        const int ms = TT % kMetaRing;
        const int i0 = lo + t * kTM, cnt = min(kTM, hi - i0);
        mbar_wait(&bar_mempty[ms], ((TT / kMetaRing) & 1) ^ 1);
        const int tslot = (l >= 0 && l < 2 && t < 5) ? 128 + 12 * (t + 5 * l) : 1 << 30;
        tc_mark(a, tslot + 0, warp * 32);
        TcMeta<J> &m = meta[ms];
        if constexpr (C::LSTM) {
          // the slot's previous tile (TT - kMetaRing, filled by this warp) is
          // done: its children's memory-cell lines of this CTA's units were
          // read once, by that epilogue, and are dead (a tree node has one
          // parent; hoisted word rows [0, V) are shared and stay)
          if (TT >= (uint32_t)kMetaRing && discard_ok)
            for (int r = lane; r < kTM; r += 32)
#pragma unroll
              for (int k = 0; k < J; k++) {
                const int row = m.ch[k][r];
                if (row >= (hoist ? a.V : 0)) discard_l2(cs + (size_t)row * H + unit0);
              }
        }
        constexpr int RQ = kTM / 32;
        int own[RQ], sv[RQ], psv[RQ], ps1v[RQ], ch[RQ][J];
#pragma unroll
        for (int q = 0; q < RQ; q++) {  // round 1: perm, structure, children
          const int r = lane + 32 * q, i = i0 + r;
          own[q] = -1;
          sv[q] = -1;
          psv[q] = -1;
          ps1v[q] = -1;
#pragma unroll
          for (int k = 0; k < J; k++) ch[q][k] = -1;
          if (r < cnt && !(leaf && hoist) && !proj) {
            own[q] = __ldg(a.perm + i);
            if (C::SLOTS || dslots) psv[q] = __ldcg(a.pslot + i);
            if (dslots) ps1v[q] = __ldcg(a.pslot1 + i);
            if (a.root_out) sv[q] = __ldg(a.sid + i);
            if (!leaf) {
#pragma unroll
              for (int k = 0; k < J; k++) ch[q][k] = __ldg(a.chn + (size_t)k * n + i);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < RQ; q++) {  // round 2: roots, words
          const int r = lane + 32 * q, i = i0 + r;
          int root = -1, xr = -1;
          if (r < cnt) {
            if (sv[q] >= 0) root = __ldg(a.roots + sv[q]) == i ? sv[q] : -1;
            if ((leaf && hoist) || proj) {
              xr = i;  // word row
            } else if (C::XSLOT && (leaf || C::DAG)) {
              if (a.xmode == 0) {
                int w = __ldg(a.words + own[q]);
                if (w < 0 || w >= a.V) {
                  if (latch) latch_error(a.hdr, CX_E_WORD_RANGE, own[q]);
                  w = 0;
                }
                xr = w;
              } else {
                xr = i - xlo;
              }
            }
            if (!leaf) {
              int nc = 0;
              bool absent = false;
#pragma unroll
              for (int k = 0; k < J; k++) {
                absent = absent || ch[q][k] < 0;
                if (absent) ch[q][k] = -1;
                nc += ch[q][k] >= 0;
                if (ch[q][k] >= 0) ch[q][k] = hoist ? __ldcg(a.crow + ch[q][k]) : ch[q][k];  // state row
              }
              if (C::FC && nc != 2 && latch) latch_error(a.hdr, CX_E_ARITY, own[q]);
            }
          }
          m.own[r] = own[q];
          m.xr[r] = xr;
          m.root[r] = root;
          m.ps[r] = psv[q];
          m.ps1[r] = ps1v[q];
#pragma unroll
          for (int k = 0; k < J; k++) m.ch[k][r] = ch[q][k];
        }
        if (lane == 0) { m.i0 = i0; m.cnt = cnt; }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_mfull[ms]);
        tc_mark(a, tslot + 1, warp * 32);
      }
      T0m += ntiles;
    }
  } else {
    // tiles / stages / accumulator tiles (tiles with MMAs) before this level,
    // identical in every role
    uint32_t T0 = 0, Sg0 = 0, A0 = 0;
    for (int l = l0; l < L; l++) {
      const bool leaf = l == 0, proj = l < 0;
      if (l > l0) level_sync();
      if (C::BSHARE && l == 1) {  // the leaf phase's MMAs are complete: B1 replaces B0
        load_b(2, kWork);
        fence_proxy_async();
        named_bar(3, kWork);
      }
      if (C::SLOTS && discard_ok && l >= 2) {
        // level l - 1 is complete: its tiles' parent-slot operand rows (rows
        // k n + [lbeg, lbeg + lsize) of pb, loaded by every unit-group CTA) are
        // dead; every CTA drops a share of their 128-byte lines
        const int lb = __ldg(a.lbeg + l - 1), ls = __ldg(a.lsize + l - 1);
        constexpr int LPR = RW * 2 / 128;  // lines per operand row
        const long long total = (long long)J * ls * LPR;
        for (long long e = (long long)blockIdx.x * kWork + tid; e < total; e += (long long)gridDim.x * kWork) {
          const int k = (int)(e / ((long long)ls * LPR)), rem = (int)(e % ((long long)ls * LPR));
          discard_l2(a.pb + ((size_t)k * n + lb + rem / LPR) * RW + (rem % LPR) * 64);
        }
      }
      if (l == 1 && hoist) {  // the word table is complete: fill the leaves' parent slots
        leaf_pass(true);
        level_sync();
      }
      tc_mark(a, l >= 0 ? 2 + 4 * l : -1, 0);
      int lo, hi;
      level_range(l, lo, hi);
      if constexpr (C::FC) {
        if (leaf) {  // h = Emb[word]: this CTA's node chunk x unit slice
          constexpr int q4 = U / 4;
          for (int idx = tid; idx < (hi - lo) * q4; idx += kWork) {
            const int i = lo + idx / q4, c = idx % q4;
            const int own = __ldg(a.perm + i);
            int w = __ldg(a.words + own);
            if (w < 0 || w >= a.V) {
              if (latch && c == 0) latch_error(a.hdr, CX_E_WORD_RANGE, own);
              w = 0;
            }
            const float4 v = __ldg(reinterpret_cast<const float4 *>(a.emb + (size_t)w * H + unit0) + c);
            *reinterpret_cast<float4 *>(a.h_out + (size_t)own * H + unit0 + 4 * c) = v;
            const int ps = __ldcg(a.pslot + i);  // the parent's child-slot row (-1: a root)
            if (ps >= 0) {
              unsigned short *prow = a.pb + (size_t)ps * RW;
              *reinterpret_cast<uint2 *>(prow + unit0 + 4 * c) = make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
              if constexpr (SP == 2) {
                const float4 l4 = make_float4(v.x - bf16_round(v.x), v.y - bf16_round(v.y),
                                              v.z - bf16_round(v.z), v.w - bf16_round(v.w));
                *reinterpret_cast<uint2 *>(prow + H + unit0 + 4 * c) =
                    make_uint2(pack_bf16(l4.x, l4.y), pack_bf16(l4.z, l4.w));
              }
            }
            if (a.root_out) {
              const int r = __ldg(a.sid + i);
              if (__ldg(a.roots + r) == i)
                *reinterpret_cast<float4 *>(a.root_out + (size_t)r * H + unit0 + 4 * c) = v;
            }
          }
          continue;
        }
      }
      const bool fma_l = is_fma(l);
      const int ntiles = fma_l ? 0 : (hi - lo + kTM - 1) / kTM;
      const int nsl = nsl_of(l);
      if (fma_l && warp < kEpiWarps) fma_level(l, lo, hi);

      if ((C::SLOTS || dslots) && warp == kFeed0) {
        // ========================= TMA tile loads ================================
        // per stage: NAB K-atoms (64 bf16 each) of one slot for the tile's 128
        // rows with one tile load: TreeLSTM / TreeFC operands are contiguous
        // (h stored in the parent's child-slot row, x rows word- or
        // node-ordered); rows of absent children / padding rows are not read
        // by the epilogue
        // TPL lanes issue consecutive stages side by side (a thread completes
        // about one TMA load per 0.36 us, tools/micro/tma_rate.cu): stage
        // q = (t * nka + ka / NAB) * nsl + s of this level goes to lane q % TPL
        constexpr int TPL = CX_TC_TMA_LANES < S ? CX_TC_TMA_LANES : S;  // <= S stages at once
        const int nka = KAA / C::NAB, total = ntiles * nka * nsl;
        for (int q0 = 0; q0 < total; q0 += TPL) {
          const int q = q0 + lane;
          if (lane < TPL && q < total) {
            const int s = q % nsl, kq = (q / nsl) % nka, t = q / (nsl * nka);
            const int ka = kq * C::NAB, i0 = lo + t * kTM;
            const uint32_t Sg = Sg0 + (uint32_t)q;
            int src, bm, acc;
            slot_of(l, s, src, bm, acc);
            const int st = Sg % S;
            const int sslot = (l == 1 && q < 16) ? 64 + 4 * q : 1 << 30;
            mbar_wait(&bar_empty[st], ((Sg / S) & 1) ^ 1);
            tc_mark(a, sslot + 0, kFeed0 * 32);
            mbar_arrive_expect_tx(&bar_full[st], C::STB);
            // child slot k: rows k*n + i0 + ..; x: word rows (hoisted) or node-order rows
            const int row0 = src >= 0 ? src * n + i0 : (hoist ? i0 : i0 - xlo);
            const void *tm = src >= 0 ? (const void *)&ta.tm_p : (const void *)&ta.tm_x;
            const uint32_t dst = smem_u32(sStage + (size_t)st * C::STB);
            if (C::NAB > 1)  // atoms ka .. ka + NAB - 1 of the 128 rows, atom after atom
              tma_tile3d(dst, tm, &bar_full[st], 0, row0, ka);
            else if (C::CL == 1 && !CX_TC_TMA_MC)
              tma_tile2d(dst, tm, &bar_full[st], ka * 64, row0);
            else
              tma_tile2d_mc(dst, tm, &bar_full[st], ka * 64, row0, (uint16_t)1);
            if (CX_TC_L2PF > 0 && q + CX_TC_L2PF < total) {  // warm L2 for a later stage
              const int qp = q + CX_TC_L2PF;
              const int sp = qp % nsl, kp = ((qp / nsl) % nka) * C::NAB, tp = qp / (nsl * nka);
              int srcp, bmp, accp;
              slot_of(l, sp, srcp, bmp, accp);
              const int i0p = lo + tp * kTM;
              const int rowp = srcp >= 0 ? srcp * n + i0p : (hoist ? i0p : i0p - xlo);
              const void *tmp = srcp >= 0 ? (const void *)&ta.tm_p : (const void *)&ta.tm_x;
              if (C::NAB > 1) tma_prefetch3d(tmp, 0, rowp, kp);
              else tma_prefetch2d(tmp, kp * 64, rowp);
            }
            tc_mark(a, sslot + 1, kFeed0 * 32);
          }
          __syncwarp();
        }
        tc_mark(a, l >= 0 ? 3 + 4 * l : -1, kFeed0 * 32);
      } else if (!C::SLOTS && !dslots && warp >= kFeed0 && warp < kMeta0) {
        // ========================= cp.async gathers ==============================
        // per stage: one K-atom of one slot for the tile's 128 rows, 16-byte
        // cp.async into the swizzled layout (zero-fill: absent child, unused
        // row); each thread's cp.async.mbarrier.arrive fires when its copies land
        constexpr int FT = 32 * C::FEEDW, kChunks = kTM * 8 / FT;
        const int p = tid - kFeed0 * 32;
        uint32_t Sg = Sg0;
        for (int t = 0; t < ntiles; t++) {
          const uint32_t TT = T0 + t;
          const int ms = TT % kMetaRing;
          mbar_wait(&bar_mfull[ms], (TT / kMetaRing) & 1);
          const TcMeta<J> &m = meta[ms];
          for (int ka = 0; ka < KAA; ka += C::NAB) {
            for (int s = 0; s < nsl; s++) {
              int src, bm, acc;
              slot_of(l, s, src, bm, acc);
              const int st = Sg % S;
              mbar_wait(&bar_empty[st], ((Sg / S) & 1) ^ 1);
              const uint32_t dst0 = smem_u32(sStage + (size_t)st * C::STB);
              const int *rows = src < 0 ? m.xr : m.ch[src];
              const unsigned short *base = src < 0 ? xb : hb;
#pragma unroll
              for (int aj = 0; aj < C::NAB; aj++)  // the stage's K-atoms, atom after atom
#pragma unroll
                for (int e = 0; e < kChunks; e++) {
                  const int q = p + FT * e, r = q >> 3, c = q & 7;
                  const int row = rows[r];
                  const bool valid = row >= 0;
                  cp16_zfill(dst0 + aj * kStageBytes + sw128_off(r, c),
                             base + (size_t)(valid ? row : 0) * RW + (ka + aj) * 64 + c * 8, valid);
                }
              mbar_arrive_cpasync(&bar_full[st]);
              Sg++;
            }
          }
        }
      } else if (warp == kMmaWarp) {
        // =========================== MMA issuer ==================================
        if (lane == 0 && nsl > 0) {  // (no MMAs in a hoisted DAG-RNN leaf level)
          const uint32_t idesc = idesc_bf16(kTM, leaf ? C::NLEAF : C::NLVL);
          const uint32_t idesc2 = idesc_bf16(kTM, (leaf ? C::NLEAF : C::NLVL) * C::MW);  // MERGE hi atoms
          const int ncol = (leaf ? C::NLEAF : C::NLVL) * C::MW;
          uint32_t Sg = Sg0;
          for (int t = 0; t < ntiles; t++) {
            const uint32_t TA = A0 + t, buf = TA & 1;
            mbar_wait(&bar_tempty[buf], ((TA >> 1) & 1) ^ 1);
            fence_after();
            const int tslot = (l >= 0 && l < 2 && t < 5) ? 128 + 12 * (t + 5 * l) : 1 << 30;
            tc_mark(a, tslot + 2, kMmaWarp * 32);
            uint32_t started = 0;
            for (int ka0 = 0; ka0 < KAA; ka0 += C::NAB) {
              for (int s = 0; s < nsl; s++) {
                int src, bm, acc;
                slot_of(l, s, src, bm, acc);
                const int st = Sg % S;
                const int kst = (int)(Sg - Sg0);
                const int sslot = (l == 1 && kst < 16) ? 64 + 4 * kst : 1 << 30;
                mbar_wait(&bar_full[st], (Sg / S) & 1);
                tc_mark(a, sslot + 2, kMmaWarp * 32);
                if (!C::SLOTS) fence_proxy_async();  // landed cp.async data (generic proxy) -> tensor core
                fence_after();
                for (int aj = 0; aj < C::NAB; aj++) {  // the stage's K-atoms
                  const int ka = ka0 + aj;
                  const uint32_t a0 = smem_u32(sStage + (size_t)st * C::STB + (size_t)aj * kStageBytes);
                  const size_t brows = bm ? C::B1 : C::B0;
                  unsigned char *bbase = bm ? sB1 : sB0;
                  // SP = 2: a hi atom (ka < KA) meets B_hi and B_lo, a lo atom B_hi
                  const int kb = ka < KA ? ka : ka - KA;
                  const uint32_t b0 = smem_u32(bbase + (size_t)kb * brows * C::MW * 128);
                  const uint32_t d = tmem + buf * C::BUFC + acc * ncol;
                  const uint32_t idk = (C::MERGE && ka < KA) ? idesc2 : idesc;  // N = 2R: B_hi and B_lo at once
    #pragma unroll
                  for (int kk = 0; kk < 4; kk++) {
                    const uint32_t accum = ((started >> acc) & 1u) | (kk > 0 ? 1u : 0u);
                    mma_bf16(d, sdesc_sw128(a0 + kk * 32), sdesc_sw128(b0 + kk * 32), idk, accum);
                  }
                  if (SP == 2 && !C::MERGE && ka < KA && !CX_TC_SKIP_LO) {
                    const uint32_t b1 = smem_u32(bbase + (size_t)(kb + KA) * brows * 128);
    #pragma unroll
                    for (int kk = 0; kk < 4; kk++)
                      mma_bf16(d, sdesc_sw128(a0 + kk * 32), sdesc_sw128(b1 + kk * 32), idesc, 1u);
                  }
                  started |= 1u << acc;
                }
                if (C::CL == 1 && !CX_TC_TMA_MC) mma_commit(&bar_empty[st]);  // frees the slot
                else mma_commit_mc(&bar_empty[st], (uint16_t)((1u << C::CL) - 1));  // ... cluster-wide
                tc_mark(a, sslot + 3, kMmaWarp * 32);
                Sg++;
              }
            }
            mma_commit(&bar_tfull[buf]);
            tc_mark(a, tslot + 3, kMmaWarp * 32);
          }
          tc_mark(a, l >= 0 ? 4 + 4 * l : -1, kMmaWarp * 32);
        }
        __syncwarp();
      } else if (warp < kEpiWarps) {  // (idle feed warps of a DAG slot run skip all roles)
        // =========================== epilogue ====================================
        // thread = tile row r (TMEM lane) x column half hh: units [u0, u0 + U/2)
        constexpr int UC = U / 2;
        const int q4 = warp & 3, hh = warp >> 2;
        const int r = q4 * 32 + lane, u0 = hh * UC;
        for (int t = 0; t < ntiles; t++) {
          const uint32_t TT = T0 + t, TA = A0 + t, buf = TA & 1;
          const int ms = TT % kMetaRing;
          mbar_wait(&bar_mfull[ms], (TT / kMetaRing) & 1);
          const TcMeta<J> &m = meta[ms];
          const bool valid = r < m.cnt;
          const int i = m.i0 + r, own = m.own[r], root = m.root[r];
          const int tslot = (l >= 0 && l < 2 && t < 5) ? 128 + 12 * (t + 5 * l) : 1 << 30;
          const uint32_t tb = tmem + ((uint32_t)(q4 * 32) << 16) + buf * C::BUFC + u0;
          if constexpr (C::LSTM) {
            static_assert(UC == 16, "TreeLSTM epilogue: 16 units per thread");
            constexpr int NL = C::NLVL;
            float c[16], h[16], v[16], w[16];
            float cp[J][16];  // children's memory cells (prefetched before the MMA wait)
            int ck[J];
  #pragma unroll
            for (int k = 0; k < J; k++) {
              ck[k] = (valid && !leaf) ? m.ch[k][r] : -1;
              if (ck[k] >= 0) {
                // L1-allocating loads: a child's row slice (128 B = one line) is
                // written once, at an earlier level, and read by nobody before,
                // so no SM can hold a stale copy; the line's 4 (x 2 column
                // halves) 16-byte pieces then cost one L2 request instead of 8
                const float *src = cs + (size_t)ck[k] * H + unit0 + u0;
                ld256(src, cp[k]);
                ld256(src + 8, cp[k] + 8);
              }
            }
            mbar_wait(&bar_tfull[buf], (TA >> 1) & 1);
            fence_after();
            tc_mark(a, tslot + 4, 0);
            const float *bi = s_bias + u0, *bo = bi + U, *bu = bi + 2 * U, *bf = bi + 3 * U;
            if (leaf) {
              tmem_ld<16>(tb + 0, v);        // i
              tmem_ld<16>(tb + 2 * U, w);    // u
  #pragma unroll
              for (int j = 0; j < 16; j++) c[j] = act_sig<SP>(v[j] + bi[j]) * act_tanh<SP>(w[j] + bu[j]);
              tmem_ld<16>(tb + U, v);        // o
  #pragma unroll
              for (int j = 0; j < 16; j++) h[j] = act_sig<SP>(v[j] + bo[j]) * act_tanh<SP>(c[j]);
            } else {
  #pragma unroll
              for (int j = 0; j < 16; j++) c[j] = 0.f;
  #pragma unroll
              for (int k = 0; k < J; k++) {  // sum_k f_k * c_k
                tmem_ld<16>(tb + k * NL + 3 * U, v);
                if (ck[k] >= 0) {
  #pragma unroll
                  for (int j = 0; j < 16; j++) c[j] = fmaf(act_sig<SP>(v[j] + bf[j]), cp[k][j], c[j]);
                }
              }
              tmem_ld<16>(tb + 0, v);        // i = sum_k acc_k[i], u = sum_k acc_k[u]
              tmem_ld<16>(tb + 2 * U, w);
  #pragma unroll
              for (int k = 1; k < J; k++) {  // absent children's accumulators are not read
                tmem_ld<16>(tb + k * NL + 0, h);
                if (ck[k] >= 0) {
  #pragma unroll
                  for (int j = 0; j < 16; j++) v[j] += h[j];
                }
                tmem_ld<16>(tb + k * NL + 2 * U, h);
                if (ck[k] >= 0) {
  #pragma unroll
                  for (int j = 0; j < 16; j++) w[j] += h[j];
                }
              }
  #pragma unroll
              for (int j = 0; j < 16; j++) c[j] = fmaf(act_sig<SP>(v[j] + bi[j]), act_tanh<SP>(w[j] + bu[j]), c[j]);
              tmem_ld<16>(tb + U, v);        // o
  #pragma unroll
              for (int k = 1; k < J; k++) {
                tmem_ld<16>(tb + k * NL + U, h);
                if (ck[k] >= 0) {
  #pragma unroll
                  for (int j = 0; j < 16; j++) v[j] += h[j];
                }
              }
  #pragma unroll
              for (int j = 0; j < 16; j++) h[j] = act_sig<SP>(v[j] + bo[j]) * act_tanh<SP>(c[j]);
            }
            if (valid) {
              const bool wordrow = leaf && hoist;  // hoisted leaf cell: row i = word i
              const size_t rowi = (size_t)(wordrow ? i : sbase + i);
              const size_t ui = rowi * H + unit0 + u0;
              if (wordrow) st_op<SP, H, 16>(hb + rowi * RW, unit0 + u0, h);  // the word table (copied to slots below)
              else if (m.ps[r] >= 0) st_op<SP, H, 16>(a.pb + (size_t)m.ps[r] * RW, unit0 + u0, h);
              st_row<16>(cs + ui, c);
              if (wordrow) {
                st_row<16>(a.hf + (size_t)i * H + unit0 + u0, h);
              } else {
                const size_t uo = (size_t)own * H + unit0 + u0;
                st_row_cs<16>(a.h_out + uo, h);
                if (a.aux_out) st_row_cs<16>(a.aux_out + uo, c);
                if (root >= 0) st_row_cs<16>(a.root_out + (size_t)root * H + unit0 + u0, h);
              }
            }
          } else {  // DAG-RNN / TreeFC: h = tanh(acc + b)
            constexpr int CW = UC < 32 ? UC : 32;
            // hoisted DAG-RNN: this row's word projection (bias included),
            // first chunk loaded before the accumulator wait
            const int xrow = (hx && !proj && valid) ? m.xr[r] : -1;
            float pv[CW];
            if (xrow >= 0) {
              const float *pr = a.hf + (size_t)xrow * H + unit0 + u0;
  #pragma unroll
              for (int j = 0; j < CW; j += 8) ld256(pr + j, pv + j);
            }
            if (nsl > 0) {
              mbar_wait(&bar_tfull[buf], (TA >> 1) & 1);
              fence_after();
            }
            tc_mark(a, tslot + 4, 0);
  #pragma unroll 1
            for (int q = 0; q < UC / CW; q++) {
              float v[CW];
              if (nsl > 0) {
                tmem_ld<CW>(tb + q * CW, v);
                if constexpr (C::MERGE) {  // + the A_hi B_lo columns
                  float v2[CW];
                  tmem_ld<CW>(tb + U + q * CW, v2);
  #pragma unroll
                  for (int j = 0; j < CW; j++) v[j] += v2[j];
                }
              } else {
  #pragma unroll
                for (int j = 0; j < CW; j++) v[j] = 0.f;
              }
              if (proj) {  // W_x x + b of word i -> the table (no outputs)
                if (valid) {
  #pragma unroll
                  for (int j = 0; j < CW; j++) v[j] += s_bias[u0 + q * CW + j];
                  st_row<CW>(a.hf + (size_t)i * H + unit0 + u0 + q * CW, v);
                }
                continue;
              }
              if (hx) {
                if (q > 0 && xrow >= 0) {
  #pragma unroll
                  for (int j = 0; j < CW; j += 8) ld256(a.hf + (size_t)xrow * H + unit0 + u0 + q * CW + j, pv + j);
                }
  #pragma unroll
                for (int j = 0; j < CW; j++) v[j] = act_tanh<SP>(v[j] + pv[j]);
              } else {
  #pragma unroll
                for (int j = 0; j < CW; j++) v[j] = act_tanh<SP>(v[j] + s_bias[u0 + q * CW + j]);
              }
              if (valid) {
                const int uu = unit0 + u0 + q * CW;
                st_row_cs<CW>(a.h_out + (size_t)own * H + uu, v);
                if (C::SLOTS || dslots) {  // TreeFC / DAG slots: the parents' child-slot rows
                  if (m.ps[r] >= 0) st_op<SP, H, CW>(a.pb + (size_t)m.ps[r] * RW, uu, v);
                  if (dslots && m.ps1[r] >= 0) st_op<SP, H, CW>(a.pb + (size_t)m.ps1[r] * RW, uu, v);
                } else {
                  st_op<SP, H, CW>(hb + (size_t)i * RW, uu, v);
                }
                if (root >= 0) st_row_cs<CW>(a.root_out + (size_t)root * H + uu, v);
              }
            }
          }
          fence_before();
          if (nsl > 0) mbar_arrive(&bar_tempty[buf]);
          mbar_arrive(&bar_mempty[ms]);
          tc_mark(a, tslot + 5, 0);
        }
        tc_mark(a, l >= 0 ? 5 + 4 * l : -1, 0);
      }
      T0 += ntiles;
      Sg0 += (uint32_t)ntiles * (KAA / C::NAB) * nsl;
      if (nsl > 0) A0 += ntiles;
    }

    if (hoist && L > 0) {  // leaves' caller outputs (the table is complete since level 1)
      if (L == 1) level_sync();  // single level: no barrier yet
      tc_mark(a, 62, 0);
      leaf_pass(false);
      tc_mark(a, 63, 0);
    }

  }


  // ---- hoisted leaves: outputs copied from the word table -------------------
  // (the table was complete at the level-1 barrier; every CTA copies a share)
  // ---- teardown -------------------------------------------------------------
  fence_before();
  __syncthreads();
  cluster_sync_all();  // no peer still signals this CTA's barriers
  if (warp == kMmaWarp) {
    fence_after();
    tmem_free<C::TCOLS>(tmem);
  }
  publish_and_exit(a);
}

template <int CELL, int H, int MAXC, int SP>
bool tc_plan_one(int num_sms, FwdPlan *p, int *Gn, int *Gu) {
  using C = TcCfg<CELL, H, MAXC, SP>;
  static_assert(C::S >= 2, "at least two pipeline stages");
  auto k = tc_kernel<CELL, H, MAXC, SP>;
  // per-device caches (attributes and occupancy are per device context)
  static bool set[kMaxDevices];
  static int max_clusters_dev[kMaxDevices];
  const int dev = device_slot();
  if (dev < 0) return false;
  if (!set[dev]) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::dyn_bytes) !=
        cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    set[dev] = true;
    max_clusters_dev[dev] = -1;
  }
  int &max_clusters = max_clusters_dev[dev];  // co-resident clusters (the grid barrier needs all)
  if (max_clusters < 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C::CL * 64);
    cfg.blockDim = dim3(C::THREADS);
    cfg.dynamicSmemBytes = C::dyn_bytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C::CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, (const void *)k, &cfg) != cudaSuccess) {
      cudaGetLastError();
      nc = 0;
    }
    max_clusters = nc;
  }
  *Gu = C::GU;
  *Gn = min(num_sms / C::GU, max_clusters * C::CL / C::GU);
  if (*Gn < 1) return false;
  p->ctas = *Gn * *Gu;
  p->threads = C::THREADS;
  p->smem = C::dyn_bytes;
  p->kernel = (const void *)k;
  p->cluster = C::CL;
  p->family = SP == 2 ? 8 : 6;
  p->big = false;
  p->tc = true;
  p->tc_sp = SP;
  p->tc_nab = C::NAB;
  return true;
}

template <int CELL, int H, int SP>
bool tc_plan_c(int maxc, int num_sms, FwdPlan *p, int *Gn, int *Gu) {
  if constexpr (CELL == CX_TREEFC) {
    return maxc == 2 && tc_plan_one<CELL, H, 2, SP>(num_sms, p, Gn, Gu);
  } else {
    if (maxc == 1) return tc_plan_one<CELL, H, 1, SP>(num_sms, p, Gn, Gu);
    if (maxc == 2) return tc_plan_one<CELL, H, 2, SP>(num_sms, p, Gn, Gu);
    return false;
  }
}
template <int SP>
bool tc_plan_sp(int cell, int H, int maxc, int num_sms, FwdPlan *p, int *Gn, int *Gu) {
  switch (cell) {
    case CX_TREELSTM:
      if (H == 256) return tc_plan_c<CX_TREELSTM, 256, SP>(maxc, num_sms, p, Gn, Gu);
      if (H == 128) return tc_plan_c<CX_TREELSTM, 128, SP>(maxc, num_sms, p, Gn, Gu);
      return false;
    case CX_DAGRNN:
      if (H == 256) return tc_plan_c<CX_DAGRNN, 256, SP>(maxc, num_sms, p, Gn, Gu);
      if (H == 128) return tc_plan_c<CX_DAGRNN, 128, SP>(maxc, num_sms, p, Gn, Gu);
      return false;
    case CX_TREEFC:
      if (H == 512) return tc_plan_c<CX_TREEFC, 512, SP>(maxc, num_sms, p, Gn, Gu);
      if (H == 256) return tc_plan_c<CX_TREEFC, 256, SP>(maxc, num_sms, p, Gn, Gu);
      return false;
  }
  return false;
}

}  // namespace

// Tensor-core path: TreeLSTM / DAG-RNN H in {128, 256}, TreeFC H in {256, 512};
// max_children <= 2 (TMEM holds two accumulator buffers of max_children x 4U
// columns). sp = 1: bf16 operands; sp = 2: split fp32 operands (TcCfg).
bool tc_plan(int cell, int H, int maxc, int sp, int num_sms, FwdPlan *p, int *Gn, int *Gu) {
  return sp == 2 ? tc_plan_sp<2>(cell, H, maxc, num_sms, p, Gn, Gu)
                 : tc_plan_sp<1>(cell, H, maxc, num_sms, p, Gn, Gu);
}

// ---- launch: tensor maps of the gathered operands + cooperative launch --------
namespace {
using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                   const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                   const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static std::once_flag once;
  static EncodeTiledFn fn = nullptr;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
    cudaGetLastError();
  });
  return fn;
}

// [rows][H] bf16 row-major, box = 64 columns x box_rows rows, 128-byte swizzle
bool encode_rows(TmaDesc *d, const void *base, int H, long long rows, int box_rows = 1) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || rows < 1) return false;
  cuuint64_t dims[2] = {(cuuint64_t)H, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)H * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows}, es[2] = {1, 1};
  return fn(reinterpret_cast<CUtensorMap *>(d), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
            const_cast<void *>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// the same rows as a 3D tensor {64 columns, rows, K-atoms} (strides: row =
// H * 2 bytes, atom = 128 bytes), box {64, box_rows, nab}: nab K-atoms of
// box_rows rows per load, landing atom after atom (each a K-major SW128 block)
bool encode_rows3(TmaDesc *d, const void *base, int H, long long rows, int box_rows, int nab) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || rows < 1 || H % 64) return false;
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(H / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)H * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)nab}, es[3] = {1, 1, 1};
  return fn(reinterpret_cast<CUtensorMap *>(d), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
            const_cast<void *>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

cudaError_t tc_launch(const FwdPlan &plan, const FwdArgs &f, cudaStream_t stream) {
  static_assert(sizeof(TmaDesc) == sizeof(CUtensorMap), "tensor map size");
  TcArgs ta;
  std::memset(&ta, 0, sizeof ta);
  ta.f = f;
  const long long xrows = f.xmode ? f.n : f.V;
  if (f.pb) {  // TreeLSTM: contiguous operands, 128-row tile loads of rows of sp x H bf16
    const int rw = plan.tc_sp * f.H;
    if (plan.tc_nab > 1) {  // NAB K-atoms per load (3D box)
      if (!encode_rows3(&ta.tm_p, f.pb, rw, 2LL * f.n, kTM, plan.tc_nab)) return cudaErrorInvalidValue;
      if (f.xb && !encode_rows3(&ta.tm_x, f.xb, rw, xrows, kTM, plan.tc_nab)) return cudaErrorInvalidValue;
    } else {
      if (!encode_rows(&ta.tm_p, f.pb, rw, 2LL * f.n, kTM)) return cudaErrorInvalidValue;
      if (f.xb && !encode_rows(&ta.tm_x, f.xb, rw, xrows, kTM)) return cudaErrorInvalidValue;
    }
  }
  void *params[] = {&ta};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(plan.ctas);
  cfg.blockDim = dim3(plan.threads);
  cfg.dynamicSmemBytes = plan.smem;
  cfg.stream = stream;
  // thread-block clusters (no cooperative attribute: the grid was sized from
  // cudaOccupancyMaxActiveClusters so every CTA is co-resident)
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = plan.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap cx_linearize
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelExC(&cfg, plan.kernel, params);
}

// x rows in node order when the batch has at most V/2 of them, else the table
int tc_xmode(int n, int V) { return (size_t)n * 2 <= (size_t)V ? 1 : 0; }

// workspace bytes of the tensor-core path (after the GridBar): hb, cs, xb
// Computation hoisting of the TreeLSTM leaf cell (PAPER §4.3 P:1127-1132,
// SURVEY §8(f) f1): a leaf's (h, c) depends only on its word, so when the batch
// has more leaves' worth of x rows than V/2 (table mode) the leaf level is
// evaluated once per vocabulary word and parents read leaf children from that
// table.
// DAG-RNN (split fp32 operands only: on bf16 operands the extra phase and the
// epilogue's table loads cost more than the removed x slot, measured): the
// input projection W_x x + b once per word (a [V][H] fp32 table) in the same
// condition. CX_TC_HOIST=0 disables both (measurement).
bool tc_hoist(int cell, int n, int V, int sp) {
  const char *e = std::getenv("CX_TC_HOIST");
  if (e && e[0] == '0') return false;
  return (cell == CX_TREELSTM || (cell == CX_DAGRNN && sp == 2)) && tc_xmode(n, V) == 0;
}

// State rows: hoisted TreeLSTM keeps the V word rows first, node i at row V + i.
size_t tc_state_rows(int cell, int n, int V) {
  return (size_t)(n > 0 ? n : 1) + (cell == CX_TREELSTM && tc_hoist(cell, n, V, 1) ? (size_t)V : 0);
}

// workspace bytes of the tensor-core path (after the GridBar); forward_impl in
// api.cu lays the buffers out in this order. Operand rows (hb, xb, pb) hold
// sp x H bf16 (sp = 2: the split fp32 path).
size_t tc_workspace_bytes(int cell, int H, int V, int n, int sp) {
  const size_t N = (size_t)(n > 0 ? n : 1), h = (size_t)H, R = tc_state_rows(cell, n, V);
  const size_t rw = h * (sp == 2 ? 2 : 1);                     // bf16 per operand row
  size_t b = 2 * R * rw + 256;                                  // hb
  if (cell == CX_TREELSTM) b += 4 * R * h + 256;                // cs
  if (cell == CX_TREELSTM || cell == CX_DAGRNN)                 // xb
    b += 2 * (tc_xmode(n, V) ? N : (size_t)V) * rw + 256;
  if (tc_hoist(cell, n, V, sp)) b += 4 * (size_t)V * h + 4 * N + 512;  // hf, crow
  if (cell == CX_TREELSTM || cell == CX_TREEFC || (cell == CX_DAGRNN && sp == 2))
    b += 2 * (2 * N) * rw + 4 * N + 512;                                     // pb (J <= 2), pslot
  if (cell == CX_DAGRNN && sp == 2) b += 8 * N + 512;                           // pslot1, pcnt
  return b;
}

}  // namespace cx
