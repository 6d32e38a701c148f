// lin_warp.cuh -- the linearizer for tiny forests, n <= 32
// nodes and max_children <= 4, run by ONE warp: lane v owns node v, every
// cross-node step is a shuffle or a ballot, and there is no block barrier and
// no shared-memory atomic until the results are stored. The single-CTA
// linearizer's phases are bounded by instruction fetch and block barriers
// (~1,000-3,700 cycles each whatever n is); this path replaces
// them for the tiny latency configs (cfg1: 15 nodes).
//
// Same definitions and outputs as lin_single.cuh (§4.2 P:1060-1085,
// App. B, readings Q4-Q7): heights by Jacobi rounds (round r
// finalises exactly the nodes of height r, for trees and DAGs alike: a node's
// height is undefined iff it is on or above a cycle, the lowest such id is the
// CX_E_CYCLE node), new id = #{higher level} + #{same level, smaller input id},
// roots in ascending input id, structure = the smallest root index reaching
// the node (trees: their root, found by pointer jumping). Errors: the lowest
// (code, input id) key, a1 before a2.
#pragma once
#include <cuda_runtime.h>

#include <climits>

#include "lin_single.cuh"

namespace cx {

constexpr int kLinWarpMaxN = 32, kLinWarpMaxC = 4;

__host__ __device__ inline bool lin_warp_applies(int n, int maxc) {
  return n >= 1 && n <= kLinWarpMaxN && maxc <= kLinWarpMaxC;
}

// Run by the whole CTA (only warp 0 works; the others wait at the final
// barrier). Fills the LinSm arrays of `sm` (the layout of lin_single_body)
// and, when write_global, the cx_linearization outputs and header of `a`;
// chn_s (optional): remapped children [maxc][n] in shared memory.
__device__ __forceinline__ LinOut lin_warp_body(const LinArgs &a, int *sm, bool write_global,
                                                int *chn_s) {
  __shared__ LinOut s_out;
  const int n = a.n, maxc = a.maxc, lane = threadIdx.x & 31;
  const LinSm s = lin_carve(sm, n, maxc);
  if (threadIdx.x < 32) {
    const unsigned FULL = 0xffffffffu;
    const bool in = lane < n;
    const unsigned below = (1u << lane) - 1u;
    const bool tree_like = a.kind != CX_DAG;
    int c[kLinWarpMaxC];
#pragma unroll
    for (int k = 0; k < kLinWarpMaxC; k++) c[k] = (in && k < maxc) ? __ldg(a.ch + (size_t)k * n + lane) : -1;
    // ---- a1: layout, range, duplicate child; in-degree and parent by shuffles
    unsigned long long key = kNoError;
    auto latch = [&](int code) {
      const unsigned long long kk = ((unsigned long long)(unsigned)code << 32) | (unsigned)lane;
      if (kk < key) key = kk;
    };
    int nc = 0;
    bool absent = false;
#pragma unroll
    for (int k = 0; k < kLinWarpMaxC; k++) {
      if (!in || k >= maxc) continue;
      if (c[k] == -1) {
        absent = true;
        continue;
      }
      nc++;
      if (absent) latch(CX_E_CHILD_LAYOUT);
      if (c[k] < 0 || c[k] >= n) {
        latch(CX_E_CHILD_RANGE);
        c[k] = -2;  // not an edge (the in-degree and remap skip it)
        continue;
      }
#pragma unroll
      for (int k2 = 0; k2 < kLinWarpMaxC; k2++)
        if (k2 < k && c[k2] == c[k]) latch(CX_E_KIND);
    }
    int indeg = 0, parent = -1;
    for (int u = 0; u < n; u++) {
#pragma unroll
      for (int k = 0; k < kLinWarpMaxC; k++) {
        const int cu = __shfl_sync(FULL, c[k], u);
        if (cu == lane) {
          indeg++;
          parent = u;
        }
      }
    }
    if (in && tree_like && indeg > 1) latch(CX_E_KIND);
    for (int o = 16; o; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(FULL, key, o);
      key = other < key ? other : key;
    }
    bool ok = key == kNoError;
    // ---- a2: heights, Jacobi rounds over shuffled child heights --------------
    int h = (in && nc == 0) ? 0 : -1;
    int L = 0;
    if (ok) {
      for (int r = 1; r <= n; r++) {
        bool ready = in && h < 0;
#pragma unroll
        for (int k = 0; k < kLinWarpMaxC; k++) {
          const int hk = __shfl_sync(FULL, h, c[k] >= 0 ? c[k] : 0);
          if (c[k] >= 0 && (hk < 0 || hk >= r)) ready = false;
        }
        if (ready) h = r;
        if (!__any_sync(FULL, ready)) break;
      }
      const unsigned undef = __ballot_sync(FULL, in && h < 0);
      if (undef) {
        key = ((unsigned long long)CX_E_CYCLE << 32) | (unsigned)(__ffs(undef) - 1);
        ok = false;
      }
      int hm = in ? h : 0;
      for (int o = 16; o; o >>= 1) hm = max(hm, __shfl_xor_sync(FULL, hm, o));
      L = hm + 1;
    }
    LinOut out;
    out.ok = ok;
    out.L = ok ? L : 0;
    out.num_roots = 0;
    out.first_leaf = 0;
    if (ok) {
      // ---- a3/a4: level sizes and the stable numbering ----------------------
      int nid = 0;
      for (int u = 0; u < n; u++) {
        const int hu = __shfl_sync(FULL, h, u);
        nid += (hu > h) || (hu == h && u < lane);
      }
      int lsz = 0, lbg = 0, mx = 0;  // lane l < L: level l
      for (int l = 0; l < L; l++) {
        const int cnt = __popc(__ballot_sync(FULL, in && h == l));
        const int higher = __popc(__ballot_sync(FULL, in && h > l));
        if (lane == l) {
          lsz = cnt;
          lbg = higher;
        }
        mx = max(mx, cnt);
      }
      const unsigned rootm = __ballot_sync(FULL, in && indeg == 0);
      const int ridx = __popc(rootm & below);
      out.num_roots = __popc(rootm);
      out.first_leaf = n - __shfl_sync(FULL, lsz, 0);
      // ---- a5: remapped children; a6: structures ----------------------------
      int cn[kLinWarpMaxC];
#pragma unroll
      for (int k = 0; k < kLinWarpMaxC; k++) {
        const int m = __shfl_sync(FULL, nid, c[k] >= 0 ? c[k] : 0);
        cn[k] = c[k] >= 0 ? m : -1;
      }
      int sid;
      if (tree_like) {  // the root by pointer jumping
        int r = parent >= 0 ? parent : lane;
        for (int it = 0; it < 5; it++) r = __shfl_sync(FULL, r, r);
        sid = __shfl_sync(FULL, ridx, r);
      } else {  // smallest root index reaching the node: min over the parents, to a fixed point
        sid = (in && indeg == 0) ? ridx : INT_MAX;
        for (int it = 0; it < n; it++) {
          int m = sid;
          for (int u = 0; u < n; u++) {
            const int su = __shfl_sync(FULL, sid, u);
#pragma unroll
            for (int k = 0; k < kLinWarpMaxC; k++)
              if (__shfl_sync(FULL, c[k], u) == lane) m = min(m, su);
          }
          const bool changed = m != sid;
          sid = m;
          if (!__any_sync(FULL, changed)) break;
        }
      }
      // ---- stores: shared-memory arrays (for the fused kernels) + outputs ----
      if (in) {
        s.perm[nid] = lane;
        s.inv[lane] = nid;
        s.hgt[lane] = h;
        s.indeg[lane] = indeg;
        s.par[lane] = tree_like ? parent : -1;
        s.sid[nid] = sid;
#pragma unroll
        for (int k = 0; k < kLinWarpMaxC; k++)
          if (k < maxc) {
            s.ch[(size_t)k * n + lane] = c[k] >= 0 ? c[k] : -1;
            if (chn_s) chn_s[(size_t)k * n + nid] = cn[k];
          }
      }
      if (lane < L) {
        s.lb[lane] = lbg;
        s.ls[lane] = lsz;
      }
      if (write_global) {
        if (in) {
          a.perm[nid] = lane;
          a.inv[lane] = nid;
          a.hnew[nid] = h;
          a.sid[nid] = sid;
#pragma unroll
          for (int k = 0; k < kLinWarpMaxC; k++)
            if (k < maxc) a.chn[(size_t)k * n + nid] = cn[k];
          if (indeg == 0) a.roots[ridx] = nid;
        }
        if (lane < L) {
          a.lbeg[lane] = lbg;
          a.lsize[lane] = lsz;
        }
      }
      if (write_global && lane == 0) {
        cx_lin_header *hd = a.hdr;
        hd->err_key = kNoError;
        hd->num_nodes = n;
        hd->status = CX_OK;
        hd->bad_node = -1;
        hd->num_levels = L;
        hd->num_roots = out.num_roots;
        hd->num_leaves = n - out.first_leaf;
        hd->first_leaf = out.first_leaf;
        hd->max_level_size = mx;
      }
    } else if (write_global && lane == 0) {
      cx_lin_header *hd = a.hdr;
      hd->err_key = key;
      hd->num_nodes = n;
      hd->status = (int)(key >> 32);
      hd->bad_node = (int)(key & 0xffffffffu);
      hd->num_levels = 0;
    }
    if (lane == 0) s_out = out;
  }
  __syncthreads();
  return s_out;
}

}  // namespace cx
