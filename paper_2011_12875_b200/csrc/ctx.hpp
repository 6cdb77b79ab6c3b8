// ctx.hpp -- the engine context, shared by the host translation unit
// (snapgpu.cu: C-ABI, planning, graph) and the per-twojmax kernel units
// (launch_t.cu compiled once per 2J, so the build runs in parallel).
// Internal header: not part of the C-ABI (include/snapgpu.h).
//
// A context mirrors the reference's DescriptorState (snap_core.hpp:130-172):
// it owns every per-atom array, here in HBM, plus the host-built tables
// (tables.cpp).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/snapgpu.h"
#include "kernels.cuh"
#include "tables.hpp"

namespace snapgpu {
namespace host {

struct CudaError {
  std::string msg;
};

#define CK(expr)                                                                        \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      throw ::snapgpu::host::CudaError{std::string(#expr) + ": " + cudaGetErrorString(_e)}; \
  } while (0)

struct InvalidArg {
  std::string msg;
};
struct StateErr {
  std::string msg;
};

inline void require(bool ok, const char* m) {
  if (!ok) throw InvalidArg{m};
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  bool own = true;  // false: a view into another buffer
  void alloc(size_t count) {
    if (count <= n && p && own) return;
    release();
    if (count == 0) return;
    CK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void view(T* ptr, size_t count) {
    release();
    p = ptr;
    n = count;
    own = false;
  }
  void release() {
    if (p && own) cudaFree(p);
    p = nullptr;
    n = 0;
    own = true;
  }
};

}  // namespace host
}  // namespace snapgpu

struct snapgpu_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  std::string err;

  // parameters (SnapParams, snap_core.hpp:48-57)
  int T = 0;
  snapgpu::GeoParams gp{};
  std::vector<double> beta, weights;
  snapgpu::IndexMaps maps;
  std::vector<double> cg, hf, ywgt;

  // device tables
  snapgpu::host::DevBuf<double> d_weights, d_cw;
  snapgpu::host::DevBuf<double> d_cwp;    // padded windowed C' of k_compute_Y_cwin
  snapgpu::host::DevBuf<uint4> d_yunits;  // its unit records (YUnit: 2 x uint4, W included)
  std::vector<uint4> yunit_rec;           // beta-independent half of the records
  snapgpu::host::DevBuf<int> d_tasks, d_expand;
  snapgpu::YPlan yplan;
  snapgpu::YCoopPlan ycplan;     // constant-window units, LPT-split over 4 warps per row
  snapgpu::YQuadPlan yqplan;     // quad units (2J > 8)
  snapgpu::host::DevBuf<int4> d_qunits;
  snapgpu::host::DevBuf<double> d_qitw;
  snapgpu::host::DevBuf<double> d_cwq;  // the quad kernel's padded windowed C' (yquad_cw)
  snapgpu::host::DevBuf<int> d_qrw, d_qrows;
  int y_parts = 0;        // compute_Y CTAs per 32-atom tile forced by snapgpu_tune (0 = automatic)
  int y_parts_max = 1;    // the most parts any tile has in the current plan
  int y_ctas = 0;         // compute_Y grid (2J <= 8): one CTA per (tile, part)
  snapgpu::host::DevBuf<int4> d_ycta;    // per CTA {tile, part | parts << 8, row list, stride}
  snapgpu::host::DevBuf<unsigned> d_ready;  // [ntiles] tile flags (Y -> dE hand-off)
  // compute_fused_dE starts per tile while compute_Y still runs (2J <= 8).
  // Off when a tool is injected (ncu: CUDA_INJECTION64_PATH, compute-
  // sanitizer: NV_SANITIZER_INJECTION_*): tools may serialize the grids, and
  // a dE CTA waiting for a tile would then wait for a CTA that cannot run.
  bool y_overlap = true;
  // the hand-off in use: on, and a single force chunk (the chunked multi-GPU
  // layout copies compute_Y's etotal in the gather, after the grid-wide wait)
  bool overlap_now() const { return y_overlap && nchunks == 1; }

  // problem shape
  int natoms_total = 0, atom_lo = 0, nlocal = 0, stride = 0, ntiles = 0;
  bool have_lists = false, have_U = false, have_Y = false, have_dE = false, have_forces = false;

  // device arrays
  snapgpu::host::DevBuf<int> d_numneigh, d_nbr, d_types;
  snapgpu::host::DevBuf<double> d_disp, d_V, d_Y, d_dedr, d_forces, d_eatom, d_etotal;
  snapgpu::host::DevBuf<double> d_virial;  // virial partial sums + result
  snapgpu::host::DevBuf<double> d_out;     // [forces | eatom | etotal]: one D2H per step
  snapgpu::host::DevBuf<double> d_nlpos;   // device neighbor-list build: positions, wrapped
  snapgpu::host::DevBuf<int> d_nlint;      // cell_of | members | counts | head | fill | max
  snapgpu::host::DevBuf<unsigned> d_err;   // device validation flags (kErr*)
  unsigned* h_err = nullptr;               // pinned readback of d_err
  double* h_out = nullptr;                 // pinned staging of d_out (one-call API)
  size_t h_out_n = 0;

  // direct bispectrum components (kernels.cuh k_compute_B), built on first use
  snapgpu::host::DevBuf<int4> d_bitems;
  snapgpu::host::DevBuf<int> d_bcwoff, d_btbeg;
  snapgpu::host::DevBuf<double> d_bwgt, d_blist;

  // deterministic energy epilogue (kernels.cuh energy_epilogue)
  snapgpu::host::DevBuf<double> d_epart, d_tile_sum;
  snapgpu::host::DevBuf<unsigned> d_tickets;  // [0]: global ticket, [1..]: per tile

  // deterministic force gather (kernels.cuh k_gather_forces): reverse
  // neighbor index, rebuilt when the lists change
  snapgpu::host::DevBuf<int> d_rev_off, d_rev_cur, d_rev;
  bool csr_dirty = true;
  bool sym_lists = false;  // lists built on the device: symmetric, partner slots in d_rev
  // force output layout: nchunks chunks of chunk_rows atoms (+ energy slot
  // when nchunks > 1), into the caller's device buffer when ext_forces is set
  int nchunks = 1;
  double* ext_forces = nullptr;
  // one-call step from pinned host lists: mapped host sources compute_U pulls
  // the lists from (UArgs::src_*); set only for the duration of that launch
  const int* zc_numneigh = nullptr;
  const int* zc_nbr = nullptr;
  const double* zc_disp = nullptr;
  // ... and its mapped host outputs, written by the kernels beside the
  // device copies (EnergyOut / GatherArgs second sinks); null otherwise
  double* sink_forces = nullptr;
  double* sink_eatom = nullptr;
  double* sink_etotal = nullptr;
  unsigned* sink_flags = nullptr;
  int chunk_rows() const {
    return nchunks > 1 ? (natoms_total + nchunks - 1) / nchunks : (natoms_total > 0 ? natoms_total : 1);
  }
  int chunk_stride() const { return nchunks > 1 ? 3 * chunk_rows() + 1 : 3 * chunk_rows(); }

  // the one-call pull step (pinned lists and outputs) as a graph; the host
  // pointers of each call are patched into its U / Y / gather nodes
  cudaGraph_t pull_graph = nullptr;
  cudaGraphExec_t pull_gexec = nullptr;
  cudaGraphNode_t pull_node[3] = {nullptr, nullptr, nullptr};  // U, Y, gather
  cudaKernelNodeParams pull_kp[3] = {};
  snapgpu::UArgs pull_u{};
  snapgpu::YWArgs pull_y{};
  alignas(16) unsigned char pull_g[256];  // the GatherArgs (host translation unit only)
  // the one-call positions step with pinned positions and outputs: the
  // binning kernel reads the positions from host memory, the kernels write
  // the results into the outputs; per-call pointers patched into its
  // binning / Y / gather nodes
  cudaGraph_t ppos_graph = nullptr;
  cudaGraphExec_t ppos_gexec = nullptr;
  cudaGraphNode_t ppos_node[3] = {nullptr, nullptr, nullptr};  // bin, Y, gather
  cudaKernelNodeParams ppos_kp[3] = {};
  alignas(16) unsigned char ppos_nl[256];  // the NLArgs (host translation unit only)
  snapgpu::YWArgs ppos_y{};
  alignas(16) unsigned char ppos_g[256];
  // graphs: the force step, and the reverse-index build
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  bool graph_valid = false;
  cudaGraph_t csr_graph = nullptr;
  cudaGraphExec_t csr_gexec = nullptr;
  // the force step after a list upload: the reverse-index build forked onto
  // side_stream, joined only before the force gather (its one consumer)
  cudaGraph_t fork_graph = nullptr;
  cudaGraphExec_t fork_gexec = nullptr;
  cudaStream_t side_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // one-call positions step (snapgpu_run_positions): pinned staging + graph
  cudaGraph_t pos_graph = nullptr;
  cudaGraphExec_t pos_gexec = nullptr;
  double* h_pos = nullptr;
  size_t h_pos_n = 0;
  double nl_box[3] = {0, 0, 0};

  // timing
  bool timing = false;
  cudaEvent_t ev[5] = {};
  float stage_ms[4] = {0, 0, 0, 0};
};

namespace snapgpu {
namespace host {

// Launch with programmatic stream serialization (PDL): the kernel may start
// while the previous kernel in the stream drains; it calls pdl_wait() before
// reading that kernel's outputs (kernels.cuh).
template <class... KArgs, class... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

inline PairArgs pair_args(const snapgpu_ctx* c) {
  PairArgs p;
  p.nlocal = c->nlocal;
  p.stride = c->stride;
  p.atom_lo = c->atom_lo;
  p.numneigh = c->d_numneigh.p;
  p.nbr = c->d_nbr.p;
  p.disp = c->d_disp.p;
  p.types = c->d_types.p;
  p.weights = c->d_weights.p;
  p.natoms_total = c->natoms_total;
  p.nweights = static_cast<int>(c->weights.size());
  p.rc2 = c->gp.rcut * c->gp.rcut;
  p.err = c->d_err.p;
  return p;
}

inline EnergyOut energy_out(snapgpu_ctx* c) {
  EnergyOut E;
  E.eatom = c->d_eatom.p;
  E.epart = c->d_epart.p;
  E.tile_sum = c->d_tile_sum.p;
  E.ticket = c->d_tickets.p;
  E.tile_ticket = c->d_tickets.p + 1;
  E.etotal = c->d_etotal.p;
  E.eatom_host = c->sink_eatom;
  E.etotal_host = c->sink_etotal;
  E.pstride = c->y_parts_max;
  E.ready = nullptr;  // set by the 2J <= 8 compute_Y launch
  return E;
}

// Per-2J launchers, explicitly instantiated in launch_t.cu (one object file
// per 2J).  upload_ytables_t fills that object's own constant bank.
template <int T> void launch_U_t(snapgpu_ctx* c);
template <int T> void launch_Y_t(snapgpu_ctx* c);
template <int T> void launch_DE_t(snapgpu_ctx* c);
template <int T> void launch_B_t(snapgpu_ctx* c, double* blist);
struct YTablesHost {  // constant-bank tables of k_compute_Y_cwin (kernels.cuh)
  std::vector<int> rw;
};
template <int T> void upload_ytables_t(int device, const YTablesHost& t);
#ifdef SNAP_Y_PROFILE
extern long long* g_yprof;  // per-row cycle sums of k_compute_Y_cwin (calibration builds)
#endif

}  // namespace host
}  // namespace snapgpu
