// snapgpu.cu -- context lifetime, planning, stage sequencing, CUDA graph and
// the C-ABI (include/snapgpu.h).  The kernels are launched from the per-2J
// objects built from launch_t.cu; snapgpu_run replays the whole force step
// from a CUDA graph.
#include <cstdarg>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: named ranges for nsys / ncu

#include "ctx.hpp"

using namespace snapgpu;
using namespace snapgpu::host;

namespace {

thread_local std::string g_err = "";

// NVTX range over a C-ABI call (a no-op unless a tool is attached)
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

void invalidate_graph(snapgpu_ctx* c) {
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->graph) cudaGraphDestroy(c->graph);
  c->gexec = nullptr;
  c->graph = nullptr;
  c->graph_valid = false;
  if (c->fork_gexec) cudaGraphExecDestroy(c->fork_gexec);
  if (c->fork_graph) cudaGraphDestroy(c->fork_graph);
  c->fork_gexec = nullptr;
  c->fork_graph = nullptr;
  if (c->pull_gexec) cudaGraphExecDestroy(c->pull_gexec);
  if (c->pull_graph) cudaGraphDestroy(c->pull_graph);
  c->pull_gexec = nullptr;
  c->pull_graph = nullptr;
}

void invalidate_pos_graph(snapgpu_ctx* c) {
  if (c->pos_gexec) cudaGraphExecDestroy(c->pos_gexec);
  if (c->pos_graph) cudaGraphDestroy(c->pos_graph);
  c->pos_gexec = nullptr;
  c->pos_graph = nullptr;
  if (c->ppos_gexec) cudaGraphExecDestroy(c->ppos_gexec);
  if (c->ppos_graph) cudaGraphDestroy(c->ppos_graph);
  c->ppos_gexec = nullptr;
  c->ppos_graph = nullptr;
}

template <class F>
int guarded(snapgpu_ctx* c, F&& f) {
  try {
    if (c) CK(cudaSetDevice(c->device));
    f();
    return SNAPGPU_OK;
  } catch (const InvalidArg& e) {
    (c ? c->err : g_err) = e.msg;
    return SNAPGPU_EINVAL;
  } catch (const StateErr& e) {
    (c ? c->err : g_err) = e.msg;
    return SNAPGPU_ESTATE;
  } catch (const CudaError& e) {
    (c ? c->err : g_err) = e.msg;
    return SNAPGPU_ECUDA;
  } catch (const std::exception& e) {
    (c ? c->err : g_err) = e.what();
    return SNAPGPU_EPIPELINE;
  }
}

// ---------------------------------------------------------------------------
// template dispatch over twojmax
// ---------------------------------------------------------------------------
template <class Fn>
Fn pick_T(int T, Fn f0, Fn f1, Fn f2, Fn f3, Fn f4, Fn f5, Fn f6, Fn f7, Fn f8, Fn f9,
          Fn f10, Fn f11, Fn f12, Fn f13, Fn f14) {
  const Fn tab[15] = {f0, f1, f2, f3, f4, f5, f6, f7, f8, f9, f10, f11, f12, f13, f14};
  if (T < 0 || T > 14) throw InvalidArg{"twojmax outside [0, 14]"};
  return tab[T];
}
#define SNAP_PICK(name, T)                                                              \
  pick_T<void (*)(snapgpu_ctx*)>(T, name<0>, name<1>, name<2>, name<3>, name<4>, name<5>, \
                                 name<6>, name<7>, name<8>, name<9>, name<10>, name<11>, \
                                 name<12>, name<13>, name<14>)

void upload_ytables(int device, int T, const YTablesHost& t) {
  using Fn = void (*)(int, const YTablesHost&);
  pick_T<Fn>(T, upload_ytables_t<0>, upload_ytables_t<1>, upload_ytables_t<2>,
             upload_ytables_t<3>, upload_ytables_t<4>, upload_ytables_t<5>, upload_ytables_t<6>,
             upload_ytables_t<7>, upload_ytables_t<8>, upload_ytables_t<9>, upload_ytables_t<10>,
             upload_ytables_t<11>, upload_ytables_t<12>, upload_ytables_t<13>,
             upload_ytables_t<14>)(device, t);
}

// compute_Y work split (2J <= 8): one CTA per 32-atom tile, or, when the
// tiles are too few to fill the SMs, P CTAs per tile splitting its target
// rows (LPT on measured row costs); 2J > 8: one CTA per 8 atoms, fixed rows.
void build_ycoop(snapgpu_ctx* c);

void plan_y(snapgpu_ctx* c) {
  int pmax = 1;
  const int ntiles = std::max(1, c->ntiles);
  if (c->T <= SNAP_CWIN_MAXT) {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
    // per-tile part counts, row lists and the part-major CTA table
    // (tables.cpp y_cta_plan)
    const YCtaPlan yp = y_cta_plan(c->maps, c->ycplan.row_cost, ntiles, nsm, c->y_parts,
                                   kMaxYParts, kYGroups);
    pmax = yp.pmax;
    const std::vector<int>& tasks = yp.tasks;
    std::vector<int4> cta(yp.cta.size());
    for (size_t k = 0; k < cta.size(); ++k)
      cta[k] = make_int4(yp.cta[k][0], yp.cta[k][1], yp.cta[k][2], yp.cta[k][3]);
    c->y_ctas = static_cast<int>(cta.size());
    c->d_tasks.alloc(tasks.size());
    CK(cudaMemcpy(c->d_tasks.p, tasks.data(), tasks.size() * sizeof(int), cudaMemcpyHostToDevice));
    c->d_ycta.alloc(cta.size());
    CK(cudaMemcpy(c->d_ycta.p, cta.data(), cta.size() * sizeof(int4), cudaMemcpyHostToDevice));
    c->d_ready.alloc((size_t)ntiles);
    CK(cudaMemsetAsync(c->d_ready.p, 0, sizeof(unsigned) * (size_t)ntiles, c->stream));
  } else if (c->y_parts > 0) {
    pmax = c->y_parts;
  }
  c->y_parts_max = pmax;
  // energy epilogue: per-CTA lane energies, per-tile sums and tickets (the
  // 2J > 8 kernel has 4 tiles of 8 atoms per 32-atom V tile)
  const size_t nt = (size_t)ntiles;
  c->d_epart.alloc((size_t)pmax * 4 * nt * 32);
  c->d_tile_sum.alloc(4 * nt);
  c->d_tickets.alloc(1 + 4 * nt);
  CK(cudaMemsetAsync(c->d_tickets.p, 0, sizeof(unsigned) * (1 + 4 * nt), c->stream));
}

void upload_beta(snapgpu_ctx* c) {
  const std::vector<double> W = w_table(c->maps, c->cg, c->beta.data(), false);
  if (c->T <= SNAP_CWIN_MAXT) {
    // unit records: the beta-independent half + the W of the unit's items
    const std::vector<double> itw = ycoop_weights(c->ycplan, c->maps, W);
    const size_t nu = c->ycplan.units.size();
    std::vector<YUnit> u(nu);
    for (size_t q = 0; q < nu; ++q) {
      const int i0 = c->ycplan.units[q][0], n = c->ycplan.units[q][1];
      u[q].m = c->yunit_rec[q];
      u[q].w = make_double2(itw[i0], n == 2 ? itw[i0 + 1] : 0.0);
    }
    c->d_yunits.alloc(std::max<size_t>(1, 2 * nu));
    CK(cudaMemcpy(c->d_yunits.p, u.data(), nu * sizeof(YUnit), cudaMemcpyHostToDevice));
    return;
  }
  const std::vector<double> itw = yquad_weights(c->yqplan, c->maps, W);
  c->d_qitw.alloc(std::max<size_t>(1, itw.size()));
  CK(cudaMemcpy(c->d_qitw.p, itw.data(), itw.size() * sizeof(double), cudaMemcpyHostToDevice));
}

// constant-window units (kernels.cuh YUnit): the beta-independent record
// half; C' offsets index the padded windowed table (rows of cw_row(j))
static std::vector<uint4> pack_units(const snapgpu_ctx* c, const YCoopPlan& p) {
  std::vector<int> cwoff(c->maps.tuples.size());
  int o = 0;
  for (size_t q = 0; q < cwoff.size(); ++q) {
    cwoff[q] = o;
    o += (c->maps.tuples[q].j2 + 1) * cw_row(c->maps.tuples[q].j);
  }
  auto rows = [&](int i) {  // x1 window base | x2 row base << 16 of item i
    const Tuple& tp = c->maps.tuples[p.items[i][0]];
    const int D = (tp.j1 + tp.j2 - tp.j) / 2;
    const int mb1 = p.items[i][1], mb2 = p.items[i][2];
    const unsigned x1 = c->maps.full_off[tp.j1] + mb1 * (tp.j1 + 1) + D;
    const unsigned x2 = c->maps.full_off[tp.j2] + mb2 * (tp.j2 + 1);
    return x1 | (x2 << 16);
  };
  std::vector<uint4> out(p.units.size());
  for (size_t u = 0; u < out.size(); ++u) {
    const int i0 = p.units[u][0], n = p.units[u][1];
    const Tuple& tp = c->maps.tuples[p.items[i0][0]];
    out[u] = make_uint4(rows(i0), tp.j2 | (cwoff[p.items[i0][0]] << 8),
                        rows(n == 2 ? i0 + 1 : i0), 0u);
  }
  return out;
}

// y_plan's windowed C' (per tuple (j2+1) rows of j+1) with rows padded to
// cw_row(j) doubles (16-byte aligned coefficient pairs)
static std::vector<double> pad_cw(const snapgpu_ctx* c) {
  std::vector<double> out;
  size_t src = 0;
  for (const Tuple& tp : c->maps.tuples)
    for (int a2 = 0; a2 <= tp.j2; ++a2) {
      for (int ma = 0; ma < cw_row(tp.j); ++ma) out.push_back(ma <= tp.j ? c->yplan.cw[src + ma] : 0.0);
      src += tp.j + 1;
    }
  return out;
}

void build_ycoop(snapgpu_ctx* c) {
  c->ycplan = ycoop_pair_plan(c->maps, kYGroupWarps);
  c->yunit_rec = pack_units(c, c->ycplan);
  const std::vector<double> cwp = pad_cw(c);
  require(cwp.size() == (size_t)c_cwp_total(c->T), "compute_Y: C' table size mismatch");
  c->d_cwp.alloc(cwp.size());
  CK(cudaMemcpy(c->d_cwp.p, cwp.data(), cwp.size() * sizeof(double), cudaMemcpyHostToDevice));
  YTablesHost t;
  t.rw = c->ycplan.rw_begin;
  upload_ytables(c->device, c->T, t);
  upload_beta(c);
}

void launch_U(snapgpu_ctx* c) {
  if (c->nlocal > 0) SNAP_PICK(launch_U_t, c->T)(c);
}
void launch_Y(snapgpu_ctx* c) {
  if (c->nlocal > 0) {
    SNAP_PICK(launch_Y_t, c->T)(c);  // eatom and the total from the kernel's epilogue
  } else {
    CK(cudaMemsetAsync(c->d_etotal.p, 0, sizeof(double), c->stream));
  }
}
void launch_dE(snapgpu_ctx* c) {
  if (c->nlocal > 0) SNAP_PICK(launch_DE_t, c->T)(c);
}

double* forces_ptr(snapgpu_ctx* c) { return c->ext_forces ? c->ext_forces : c->d_forces.p; }
// doubles of the force output: natoms x 3, or nchunks x (3 chunk_rows + 1)
size_t force_doubles(const snapgpu_ctx* c) {
  return c->natoms_total > 0 ? (size_t)c->nchunks * c->chunk_stride() : 0;
}

RevArgs rev_args(snapgpu_ctx* c) {
  RevArgs a;
  a.pr = pair_args(c);
  a.off = c->d_rev_off.p;
  a.cur = c->d_rev_cur.p;
  a.rev = c->d_rev.p;
  a.nslots = c->nlocal * c->stride;
  return a;
}

// reverse-neighbor index of the current lists (kernels.cuh k_rev_*)
void launch_rev_build(snapgpu_ctx* c) {
  const int n = c->natoms_total;
  CK(cudaMemsetAsync(c->d_rev_off.p, 0, sizeof(int) * (n + 1), c->stream));
  const RevArgs a = rev_args(c);
  if (a.nslots > 0) {
    const int blk = (a.nslots + 255) / 256;
    k_rev_count<<<blk, 256, 0, c->stream>>>(a);
    k_nl_scan<<<1, 1024, 0, c->stream>>>(a.off, n, a.cur);
    k_rev_fill<<<blk, 256, 0, c->stream>>>(a);
    if (n > 0) k_rev_sort<<<(n + 7) / 8, 256, 0, c->stream>>>(a);
    CK(cudaGetLastError());
  }
}

void invalidate_csr_graph(snapgpu_ctx* c) {
  if (c->csr_gexec) cudaGraphExecDestroy(c->csr_gexec);
  if (c->csr_graph) cudaGraphDestroy(c->csr_graph);
  c->csr_gexec = nullptr;
  c->csr_graph = nullptr;
}

// Rebuild the reverse index if the lists changed since the last build (a
// captured graph of its five stream operations, replayed per list upload).
void ensure_csr(snapgpu_ctx* c) {
  if (!c->csr_dirty || c->sym_lists) return;
  if (!c->csr_gexec) {
    cudaStream_t user = c->stream;
    c->stream = c->own_stream;
    CK(cudaStreamSynchronize(user));
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    try {
      launch_rev_build(c);
    } catch (...) {
      cudaGraph_t g;
      cudaStreamEndCapture(c->stream, &g);
      if (g) cudaGraphDestroy(g);
      c->stream = user;
      throw;
    }
    CK(cudaStreamEndCapture(c->stream, &c->csr_graph));
    CK(cudaGraphInstantiate(&c->csr_gexec, c->csr_graph, 0));
    c->stream = user;
  }
  CK(cudaGraphLaunch(c->csr_gexec, c->stream));
  c->csr_dirty = false;
}

void launch_gather(snapgpu_ctx* c) {
  GatherArgs a;
  a.pr = pair_args(c);
  a.off = c->d_rev_off.p;
  a.rev = c->d_rev.p;
  a.rev_stride = c->sym_lists ? c->stride : 0;
  a.dedr = c->d_dedr.p;
  a.forces = forces_ptr(c);
  a.chunk_rows = c->chunk_rows();
  a.chunk_stride = c->chunk_stride();
  a.nchunks = c->nchunks;
  a.etotal = c->d_etotal.p;
  a.flags_out = reinterpret_cast<unsigned*>(c->d_out.p + c->d_forces.n + c->d_eatom.n + 1);
  a.forces_host = c->sink_forces;
  a.flags_host = c->sink_flags;
  const int nthr = std::max(3 * c->natoms_total, c->nchunks);
  if (c->natoms_total > 0) {  // one thread per force component
    launch_pdl(k_gather_forces, dim3((nthr + 127) / 128), dim3(128), 0, c->stream, a);
    CK(cudaGetLastError());
  }
}

void need(bool ok, const char* what) {
  if (!ok) throw StateErr{std::string("stage called out of order: ") + what};
}

const char* device_error_message(unsigned f) {
  if (f & kErrType) return "problem: atom type outside weight table";
  if (f & kErrCount) return "problem: neighbor count outside stride";
  if (f & kErrIndex) return "problem: neighbor index out of range";
  if (f & kErrSelf) return "problem: self neighbor";
  if (f & kErrZero) return "problem: zero-length neighbor displacement";
  return "problem: neighbor at or beyond Rcut";
}

// host_validate = false defers Problem::validate to the U kernel's checks
// (snapgpu_run_host reads the flags back with the results).
void set_lists(snapgpu_ctx* c, int natoms_total, int atom_lo, int nlocal, int stride,
               const int* numneigh, const int* nbr, const double* disp, const int* types,
               bool host_validate = true, bool upload = true) {
  require(natoms_total >= 0 && nlocal >= 0 && atom_lo >= 0 && atom_lo + nlocal <= natoms_total,
          "problem: owned range outside the atom count");
  require(nlocal == 0 || natoms_total > 0, "problem: no atoms");
  require(stride >= 0, "problem: negative neighbor stride");
  require((size_t)nlocal * stride < (size_t)INT32_MAX / 3, "problem: too many neighbor slots");
  require(!upload || nlocal == 0 || stride == 0 || (numneigh && nbr && disp),
          "problem: null neighbor arrays");
  c->have_lists = c->have_U = c->have_Y = c->have_dE = c->have_forces = false;
  c->csr_dirty = true;
  c->sym_lists = false;
  const bool reshape = natoms_total != c->natoms_total || nlocal != c->nlocal ||
                       stride != c->stride || atom_lo != c->atom_lo ||
                       (types != nullptr) != (c->d_types.p != nullptr);
  if (reshape) {
    invalidate_graph(c);
    invalidate_csr_graph(c);
    invalidate_pos_graph(c);
  }
  c->natoms_total = natoms_total;
  c->atom_lo = atom_lo;
  c->nlocal = nlocal;
  c->stride = stride;
  const int ntiles = (nlocal + 31) / 32;
  const size_t nslots = (size_t)nlocal * stride;
  const int NH = c->maps.nhalf;
  const size_t vsz = (size_t)std::max(1, ntiles) * 2 * NH * 32;
  if (reshape || ntiles != c->ntiles) {
    c->d_numneigh.alloc(std::max(1, nlocal));
    c->d_nbr.alloc(std::max<size_t>(1, nslots));
    c->d_disp.alloc(std::max<size_t>(1, nslots * 3));
    c->d_dedr.alloc(std::max<size_t>(1, nslots * 3));
    c->d_rev_off.alloc((size_t)natoms_total + 1);
    c->d_rev_cur.alloc(std::max(1, natoms_total));
    c->d_rev.alloc(std::max<size_t>(1, nslots));
    // forces, eatom and etotal are contiguous so the one-call API reads them
    // back with a single copy
    const size_t nf = (size_t)std::max(1, c->nchunks) * c->chunk_stride(),
                 ne = std::max(1, nlocal);
    c->d_forces.release();
    c->d_eatom.release();
    c->d_etotal.release();
    // [forces | eatom | etotal | validation flags]: the gather copies the
    // flags into the last slot, so a one-call step reads everything back
    // with one D2H
    c->d_out.alloc(nf + ne + 2);
    CK(cudaMemsetAsync(c->d_out.p, 0, (nf + ne + 2) * sizeof(double), c->stream));
    c->d_forces.view(c->d_out.p, nf);
    c->d_eatom.view(c->d_out.p + nf, ne);
    c->d_etotal.view(c->d_out.p + nf + ne, 1);
    const bool grow = vsz > c->d_V.n;
    c->d_V.alloc(vsz);
    c->d_Y.alloc(vsz);
    if (grow || ntiles != c->ntiles) {
      CK(cudaMemsetAsync(c->d_V.p, 0, vsz * sizeof(double), c->stream));
      CK(cudaMemsetAsync(c->d_Y.p, 0, vsz * sizeof(double), c->stream));
    }
    if (types) {
      c->d_types.alloc(std::max(1, natoms_total));
    } else {
      c->d_types.release();
    }
    c->ntiles = ntiles;
    plan_y(c);
  }
  // Enqueue the uploads first (asynchronous from pinned memory) and validate
  // on the host while they are in flight; a failed validation leaves the
  // context without lists, so nothing runs on the uploaded data.
  if (nlocal > 0 && upload) {
    CK(cudaMemcpyAsync(c->d_numneigh.p, numneigh, sizeof(int) * nlocal, cudaMemcpyHostToDevice,
                       c->stream));
    if (nslots > 0) {
      CK(cudaMemcpyAsync(c->d_nbr.p, nbr, sizeof(int) * nslots, cudaMemcpyHostToDevice,
                         c->stream));
      CK(cudaMemcpyAsync(c->d_disp.p, disp, sizeof(double) * nslots * 3, cudaMemcpyHostToDevice,
                         c->stream));
    }
  }
  if (types)
    CK(cudaMemcpyAsync(c->d_types.p, types, sizeof(int) * natoms_total, cudaMemcpyHostToDevice,
                       c->stream));
  if (!host_validate) {
    c->have_lists = true;
    return;
  }
  // Problem::validate (snap_core.hpp:89-118)
  const double rc2 = c->gp.rcut * c->gp.rcut;
  const int nw = static_cast<int>(c->weights.size());
  if (types)
    for (int a = 0; a < natoms_total; ++a)
      require(types[a] >= 0 && types[a] < nw, "problem: atom type outside weight table");
  for (int i = 0; i < nlocal; ++i) {
    const int nn = numneigh[i];
    require(nn >= 0 && nn <= stride, "problem: neighbor count outside stride");
    const int* ip = nbr + (size_t)i * stride;
    const double* dp = disp + (size_t)i * stride * 3;
    bool idx_ok = true, self_ok = true, pos_ok = true, cut_ok = true;
    for (int k = 0; k < nn; ++k) {
      const int j = ip[k];
      idx_ok &= (j >= 0) & (j < natoms_total);
      self_ok &= (j != atom_lo + i);
      const double r2 = dp[3 * k] * dp[3 * k] + dp[3 * k + 1] * dp[3 * k + 1] +
                        dp[3 * k + 2] * dp[3 * k + 2];
      pos_ok &= r2 > 0.0;
      cut_ok &= r2 < rc2;
    }
    require(idx_ok, "problem: neighbor index out of range");
    require(self_ok, "problem: self neighbor");
    require(pos_ok, "problem: zero-length neighbor displacement");
    require(cut_ok, "problem: neighbor at or beyond Rcut");
  }
  c->have_lists = true;
}

// Device neighbor lists (kernels.cuh k_nl_*): argument block, scratch
// allocations and the front half (positions upload, cell binning, cell
// offsets, members) shared by set_positions and the one-call positions step.
NLArgs nl_setup(snapgpu_ctx* c, int natoms, const double* pos, const double* box) {
  require(natoms >= 0 && (natoms == 0 || pos) && box, "set_positions: bad arguments");
  const double rcut = c->gp.rcut;
  NLArgs a{};
  for (int d = 0; d < 3; ++d) {  // harness.hpp:119-125 preconditions
    require(box[d] > 0.0 && rcut > 0.0, "build_neighborlist: box and Rcut must be positive");
    require(rcut <= 0.5 * box[d], "build_neighborlist: Rcut must not exceed box/2");
    a.box[d] = box[d];
    a.nc[d] = static_cast<int>(std::floor(box[d] / rcut));
  }
  a.cells = (a.nc[0] >= 3 && a.nc[1] >= 3 && a.nc[2] >= 3) ? 1 : 0;
  a.n = natoms;
  a.rc2 = rcut * rcut;
  const long ncell = a.cells ? (long)a.nc[0] * a.nc[1] * a.nc[2] : 0;
  c->d_nlpos.alloc(std::max<size_t>(1, (size_t)natoms * 6));
  c->d_nlint.alloc((size_t)std::max(1, natoms) * 3 + 2 * (size_t)ncell + 4);
  double* dpos = c->d_nlpos.p;
  a.pos = dpos;
  a.w = dpos + (size_t)natoms * 3;
  int* ib = c->d_nlint.p;
  a.cell_of = ib;
  a.members = ib + natoms;
  a.numneigh = ib + 2 * (size_t)natoms;
  a.head = ib + 3 * (size_t)natoms;
  a.fill = a.head + ncell + 1;
  a.maxcount = a.fill + ncell;
  return a;
}

void nl_front(snapgpu_ctx* c, const NLArgs& a, const double* host_pos) {
  const long ncell = a.cells ? (long)a.nc[0] * a.nc[1] * a.nc[2] : 0;
  if (a.n > 0)
    CK(cudaMemcpyAsync(const_cast<double*>(a.pos), host_pos, sizeof(double) * 3 * a.n,
                       cudaMemcpyHostToDevice, c->stream));
  if (a.n > 0 && a.n <= kNLSmallAtoms && ncell <= kNLSmallCells) {  // one launch
    k_nl_front_small<<<1, 1024, 0, c->stream>>>(a);
    CK(cudaGetLastError());
    return;
  }
  CK(cudaMemsetAsync(a.head, 0, sizeof(int) * (ncell + 1), c->stream));
  const int blk = (a.n + 127) / 128;
  if (a.n > 0) {
    k_nl_bin<<<blk, 128, 0, c->stream>>>(a);
    if (a.cells) {
      k_nl_scan<<<1, 1024, 0, c->stream>>>(a.head, (int)ncell, a.fill);
      k_nl_members<<<blk, 128, 0, c->stream>>>(a);
    }
    CK(cudaGetLastError());
  }
}

// partner slots of the (symmetric) device-built lists into d_rev
void launch_partner(snapgpu_ctx* c) {
  const int ns = c->nlocal * c->stride;
  if (ns > 0) {
    k_nl_partner<<<(ns + 255) / 256, 256, 0, c->stream>>>(c->d_numneigh.p, c->d_nbr.p,
                                                          c->nlocal, c->stride, c->d_rev.p,
                                                          c->d_err.p);
    CK(cudaGetLastError());
  }
}

void record(snapgpu_ctx* c, int k) {
  if (c->timing) CK(cudaEventRecord(c->ev[k], c->stream));
}

// Device address of a mapped (pinned) host array, or null for pageable memory.
const void* mapped_ptr(const void* p) {
  if (!p) return nullptr;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return (at.type == cudaMemoryTypeHost) ? at.devicePointer : nullptr;
}

// The one-call step from pinned host lists: compute_U pulls the lists over
// PCIe while it computes (UArgs::src_*) and leaves the device copies; the
// reverse-index build forks onto side_stream after it and joins before the
// force gather.  Direct launches (the sources change every call).
void run_pull(snapgpu_ctx* c, const int* nn, const int* nb, const double* dp) {
  cudaStream_t main = c->stream;
  c->zc_numneigh = nn;
  c->zc_nbr = nb;
  c->zc_disp = dp;
  try {
    launch_U(c);
    c->zc_numneigh = c->zc_nbr = nullptr;
    c->zc_disp = nullptr;
    CK(cudaEventRecord(c->ev_fork, main));
    CK(cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
    c->stream = c->side_stream;
    launch_rev_build(c);
    CK(cudaEventRecord(c->ev_join, c->side_stream));
    c->stream = main;
    launch_Y(c);
    launch_dE(c);
    CK(cudaStreamWaitEvent(main, c->ev_join, 0));
    launch_gather(c);
  } catch (...) {
    c->stream = main;
    c->zc_numneigh = c->zc_nbr = nullptr;
    c->zc_disp = nullptr;
    throw;
  }
  c->csr_dirty = false;
}

// The node the capture on `s` just added (its single current dependency).
cudaGraphNode_t last_node(cudaStream_t s) {
  cudaStreamCaptureStatus st;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CK(cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &deps, &nd));
  if (st != cudaStreamCaptureStatusActive || nd != 1) throw CudaError{"pull graph: capture state"};
  return deps[0];
}

// run_pull as one graph (pinned lists and pinned outputs): captured once per
// shape, then each call patches its host pointers into the U node (list
// sources), the Y node (eatom / etotal sinks) and the gather node (forces /
// flags sinks) and replays it -- no per-kernel launch overhead, no gaps.
void run_pull_graph(snapgpu_ctx* c, const int* nn, const int* nb, const double* dp) {
  if (!c->pull_gexec) {
    cudaStream_t user = c->stream;
    c->stream = c->own_stream;
    CK(cudaStreamSynchronize(user));
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    try {
      c->zc_numneigh = nn;
      c->zc_nbr = nb;
      c->zc_disp = dp;
      launch_U(c);
      c->pull_node[0] = last_node(c->stream);
      c->zc_numneigh = c->zc_nbr = nullptr;
      c->zc_disp = nullptr;
      CK(cudaEventRecord(c->ev_fork, c->own_stream));
      CK(cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
      c->stream = c->side_stream;
      launch_rev_build(c);
      CK(cudaEventRecord(c->ev_join, c->side_stream));
      c->stream = c->own_stream;
      launch_Y(c);
      c->pull_node[1] = last_node(c->stream);
      launch_dE(c);
      CK(cudaStreamWaitEvent(c->own_stream, c->ev_join, 0));
      launch_gather(c);
      c->pull_node[2] = last_node(c->stream);
    } catch (...) {
      c->stream = c->own_stream;
      c->zc_numneigh = c->zc_nbr = nullptr;
      c->zc_disp = nullptr;
      cudaGraph_t g;
      cudaStreamEndCapture(c->stream, &g);
      if (g) cudaGraphDestroy(g);
      c->stream = user;
      throw;
    }
    CK(cudaStreamEndCapture(c->stream, &c->pull_graph));
    CK(cudaGraphInstantiate(&c->pull_gexec, c->pull_graph, 0));
    c->stream = user;
    for (int k = 0; k < 3; ++k) CK(cudaGraphKernelNodeGetParams(c->pull_node[k], &c->pull_kp[k]));
    std::memcpy(&c->pull_u, c->pull_kp[0].kernelParams[0], sizeof(UArgs));
    std::memcpy(&c->pull_y, c->pull_kp[1].kernelParams[0], sizeof(YWArgs));
    static_assert(sizeof(GatherArgs) <= sizeof(c->pull_g), "pull graph: gather args storage");
    std::memcpy(c->pull_g, c->pull_kp[2].kernelParams[0], sizeof(GatherArgs));
  }
  // patch the nodes whose host pointers differ from the last replay (an MD
  // loop passes the same pinned buffers every step: no patch at all)
  UArgs& u = c->pull_u;
  YWArgs& y = c->pull_y;
  GatherArgs g;
  std::memcpy(&g, c->pull_g, sizeof(GatherArgs));
  const bool du = u.src_numneigh != nn || u.src_nbr != nb || u.src_disp != dp;
  const bool dy = y.E.eatom_host != c->sink_eatom || y.E.etotal_host != c->sink_etotal;
  const bool dg = g.forces_host != c->sink_forces || g.flags_host != c->sink_flags;
  u.src_numneigh = nn;
  u.src_nbr = nb;
  u.src_disp = dp;
  y.E.eatom_host = c->sink_eatom;
  y.E.etotal_host = c->sink_etotal;
  g.forces_host = c->sink_forces;
  g.flags_host = c->sink_flags;
  std::memcpy(c->pull_g, &g, sizeof(GatherArgs));
  void* pp[3] = {&u, &y, &g};
  const bool dirty[3] = {du, dy, dg};
  for (int k = 0; k < 3; ++k) {
    if (!dirty[k]) continue;
    cudaKernelNodeParams kp = c->pull_kp[k];
    kp.kernelParams = &pp[k];
    CK(cudaGraphExecKernelNodeSetParams(c->pull_gexec, c->pull_node[k], &kp));
  }
  CK(cudaGraphLaunch(c->pull_gexec, c->stream));
  c->csr_dirty = false;
}

// The one-call positions step from pinned positions into pinned outputs
// (host pointers already device-mapped; sinks set by the caller): binning
// reads the positions over PCIe, lists, partner slots, U, Y, dE, gather with
// the result sinks -- one graph, no copies; per-call pointers patched into
// the binning, Y and gather nodes when they change.
void run_positions_pull(snapgpu_ctx* c, int natoms, const double* pos) {
  if (!c->ppos_gexec) {
    cudaStream_t user = c->stream;
    c->stream = c->own_stream;
    CK(cudaStreamSynchronize(user));
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    try {
      NLArgs a = nl_setup(c, natoms, pos, c->nl_box);
      a.pos = pos;  // mapped host positions (the binning kernel's only input)
      const long ncell = a.cells ? (long)a.nc[0] * a.nc[1] * a.nc[2] : 0;
      if (a.n <= kNLSmallAtoms && ncell <= kNLSmallCells) {
        k_nl_front_small<<<1, 1024, 0, c->stream>>>(a);
        CK(cudaGetLastError());
        c->ppos_node[0] = last_node(c->stream);
      } else {
        CK(cudaMemsetAsync(a.head, 0, sizeof(int) * (ncell + 1), c->stream));
        const int blk = (a.n + 127) / 128;
        k_nl_bin<<<blk, 128, 0, c->stream>>>(a);
        CK(cudaGetLastError());
        c->ppos_node[0] = last_node(c->stream);
        if (a.cells) {
          k_nl_scan<<<1, 1024, 0, c->stream>>>(a.head, (int)ncell, a.fill);
          k_nl_members<<<blk, 128, 0, c->stream>>>(a);
        }
      }
      a.numneigh = c->d_numneigh.p;
      a.nbr = c->d_nbr.p;
      a.disp = c->d_disp.p;
      a.stride = c->stride;
      a.maxcount = nullptr;
      k_nl_lists_warp<<<(natoms + kNLWarps - 1) / kNLWarps, kNLWarps * 32, 0, c->stream>>>(
          a, c->d_err.p);
      CK(cudaGetLastError());
      // the partner slots only feed the gather: built beside U / Y / dE
      CK(cudaEventRecord(c->ev_fork, c->stream));
      CK(cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
      c->stream = c->side_stream;
      launch_partner(c);
      CK(cudaEventRecord(c->ev_join, c->side_stream));
      c->stream = c->own_stream;
      launch_U(c);
      launch_Y(c);
      c->ppos_node[1] = last_node(c->stream);
      launch_dE(c);
      CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
      launch_gather(c);
      c->ppos_node[2] = last_node(c->stream);
    } catch (...) {
      c->stream = c->own_stream;
      cudaGraph_t g;
      cudaStreamEndCapture(c->stream, &g);
      if (g) cudaGraphDestroy(g);
      c->stream = user;
      throw;
    }
    CK(cudaStreamEndCapture(c->stream, &c->ppos_graph));
    CK(cudaGraphInstantiate(&c->ppos_gexec, c->ppos_graph, 0));
    c->stream = user;
    for (int k = 0; k < 3; ++k) CK(cudaGraphKernelNodeGetParams(c->ppos_node[k], &c->ppos_kp[k]));
    static_assert(sizeof(NLArgs) <= sizeof(c->ppos_nl), "positions graph: binning args storage");
    std::memcpy(c->ppos_nl, c->ppos_kp[0].kernelParams[0], sizeof(NLArgs));
    std::memcpy(&c->ppos_y, c->ppos_kp[1].kernelParams[0], sizeof(YWArgs));
    static_assert(sizeof(GatherArgs) <= sizeof(c->ppos_g), "positions graph: gather args storage");
    std::memcpy(c->ppos_g, c->ppos_kp[2].kernelParams[0], sizeof(GatherArgs));
  }
  NLArgs a;
  std::memcpy(&a, c->ppos_nl, sizeof(NLArgs));
  YWArgs& y = c->ppos_y;
  GatherArgs g;
  std::memcpy(&g, c->ppos_g, sizeof(GatherArgs));
  const bool da = a.pos != pos;
  const bool dy = y.E.eatom_host != c->sink_eatom || y.E.etotal_host != c->sink_etotal;
  const bool dg = g.forces_host != c->sink_forces || g.flags_host != c->sink_flags;
  a.pos = pos;
  y.E.eatom_host = c->sink_eatom;
  y.E.etotal_host = c->sink_etotal;
  g.forces_host = c->sink_forces;
  g.flags_host = c->sink_flags;
  std::memcpy(c->ppos_g, &g, sizeof(GatherArgs));
  std::memcpy(c->ppos_nl, &a, sizeof(NLArgs));
  void* pp[3] = {&a, &y, &g};
  const bool dirty[3] = {da, dy, dg};
  for (int k = 0; k < 3; ++k) {
    if (!dirty[k]) continue;
    cudaKernelNodeParams kp = c->ppos_kp[k];
    kp.kernelParams = &pp[k];
    CK(cudaGraphExecKernelNodeSetParams(c->ppos_gexec, c->ppos_node[k], &kp));
  }
  CK(cudaGraphLaunch(c->ppos_gexec, c->stream));
}

void run_direct(snapgpu_ctx* c) {
  record(c, 0);
  launch_U(c);
  record(c, 1);
  launch_Y(c);
  record(c, 2);
  launch_dE(c);
  record(c, 3);
  launch_gather(c);
  record(c, 4);
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
#ifdef SNAP_Y_PROFILE
long long* snapgpu::host::g_yprof = nullptr;
extern "C" int snapgpu_debug_yprof(long long* out, int n) {
  if (!g_yprof) return -1;
  cudaDeviceSynchronize();
  cudaMemcpy(out, g_yprof, sizeof(long long) * n, cudaMemcpyDeviceToHost);
  cudaMemset(g_yprof, 0, sizeof(long long) * 2112);
  return 0;
}
#endif

extern "C" {

const char* snapgpu_last_error(const snapgpu_ctx* c) {
  return c ? c->err.c_str() : g_err.c_str();
}

const char* snapgpu_version(void) { return "snapgpu 0.1 (sm_100a, FP64 SIMT, v-space)"; }

int snapgpu_debug_y_plan(int twojmax, int ntiles, int nsm, int y_parts, int* cta, int cta_cap,
                         int* tasks, int tasks_cap) {
  int n = 0;
  const int rc = guarded(nullptr, [&] {
    require(twojmax >= 0 && twojmax <= SNAP_CWIN_MAXT, "debug_y_plan: twojmax outside [0, 8]");
    require(ntiles > 0 && nsm > 0 && y_parts >= 0 && y_parts <= kMaxYParts,
            "debug_y_plan: bad arguments");
    const IndexMaps m = IndexMaps::build(twojmax);
    const YCoopPlan cp = ycoop_pair_plan(m, kYGroupWarps);
    const YCtaPlan yp = y_cta_plan(m, cp.row_cost, ntiles, nsm, y_parts, kMaxYParts, kYGroups);
    n = static_cast<int>(yp.cta.size());
    require(cta && cta_cap >= 4 * n && tasks && tasks_cap >= static_cast<int>(yp.tasks.size()),
            "debug_y_plan: output too small");
    for (int k = 0; k < n; ++k)
      for (int q = 0; q < 4; ++q) cta[4 * k + q] = yp.cta[k][q];
    std::copy(yp.tasks.begin(), yp.tasks.end(), tasks);
  });
  return rc == SNAPGPU_OK ? n : rc;
}

int snapgpu_counts(int twojmax, int* out) {
  return guarded(nullptr, [&] {
    require(twojmax >= 0 && twojmax <= 64, "twojmax out of range");
    require(out != nullptr, "null output");
    IndexMaps m = IndexMaps::build(twojmax);
    out[0] = static_cast<int>(m.triples.size());
    out[1] = static_cast<int>(m.tuples.size());
    out[2] = m.nfull;
    out[3] = m.nhalf;
    out[4] = m.zelems;
    out[5] = m.cgtot;
  });
}

int snapgpu_create(int device, int twojmax, double rcut, double rmin0, double rfac0,
                   double wself, int self_flag, const double* beta, int nbeta,
                   const double* weights, int nweights, snapgpu_ctx** out) {
  snapgpu_ctx* c = nullptr;
  const int rc = guarded(nullptr, [&] {
    require(out != nullptr, "snapgpu_create: null output handle");
    require(twojmax >= 0 && twojmax <= SNAPGPU_MAX_TWOJMAX,
            "snapgpu_create: twojmax outside [0, 14]");
    require(rcut > rmin0, "problem: Rcut must exceed rmin0");  // snap_core.hpp:98
    require(nweights > 0 && weights, "problem: empty weight table");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    require(device >= 0 && device < ndev, "snapgpu_create: no such CUDA device");
    CK(cudaSetDevice(device));
    c = new snapgpu_ctx();
    c->device = device;
    {  // tools that inject themselves (ncu: CUDA_INJECTION64_PATH;
       // compute-sanitizer: NV_SANITIZER_INJECTION_*) may serialize grids
      const char* inj = std::getenv("CUDA_INJECTION64_PATH");
      const char* san = std::getenv("NV_SANITIZER_INJECTION_PORT_BASE");
      c->y_overlap = !((inj && *inj) || (san && *san));
    }
    c->T = twojmax;
    c->d_err.alloc(1);
    CK(cudaMemset(c->d_err.p, 0, sizeof(unsigned)));
    CK(cudaMallocHost(&c->h_err, sizeof(unsigned)));
    *c->h_err = 0u;
    c->maps = IndexMaps::build(twojmax);
    require(nbeta == static_cast<int>(c->maps.triples.size()) && beta,
            "problem: beta length must match the triple count");
    c->gp.rcut = rcut;
    c->gp.rmin0 = rmin0;
    c->gp.rfac0 = rfac0;
    c->gp.wself = wself;
    c->gp.self_flag = self_flag ? 1 : 0;
    c->beta.assign(beta, beta + nbeta);
    c->weights.assign(weights, weights + nweights);
    c->cg = cg_table(c->maps);
    c->hf = half_f(c->maps);
    c->ywgt = half_ywgt(c->maps);
    CK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    {  // the reverse-index build runs beside compute_Y, which fills every SM:
       // its small kernels take SMs ahead of the waiting compute_fused_dE CTAs
      int lo = 0, hi = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      CK(cudaStreamCreateWithPriority(&c->side_stream, cudaStreamNonBlocking, hi));
    }
    CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    c->stream = c->own_stream;
    for (auto& e : c->ev) CK(cudaEventCreate(&e));
    auto up = [](auto& buf, const auto& v) {
      using E = typename std::decay_t<decltype(v)>::value_type;
      buf.alloc(std::max<size_t>(1, v.size()));
      CK(cudaMemcpy(buf.p, v.data(), v.size() * sizeof(E), cudaMemcpyHostToDevice));
    };
    up(c->d_weights, c->weights);
    c->yplan = y_plan(c->maps, cprime_table(c->maps, c->cg));
    up(c->d_expand, half_scatter_map(c->maps));
    if (twojmax <= SNAP_CWIN_MAXT) {
      // constant-window compute_Y: the windowed C' and the unit tables live
      // in the per-2J object's constant bank
      build_ycoop(c);
    } else {
      // quad-unit compute_Y: C' and the beta-independent unit tables in HBM
      up(c->d_cw, c->yplan.cw);  // (the descriptor kernel's layout)
      up(c->d_cwq, yquad_cw(c->maps, c->yplan.cw));
      c->yqplan = yquad_plan(c->maps, kQWarps / kQGroups, kQGroups);
      std::vector<int4> u(c->yqplan.units.size());
      for (size_t q = 0; q < u.size(); ++q)
        u[q] = make_int4(c->yqplan.units[q][0], c->yqplan.units[q][1], c->yqplan.units[q][2],
                         c->yqplan.units[q][3]);
      up(c->d_qunits, u);
      up(c->d_qrw, c->yqplan.rw);
      up(c->d_qrows, c->yqplan.rows);
      upload_beta(c);
    }
    *out = c;
  });
  if (rc != SNAPGPU_OK && c) {
    snapgpu_destroy(c);
    if (out) *out = nullptr;
  }
  return rc;
}

int snapgpu_destroy(snapgpu_ctx* c) {
  if (!c) return SNAPGPU_OK;
  cudaSetDevice(c->device);
  invalidate_graph(c);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  invalidate_csr_graph(c);
  invalidate_pos_graph(c);
  if (c->h_pos) cudaFreeHost(c->h_pos);
  c->d_weights.release();
  c->d_cw.release();

  c->d_cwp.release();
  c->d_yunits.release();
  c->d_qunits.release();
  c->d_qitw.release();
  c->d_cwq.release();
  c->d_qrw.release();
  c->d_qrows.release();
  c->d_nlpos.release();
  c->d_nlint.release();
  c->d_virial.release();
  c->d_expand.release();
  c->d_tasks.release();
  c->d_ycta.release();
  c->d_ready.release();
  c->d_numneigh.release();
  c->d_nbr.release();
  c->d_types.release();
  c->d_disp.release();
  c->d_V.release();
  c->d_Y.release();
  c->d_dedr.release();
  c->d_forces.release();
  c->d_eatom.release();
  c->d_etotal.release();
  c->d_out.release();
  if (c->h_out) cudaFreeHost(c->h_out);
  c->d_bitems.release();
  c->d_bcwoff.release();
  c->d_btbeg.release();
  c->d_bwgt.release();
  c->d_blist.release();
  c->d_epart.release();
  c->d_tile_sum.release();
  c->d_tickets.release();
  c->d_rev_off.release();
  c->d_rev_cur.release();
  c->d_rev.release();
  c->d_err.release();
  if (c->h_err) cudaFreeHost(c->h_err);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->side_stream) cudaStreamDestroy(c->side_stream);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  delete c;
  return SNAPGPU_OK;
}

int snapgpu_set_beta(snapgpu_ctx* c, const double* beta, int nbeta) {
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    require(beta && nbeta == static_cast<int>(c->maps.triples.size()),
            "problem: beta length must match the triple count");
    CK(cudaStreamSynchronize(c->stream));
    c->beta.assign(beta, beta + nbeta);
    upload_beta(c);
    c->have_Y = c->have_dE = false;
  });
}

int snapgpu_compute_descriptors(snapgpu_ctx* c, double* blist) {
  const Nvtx nvtx_range("snapgpu_compute_descriptors");
  if (!c || !blist) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    need(c->have_lists, "compute_descriptors: no neighbor lists");
    // B_l(i) (compute_B_from_U, snap_core.hpp:642-681) in one pass over V
    if (!c->d_bitems.p) {
      const BPlan bp = b_plan(c->maps, c->cg);
      std::vector<int4> it(bp.items.size());
      for (size_t q = 0; q < it.size(); ++q)
        it[q] = make_int4(bp.items[q][0], bp.items[q][1], bp.items[q][2], bp.items[q][3]);
      auto up = [](auto& buf, const auto& v) {
        using E = typename std::decay_t<decltype(v)>::value_type;
        buf.alloc(std::max<size_t>(1, v.size()));
        CK(cudaMemcpy(buf.p, v.data(), v.size() * sizeof(E), cudaMemcpyHostToDevice));
      };
      up(c->d_bitems, it);
      up(c->d_bcwoff, bp.cwoff);
      up(c->d_bwgt, bp.wgt);
      up(c->d_btbeg, bp.triple_begin);
      if (!c->d_cw.p) up(c->d_cw, c->yplan.cw);
    }
    if (!c->have_U) launch_U(c);
    c->have_U = true;
    const size_t nb = (size_t)std::max(1, c->nlocal) * c->maps.triples.size();
    c->d_blist.alloc(nb);
    if (c->nlocal > 0) {
      using Fn = void (*)(snapgpu_ctx*, double*);
      pick_T<Fn>(c->T, launch_B_t<0>, launch_B_t<1>, launch_B_t<2>, launch_B_t<3>,
                 launch_B_t<4>, launch_B_t<5>, launch_B_t<6>, launch_B_t<7>, launch_B_t<8>,
                 launch_B_t<9>, launch_B_t<10>, launch_B_t<11>, launch_B_t<12>, launch_B_t<13>,
                 launch_B_t<14>)(c, c->d_blist.p);
      CK(cudaMemcpyAsync(blist, c->d_blist.p,
                         sizeof(double) * (size_t)c->nlocal * c->maps.triples.size(),
                         cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
  });
}

int snapgpu_set_stream(snapgpu_ctx* c, void* s) {
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    c->stream = s ? static_cast<cudaStream_t>(s) : c->own_stream;
  });
}

int snapgpu_set_neighbors(snapgpu_ctx* c, int natoms, int stride, const int* numneigh,
                          const int* nbr, const double* disp, const int* types) {
  const Nvtx nvtx_range("snapgpu_set_neighbors");
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    set_lists(c, natoms, 0, natoms, stride, numneigh, nbr, disp, types);
  });
}

int snapgpu_set_neighbors_partition(snapgpu_ctx* c, int natoms_total, int atom_lo, int nlocal,
                                    int stride, const int* numneigh, const int* nbr,
                                    const double* disp, const int* types) {
  const Nvtx nvtx_range("snapgpu_set_neighbors_partition");
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    set_lists(c, natoms_total, atom_lo, nlocal, stride, numneigh, nbr, disp, types);
  });
}

int snapgpu_compute_U(snapgpu_ctx* c) {
  const Nvtx nvtx_range("snapgpu_compute_U");
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    need(c->have_lists, "compute_U needs neighbor lists");
    launch_U(c);
    c->have_U = true;
    c->have_Y = c->have_dE = false;
  });
}

int snapgpu_compute_Y(snapgpu_ctx* c) {
  const Nvtx nvtx_range("snapgpu_compute_Y");
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    need(c->have_U, "compute_Y: no Ulisttot");  // snap_core.hpp:1089
    launch_Y(c);
    c->have_Y = true;
  });
}

int snapgpu_compute_dU_deidrj(snapgpu_ctx* c) {
  const Nvtx nvtx_range("snapgpu_compute_dU_deidrj");
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    need(c->have_Y, "compute_fused_dE: requires Ylist");  // snap_core.hpp:1278
    launch_dE(c);
    c->have_dE = true;
  });
}

int snapgpu_scatter_forces(snapgpu_ctx* c) {
  const Nvtx nvtx_range("snapgpu_scatter_forces");
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    need(c->have_dE, "scatter_forces: no dElist");  // snap_core.hpp:876
    ensure_csr(c);
    launch_gather(c);
    c->have_forces = true;
  });
}

int snapgpu_run(snapgpu_ctx* c) {
  const Nvtx nvtx_range("snapgpu_run");
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    need(c->have_lists, "run: no neighbor lists");
    if (c->timing) {
      ensure_csr(c);
      run_direct(c);
      CK(cudaEventSynchronize(c->ev[4]));
      for (int s = 0; s < 4; ++s) CK(cudaEventElapsedTime(&c->stage_ms[s], c->ev[s], c->ev[s + 1]));
    } else if (c->csr_dirty && !c->sym_lists) {
      // new lists: the reverse-index build runs beside U / Y / dE (it only
      // feeds the force gather), one graph with a fork and a join
      if (!c->fork_gexec) {
        cudaStream_t user = c->stream;
        c->stream = c->own_stream;
        CK(cudaStreamSynchronize(user));
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        try {
          CK(cudaEventRecord(c->ev_fork, c->own_stream));
          CK(cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
          c->stream = c->side_stream;
          launch_rev_build(c);
          CK(cudaEventRecord(c->ev_join, c->side_stream));
          c->stream = c->own_stream;
          launch_U(c);
          launch_Y(c);
          launch_dE(c);
          CK(cudaStreamWaitEvent(c->own_stream, c->ev_join, 0));
          launch_gather(c);
        } catch (...) {
          c->stream = c->own_stream;
          cudaGraph_t g;
          cudaStreamEndCapture(c->stream, &g);
          if (g) cudaGraphDestroy(g);
          c->stream = user;
          throw;
        }
        CK(cudaStreamEndCapture(c->stream, &c->fork_graph));
        CK(cudaGraphInstantiate(&c->fork_gexec, c->fork_graph, 0));
        c->stream = user;
      }
      CK(cudaGraphLaunch(c->fork_gexec, c->stream));
      c->csr_dirty = false;
    } else {
      if (!c->graph_valid) {
        if (c->gexec) cudaGraphExecDestroy(c->gexec);
        if (c->graph) cudaGraphDestroy(c->graph);
        c->gexec = nullptr;
        c->graph = nullptr;
        cudaStream_t user = c->stream;
        c->stream = c->own_stream;  // capture on our own (non-legacy) stream
        CK(cudaStreamSynchronize(user));
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        try {
          run_direct(c);
        } catch (...) {
          cudaGraph_t g;
          cudaStreamEndCapture(c->stream, &g);
          if (g) cudaGraphDestroy(g);
          c->stream = user;
          throw;
        }
        CK(cudaStreamEndCapture(c->stream, &c->graph));
        CK(cudaGraphInstantiate(&c->gexec, c->graph, 0));
        c->stream = user;
        c->graph_valid = true;
      }
      CK(cudaGraphLaunch(c->gexec, c->stream));
    }
    c->have_U = c->have_Y = c->have_dE = c->have_forces = true;
  });
}

int snapgpu_run_host(snapgpu_ctx* c, int natoms_total, int atom_lo, int nlocal, int stride,
                     const int* numneigh, const int* nbr, const double* disp,
                     const int* types, double* forces, double* eatom, double* etotal) {
  const Nvtx nvtx_range("snapgpu_run_host");
  if (!c) return SNAPGPU_EINVAL;
  bool pulled = false, sunk = false;
  const int rc = guarded(c, [&] {
    // pinned (mapped) host lists: no upload, compute_U pulls them itself
    const void* zn = nullptr;
    const void* zb = nullptr;
    const void* zd = nullptr;
    if (c->T <= 8 && nlocal > 0 && stride > 0 && !c->timing) {  // k_compute_U2
      zn = mapped_ptr(numneigh);
      zb = zn ? mapped_ptr(nbr) : nullptr;
      zd = zb ? mapped_ptr(disp) : nullptr;
    }
    pulled = zd != nullptr;
    set_lists(c, natoms_total, atom_lo, nlocal, stride, numneigh, nbr, disp, types, false,
              !pulled);
    if (pulled) {
      // pinned outputs too: the kernels write them beside the device copies
      // (forces by the gather, eatom / etotal by the energy epilogue, the
      // validation flags into h_err), so no read-back copy is issued
      if (c->nchunks == 1 && !c->ext_forces) {
        double* sf = forces ? static_cast<double*>(const_cast<void*>(mapped_ptr(forces))) : nullptr;
        double* se = (eatom && nlocal > 0)
                         ? static_cast<double*>(const_cast<void*>(mapped_ptr(eatom))) : nullptr;
        double* st = etotal ? static_cast<double*>(const_cast<void*>(mapped_ptr(etotal))) : nullptr;
        unsigned* sg = static_cast<unsigned*>(const_cast<void*>(mapped_ptr(c->h_err)));
        sunk = (!forces || sf) && (!(eatom && nlocal > 0) || se) && (!etotal || st) && sg;
        if (sunk) {
          c->sink_forces = sf;
          c->sink_eatom = se;
          c->sink_etotal = st;
          c->sink_flags = sg;
        }
      }
      try {
        if (sunk && c->T <= SNAP_CWIN_MAXT)
          run_pull_graph(c, static_cast<const int*>(zn), static_cast<const int*>(zb),
                         static_cast<const double*>(zd));
        else
          run_pull(c, static_cast<const int*>(zn), static_cast<const int*>(zb),
                   static_cast<const double*>(zd));
      } catch (...) {
        c->sink_forces = c->sink_eatom = c->sink_etotal = nullptr;
        c->sink_flags = nullptr;
        throw;
      }
      c->sink_forces = c->sink_eatom = c->sink_etotal = nullptr;
      c->sink_flags = nullptr;
      c->have_U = c->have_Y = c->have_dE = c->have_forces = true;
    }
  });
  if (rc != SNAPGPU_OK) return rc;
  if (!pulled) {
    const int rr = snapgpu_run(c);
    if (rr != SNAPGPU_OK) return rr;
  }
  if (sunk)
    return guarded(c, [&] {
      CK(cudaStreamSynchronize(c->stream));
      const unsigned f = *static_cast<volatile unsigned*>(c->h_err);
      if (f) {
        *c->h_err = 0u;
        CK(cudaMemsetAsync(c->d_err.p, 0, sizeof(unsigned), c->stream));
        CK(cudaStreamSynchronize(c->stream));
        c->have_lists = c->have_U = c->have_Y = c->have_dE = c->have_forces = false;
        throw InvalidArg{device_error_message(f)};
      }
    });
  return guarded(c, [&] {
    // one D2H of [forces | eatom | etotal | flags] into pinned staging, then
    // host copies
    const size_t nf = c->d_forces.n, ne = c->d_eatom.n, nout = nf + ne + 2;
    if (c->natoms_total <= 0)  // no gather launched: flags straight into their slot
      CK(cudaMemcpyAsync(c->d_out.p + nf + ne + 1, c->d_err.p, sizeof(unsigned),
                         cudaMemcpyDeviceToDevice, c->stream));
    if (c->h_out_n < nout) {
      if (c->h_out) cudaFreeHost(c->h_out);
      c->h_out = nullptr;
      c->h_out_n = 0;
      CK(cudaMallocHost(&c->h_out, nout * sizeof(double)));
      c->h_out_n = nout;
    }
    CK(cudaMemcpyAsync(c->h_out, c->d_out.p, nout * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream));
    if (c->ext_forces && forces)
      CK(cudaMemcpyAsync(forces, c->ext_forces, sizeof(double) * force_doubles(c),
                         cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (forces && !c->ext_forces) std::memcpy(forces, c->h_out, sizeof(double) * force_doubles(c));
    if (eatom && c->nlocal > 0) std::memcpy(eatom, c->h_out + nf, sizeof(double) * c->nlocal);
    if (etotal) *etotal = c->h_out[nf + ne];
    unsigned flags;
    std::memcpy(&flags, c->h_out + nf + ne + 1, sizeof(unsigned));
    if (flags) {
      const unsigned f = flags;
      CK(cudaMemsetAsync(c->d_err.p, 0, sizeof(unsigned), c->stream));
      CK(cudaStreamSynchronize(c->stream));
      c->have_lists = c->have_U = c->have_Y = c->have_dE = c->have_forces = false;
      throw InvalidArg{device_error_message(f)};
    }
  });
}

int snapgpu_synchronize(snapgpu_ctx* c) {
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] { CK(cudaStreamSynchronize(c->stream)); });
}

int snapgpu_get_forces(snapgpu_ctx* c, double* f) {
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    need(c->have_forces, "get_forces before scatter_forces");
    require(f != nullptr, "null output");
    CK(cudaMemcpyAsync(f, forces_ptr(c), sizeof(double) * force_doubles(c),
                       cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int snapgpu_get_energy(snapgpu_ctx* c, double* eatom, double* etotal) {
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    need(c->have_Y, "get_energy before compute_Y");
    if (eatom && c->nlocal > 0)
      CK(cudaMemcpyAsync(eatom, c->d_eatom.p, sizeof(double) * c->nlocal, cudaMemcpyDeviceToHost,
                         c->stream));
    if (etotal)
      CK(cudaMemcpyAsync(etotal, c->d_etotal.p, sizeof(double), cudaMemcpyDeviceToHost,
                         c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

// Readback of V / Y' converted to the reference's logical u-space half arrays.
static void read_tiles(snapgpu_ctx* c, const double* dev, std::vector<double>& host) {
  const int NH = c->maps.nhalf;
  host.resize((size_t)c->ntiles * 2 * NH * 32);
  CK(cudaMemcpyAsync(host.data(), dev, host.size() * sizeof(double), cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

int snapgpu_get_ulisttot(snapgpu_ctx* c, double* out) {
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    need(c->have_U, "get_ulisttot before compute_U");
    std::vector<double> h;
    read_tiles(c, c->d_V.p, h);
    const int NH = c->maps.nhalf;
    for (int a = 0; a < c->nlocal; ++a)
      for (int e = 0; e < NH; ++e) {
        const size_t base = (size_t)(a >> 5) * 2 * NH * 32 + (a & 31);
        const double inv = 1.0 / c->hf[e];
        out[((size_t)a * NH + e) * 2] = h[base + (size_t)e * 32] * inv;
        out[((size_t)a * NH + e) * 2 + 1] = h[base + (size_t)(NH + e) * 32] * inv;
      }
  });
}

int snapgpu_get_ylist(snapgpu_ctx* c, double* out) {
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    need(c->have_Y, "get_ylist before compute_Y");
    std::vector<double> h;
    read_tiles(c, c->d_Y.p, h);
    const IndexMaps& m = c->maps;
    const int NH = m.nhalf;
    for (int a = 0; a < c->nlocal; ++a) {
      const size_t base = (size_t)a * NH * 2;  // Y' atom-major, interleaved complex
      double* o = out + (size_t)a * NH * 2;
      for (int t = 0; t <= m.T; ++t)
        for (int mb = 0; 2 * mb <= t; ++mb)
          for (int ma = 0; ma <= t; ++ma) {
            const int e = m.half_off[t] + mb * (t + 1) + ma;
            if (c->ywgt[e] != 0.0) {
              const double s = c->hf[e] / c->ywgt[e];
              o[2 * e] = h[base + 2 * e] * s;
              o[2 * e + 1] = h[base + 2 * e + 1] * s;
            }
          }
      // middle-row elements ma > t/2 are never computed on the device; they
      // follow from the index-reversal symmetry (halfint_index.hpp:22-25)
      for (int t = 0; t <= m.T; t += 2) {
        const int mb = t / 2;
        for (int ma = t / 2 + 1; ma <= t; ++ma) {
          const int e = m.half_off[t] + mb * (t + 1) + ma;
          const int src = m.half_off[t] + mb * (t + 1) + (t - ma);
          const double sg = ((ma + mb) & 1) ? -1.0 : 1.0;
          o[2 * e] = sg * o[2 * src];
          o[2 * e + 1] = -sg * o[2 * src + 1];
        }
      }
    }
  });
}

int snapgpu_set_positions(snapgpu_ctx* c, int natoms, const double* pos, const double* box) {
  const Nvtx nvtx_range("snapgpu_set_positions");
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    NLArgs a = nl_setup(c, natoms, pos, box);
    nl_front(c, a, pos);
    CK(cudaMemsetAsync(a.maxcount, 0, sizeof(int), c->stream));
    const int wblk = (natoms + kNLWarps - 1) / kNLWarps;
    if (natoms > 0) {  // count pass (a.nbr == nullptr)
      k_nl_lists_warp<<<wblk, kNLWarps * 32, 0, c->stream>>>(a, c->d_err.p);
      CK(cudaGetLastError());
    }
    int mx = 0;
    CK(cudaMemcpyAsync(&mx, a.maxcount, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    require(mx <= 128, "set_positions: more than 128 neighbors within Rcut");
    // shapes/allocations of the context (nothing uploaded: the lists are built in place)
    set_lists(c, natoms, 0, natoms, mx, nullptr, nullptr, nullptr, nullptr, false, false);
    a.nbr = c->d_nbr.p;
    a.disp = c->d_disp.p;
    a.stride = mx;
    if (natoms > 0) {
      CK(cudaMemcpyAsync(c->d_numneigh.p, a.numneigh, sizeof(int) * natoms,
                         cudaMemcpyDeviceToDevice, c->stream));
      if (mx > 0) {
        CK(cudaMemsetAsync(c->d_nbr.p, 0, sizeof(int) * (size_t)natoms * mx, c->stream));
        CK(cudaMemsetAsync(c->d_disp.p, 0, sizeof(double) * (size_t)natoms * mx * 3, c->stream));
        a.maxcount = nullptr;
        k_nl_lists_warp<<<wblk, kNLWarps * 32, 0, c->stream>>>(a, c->d_err.p);
        CK(cudaGetLastError());
        launch_partner(c);
      }
    }
    // device-built lists are symmetric and sorted: the force gather takes the
    // partner slots instead of a reverse-neighbor CSR
    c->sym_lists = true;
    c->csr_dirty = false;
    // the positions graphs embed the box (cells, minimum image)
    if (box[0] != c->nl_box[0] || box[1] != c->nl_box[1] || box[2] != c->nl_box[2])
      invalidate_pos_graph(c);
    for (int d = 0; d < 3; ++d) c->nl_box[d] = box[d];
  });
}

int snapgpu_run_positions(snapgpu_ctx* c, int natoms, const double* pos, const double* box,
                          double* forces, double* eatom, double* etotal) {
  const Nvtx nvtx_range("snapgpu_run_positions");
  if (!c) return SNAPGPU_EINVAL;
  bool fast = c->have_lists && c->sym_lists && natoms == c->natoms_total &&
              natoms == c->nlocal && c->atom_lo == 0 && c->nchunks == 1 && !c->timing &&
              box != nullptr && pos != nullptr;
  if (fast)
    for (int d = 0; d < 3; ++d) fast = fast && box[d] == c->nl_box[d];
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (!fast) {  // (re)establish stride, cells and shapes: lists with a host sync
      const int rc = snapgpu_set_positions(c, natoms, pos, box);
      if (rc != SNAPGPU_OK) return rc;
    }
    bool overflow = false, done = false;
    // pinned positions and outputs (2J <= 8): the copy-free graph
    const int rp = guarded(c, [&] {
      require(natoms > 0, "run_positions: no atoms");
      if (c->T > SNAP_CWIN_MAXT || c->nchunks != 1 || c->ext_forces) return;
      const double* mp = static_cast<const double*>(mapped_ptr(pos));
      double* sf = forces ? static_cast<double*>(const_cast<void*>(mapped_ptr(forces))) : nullptr;
      double* se = eatom ? static_cast<double*>(const_cast<void*>(mapped_ptr(eatom))) : nullptr;
      double* st = etotal ? static_cast<double*>(const_cast<void*>(mapped_ptr(etotal))) : nullptr;
      unsigned* sg = static_cast<unsigned*>(const_cast<void*>(mapped_ptr(c->h_err)));
      if (!mp || !sg || (forces && !sf) || (eatom && !se) || (etotal && !st)) return;
      c->sink_forces = sf;
      c->sink_eatom = se;
      c->sink_etotal = st;
      c->sink_flags = sg;
      try {
        run_positions_pull(c, natoms, mp);
      } catch (...) {
        c->sink_forces = c->sink_eatom = c->sink_etotal = nullptr;
        c->sink_flags = nullptr;
        throw;
      }
      c->sink_forces = c->sink_eatom = c->sink_etotal = nullptr;
      c->sink_flags = nullptr;
      CK(cudaStreamSynchronize(c->stream));
      c->have_U = c->have_Y = c->have_dE = c->have_forces = true;
      const unsigned f = *static_cast<volatile unsigned*>(c->h_err);
      done = true;
      if (f) {
        *c->h_err = 0u;
        CK(cudaMemsetAsync(c->d_err.p, 0, sizeof(unsigned), c->stream));
        CK(cudaStreamSynchronize(c->stream));
        c->have_U = c->have_Y = c->have_dE = c->have_forces = false;
        if ((f & kErrCount) && attempt == 0) {  // a list outgrew the stride: rebuild
          overflow = true;
          return;
        }
        c->have_lists = false;
        throw InvalidArg{device_error_message(f)};
      }
    });
    if (rp != SNAPGPU_OK) return rp;
    if (done && !overflow) return SNAPGPU_OK;
    if (overflow) {
      fast = false;
      continue;
    }
    const int rc = guarded(c, [&] {
      require(natoms > 0, "run_positions: no atoms");
      const size_t nf = c->d_forces.n, ne = c->d_eatom.n, nout = nf + ne + 2;
      if (c->h_out_n < nout) {
        if (c->h_out) cudaFreeHost(c->h_out);
        c->h_out = nullptr;
        c->h_out_n = 0;
        CK(cudaMallocHost(&c->h_out, nout * sizeof(double)));
        c->h_out_n = nout;
        invalidate_pos_graph(c);
      }
      if (c->h_pos_n < (size_t)natoms * 3) {
        if (c->h_pos) cudaFreeHost(c->h_pos);
        c->h_pos = nullptr;
        c->h_pos_n = 0;
        CK(cudaMallocHost(&c->h_pos, sizeof(double) * 3 * natoms));
        c->h_pos_n = (size_t)natoms * 3;
        invalidate_pos_graph(c);
      }
      std::memcpy(c->h_pos, pos, sizeof(double) * 3 * natoms);
      if (!c->pos_gexec) {  // one graph: H2D, lists, partners, U, Y, dE, gather, D2H
        cudaStream_t user = c->stream;
        c->stream = c->own_stream;
        CK(cudaStreamSynchronize(user));
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        try {
          NLArgs a = nl_setup(c, natoms, c->h_pos, c->nl_box);
          nl_front(c, a, c->h_pos);
          a.numneigh = c->d_numneigh.p;
          a.nbr = c->d_nbr.p;
          a.disp = c->d_disp.p;
          a.stride = c->stride;
          a.maxcount = nullptr;
          k_nl_lists_warp<<<(natoms + kNLWarps - 1) / kNLWarps, kNLWarps * 32, 0, c->stream>>>(
              a, c->d_err.p);
          CK(cudaGetLastError());
          launch_partner(c);
          run_direct(c);
          CK(cudaMemcpyAsync(c->h_out, c->d_out.p, nout * sizeof(double), cudaMemcpyDeviceToHost,
                             c->stream));
        } catch (...) {
          cudaGraph_t g;
          cudaStreamEndCapture(c->stream, &g);
          if (g) cudaGraphDestroy(g);
          c->stream = user;
          throw;
        }
        CK(cudaStreamEndCapture(c->stream, &c->pos_graph));
        CK(cudaGraphInstantiate(&c->pos_gexec, c->pos_graph, 0));
        c->stream = user;
      }
      CK(cudaGraphLaunch(c->pos_gexec, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      c->have_U = c->have_Y = c->have_dE = c->have_forces = true;
      unsigned flags;
      std::memcpy(&flags, c->h_out + nf + ne + 1, sizeof(unsigned));
      if (flags) {
        const unsigned f = flags;
        CK(cudaMemsetAsync(c->d_err.p, 0, sizeof(unsigned), c->stream));
        CK(cudaStreamSynchronize(c->stream));
        c->have_U = c->have_Y = c->have_dE = c->have_forces = false;
        if ((f & kErrCount) && attempt == 0) {  // a list outgrew the stride: rebuild
          overflow = true;
          return;
        }
        c->have_lists = false;
        throw InvalidArg{device_error_message(f)};
      }
      if (forces) std::memcpy(forces, c->h_out, sizeof(double) * force_doubles(c));
      if (eatom) std::memcpy(eatom, c->h_out + nf, sizeof(double) * c->nlocal);
      if (etotal) *etotal = c->h_out[nf + ne];
    });
    if (rc != SNAPGPU_OK) return rc;
    if (!overflow) return SNAPGPU_OK;
    fast = false;
  }
  return SNAPGPU_OK;
}

int snapgpu_get_neighbors(snapgpu_ctx* c, int* numneigh, int* nbr, double* disp) {
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    need(c->have_lists, "get_neighbors: no neighbor lists");
    const size_t n = (size_t)c->nlocal, ns = n * c->stride;
    if (numneigh && n)
      CK(cudaMemcpyAsync(numneigh, c->d_numneigh.p, sizeof(int) * n, cudaMemcpyDeviceToHost,
                         c->stream));
    if (nbr && ns)
      CK(cudaMemcpyAsync(nbr, c->d_nbr.p, sizeof(int) * ns, cudaMemcpyDeviceToHost, c->stream));
    if (disp && ns)
      CK(cudaMemcpyAsync(disp, c->d_disp.p, sizeof(double) * ns * 3, cudaMemcpyDeviceToHost,
                         c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int snapgpu_get_virial(snapgpu_ctx* c, double* out6) {
  if (!c || !out6) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    need(c->have_dE, "get_virial before the force pass");
    constexpr int kBlk = 148;
    c->d_virial.alloc(kBlk * 6 + 6);
    VirialArgs a;
    a.numneigh = c->d_numneigh.p;
    a.disp = c->d_disp.p;
    a.dedr = c->d_dedr.p;
    a.nlocal = c->nlocal;
    a.stride = c->stride;
    a.part = c->d_virial.p;
    a.out = c->d_virial.p + kBlk * 6;
    k_virial_partial<<<kBlk, 256, 0, c->stream>>>(a);
    CK(cudaGetLastError());
    k_virial_final<<<1, 32, 0, c->stream>>>(a.part, kBlk, a.out);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out6, a.out, 6 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int snapgpu_get_dedr(snapgpu_ctx* c, double* out) {
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    need(c->have_dE, "get_dedr before the force pass");
    const size_t n = (size_t)c->nlocal * c->stride * 3;
    std::vector<double> h(n);
    std::vector<int> nnh(c->nlocal);
    if (n) {
      CK(cudaMemcpyAsync(h.data(), c->d_dedr.p, n * sizeof(double), cudaMemcpyDeviceToHost,
                         c->stream));
      CK(cudaMemcpyAsync(nnh.data(), c->d_numneigh.p, sizeof(int) * c->nlocal,
                         cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
    }
    // zero the unused (padding) slots like the reference's zero-filled dElist
    for (int i = 0; i < c->nlocal; ++i) {
      const int nn = nnh[i];
      for (int k = 0; k < c->stride; ++k)
        for (int d = 0; d < 3; ++d) {
          const size_t s = ((size_t)i * c->stride + k) * 3 + d;
          out[s] = k < nn ? h[s] : 0.0;
        }
    }
  });
}

int snapgpu_get_forces_device(snapgpu_ctx* c, double* dst) {
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    need(c->have_forces, "get_forces_device before scatter_forces");
    require(dst != nullptr, "null output");
    CK(cudaMemcpyAsync(dst, forces_ptr(c), sizeof(double) * force_doubles(c),
                       cudaMemcpyDeviceToDevice, c->stream));
  });
}

int snapgpu_get_energy_device(snapgpu_ctx* c, double* eatom, double* etotal) {
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    need(c->have_Y, "get_energy_device before compute_Y");
    if (eatom && c->nlocal > 0)
      CK(cudaMemcpyAsync(eatom, c->d_eatom.p, sizeof(double) * c->nlocal,
                         cudaMemcpyDeviceToDevice, c->stream));
    if (etotal)
      CK(cudaMemcpyAsync(etotal, c->d_etotal.p, sizeof(double), cudaMemcpyDeviceToDevice,
                         c->stream));
  });
}

int snapgpu_fp64_peak(int device, int iters, double* tflops, double* ms) {
  return guarded(nullptr, [&] {
    CK(cudaSetDevice(device));
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    double* d = nullptr;
    CK(cudaMalloc(&d, sizeof(double)));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int blocks = nsm * 8, threads = 256;
    k_fp64_peak<<<blocks, threads>>>(d, 1000, 1.0);  // warm-up
    CK(cudaEventRecord(e0));
    k_fp64_peak<<<blocks, threads>>>(d, iters, 1.0);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, e0, e1));
    const double flops = 2.0 * 8.0 * (double)iters * blocks * threads;
    if (tflops) *tflops = flops / (t * 1e-3) / 1e12;
    if (ms) *ms = t;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
  });
}

int snapgpu_device_outputs(snapgpu_ctx* c, double** forces, double** eatom, double** etotal) {
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    if (forces) *forces = forces_ptr(c);
    if (eatom) *eatom = c->d_eatom.p;
    if (etotal) *etotal = c->d_etotal.p;
  });
}

int snapgpu_enable_stage_timing(snapgpu_ctx* c, int on) {
  if (!c) return SNAPGPU_EINVAL;
  c->timing = on != 0;
  return SNAPGPU_OK;
}

int snapgpu_stage_times(snapgpu_ctx* c, float* out4) {
  if (!c) return SNAPGPU_EINVAL;
  for (int s = 0; s < 4; ++s) out4[s] = c->stage_ms[s];
  return SNAPGPU_OK;
}

int snapgpu_tune(snapgpu_ctx* c, int y_parts) {
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    require(y_parts >= 0 && y_parts <= kMaxYParts, "tune: y_parts must be in [0, 8]");
    c->y_parts = y_parts;
    invalidate_graph(c);
    invalidate_pos_graph(c);
    if (c->have_lists) plan_y(c);
  });
}

int snapgpu_set_overlap(snapgpu_ctx* c, int on) {
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    CK(cudaStreamSynchronize(c->stream));
    c->y_overlap = on != 0;
    invalidate_graph(c);
    invalidate_pos_graph(c);
  });
}

int snapgpu_set_force_layout(snapgpu_ctx* c, int nchunks, double* ext_forces) {
  if (!c) return SNAPGPU_EINVAL;
  return guarded(c, [&] {
    require(nchunks >= 1 && nchunks <= 256, "set_force_layout: nchunks must be in [1, 256]");
    CK(cudaStreamSynchronize(c->stream));
    c->nchunks = nchunks;
    c->ext_forces = ext_forces;
    invalidate_graph(c);
    // re-shape the output buffers on the next list upload
    c->natoms_total = -1;
    c->have_lists = c->have_U = c->have_Y = c->have_dE = c->have_forces = false;
  });
}

int snapgpu_build_neighborlist(const double* pos, int n, const double box[3], double rcut,
                               int maxstride, int* numneigh, int* nbr, double* disp) {
  int mx = -1;
  const int rc = guarded(nullptr, [&] {
    require(n >= 0 && (n == 0 || pos) && box, "build_neighborlist: null input");
    std::string err;
    mx = build_neighborlist(pos, n, box, rcut, maxstride, numneigh, nbr, disp, &err);
    if (mx < 0) throw InvalidArg{err};
  });
  return rc == SNAPGPU_OK ? mx : -rc;
}

int snapgpu_bcc_lattice(int nx, int ny, int nz, double a, double jitter, uint64_t seed,
                        int twojmax, double* pos, double* beta) {
  int n = -1;
  const int rc = guarded(nullptr, [&] {
    require(nx > 0 && ny > 0 && nz > 0 && a > 0.0 && pos && beta, "bcc_lattice: bad arguments");
    n = bcc_lattice(nx, ny, nz, a, jitter, seed, twojmax, pos, beta);
  });
  return rc == SNAPGPU_OK ? n : -rc;
}

}  // extern "C"
