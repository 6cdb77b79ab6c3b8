// launch_t.cu -- kernel launches for ONE band limit 2J = SNAP_T.
//
// Compiled once per 2J (Makefile: -DSNAP_T=0..14) so the sm_100a kernels of
// the different band limits build in parallel; snapgpu.cu dispatches on the
// context's twojmax to the instantiations below.
#include "ctx.hpp"

#ifndef SNAP_U2_PP
#define SNAP_U2_PP 1  // pairs per lane per compute_U pass
#endif

#ifndef SNAP_T
#error "compile with -DSNAP_T=<twojmax>"
#endif

namespace snapgpu {
namespace host {

// compute_Y's read-only tables, prefetched into L2 by compute_U
template <int T>
static L2Prefetch y_prefetch(snapgpu_ctx* c) {
  L2Prefetch P{};
#if SNAP_T <= SNAP_CWIN_MAXT
  {
    void* rw = nullptr;
    CK(cudaGetSymbolAddress(&rw, cYRowW));
    const void* a[3] = {c->d_yunits.p, c->d_cwp.p, rw};
    const int b[3] = {(int)(c->ycplan.units.size() * sizeof(YUnit)),
                      (int)(c_cwp_total(T) * sizeof(double)),
                      (int)(c->ycplan.rw_begin.size() * sizeof(int))};
    for (int r = 0; r < 3; ++r) {
      P.p[r] = static_cast<const char*>(a[r]);
      P.bytes[r] = a[r] ? b[r] : 0;
    }
  }
#else
  (void)c;
#endif
  return P;
}

template <int T, int SL, int PP = SNAP_U2_PP>
static void launch_U2(snapgpu_ctx* c) {
  using C2 = U2Cfg<T, SL>;
  UArgs a;
  a.pr = pair_args(c);
  a.gp = c->gp;
  a.V = c->d_V.p;
  a.pf = y_prefetch<T>(c);
  a.src_numneigh = c->zc_numneigh;
  a.src_nbr = c->zc_nbr;
  a.src_disp = c->zc_disp;
  const size_t smem = sizeof(double) * (size_t)C2::WARPS * C2::APW * c->stride * 5;
  CK(cudaFuncSetAttribute(k_compute_U2<T, SL, PP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)std::max<size_t>(smem, 48 * 1024)));
  const int per_block = C2::WARPS * C2::APW;
  const int blocks = (c->nlocal + per_block - 1) / per_block;
  k_compute_U2<T, SL, PP><<<blocks, C2::WARPS * 32, smem, c->stream>>>(a);
  CK(cudaGetLastError());
}

template <int T>
void launch_U_t(snapgpu_ctx* c) {
  if constexpr (T <= 8) {  // row-lane kernel
    // two pair slots per atom when the atoms fill the SMs, else four
    // (measured at 2000 atoms: 2 / 4 / 8 slots -> 28.7 / 26.4 / 31.6 us)
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
    if (c->nlocal / U2Cfg<T, 2>::APW >= 8 * nsm) return launch_U2<T, 2>(c);
    return launch_U2<T, 4>(c);
  } else {  // column-lane kernel
    using C = UCfg<T>;
    UArgs a;
    a.pr = pair_args(c);
    a.gp = c->gp;
    a.V = c->d_V.p;
    a.pf = L2Prefetch{};
    a.src_numneigh = a.src_nbr = nullptr;  // (the one-call pull is T <= 8 only)
    a.src_disp = nullptr;
    const size_t smem = sizeof(double) * ((size_t)C::WARPS * c->stride * 5 +
                                          (C::REGACC ? 0 : (size_t)C::WARPS * 2 * C::NACC * 32));
    CK(cudaFuncSetAttribute(k_compute_U<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)std::max<size_t>(smem, 48 * 1024)));
    const int blocks = (c->nlocal + C::WARPS - 1) / C::WARPS;
    k_compute_U<T><<<blocks, C::WARPS * 32, smem, c->stream>>>(a);
    CK(cudaGetLastError());
  }
}

template <int T>
void launch_Y_t(snapgpu_ctx* c) {
#if SNAP_T <= SNAP_CWIN_MAXT
  constexpr int NF = c_full_off(T + 1);
  constexpr int NP = NF + 2 * kXPad;
  YWArgs a;
  a.V = c->d_V.p;
  a.Y = c->d_Y.p;
  a.expand = c->d_expand.p;
  a.units = reinterpret_cast<const YUnit*>(c->d_yunits.p);
  a.cw = c->d_cwp.p;
  a.prof = nullptr;
#ifdef SNAP_Y_PROFILE
  if (!g_yprof) {
    CK(cudaMalloc(&g_yprof, 2112 * sizeof(long long)));
    CK(cudaMemset(g_yprof, 0, 2112 * sizeof(long long)));
  }
  a.prof = g_yprof;
#endif
  a.tasks = c->d_tasks.p;
  a.cta = c->d_ycta.p;
  a.ntiles = c->ntiles;
  a.early = c->overlap_now() ? 1 : 0;
  a.nlocal = c->nlocal;
  a.E = energy_out(c);
  a.E.ready = c->d_ready.p;  // the per-tile hand-off to compute_fused_dE
  const size_t smem = sizeof(double) * (2 * NP * 32 + (size_t)kYRedSlots * (T + 1) * 2 * 32 +
                                        (size_t)c_cwp_total(T));
  dim3 grid(c->y_ctas);
  CK(cudaFuncSetAttribute(k_compute_Y_cwin<T, kYGroups>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  launch_pdl(k_compute_Y_cwin<T, kYGroups>, grid, dim3(kYWarps * 32), smem, c->stream, a);
  CK(cudaGetLastError());
#else
  constexpr int NF = c_full_off(T + 1);
  constexpr int NP = NF + 2 * kQPad;
  YQArgs a;
  a.V = c->d_V.p;
  a.Y = c->d_Y.p;
  a.expand = c->d_expand.p;
  a.units = c->d_qunits.p;
  a.itw = c->d_qitw.p;
  a.rw = c->d_qrw.p;
  a.cw = c->d_cwq.p;
  a.rows = c->d_qrows.p;
  a.rows_cap = c->yqplan.rows_cap;
  a.nlocal = c->nlocal;
  a.E = energy_out(c);
  const size_t smem = sizeof(double) * (2 * NP * 8 + (size_t)kQWarps * (T + 1) * 2 * 8);
  CK(cudaFuncSetAttribute(k_compute_Y_quad<T, kQGroups>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  launch_pdl(k_compute_Y_quad<T, kQGroups>, dim3(c->ntiles * 4), dim3(kQWarps * 32), smem,
             c->stream, a);
  CK(cudaGetLastError());
#endif
}

template <int T>
void launch_B_t(snapgpu_ctx* c, double* blist) {
  constexpr int TA = T <= 8 ? 32 : 8;
  constexpr int NP = c_full_off(T + 1) + 2 * 16;
  BArgs a;
  a.V = c->d_V.p;
  a.expand = c->d_expand.p;
  a.items = c->d_bitems.p;
  a.cwoff = c->d_bcwoff.p;
  a.wgt = c->d_bwgt.p;
  a.tbeg = c->d_btbeg.p;
  a.cw = c->d_cw.p;
  a.ntriples = static_cast<int>(c->maps.triples.size());
  a.nlocal = c->nlocal;
  a.blist = blist;
  const size_t smem = sizeof(double) * 2 * NP * TA;
  CK(cudaFuncSetAttribute(k_compute_B<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  k_compute_B<T><<<(c->nlocal + TA - 1) / TA, 384, smem, c->stream>>>(a);
  CK(cudaGetLastError());
}

template <int T>
void launch_DE_t(snapgpu_ctx* c) {
  using R = DERCfg<T>;
  DEArgs a;
  a.pr = pair_args(c);
  a.gp = c->gp;
  a.Y = c->d_Y.p;
  a.dedr = c->d_dedr.p;
  a.nslots = c->nlocal * c->stride;
  // 2J <= 8: wait per tile on compute_Y's flags instead of for its whole grid
  a.ready = (T <= SNAP_CWIN_MAXT && c->overlap_now()) ? c->d_ready.p : nullptr;
  const int per_block = R::WARPS * R::PPW;
  const int blocks = (a.nslots + per_block - 1) / per_block;
  if (blocks > 0) {
    CK(cudaFuncSetAttribute(k_fused_dE_rev<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            R::SMEM));
    launch_pdl(k_fused_dE_rev<T>, dim3(blocks), dim3(R::WARPS * 32), (size_t)R::SMEM, c->stream, a);
    CK(cudaGetLastError());
  }
}

// The beta-independent [row][warp] unit ranges of the constant-window
// compute_Y live in this object's constant bank (kernels.cuh), uploaded once
// per device.
template <int T>
void upload_ytables_t(int device, const YTablesHost& t) {
#if SNAP_T <= SNAP_CWIN_MAXT
  {
    static std::mutex mu;
    static std::vector<int> done;
    std::lock_guard<std::mutex> lk(mu);
    for (int d : done)
      if (d == device) return;
    require(t.rw.size() == (size_t)c_acc_off(T + 1) * (2 * kYGroupWarps + 1),
            "compute_Y: row/warp table size mismatch");
    CK(cudaMemcpyToSymbol(cYRowW, t.rw.data(), t.rw.size() * sizeof(int)));
    done.push_back(device);
  }
#else
  (void)device;
  (void)t;
#endif
}

template void launch_U_t<SNAP_T>(snapgpu_ctx*);
template void launch_Y_t<SNAP_T>(snapgpu_ctx*);
template void launch_DE_t<SNAP_T>(snapgpu_ctx*);
template void launch_B_t<SNAP_T>(snapgpu_ctx*, double*);
template void upload_ytables_t<SNAP_T>(int, const YTablesHost&);

}  // namespace host
}  // namespace snapgpu
