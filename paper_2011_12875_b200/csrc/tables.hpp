// tables.hpp -- host-side setup for the B200 SNAP engine.
//
// Everything here runs once per context (or once per neighbor-list upload)
// on the host: the integer index bookkeeping of the reference
// (halfint_index.hpp), the Clebsch-Gordan table (angular_basis.hpp:151-196),
// the beta multiplicity fold (snap_core.hpp:308-322), and the tables that
// are specific to this engine's "v-space" formulation:
//
//   v(t,mb,ma) = f(t,mb,ma) u(t,mb,ma),  f = g(t,mb) h(t,ma),
//   g(t,mb) = sqrt((t-mb)!),  h(t,ma) = 1/sqrt((t-ma)! ma!),
//
// under which the Wigner level recursion (angular_basis.hpp:232-257) loses
// its sqrt(p/q) weights:  v(t,mb,ma) = conj(a) v(t-1,mb,ma)
//                                       - conj(b) v(t-1,mb,ma-1).
// The per-element scale factors are folded into the coupling tables (C')
// and the beta-weighted row tables (W) consumed by the compute_Y kernel.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

namespace snapgpu {

struct Tuple {
  int j1, j2, j, elem_off, cg_off;
};

// HalfIntIndexMaps (halfint_index.hpp:64-128), same enumeration order.
struct IndexMaps {
  int T = 0;
  int nhalf = 0, nfull = 0, cgtot = 0, zelems = 0;
  std::vector<int> half_off, full_off;           // T+2 entries
  std::vector<std::array<int, 3>> triples;       // canonical (j1, j2, j)
  std::vector<Tuple> tuples;                     // all coupling tuples
  std::vector<int> triple_flat, tuple_flat, cg_flat;  // dense (T+1)^3 lookups

  static IndexMaps build(int T);
  int dense(int a, int b, int c) const { return (a * (T + 1) + b) * (T + 1) + c; }
  int triple_index(int a, int b, int c) const { return triple_flat[dense(a, b, c)]; }
};

double factorial(int n);
std::vector<double> cg_table(const IndexMaps& m);  // angular_basis.hpp:151-196
double fold_beta(const IndexMaps& m, const double* beta, int j1, int j2, int j);

// v-space scale factors.
double g_scale(int t, int mb);   // sqrt((t-mb)!)
double h_scale(int t, int ma);   // 1/sqrt((t-ma)! ma!)
double f_scale(int t, int mb, int ma);  // g*h

// C'(tuple; ma1, ma2) = cg / (h(j1,ma1) h(j2,ma2) h(j, ma1+ma2-D)); same layout
// as the CG table (cg_offset + ma1*(j2+1) + ma2).
std::vector<double> cprime_table(const IndexMaps& m, const std::vector<double>& cg);
// W(tuple; mb1, mb2) = fold_beta * cg / (G(j1,mb1) G(j2,mb2) g(j, mb)),
// G(t,m) = g(t, min(m, t-m)); zero where the target row is not stored.
// With mirror_signs, the (-1)^mb factor of mirrored factor rows is folded in
// (the kernel then applies only (-1)^ma and the conjugation).
std::vector<double> w_table(const IndexMaps& m, const std::vector<double>& cg,
                            const double* beta, bool mirror_signs);

// Per-half-index scale 1/f (u = v/f) and f, in half index order.
std::vector<double> half_f(const IndexMaps& m);
// Weight of a stored Y' element: 1 on strict rows, on the middle row of even
// levels 1 (ma < t/2), 0.5 (ma == t/2), 0 (ma > t/2).
std::vector<double> half_ywgt(const IndexMaps& m);

// Full-index expansion map for the Y kernel: for full index (t,mb,ma),
// src half index and sign (+1, or -1 with conj when mirrored).  Encoded
// as src*4 + (mirrored?2:0) + (negative?1:0).
std::vector<int> half_scatter_map(const IndexMaps& m);


// compute_Y row-pair items (sliding-window kernel, kernels.cuh k_compute_Y).
// Target rows (j, mb <= j/2) are numbered rid = sum_{s<j}(s/2+1) + mb; row
// rid owns items [row_begin[rid], row_begin[rid+1]), one per contributing
// (tuple, mb1).  Item: x = half-storage start of factor row mb1 of level j1
// (or of its mirror source), y = same for row mb2 of level j2, z = packed
// j1 | j2<<8 | D<<16 | mirrored1<<24 | mirrored2<<25 | (j+1)<<26, w = offset
// of the tuple's windowed coefficient block.  itw = W' (beta-dependent).
struct YPlan {
  std::vector<std::array<int, 4>> items;
  std::vector<int> row_begin;
  std::vector<double> cw;       // windowed C': per tuple (j2+1) x (j+1)
  std::vector<double> row_cost; // per row (FP64 instructions, for scheduling)
};
YPlan y_plan(const IndexMaps& m, const std::vector<double>& cprime);
std::vector<double> y_item_weights(const IndexMaps& m, const std::vector<double>& wtab);
// Unrolled cooperative compute_Y (2J <= 8): per target row, the row-pair
// items {tuple q, mb1, mb2} are LPT-split over `warps` warps; items of row
// rid, warp w live in [rw_begin[rid*(warps+1)+w], rw_begin[rid*(warps+1)+w+1]).
struct YCoopPlan {
  int warps = 0;
  std::vector<std::array<int, 4>> items;
  std::vector<int> rw_begin;
  std::vector<double> row_cost;
  // paired plan only: units {first item, item count 1|2}; the two items of a
  // pair share (tuple, target row), so they share every C' coefficient.
  // rw_begin then holds 2*warps+1 bounds per row: [pairs of warp 0, singles
  // of warp 0, pairs of warp 1, ...].
  std::vector<std::array<int, 2>> units;
};
YCoopPlan ycoop_plan(const IndexMaps& m, int warps, bool lpt_split);
YCoopPlan ycoop_pair_plan(const IndexMaps& m, int warps);
std::vector<double> ycoop_weights(const YCoopPlan& p, const IndexMaps& m,
                                  const std::vector<double>& wtab);
// Quad units for the 2J > 8 compute_Y (kernels.cuh k_compute_Y_quad): per
// target row, up to 4 consecutive mb1 items of one tuple form a unit (they
// share every C' coefficient); units are LPT-split over `warps` warps.
// unit = {x1_0 | x2_0 << 16, J2 | J1 << 8 | count << 16, C' offset, item0};
// items = {tuple, mb1, mb2} (W order); rw = [row][warps + 1] unit ranges.
struct YQuadPlan {
  std::vector<std::array<int, 4>> units;
  std::vector<std::array<int, 3>> items;
  std::vector<int> rw;
  std::vector<int> rows;  // [group][rows_cap] row codes j*64+mb, -1 terminated
  int rows_cap = 0;
};
YQuadPlan yquad_plan(const IndexMaps& m, int warps, int groups);
// y_plan's windowed C' with every row padded to even length (the quad
// kernel loads coefficient pairs)
std::vector<double> yquad_cw(const IndexMaps& m, const std::vector<double>& cw);
std::vector<double> yquad_weights(const YQuadPlan& p, const IndexMaps& m,
                                  const std::vector<double>& wtab);

// Direct bispectrum components B_l (compute_B_from_U, snap_core.hpp:642-681;
// kernels.cuh k_compute_B).  Per canonical triple l = tuple (j1, j2, j):
// items {x1 window base (full idx + D), x2 row base (full idx), (j, mb) row
// base (full idx), j2 | j << 8}, the C' block offset (y_plan windowed
// layout) and the weight w' W_B(mb1, mb2), with W_B the beta-free W table
// (w_table with every folded beta = 1) and w' = 2 on strict rows, 1 on the
// middle row (b_contract, snap_core.hpp:556-575: the middle row runs over all
// ma).  triple_begin[l] .. [l+1]: the triple's items.
struct BPlan {
  std::vector<std::array<int, 4>> items;
  std::vector<int> cwoff;
  std::vector<double> wgt;
  std::vector<int> triple_begin;
};
BPlan b_plan(const IndexMaps& m, const std::vector<double>& cg);

// LPT assignment of rows to workers: [worker][cap] row codes j*64+mb, -1 end.
std::vector<int> y_row_schedule(const IndexMaps& m, const std::vector<double>& row_cost,
                                int workers, int* cap);

// compute_Y (2J <= 8) launch plan: the part count of every 32-atom tile, the
// per-(parts, part, group) row lists and the CTA table {tile, part | parts <<
// 8, first row list, list stride} in part-major order (snapgpu.cu plan_y).
struct YCtaPlan {
  std::vector<int> tasks;
  std::vector<std::array<int, 4>> cta;
  int pmax = 1;
};
YCtaPlan y_cta_plan(const IndexMaps& m, const std::vector<double>& row_cost, int ntiles,
                    int nsm, int forced_parts, int max_parts, int groups);

// Reference-order neighbor list builder (harness.hpp:119-202, orthorhombic).
// Returns max neighbor count or -1 (err set).
int build_neighborlist(const double* pos, int n, const double box[3], double rcut,
                       int maxstride, int* numneigh, int* nbr, double* disp,
                       std::string* err);

int bcc_lattice(int nx, int ny, int nz, double a, double jitter, std::uint64_t seed,
                int T, double* pos, double* beta);

}  // namespace snapgpu
