// tables.cpp -- host-side setup for the B200 SNAP engine (see tables.hpp).
//
// Reference citations are relative to /root/reference/proj/include/snapforge/.
#include "tables.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <queue>
#include <random>

namespace snapgpu {

namespace {
int full_block(int t) { return (t + 1) * (t + 1); }
int half_block(int t) { return (t / 2 + 1) * (t + 1); }
}  // namespace

// HalfIntIndexMaps::build (halfint_index.hpp:155-200); triples and tuples are
// enumerated in the same lexicographic order (:132-141, :184-198).
IndexMaps IndexMaps::build(int T) {
  IndexMaps m;
  m.T = T;
  m.half_off.assign(T + 2, 0);
  m.full_off.assign(T + 2, 0);
  for (int t = 0; t <= T; ++t) {
    m.full_off[t + 1] = m.full_off[t] + full_block(t);
    m.half_off[t + 1] = m.half_off[t] + half_block(t);
  }
  m.nhalf = m.half_off[T + 1];
  m.nfull = m.full_off[T + 1];
  const int nd = (T + 1) * (T + 1) * (T + 1);
  m.triple_flat.assign(nd, -1);
  m.tuple_flat.assign(nd, -1);
  m.cg_flat.assign(nd, -1);
  int elem = 0, cgo = 0;
  for (int j1 = 0; j1 <= T; ++j1)
    for (int j2 = 0; j2 <= j1; ++j2)
      for (int j = j1 - j2; j <= std::min(j1 + j2, T); j += 2) {
        if (j >= j1) {
          m.triple_flat[m.dense(j1, j2, j)] = static_cast<int>(m.triples.size());
          m.triples.push_back({j1, j2, j});
        }
        m.tuple_flat[m.dense(j1, j2, j)] = static_cast<int>(m.tuples.size());
        m.cg_flat[m.dense(j1, j2, j)] = cgo;
        m.tuples.push_back({j1, j2, j, elem, cgo});
        elem += half_block(j);
        cgo += (j1 + 1) * (j2 + 1);
      }
  m.zelems = elem;
  m.cgtot = cgo;
  return m;
}

double factorial(int n) {  // angular_basis.hpp:38-47
  static const std::array<double, 65> table = [] {
    std::array<double, 65> t{};
    t[0] = 1.0;
    for (int i = 1; i <= 64; ++i) t[i] = t[i - 1] * i;
    return t;
  }();
  return table[n];
}

static double deltacg(int j1, int j2, int j) {  // angular_basis.hpp:66-70
  const double sfaccg = factorial((j1 + j2 + j) / 2 + 1);
  return std::sqrt(factorial((j1 + j2 - j) / 2) * factorial((j1 - j2 + j) / 2) *
                   factorial((-j1 + j2 + j) / 2) / sfaccg);
}

// Racah closed form, identical arithmetic to compute_cg_table
// (angular_basis.hpp:151-196) so the table is bitwise equal.
std::vector<double> cg_table(const IndexMaps& m) {
  std::vector<double> cg(m.cgtot, 0.0);
  for (const Tuple& tp : m.tuples) {
    const int j1 = tp.j1, j2 = tp.j2, j = tp.j;
    int idx = tp.cg_off;
    for (int m1 = 0; m1 <= j1; ++m1) {
      const int aa2 = 2 * m1 - j1;
      for (int m2 = 0; m2 <= j2; ++m2, ++idx) {
        const int bb2 = 2 * m2 - j2;
        const int mm = (aa2 + bb2 + j) / 2;
        if (mm < 0 || mm > j) continue;
        double sum = 0.0;
        const int zlo = std::max(0, std::max(-(j - j2 + aa2) / 2, -(j - j1 - bb2) / 2));
        const int zhi = std::min((j1 + j2 - j) / 2, std::min((j1 - aa2) / 2, (j2 + bb2) / 2));
        for (int zz = zlo; zz <= zhi; ++zz) {
          const double ifac = (zz % 2) ? -1.0 : 1.0;
          sum += ifac / (factorial(zz) * factorial((j1 + j2 - j) / 2 - zz) *
                         factorial((j1 - aa2) / 2 - zz) * factorial((j2 + bb2) / 2 - zz) *
                         factorial((j - j2 + aa2) / 2 + zz) *
                         factorial((j - j1 - bb2) / 2 + zz));
        }
        const int cc2 = 2 * mm - j;
        const double norm =
            std::sqrt(factorial((j1 + aa2) / 2) * factorial((j1 - aa2) / 2) *
                      factorial((j2 + bb2) / 2) * factorial((j2 - bb2) / 2) *
                      factorial((j + cc2) / 2) * factorial((j - cc2) / 2) * (j + 1));
        cg[idx] = sum * deltacg(j1, j2, j) * norm;
      }
    }
  }
  return cg;
}

// fold_beta (snap_core.hpp:308-322).
double fold_beta(const IndexMaps& m, const double* beta, int j1, int j2, int j) {
  if (j >= j1) {
    const double b = beta[m.triple_index(j1, j2, j)];
    if (j1 == j) return (j2 == j) ? 3.0 * b : 2.0 * b;
    return b;
  }
  if (j >= j2) {
    const double b = beta[m.triple_index(j, j2, j1)];
    const double ratio = static_cast<double>(j1 + 1) / static_cast<double>(j + 1);
    return (j2 == j ? 2.0 * b : b) * ratio;
  }
  const double b = beta[m.triple_index(j2, j, j1)];
  return b * static_cast<double>(j1 + 1) / static_cast<double>(j + 1);
}

double g_scale(int t, int mb) { return std::sqrt(factorial(t - mb)); }
double h_scale(int t, int ma) { return 1.0 / std::sqrt(factorial(t - ma) * factorial(ma)); }
double f_scale(int t, int mb, int ma) { return g_scale(t, mb) * h_scale(t, ma); }

std::vector<double> cprime_table(const IndexMaps& m, const std::vector<double>& cg) {
  std::vector<double> out(m.cgtot, 0.0);
  for (const Tuple& tp : m.tuples) {
    const int D = (tp.j1 + tp.j2 - tp.j) / 2;
    for (int ma1 = 0; ma1 <= tp.j1; ++ma1)
      for (int ma2 = 0; ma2 <= tp.j2; ++ma2) {
        const int ma = ma1 + ma2 - D;
        const int idx = tp.cg_off + ma1 * (tp.j2 + 1) + ma2;
        if (ma < 0 || ma > tp.j) continue;
        out[idx] = cg[idx] / (h_scale(tp.j1, ma1) * h_scale(tp.j2, ma2) * h_scale(tp.j, ma));
      }
  }
  return out;
}

std::vector<double> w_table(const IndexMaps& m, const std::vector<double>& cg,
                            const double* beta, bool mirror_signs) {
  std::vector<double> out(m.cgtot, 0.0);
  auto G = [](int t, int mm) { return g_scale(t, std::min(mm, t - mm)); };
  for (const Tuple& tp : m.tuples) {
    const int D = (tp.j1 + tp.j2 - tp.j) / 2;
    const double bf = fold_beta(m, beta, tp.j1, tp.j2, tp.j);
    for (int mb1 = 0; mb1 <= tp.j1; ++mb1)
      for (int mb2 = 0; mb2 <= tp.j2; ++mb2) {
        const int mb = mb1 + mb2 - D;
        const int idx = tp.cg_off + mb1 * (tp.j2 + 1) + mb2;
        if (mb < 0 || 2 * mb > tp.j) continue;
        double s = 1.0;
        if (mirror_signs) {  // (-1)^mb of mirrored rows (halfint_index.hpp:22-25)
          if (2 * mb1 > tp.j1 && (mb1 & 1)) s = -s;
          if (2 * mb2 > tp.j2 && (mb2 & 1)) s = -s;
        }
        out[idx] = s * bf * cg[idx] / (G(tp.j1, mb1) * G(tp.j2, mb2) * g_scale(tp.j, mb));
      }
  }
  return out;
}

std::vector<double> half_f(const IndexMaps& m) {
  std::vector<double> out(m.nhalf);
  for (int t = 0; t <= m.T; ++t)
    for (int mb = 0; 2 * mb <= t; ++mb)
      for (int ma = 0; ma <= t; ++ma)
        out[m.half_off[t] + mb * (t + 1) + ma] = f_scale(t, mb, ma);
  return out;
}

std::vector<double> half_ywgt(const IndexMaps& m) {
  std::vector<double> out(m.nhalf);
  for (int t = 0; t <= m.T; ++t)
    for (int mb = 0; 2 * mb <= t; ++mb)
      for (int ma = 0; ma <= t; ++ma) {
        double w = 1.0;
        if (2 * mb == t) w = (2 * ma < t) ? 1.0 : (2 * ma == t ? 0.5 : 0.0);
        out[m.half_off[t] + mb * (t + 1) + ma] = w;
      }
  return out;
}

// Scatter map of the half stack into the full mirrored stack (compute_Y
// X tile): out[2h] = full index of half element h = (t, mb, ma); out[2h+1] =
// full index fm of its mirror (t, t-mb, t-ma) times 2 plus the sign bit
// (u(t-mb,t-ma) = (-1)^(ma+mb) conj u(mb,ma), halfint_index.hpp:22-25), or -1
// on a middle row, which the half storage holds completely.
std::vector<int> half_scatter_map(const IndexMaps& m) {
  std::vector<int> out(2 * m.nhalf);
  for (int t = 0; t <= m.T; ++t)
    for (int mb = 0; 2 * mb <= t; ++mb)
      for (int ma = 0; ma <= t; ++ma) {
        const int h = m.half_off[t] + mb * (t + 1) + ma;
        out[2 * h] = m.full_off[t] + mb * (t + 1) + ma;
        out[2 * h + 1] = (2 * mb < t)
                             ? 2 * (m.full_off[t] + (t - mb) * (t + 1) + (t - ma)) + ((ma + mb) & 1)
                             : -1;
      }
  return out;
}

static std::vector<std::vector<int>> lpt(const std::vector<std::pair<double, int>>& items,
                                         int workers) {
  std::vector<std::pair<double, int>> sorted = items;
  std::stable_sort(sorted.begin(), sorted.end(),
                   [](const auto& a, const auto& b) { return a.first > b.first; });
  std::vector<std::vector<int>> out(workers);
  using E = std::pair<double, int>;
  std::priority_queue<E, std::vector<E>, std::greater<E>> pq;
  for (int w = 0; w < workers; ++w) pq.push({0.0, w});
  for (const auto& it : sorted) {
    E e = pq.top();
    pq.pop();
    out[e.second].push_back(it.second);
    pq.push({e.first + it.first, e.second});
  }
  return out;
}

YPlan y_plan(const IndexMaps& m, const std::vector<double>& cprime) {
  YPlan p;
  std::vector<int> cwoff(m.tuples.size());
  for (std::size_t q = 0; q < m.tuples.size(); ++q) {
    const Tuple& tp = m.tuples[q];
    const int D = (tp.j1 + tp.j2 - tp.j) / 2;
    cwoff[q] = static_cast<int>(p.cw.size());
    for (int a2 = 0; a2 <= tp.j2; ++a2)
      for (int ma = 0; ma <= tp.j; ++ma) {
        const int a1 = ma + D - a2;
        double c = 0.0;
        if (a1 >= 0 && a1 <= tp.j1) c = cprime[tp.cg_off + a1 * (tp.j2 + 1) + a2];
        p.cw.push_back(c);
      }
  }
  for (int j = 0; j <= m.T; ++j)
    for (int mb = 0; 2 * mb <= j; ++mb) {
      p.row_begin.push_back(static_cast<int>(p.items.size()));
      const int L = (2 * mb == j) ? j / 2 + 1 : j + 1;
      double cost = 0.0;
      for (std::size_t q = 0; q < m.tuples.size(); ++q) {
        const Tuple& tp = m.tuples[q];
        if (tp.j != j) continue;
        const int D = (tp.j1 + tp.j2 - tp.j) / 2;
        const int lo = std::max(0, mb + D - tp.j2), hi = std::min(tp.j1, mb + D);
        for (int mb1 = lo; mb1 <= hi; ++mb1) {
          const int mb2 = mb + D - mb1;
          const bool m1 = 2 * mb1 > tp.j1, m2 = 2 * mb2 > tp.j2;
          const int r1 = m1 ? tp.j1 - mb1 : mb1, r2 = m2 ? tp.j2 - mb2 : mb2;
          const int x = m.half_off[tp.j1] + r1 * (tp.j1 + 1);
          const int y = m.half_off[tp.j2] + r2 * (tp.j2 + 1);
          const int z = tp.j1 | (tp.j2 << 8) | (D << 16) | ((m1 ? 1 : 0) << 24) |
                        ((m2 ? 1 : 0) << 25) | ((j + 1) << 26);
          p.items.push_back({x, y, z, cwoff[q]});
          cost += (tp.j2 + 1) * (6.0 * L + 12.0) + 4.0 * L + 20.0;
        }
      }
      p.row_cost.push_back(cost);
    }
  p.row_begin.push_back(static_cast<int>(p.items.size()));
  return p;
}

std::vector<double> y_item_weights(const IndexMaps& m, const std::vector<double>& wtab) {
  std::vector<double> out;
  for (int j = 0; j <= m.T; ++j)
    for (int mb = 0; 2 * mb <= j; ++mb)
      for (const Tuple& tp : m.tuples) {
        if (tp.j != j) continue;
        const int D = (tp.j1 + tp.j2 - tp.j) / 2;
        const int lo = std::max(0, mb + D - tp.j2), hi = std::min(tp.j1, mb + D);
        for (int mb1 = lo; mb1 <= hi; ++mb1)
          out.push_back(wtab[tp.cg_off + mb1 * (tp.j2 + 1) + (mb + D - mb1)]);
      }
  return out;
}

YCoopPlan ycoop_plan(const IndexMaps& m, int warps, bool lpt_split) {
  YCoopPlan p;
  p.warps = warps;
  for (int j = 0; j <= m.T; ++j)
    for (int mb = 0; 2 * mb <= j; ++mb) {
      std::vector<std::pair<double, int>> costs;
      std::vector<std::array<int, 4>> its;
      int local = -1;  // index of the tuple among those targeting j
      for (std::size_t q = 0; q < m.tuples.size(); ++q) {
        const Tuple& tp = m.tuples[q];
        if (tp.j != j) continue;
        ++local;
        const int D = (tp.j1 + tp.j2 - tp.j) / 2;
        int macs = 0;
        const int nout = (2 * mb == j) ? j / 2 + 1 : j + 1;
        for (int ma = 0; ma < nout; ++ma)
          macs += std::max(0, std::min(tp.j1, ma + D) - std::max(0, ma + D - tp.j2) + 1);
        const int lo = std::max(0, mb + D - tp.j2), hi = std::min(tp.j1, mb + D);
        for (int mb1 = lo; mb1 <= hi; ++mb1) {
          const double c_unrolled = 6.0 * macs + 2.0 * (tp.j1 + 1) + 4.0 * (tp.j1 + tp.j2 + 2) + 20.0;
          const double c_window = (tp.j2 + 1) * (7.0 * nout + 10.0) + 4.0 * nout + 30.0;
          costs.push_back({lpt_split ? c_window : c_unrolled, static_cast<int>(its.size())});
          its.push_back({static_cast<int>(q), mb1, mb + D - mb1, local});
        }
      }
      double tot = 0.0;
      for (auto& c : costs) tot += c.first;
      p.row_cost.push_back(tot);
      // Items are enumerated tuple by tuple; dealing them round-robin keeps
      // every warp on the same tuple body at the same time (instruction
      // cache locality), with per-warp counts within one of each other.
      std::vector<std::vector<int>> buckets(warps);
      if (lpt_split) {  // balance by cost (code-size-insensitive kernels)
        buckets = lpt(costs, warps);
        for (auto& bk : buckets) std::sort(bk.begin(), bk.end());
      } else {
        for (std::size_t i = 0; i < its.size(); ++i) buckets[i % warps].push_back(static_cast<int>(i));
      }
      const int base = static_cast<int>(p.items.size());
      int off = base;
      for (int w = 0; w < warps; ++w) {
        p.rw_begin.push_back(off);
        for (int idx : buckets[w]) p.items.push_back(its[idx]);
        off = static_cast<int>(p.items.size());
      }
      p.rw_begin.push_back(off);
    }
  return p;
}

YCoopPlan ycoop_pair_plan(const IndexMaps& m, int warps) {
  YCoopPlan p;
  p.warps = warps;
  for (int j = 0; j <= m.T; ++j)
    for (int mb = 0; 2 * mb <= j; ++mb) {
      const int nout = (2 * mb == j) ? j / 2 + 1 : j + 1;
      // units of this row: consecutive mb1 of one tuple paired up
      std::vector<std::vector<std::array<int, 4>>> units;
      std::vector<std::pair<double, int>> costs;
      double tot = 0.0;
      int local = -1;
      for (std::size_t q = 0; q < m.tuples.size(); ++q) {
        const Tuple& tp = m.tuples[q];
        if (tp.j != j) continue;
        ++local;
        const int D = (tp.j1 + tp.j2 - tp.j) / 2;
        const int lo = std::max(0, mb + D - tp.j2), hi = std::min(tp.j1, mb + D);
        for (int mb1 = lo; mb1 <= hi; mb1 += 2) {
          std::vector<std::array<int, 4>> u;
          u.push_back({static_cast<int>(q), mb1, mb + D - mb1, local});
          if (mb1 + 1 <= hi) u.push_back({static_cast<int>(q), mb1 + 1, mb + D - mb1 - 1, local});
          // FP64 instructions: 6 per MAC single, 10 per pair MAC; plus setup
          const double c = (tp.j2 + 1) * ((u.size() == 2 ? 10.0 : 6.0) * nout + 8.0) +
                           (u.size() == 2 ? 60.0 : 40.0);
          costs.push_back({c, static_cast<int>(units.size())});
          units.push_back(u);
          tot += c;
        }
      }
      // Row costs for the row -> (part, warp group) schedule: at 2J = 8 the
      // measured per-row cycles of k_compute_Y_cwin (tools/yprof.py on a
      // B200, 256k atoms; the model misses the per-row and per-step
      // overheads of the small-j rows), else the FP64 instruction model.
      // (k_compute_Y_cwin with direct x1 loads, GR = 3, 262k atoms, r02)
      static const double kMeasured8[25] = {
          7050,  5487,  18533, 16170, 15012, 18321, 25144, 30044, 22827, 19402, 22812, 25914, 29899,
          34546, 40189, 27725, 20532, 26596, 32257, 34000, 27325, 34365, 41883, 48782, 30904};
      const int rid = static_cast<int>(p.row_cost.size());
      p.row_cost.push_back(m.T == 8 ? kMeasured8[rid] : tot);
      std::vector<std::vector<int>> buckets = lpt(costs, warps);
      int off = static_cast<int>(p.units.size());
      for (int w = 0; w < warps; ++w) {
        std::sort(buckets[w].begin(), buckets[w].end());
        for (int kind = 2; kind >= 1; --kind) {  // pairs, then singles
          p.rw_begin.push_back(off);
          for (int idx : buckets[w]) {
            if (static_cast<int>(units[idx].size()) != kind) continue;
            p.units.push_back({static_cast<int>(p.items.size()), kind});
            for (const auto& it : units[idx]) p.items.push_back(it);
          }
          off = static_cast<int>(p.units.size());
        }
      }
      p.rw_begin.push_back(off);
    }
  return p;
}

YQuadPlan yquad_plan(const IndexMaps& m, int warps, int groups) {
  YQuadPlan p;
  // offsets into the windowed C' with rows padded to even length
  // (yquad_cw: 16-byte coefficient pairs)
  std::vector<int> cwoff(m.tuples.size());
  int o = 0;
  for (std::size_t q = 0; q < m.tuples.size(); ++q) {
    cwoff[q] = o;
    o += (m.tuples[q].j2 + 1) * ((m.tuples[q].j + 2) & ~1);
  }
  std::vector<std::pair<double, int>> rowcost;
  for (int j = 0; j <= m.T; ++j)
    for (int mb = 0; 2 * mb <= j; ++mb) {
      const int nout = (2 * mb == j) ? j / 2 + 1 : j + 1;
      std::vector<std::array<int, 4>> us;
      std::vector<std::vector<std::array<int, 3>>> uit;
      std::vector<std::pair<double, int>> costs;
      double tot = 0.0;
      for (std::size_t q = 0; q < m.tuples.size(); ++q) {
        const Tuple& tp = m.tuples[q];
        if (tp.j != j) continue;
        const int D = (tp.j1 + tp.j2 - tp.j) / 2;
        const int lo = std::max(0, mb + D - tp.j2), hi = std::min(tp.j1, mb + D);
        for (int mb1 = lo; mb1 <= hi; mb1 += 4) {
          const int cnt = std::min(4, hi - mb1 + 1);
          std::vector<std::array<int, 3>> its;
          for (int k = 0; k < cnt; ++k)
            its.push_back({static_cast<int>(q), mb1 + k, mb + D - mb1 - k});
          const int x1 = m.full_off[tp.j1] + mb1 * (tp.j1 + 1) + D;
          const int x2 = m.full_off[tp.j2] + (mb + D - mb1) * (tp.j2 + 1);
          us.push_back({x1 | (x2 << 16), tp.j2 | (tp.j1 << 8) | (cnt << 16), cwoff[q], 0});
          uit.push_back(its);
          const double c = (tp.j2 + 1) * (6.0 * nout + 24.0) + 60.0;
          costs.push_back({c, static_cast<int>(us.size()) - 1});
          tot += c;
        }
      }
      rowcost.push_back({tot, j * 64 + mb});
      std::vector<std::vector<int>> buckets = lpt(costs, warps);
      int off = static_cast<int>(p.units.size());
      for (int w = 0; w < warps; ++w) {
        std::sort(buckets[w].begin(), buckets[w].end());
        p.rw.push_back(off);
        for (int idx : buckets[w]) {
          std::array<int, 4> u = us[idx];
          u[3] = static_cast<int>(p.items.size());
          for (const auto& it : uit[idx]) p.items.push_back(it);
          p.units.push_back(u);
        }
        off = static_cast<int>(p.units.size());
      }
      p.rw.push_back(off);
    }
  // rows LPT-split over the CTA's warp groups (decreasing cost per group)
  std::vector<std::vector<int>> gb = lpt(rowcost, groups);
  p.rows_cap = 1;
  for (auto& b : gb) p.rows_cap = std::max<int>(p.rows_cap, static_cast<int>(b.size()) + 1);
  p.rows.assign(static_cast<std::size_t>(groups) * p.rows_cap, -1);
  for (int g = 0; g < groups; ++g)
    for (std::size_t q = 0; q < gb[g].size(); ++q) p.rows[g * p.rows_cap + q] = gb[g][q];
  return p;
}

std::vector<double> yquad_cw(const IndexMaps& m, const std::vector<double>& cw) {
  std::vector<double> out;
  std::size_t src = 0;
  for (const Tuple& tp : m.tuples)
    for (int a2 = 0; a2 <= tp.j2; ++a2) {
      for (int ma = 0; ma < ((tp.j + 2) & ~1); ++ma) out.push_back(ma <= tp.j ? cw[src + ma] : 0.0);
      src += tp.j + 1;
    }
  return out;
}

std::vector<double> yquad_weights(const YQuadPlan& p, const IndexMaps& m,
                                  const std::vector<double>& wtab) {
  std::vector<double> out(p.items.size());
  for (std::size_t i = 0; i < p.items.size(); ++i) {
    const Tuple& tp = m.tuples[p.items[i][0]];
    out[i] = wtab[tp.cg_off + p.items[i][1] * (tp.j2 + 1) + p.items[i][2]];
  }
  return out;
}

std::vector<double> ycoop_weights(const YCoopPlan& p, const IndexMaps& m,
                                  const std::vector<double>& wtab) {
  std::vector<double> out(p.items.size());
  for (std::size_t i = 0; i < p.items.size(); ++i) {
    const Tuple& tp = m.tuples[p.items[i][0]];
    out[i] = wtab[tp.cg_off + p.items[i][1] * (tp.j2 + 1) + p.items[i][2]];
  }
  return out;
}

BPlan b_plan(const IndexMaps& m, const std::vector<double>& cg) {
  BPlan p;
  std::vector<int> cwoff(m.tuples.size());
  int o = 0;
  for (std::size_t q = 0; q < m.tuples.size(); ++q) {  // y_plan's windowed C' layout
    cwoff[q] = o;
    o += (m.tuples[q].j2 + 1) * (m.tuples[q].j + 1);
  }
  auto G = [](int t, int mm) { return g_scale(t, std::min(mm, t - mm)); };
  for (const auto& tr : m.triples) {
    p.triple_begin.push_back(static_cast<int>(p.items.size()));
    const int j1 = tr[0], j2 = tr[1], j = tr[2];
    int q = -1;
    for (std::size_t k = 0; k < m.tuples.size(); ++k)
      if (m.tuples[k].j1 == j1 && m.tuples[k].j2 == j2 && m.tuples[k].j == j) q = static_cast<int>(k);
    const Tuple& tp = m.tuples[q];
    const int D = (j1 + j2 - j) / 2;
    for (int mb = 0; 2 * mb <= j; ++mb) {
      const double wrow = (2 * mb < j) ? 2.0 : 1.0;
      const int lo = std::max(0, mb + D - j2), hi = std::min(j1, mb + D);
      for (int mb1 = lo; mb1 <= hi; ++mb1) {
        const int mb2 = mb + D - mb1;
        const int x1 = m.full_off[j1] + mb1 * (j1 + 1) + D;
        const int x2 = m.full_off[j2] + mb2 * (j2 + 1);
        const int xr = m.full_off[j] + mb * (j + 1);
        p.items.push_back({x1, x2, xr, j2 | (j << 8)});
        p.cwoff.push_back(cwoff[q]);
        const double wb = cg[tp.cg_off + mb1 * (j2 + 1) + mb2] /
                          (G(j1, mb1) * G(j2, mb2) * g_scale(j, mb));
        p.wgt.push_back(wrow * wb);
      }
    }
  }
  p.triple_begin.push_back(static_cast<int>(p.items.size()));
  return p;
}

std::vector<int> y_row_schedule(const IndexMaps& m, const std::vector<double>& row_cost,
                                int workers, int* cap) {
  std::vector<std::pair<double, int>> items;
  int rid = 0;
  for (int j = 0; j <= m.T; ++j)
    for (int mb = 0; 2 * mb <= j; ++mb, ++rid) items.push_back({row_cost[rid], j * 64 + mb});
  auto buckets = lpt(items, workers);
  int c = 0;
  for (auto& b : buckets) c = std::max<int>(c, static_cast<int>(b.size()));
  c += 1;
  std::vector<int> out(static_cast<std::size_t>(workers) * c, -1);
  for (int w = 0; w < workers; ++w)
    for (std::size_t k = 0; k < buckets[w].size(); ++k) out[w * c + k] = buckets[w][k];
  *cap = c;
  return out;
}

// Parts (CTAs) per 32-atom tile, each taking an LPT share of the tile's rows.
// With fewer tiles than SMs the tiles get floor(nsm / ntiles) parts and the
// first tiles one more, so the grid is exactly one CTA per SM: those tiles
// finish early and their SMs take the first compute_fused_dE CTAs (which
// wait per tile) while the other tiles still run.  The base-count tiles are
// kept even, so every TPC of the long-running CTAs pairs the same (parts,
// part) row lists; forced_parts > 0 (snapgpu_tune) gives a uniform count.
// CTA order: by part count, then part, then tile -- consecutive CTAs land on
// the two SMs of a TPC, which share an instruction cache, and CTAs of the
// same (parts, part) run the same row lists, hence the same code.
YCtaPlan y_cta_plan(const IndexMaps& m, const std::vector<double>& row_cost, int ntiles,
                    int nsm, int forced_parts, int max_parts, int groups) {
  YCtaPlan p;
  ntiles = std::max(1, ntiles);
  std::vector<int> P(ntiles, 1);
  if (forced_parts > 0) {
    std::fill(P.begin(), P.end(), forced_parts);
  } else if (ntiles < nsm) {
    const int base = std::max(1, std::min(max_parts, nsm / ntiles));
    int extra = base < max_parts ? std::min(ntiles, nsm - base * ntiles) : 0;
    if (extra > 0 && ((ntiles - extra) & 1)) --extra;
    for (int t = 0; t < ntiles; ++t) P[t] = base + (t < extra ? 1 : 0);
  }
  std::vector<int> off(max_parts + 1, 0), cap(max_parts + 1, 0);
  for (int q = 1; q <= max_parts; ++q) {
    if (std::find(P.begin(), P.end(), q) == P.end()) continue;
    std::vector<int> sched = y_row_schedule(m, row_cost, q * groups, &cap[q]);
    off[q] = static_cast<int>(p.tasks.size());
    p.tasks.insert(p.tasks.end(), sched.begin(), sched.end());
    p.pmax = std::max(p.pmax, q);
  }
  for (int q = 1; q <= max_parts; ++q)
    for (int part = 0; part < q; ++part)
      for (int t = 0; t < ntiles; ++t)
        if (P[t] == q) p.cta.push_back({t, part | (q << 8), off[q] + part * groups * cap[q], cap[q]});
  return p;
}

// ---------------------------------------------------------------------------
// Neighbor lists: harness.hpp:119-202 arithmetic (wrap_coord :82-86,
// min_image :88-90, strict r2 < rc2, lists sorted by index), generalized to
// orthorhombic boxes.  Each atom scans the 27 surrounding cells of a cell
// list; the minimum-image displacement is odd-symmetric and the lists are
// sorted, so the result is bitwise identical to the reference's half-stencil
// construction (checked in tests/test_tables.py).
// ---------------------------------------------------------------------------
namespace {
double wrap_coord(double x, double box) {
  double w = x - box * std::floor(x / box);
  return w >= box ? w - box : w;
}
double min_image(double d, double box) { return d - box * std::nearbyint(d / box); }
struct Nb {
  int idx;
  double d[3];
};
}  // namespace

int build_neighborlist(const double* pos, int n, const double box[3], double rcut,
                       int maxstride, int* numneigh, int* nbr, double* disp,
                       std::string* err) {
  for (int d = 0; d < 3; ++d) {
    if (!(box[d] > 0.0) || !(rcut > 0.0)) {
      *err = "build_neighborlist: box and Rcut must be positive";
      return -1;
    }
    if (!(rcut <= 0.5 * box[d])) {
      *err = "build_neighborlist: Rcut must not exceed box/2";
      return -1;
    }
  }
  std::vector<double> w(static_cast<std::size_t>(n) * 3);
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) w[i * 3 + c] = wrap_coord(pos[i * 3 + c], box[c]);
  const double rc2 = rcut * rcut;
  std::vector<std::vector<Nb>> lists(n);
  int nc[3];
  bool cells = true;
  for (int d = 0; d < 3; ++d) {
    nc[d] = static_cast<int>(std::floor(box[d] / rcut));
    if (nc[d] < 3) cells = false;
  }
  auto try_pair = [&](int i, int k, std::vector<Nb>& out) {
    Nb e;
    for (int c = 0; c < 3; ++c) e.d[c] = min_image(w[k * 3 + c] - w[i * 3 + c], box[c]);
    const double r2 = e.d[0] * e.d[0] + e.d[1] * e.d[1] + e.d[2] * e.d[2];
    if (r2 < rc2) {
      e.idx = k;
      out.push_back(e);
    }
  };
  if (!cells) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < n; ++k)
        if (k != i) try_pair(i, k, lists[i]);
  } else {
    const long ncell = static_cast<long>(nc[0]) * nc[1] * nc[2];
    std::vector<int> cell_of(n);
    std::vector<int> head(ncell + 1, 0);
    for (int i = 0; i < n; ++i) {
      int ci[3];
      for (int d = 0; d < 3; ++d) {
        int idx = static_cast<int>(w[i * 3 + d] * (static_cast<double>(nc[d]) / box[d]));
        ci[d] = idx >= nc[d] ? nc[d] - 1 : idx;
      }
      cell_of[i] = (ci[2] * nc[1] + ci[1]) * nc[0] + ci[0];
      head[cell_of[i] + 1]++;
    }
    for (long c = 0; c < ncell; ++c) head[c + 1] += head[c];
    std::vector<int> members(n), fill(head.begin(), head.end() - 1);
    for (int i = 0; i < n; ++i) members[fill[cell_of[i]]++] = i;
#pragma omp parallel for schedule(dynamic, 256)
    for (int i = 0; i < n; ++i) {
      const int c = cell_of[i];
      const int cx = c % nc[0], cy = (c / nc[0]) % nc[1], cz = c / (nc[0] * nc[1]);
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const int ox = (cx + dx + nc[0]) % nc[0], oy = (cy + dy + nc[1]) % nc[1],
                      oz = (cz + dz + nc[2]) % nc[2];
            const long oc = (static_cast<long>(oz) * nc[1] + oy) * nc[0] + ox;
            for (int s = head[oc]; s < head[oc + 1]; ++s) {
              const int k = members[s];
              if (k != i) try_pair(i, k, lists[i]);
            }
          }
    }
  }
  int mx = 0;
  for (int i = 0; i < n; ++i) {
    std::sort(lists[i].begin(), lists[i].end(),
              [](const Nb& a, const Nb& b) { return a.idx < b.idx; });
    mx = std::max<int>(mx, static_cast<int>(lists[i].size()));
  }
  for (int i = 0; i < n; ++i) {
    if (numneigh) numneigh[i] = static_cast<int>(lists[i].size());
    if (mx > maxstride || !nbr || !disp) continue;
    for (std::size_t k = 0; k < lists[i].size(); ++k) {
      const std::size_t pk = static_cast<std::size_t>(i) * maxstride + k;
      nbr[pk] = lists[i][k].idx;
      for (int c = 0; c < 3; ++c) disp[pk * 3 + c] = lists[i][k].d[c];
    }
  }
  return mx;
}

// BCC tungsten lattice.  The reference has no lattice builder; the draws use
// its Rng mappings (rng.hpp:19-29) over std::mt19937_64 and its beta
// convention (harness.hpp:208-213: beta first).
int bcc_lattice(int nx, int ny, int nz, double a, double jitter, std::uint64_t seed,
                int T, double* pos, double* beta) {
  std::mt19937_64 eng(seed);
  auto uni = [&](double lo, double hi) {
    return lo + (hi - lo) * (static_cast<double>(eng() >> 11) * 0x1.0p-53);
  };
  const IndexMaps m = IndexMaps::build(T);
  for (std::size_t l = 0; l < m.triples.size(); ++l) beta[l] = uni(-1.0, 1.0);
  int n = 0;
  for (int cz = 0; cz < nz; ++cz)
    for (int cy = 0; cy < ny; ++cy)
      for (int cx = 0; cx < nx; ++cx)
        for (int b = 0; b < 2; ++b) {
          const double h = 0.5 * b;
          const double base[3] = {(cx + h) * a, (cy + h) * a, (cz + h) * a};
          for (int d = 0; d < 3; ++d) pos[n * 3 + d] = base[d] + uni(-jitter, jitter);
          ++n;
        }
  return n;
}

}  // namespace snapgpu
