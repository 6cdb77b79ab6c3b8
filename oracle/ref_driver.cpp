// ref_driver.cpp -- extern "C" shim over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY (see oracle/snap_oracle.h).  This file is ours; it
// contains no reference source.  It is compiled by oracle/Makefile against the
// read-only headers in /root/reference/proj/include (and the reference test
// fixture header /root/reference/proj/tests/test_support.hpp) into
// oracle/_ref/libsnapref.so, which:
//   * pins the C restatement (oracle/snap_oracle.c) bitwise,
//   * generates the golden fixtures under tests/golden/ (tests/golden/make_golden.py),
//   * is the timed CPU baseline of bench.py (`--impl reference`, cpu_baseline).
//
// Every entry point calls the reference's own public API: run_pipeline
// (pipeline.hpp:206) or the stage functions it sequences (snap_core.hpp), the
// neighbor builder (harness.hpp:119), the generators (harness.hpp:230,
// tests/test_support.hpp:21) and the oracle suite (oracle.hpp).

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "snapforge/snapforge.hpp"
#include "test_support.hpp"

using namespace snapforge;

namespace {

thread_local std::string g_err;

WorkerPool& pool_for(int workers) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<WorkerPool>> pools;
  std::lock_guard<std::mutex> lk(mu);
  auto& p = pools[workers];
  if (!p) p = std::make_unique<WorkerPool>(workers);
  return *p;
}

Problem make_problem(int twojmax, double rcut, double rmin0, double rfac0,
                     double wself, int self_flag, const double* beta, int nbeta,
                     const double* weights, int nweights, int natoms,
                     int stride, const int* numneigh, const int* nbr,
                     const double* disp, const int* types) {
  Problem p;
  p.params.twojmax = twojmax;
  p.params.rcut = rcut;
  p.params.rmin0 = rmin0;
  p.params.rfac0 = rfac0;
  p.params.wself = wself;
  p.params.self_contribution = self_flag != 0;
  p.params.weights.assign(weights, weights + nweights);
  p.params.beta.assign(beta, beta + nbeta);
  if (types) p.types.assign(types, types + natoms);
  p.neighbors.resize(static_cast<std::size_t>(natoms));
  for (int i = 0; i < natoms; ++i) {
    auto& nl = p.neighbors[static_cast<std::size_t>(i)];
    nl.resize(static_cast<std::size_t>(numneigh[i]));
    for (int k = 0; k < numneigh[i]; ++k) {
      const std::size_t pk = static_cast<std::size_t>(i) * stride + k;
      nl[static_cast<std::size_t>(k)].index = nbr[pk];
      for (int d = 0; d < 3; ++d) nl[static_cast<std::size_t>(k)].disp[d] = disp[pk * 3 + d];
    }
  }
  return p;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Stage-by-stage evaluation of a variant, mirroring run_pipeline's adjoint
// branch (pipeline.hpp:234-272) but keeping DescriptorState so the
// intermediate arrays can be read back.  Outputs may be NULL.
int ref_run(int twojmax, double rcut, double rmin0, double rfac0, double wself,
            int self_flag, const double* beta, int nbeta, const double* weights,
            int nweights, int natoms, int stride, const int* numneigh,
            const int* nbr, const double* disp, const int* types,
            const char* variant_name, int deterministic, int workers,
            double* forces, double* eatom, double* etotal, double* ulisttot,
            double* ylist, double* delist, double* blist) {
  return guarded([&] {
    Problem p = make_problem(twojmax, rcut, rmin0, rfac0, wself, self_flag, beta,
                             nbeta, weights, nweights, natoms, stride, numneigh,
                             nbr, disp, types);
    p.validate();
    const VariantSpec v = find_variant(variant_name);
    if (!v.adjoint) throw InvalidArgument("ref_run: adjoint variants only");
    WorkerPool& pool = pool_for(workers);
    const HalfIntIndexMaps maps = HalfIntIndexMaps::build(twojmax);
    const CGTable cg = compute_cg_table(twojmax, maps);
    DescriptorState st;
    const bool det = deterministic != 0;
    compute_U(p, maps, v, det, pool, st);
    if (v.transpose_before_Y) transpose_ulisttot(st, false, pool);
    if (eatom || etotal || blist) {
      compute_B_from_U(p, cg, maps, pool, st);
      EnergyReport er = compute_energy(st.blist, p.params.beta, p.natoms());
      if (eatom) std::copy(er.per_atom.begin(), er.per_atom.end(), eatom);
      if (etotal) *etotal = er.total;
      if (blist) std::copy(st.blist.begin(), st.blist.end(), blist);
    }
    if (ulisttot) {
      const detail::UtotView view{st.ulisttot.data(), &st.utot_layout, &maps,
                                  st.utot_half};
      const std::int64_t nh = maps.u_half_total();
      for (int a = 0; a < natoms; ++a)
        for (TwoJ t = 0; t <= twojmax; ++t)
          for (int mb = 0; 2 * mb <= t; ++mb)
            for (int ma = 0; ma <= t; ++ma) {
              const Complex c = view.get(a, t, mb, ma);
              const std::int64_t e = a * nh + maps.u_half_offset[t] + mb * (t + 1) + ma;
              ulisttot[2 * e] = c.re;
              ulisttot[2 * e + 1] = c.im;
            }
    }
    compute_Y(p, p.params.beta, cg, maps, v, det, pool, st);
    if (ylist) {
      const std::int64_t nh = maps.u_half_total();
      for (int a = 0; a < natoms; ++a)
        for (std::int64_t e = 0; e < nh; ++e) {
          const Complex c = st.y_layout.load(st.ylist.data(), a, e);
          ylist[2 * (a * nh + e)] = c.re;
          ylist[2 * (a * nh + e) + 1] = c.im;
        }
    }
    bool scattered = false;
    if (v.fuse_dU_with_force) {
      scattered = compute_fused_dE(p, maps, v, det, pool, st);
    } else {
      compute_dU(p, maps, v, det, pool, st);
      compute_dE_staged(p, maps, v, pool, st);
    }
    if (!scattered) scatter_forces(p, v, det, pool, st);
    if (delist) {  // re-stride from the state's max_neighbors() to ours
      for (int i = 0; i < natoms; ++i)
        for (int k = 0; k < numneigh[i]; ++k)
          for (int d = 0; d < 3; ++d)
            delist[(static_cast<std::size_t>(i) * stride + k) * 3 + d] =
                st.delist[(static_cast<std::size_t>(i) * st.nbor_stride + k) * 3 + d];
    }
    if (forces) std::copy(st.forces.begin(), st.forces.end(), forces);
  });
}

// run_pipeline timing (pipeline.hpp:206): `warmup` full evaluations (with
// energy), then `steps` force-path evaluations (with_energy = false), the
// harness protocol of harness.hpp:534-556.  step_ms[steps] receives each
// step's PipelineResult::total_ms, the sum of its stage times (what the
// harness reports, harness.hpp:540-545: the per-call Problem::validate,
// index-map and CG-table setup of run_pipeline, pipeline.hpp:211-216, are
// not part of a step); wall_ms[steps] (may be NULL) the wall clock around
// the whole call.
int ref_time(int twojmax, double rcut, double rmin0, double rfac0, double wself,
             int self_flag, const double* beta, int nbeta,
             const double* weights, int nweights, int natoms, int stride,
             const int* numneigh, const int* nbr, const double* disp,
             const int* types, const char* variant_name, int deterministic,
             int workers, int warmup, int steps, int with_energy,
             double* step_ms, double* wall_ms, double* forces, double* etotal) {
  return guarded([&] {
    Problem p = make_problem(twojmax, rcut, rmin0, rfac0, wself, self_flag, beta,
                             nbeta, weights, nweights, natoms, stride, numneigh,
                             nbr, disp, types);
    const VariantSpec v = find_variant(variant_name);
    WorkerPool& pool = pool_for(workers);
    const RunMode mode = deterministic ? RunMode::deterministic : RunMode::benchmark;
    for (int w = 0; w < warmup; ++w) {
      PipelineResult r = run_pipeline(p, v, mode, pool, 0, true);
      if (etotal) *etotal = r.energy.total;
    }
    for (int s = 0; s < steps; ++s) {
      const auto t0 = std::chrono::steady_clock::now();
      PipelineResult r = run_pipeline(p, v, mode, pool, 0, with_energy != 0);
      const auto t1 = std::chrono::steady_clock::now();
      step_ms[s] = r.total_ms;
      if (wall_ms) wall_ms[s] = std::chrono::duration<double, std::milli>(t1 - t0).count();
      if (forces && s == steps - 1) std::copy(r.forces.begin(), r.forces.end(), forces);
      if (etotal && with_energy) *etotal = r.energy.total;
    }
  });
}

// harness.hpp:119-202 (cubic boxes only, as in the reference).
int ref_build_neighborlist(const double* pos, int n, double box, double rcut,
                           int maxstride, int* numneigh, int* nbr,
                           double* disp) {
  int mx = -1;
  const int rc = guarded([&] {
    std::vector<std::array<double, 3>> P(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i)
      for (int d = 0; d < 3; ++d) P[static_cast<std::size_t>(i)][static_cast<std::size_t>(d)] = pos[i * 3 + d];
    auto lists = harness::build_neighborlist(P, box, rcut);
    mx = 0;
    for (auto& l : lists) mx = std::max<int>(mx, static_cast<int>(l.size()));
    for (int i = 0; i < n; ++i) {
      const auto& l = lists[static_cast<std::size_t>(i)];
      numneigh[i] = static_cast<int>(l.size());
      if (mx > maxstride) continue;
      for (std::size_t k = 0; k < l.size(); ++k) {
        const std::size_t pk = static_cast<std::size_t>(i) * maxstride + k;
        nbr[pk] = l[k].index;
        for (int d = 0; d < 3; ++d) disp[pk * 3 + d] = l[k].disp[d];
      }
    }
  });
  return rc == 0 ? mx : -1;
}

int ref_cg_table(int twojmax, double* out) {
  return guarded([&] {
    const auto maps = HalfIntIndexMaps::build(twojmax);
    const auto cg = compute_cg_table(twojmax, maps);
    std::copy(cg.values.begin(), cg.values.end(), out);
  });
}

// Counts pinned by tests/test_halfint_index.cpp:47-68,115-139.
int ref_counts(int twojmax, int* out6) {
  return guarded([&] {
    const auto m = HalfIntIndexMaps::build(twojmax);
    out6[0] = static_cast<int>(m.n_triples());
    out6[1] = static_cast<int>(m.z_tuples.size());
    out6[2] = static_cast<int>(m.u_full_total());
    out6[3] = static_cast<int>(m.u_half_total());
    out6[4] = static_cast<int>(m.z_total_elements);
    out6[5] = static_cast<int>(m.cg_total);
  });
}

int ref_wigner_u_half(const double* disp, double rcut, double rmin0,
                      double rfac0, int twojmax, double* out) {
  return guarded([&] {
    const SphereMap m = map_to_3sphere(disp, rcut, rmin0, rfac0);
    WignerStack s = compute_u_matrices(m, twojmax, UStorage::half);
    for (std::size_t e = 0; e < s.u.size(); ++e) {
      out[2 * e] = s.u[e].re;
      out[2 * e + 1] = s.u[e].im;
    }
  });
}

// tests/test_support.hpp:21-64, stride = natoms.
int ref_make_cluster(int natoms, int twojmax, std::uint64_t seed, int ntypes,
                     double* pos, int* types, double* weights, int* numneigh,
                     int* nbr, double* disp, double* beta) {
  int mx = -1;
  const int rc = guarded([&] {
    Problem p = testsupport::make_cluster(natoms, twojmax, seed, ntypes);
    mx = 0;
    for (int i = 0; i < natoms; ++i) {
      for (int d = 0; d < 3; ++d) pos[i * 3 + d] = p.positions[static_cast<std::size_t>(i)][static_cast<std::size_t>(d)];
      types[i] = p.types[static_cast<std::size_t>(i)];
      const auto& l = p.neighbors[static_cast<std::size_t>(i)];
      numneigh[i] = static_cast<int>(l.size());
      mx = std::max<int>(mx, numneigh[i]);
      for (std::size_t k = 0; k < l.size(); ++k) {
        const std::size_t pk = static_cast<std::size_t>(i) * natoms + k;
        nbr[pk] = l[k].index;
        for (int d = 0; d < 3; ++d) disp[pk * 3 + d] = l[k].disp[d];
      }
    }
    std::copy(p.params.weights.begin(), p.params.weights.end(), weights);
    std::copy(p.params.beta.begin(), p.params.beta.end(), beta);
  });
  return rc == 0 ? mx : -1;
}

// harness.hpp:230-262 via generate_problem with synthetic_neighbors.
int ref_generate_synthetic(int natoms, int nnbor, int twojmax, double rcut,
                           std::uint64_t seed, int* numneigh, int* nbr,
                           double* disp, double* beta) {
  return guarded([&] {
    harness::BenchConfig c;
    c.natoms = natoms;
    c.nnbor = nnbor;
    c.twojmax = twojmax;
    c.rcut = rcut;
    c.seed = seed;
    c.synthetic_neighbors = true;
    Problem p = harness::generate_problem(c);
    for (int i = 0; i < natoms; ++i) {
      const auto& l = p.neighbors[static_cast<std::size_t>(i)];
      numneigh[i] = static_cast<int>(l.size());
      for (std::size_t k = 0; k < l.size(); ++k) {
        const std::size_t pk = static_cast<std::size_t>(i) * nnbor + k;
        nbr[pk] = l[k].index;
        for (int d = 0; d < 3; ++d) disp[pk * 3 + d] = l[k].disp[d];
      }
    }
    std::copy(p.params.beta.begin(), p.params.beta.end(), beta);
  });
}

// The reference oracle checks over one problem (oracle.hpp:175-237).
// out[0] = rotation-invariance max rel err, out[1] = Newton-sum residue,
// out[2] = cross-pipeline (baseline-Z vs v1) max rel err.
int ref_oracle_checks(int twojmax, double rcut, double rmin0, double rfac0,
                      double wself, int self_flag, const double* beta,
                      int nbeta, const double* weights, int nweights,
                      int natoms, int stride, const int* numneigh,
                      const int* nbr, const double* disp, const int* types,
                      std::uint64_t seed, double* out3) {
  return guarded([&] {
    Problem p = make_problem(twojmax, rcut, rmin0, rfac0, wself, self_flag, beta,
                             nbeta, weights, nweights, natoms, stride, numneigh,
                             nbr, disp, types);
    out3[0] = oracle::rotation_invariance_check(p, seed).max_rel_err;
    WorkerPool pool(1);
    const PipelineResult r =
        run_pipeline(p, find_variant("v1"), RunMode::deterministic, pool);
    out3[1] = oracle::newton_sum_check(r.forces).max_rel_err;
    out3[2] = oracle::cross_pipeline_check(p).max_rel_err;
  });
}

// Problem file I/O through the reference's own writer / reader
// (harness.hpp:698-780, schema 1, shortest round-trip doubles):
// ref_save_problem writes the given problem (positions may be NULL);
// ref_resave_problem loads a file with harness::load_problem (which runs
// Problem::validate) and writes it back with harness::save_problem.
int ref_save_problem(int twojmax, double rcut, double rmin0, double rfac0, double wself,
                     int self_flag, const double* beta, int nbeta, const double* weights,
                     int nweights, int natoms, int stride, const int* numneigh,
                     const int* nbr, const double* disp, const int* types,
                     std::uint64_t seed, int synthetic, double box_length,
                     const double* positions, const char* path) {
  return guarded([&] {
    Problem p = make_problem(twojmax, rcut, rmin0, rfac0, wself, self_flag, beta, nbeta,
                             weights, nweights, natoms, stride, numneigh, nbr, disp, types);
    p.seed = seed;
    p.synthetic = synthetic != 0;
    p.box_length = box_length;
    if (positions)
      for (int i = 0; i < natoms; ++i)
        p.positions.push_back({positions[3 * i], positions[3 * i + 1], positions[3 * i + 2]});
    harness::save_problem(p, path);
  });
}

int ref_resave_problem(const char* in_path, const char* out_path) {
  return guarded([&] { harness::save_problem(harness::load_problem(in_path), out_path); });
}

}  // extern "C"
