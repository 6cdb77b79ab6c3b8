// adapter_test.cpp -- include/snapforge_gpu.hpp driven from the reference's
// own C++ (TEST INFRASTRUCTURE; built by tests/cpp/Makefile where
// /root/reference exists, run on the GPU box by tests/test_cpp_adapter.py).
//
// For each problem: run_pipeline_gpu (the adapter over libsnapgpu.so) vs the
// reference's run_pipeline(find_variant("v1"), RunMode::deterministic)
// (pipeline.hpp:206-303, the oracle path) -- forces max|dF|/max|F| <= 1e-10,
// total energy <= 1e-12; the stage-level Engine API equals the one-call path
// bitwise; a second run reproduces the force checksum; an invalid problem
// throws InvalidArgument.  Problems: the golden BCC-54 file written by the
// reference's save_problem (argv[1]) and the reference's make_cluster and
// generate_synthetic (tests/test_support.hpp:21-64, harness.hpp:230-262).
#include <cmath>
#include <cstdio>
#include <string>

#include "snapforge/snapforge.hpp"
#include "snapforge_gpu.hpp"
#include "test_support.hpp"

using namespace snapforge;

static int fails = 0;

static double norm_err(const std::vector<double>& a, const std::vector<double>& b) {
  double m = 0.0, d = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    m = std::max(m, std::abs(b[i]));
    d = std::max(d, std::abs(a[i] - b[i]));
  }
  return d / (m > 0 ? m : 1.0);
}

static void check_problem(const char* name, const Problem& p) {
  WorkerPool pool(4);
  const PipelineResult ref = run_pipeline(p, find_variant("v1"), RunMode::deterministic, pool);
  const PipelineResult g = gpu::run_pipeline_gpu(p);
  const double fe = norm_err(g.forces, ref.forces);
  const double ee = std::abs(g.energy.total - ref.energy.total) / std::abs(ref.energy.total);
  const double pe = norm_err(g.energy.per_atom, ref.energy.per_atom);
  gpu::Engine e(p.params);
  const PipelineResult g2 = e.run(p);
  e.set_problem(p);
  e.compute_U();
  e.compute_Y();
  e.compute_fused_dE();
  e.scatter_forces();
  const std::vector<double> fs = e.forces();
  const bool same = g2.force_checksum == g.force_checksum && fs == g.forces;
  const bool ok = fe <= 1e-10 && ee <= 1e-12 && pe <= 1e-12 && same;
  std::printf("%s natoms=%d twojmax=%d force_err=%.3e energy_err=%.3e eatom_err=%.3e "
              "checksum=%s reproducible=%d %s\n",
              name, p.natoms(), p.params.twojmax, fe, ee, pe, g.force_checksum.c_str(),
              same ? 1 : 0, ok ? "PASS" : "FAIL");
  if (!ok) ++fails;
}

int main(int argc, char** argv) {
  try {
    if (argc > 1) check_problem("bcc54_2j8(problem file)", harness::load_problem(argv[1]));
    check_problem("make_cluster(8,8,23)", testsupport::make_cluster(8, 8, 23));
    check_problem("make_cluster(7,5,915,3 types)", testsupport::make_cluster(7, 5, 915, 3));
    check_problem("make_cluster(5,14,914)", testsupport::make_cluster(5, 14, 914));
    harness::BenchConfig bc;  // the acceptance gate's problem (acceptance.cpp:249-275)
    bc.natoms = 64;
    bc.nnbor = 14;
    bc.seed = 600;
    check_problem("generate_problem(64x14, 2J=8, seed 600)", harness::generate_problem(bc));
    // Problem::validate on the device -> InvalidArgument (snap_core.hpp:112)
    Problem bad = testsupport::make_cluster(6, 4, 3);
    bad.neighbors[0][0].disp[0] = 5.0;
    bad.neighbors[0][0].disp[1] = bad.neighbors[0][0].disp[2] = 0.0;
    bool threw = false;
    try {
      gpu::run_pipeline_gpu(bad);
    } catch (const InvalidArgument& ex) {
      threw = std::string(ex.what()).find("Rcut") != std::string::npos;
    }
    std::printf("invalid problem -> InvalidArgument: %s\n", threw ? "PASS" : "FAIL");
    if (!threw) ++fails;
  } catch (const std::exception& ex) {
    std::printf("exception: %s\nFAIL\n", ex.what());
    return 2;
  }
  std::printf("%s\n", fails ? "FAILED" : "ALL PASS");
  return fails ? 1 : 0;
}
