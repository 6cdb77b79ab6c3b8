// snapforge_gpu.hpp -- the reference-side C++ binding of the B200 engine.
//
// What a snapforge maintainer adds next to pipeline.hpp to run the north-star
// path on a B200: the reference (/root/reference/proj/include/snapforge) is
// header-only C++20 without an FFI; its boundary is run_pipeline
// (pipeline.hpp:206-303) over the stage functions of snap_core.hpp.  This
// header maps that boundary onto the C-ABI of include/snapgpu.h
// (libsnapgpu.so): same inputs (Problem, snap_core.hpp:48-119), same result
// type (PipelineResult, pipeline.hpp:47-70), same exception types
// (common.hpp:21-42).
//
//   #include "snapforge/snapforge.hpp"   // -I<reference>/include
//   #include "snapforge_gpu.hpp"         // -I<repo>/include, link libsnapgpu.so
//   snapforge::PipelineResult r = snapforge::gpu::run_pipeline_gpu(problem);
//
// The GPU path is the `fused` adjoint variant (exec_variants.hpp:153-167) in
// deterministic mode: forces are the serialized pair-order scatter of dElist
// (snap_core.hpp:889-899), bitwise stable run to run.  Built and run by
// tests/cpp (Makefile) against the reference headers; the resulting binary
// is the -m gpu test tests/test_cpp_adapter.py.
#pragma once

#include <chrono>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "snapforge/common.hpp"
#include "snapforge/pipeline.hpp"
#include "snapforge/snap_core.hpp"
#include "snapgpu.h"

namespace snapforge {
namespace gpu {

// SNAPGPU_* status -> the reference's exception types (common.hpp:21-42).
inline void check(const snapgpu_ctx* c, int rc) {
  if (rc == SNAPGPU_OK) return;
  const std::string msg = snapgpu_last_error(c);
  if (rc == SNAPGPU_EINVAL) throw InvalidArgument(msg);
  throw PipelineError(msg);
}

// Problem::neighbors (vector of vectors) flattened to (atom, slot) arrays of
// stride max_neighbors(), the layout of snapgpu_set_neighbors.
struct FlatLists {
  int natoms = 0, stride = 0;
  std::vector<int> numneigh, nbr;
  std::vector<double> disp;

  explicit FlatLists(const Problem& p) : natoms(p.natoms()), stride(p.max_neighbors()) {
    numneigh.resize(static_cast<std::size_t>(natoms));
    nbr.assign(static_cast<std::size_t>(natoms) * stride, 0);
    disp.assign(static_cast<std::size_t>(natoms) * stride * 3, 0.0);
    for (int i = 0; i < natoms; ++i) {
      const auto& nl = p.neighbors[static_cast<std::size_t>(i)];
      numneigh[static_cast<std::size_t>(i)] = static_cast<int>(nl.size());
      for (std::size_t k = 0; k < nl.size(); ++k) {
        const std::size_t s = static_cast<std::size_t>(i) * stride + k;
        nbr[s] = nl[k].index;
        for (int d = 0; d < 3; ++d) disp[s * 3 + d] = nl[k].disp[d];
      }
    }
  }
};

// A device context bound to one SnapParams: tables uploaded once, then one
// force step per call (an MD loop re-uses it across steps).
class Engine {
 public:
  explicit Engine(const SnapParams& s, int device = 0) {
    check(nullptr, snapgpu_create(device, s.twojmax, s.rcut, s.rmin0, s.rfac0, s.wself,
                                  s.self_contribution ? 1 : 0, s.beta.data(),
                                  static_cast<int>(s.beta.size()), s.weights.data(),
                                  static_cast<int>(s.weights.size()), &ctx_));
  }
  ~Engine() { snapgpu_destroy(ctx_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  snapgpu_ctx* handle() const { return ctx_; }

  // run_pipeline (pipeline.hpp:206-303), fused adjoint branch: upload the
  // lists, U -> Y (+ per-atom energy) -> fused dU/dE -> deterministic force
  // scatter, read back, one stream synchronization.  Problem::validate runs
  // on the device; violations throw InvalidArgument with the reference's
  // message.  stages: one "gpu-step" entry (wall clock of the call).
  PipelineResult run(const Problem& p) {
    FlatLists f(p);
    PipelineResult r;
    r.forces.assign(static_cast<std::size_t>(f.natoms) * 3, 0.0);
    r.energy.per_atom.assign(static_cast<std::size_t>(f.natoms), 0.0);
    const auto t0 = std::chrono::steady_clock::now();
    check(ctx_, snapgpu_run_host(ctx_, f.natoms, 0, f.natoms, f.stride, f.numneigh.data(),
                                 f.nbr.data(), f.disp.data(),
                                 p.types.empty() ? nullptr : p.types.data(), r.forces.data(),
                                 r.energy.per_atom.data(), &r.energy.total));
    const auto t1 = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    r.stages.push_back({"gpu-step", ms, true});
    r.force_path_ms = r.total_ms = ms;
    r.force_checksum = checksum_hex(r.forces);
    return r;
  }

  // The stage functions (snap_core.hpp) one by one, for stage-level use like
  // tests/test_snap_core.cpp:30-62; the arrays stay on the device.
  void set_problem(const Problem& p) {
    FlatLists f(p);
    check(ctx_, snapgpu_set_neighbors(ctx_, f.natoms, f.stride, f.numneigh.data(),
                                      f.nbr.data(), f.disp.data(),
                                      p.types.empty() ? nullptr : p.types.data()));
    natoms_ = f.natoms;
  }
  void compute_U() { check(ctx_, snapgpu_compute_U(ctx_)); }              // :369
  void compute_Y() { check(ctx_, snapgpu_compute_Y(ctx_)); }              // :1085
  void compute_fused_dE() { check(ctx_, snapgpu_compute_dU_deidrj(ctx_)); }  // :1274
  void scatter_forces() { check(ctx_, snapgpu_scatter_forces(ctx_)); }    // :872
  std::vector<double> forces() {
    std::vector<double> f(static_cast<std::size_t>(natoms_) * 3);
    check(ctx_, snapgpu_get_forces(ctx_, f.data()));
    return f;
  }
  EnergyReport energy() {
    EnergyReport e;
    e.per_atom.resize(static_cast<std::size_t>(natoms_));
    check(ctx_, snapgpu_get_energy(ctx_, e.per_atom.data(), &e.total));
    return e;
  }

 private:
  snapgpu_ctx* ctx_ = nullptr;
  int natoms_ = 0;
};

// Drop-in for run_pipeline(problem, find_variant("fused"), deterministic, pool)
// on device `device`.
inline PipelineResult run_pipeline_gpu(const Problem& problem, int device = 0) {
  Engine e(problem.params, device);
  return e.run(problem);
}

}  // namespace gpu
}  // namespace snapforge
