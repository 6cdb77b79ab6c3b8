/*
 * snapgpu.h -- C-ABI of the B200-native SNAP force engine.
 *
 * Drop-in boundary for the reference's stage interface (snapforge, header-only
 * C++ under /root/reference/proj/include/snapforge).  The reference exposes
 * no FFI; its boundary is the C++ stage signatures called by run_pipeline
 * (pipeline.hpp:206-303).  Each entry point below names the reference
 * function it replaces.  Conventions:
 *
 *   - extern "C", plain pointers and sizes, no exceptions across the ABI;
 *   - every call returns an int status (SNAPGPU_OK == 0) and records a
 *     message readable through snapgpu_last_error(ctx);
 *   - a context is bound to one CUDA device and one stream, is not
 *     thread-safe, and executes stream-ordered (like DescriptorState,
 *     snap_core.hpp:130-172, it owns every per-atom array);
 *   - pointers are HOST memory unless the name says "device";
 *   - per-atom complex arrays returned by the debug getters are logical
 *     (atom, half-index) order, interleaved re/im, half index space
 *     2*mb <= t (halfint_index.hpp:16-25).
 *
 * Error codes mirror the reference exception types (common.hpp:21-42):
 *   SNAPGPU_EINVAL    <- InvalidArgument (detail::require, Problem::validate)
 *   SNAPGPU_EPIPELINE <- PipelineError
 *   SNAPGPU_ECUDA     <- CUDA runtime failure (no reference analogue)
 *   SNAPGPU_ESTATE    <- stage called before its inputs exist
 */
#ifndef SNAPGPU_H
#define SNAPGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SNAPGPU_OK 0
#define SNAPGPU_EINVAL 1
#define SNAPGPU_EPIPELINE 2
#define SNAPGPU_ECUDA 3
#define SNAPGPU_ESTATE 4

#define SNAPGPU_MAX_TWOJMAX 14

typedef struct snapgpu_ctx snapgpu_ctx;

/* Message of the last failing call on ctx (or of the last failing
 * context-free call when ctx is NULL).  Never NULL. */
const char* snapgpu_last_error(const snapgpu_ctx* ctx);
const char* snapgpu_version(void);

/* ---- setup ------------------------------------------------------------
 * Replaces SnapParams (snap_core.hpp:48-57) + HalfIntIndexMaps::build
 * (halfint_index.hpp:155-200) + compute_cg_table (angular_basis.hpp:151-196)
 * + the fold_beta table (snap_core.hpp:308-322, 1135-1138).  Builds every
 * index/coefficient table on the host and uploads it once.
 * twojmax in [0, SNAPGPU_MAX_TWOJMAX]; weights are per-type neighbor weights
 * (SnapParams::weights); beta has n_triples(twojmax) entries.
 */
int snapgpu_create(int device, int twojmax, double rcut, double rmin0,
                   double rfac0, double wself, int self_flag,
                   const double* beta, int nbeta, const double* weights,
                   int nweights, snapgpu_ctx** out);
int snapgpu_destroy(snapgpu_ctx* ctx);

/* Replace the linear model coefficients (SnapParams::beta) in place. */
int snapgpu_set_beta(snapgpu_ctx* ctx, const double* beta, int nbeta);

/* Run on a caller-owned CUDA stream (cudaStream_t passed as void*);
 * NULL restores the context's own stream. */
int snapgpu_set_stream(snapgpu_ctx* ctx, void* cuda_stream);

/* ---- neighbor lists ---------------------------------------------------
 * Replaces Problem::neighbors / Problem::types (snap_core.hpp:59-119) and
 * performs Problem::validate (:89-118).  Flattened (atom, slot) arrays:
 * nbr[i*stride+k], disp[(i*stride+k)*3+d] for k < numneigh[i]; types may be
 * NULL (all type 0).  Host->device copies run on the context stream.
 */
int snapgpu_set_neighbors(snapgpu_ctx* ctx, int natoms, int stride,
                          const int* numneigh, const int* nbr,
                          const double* disp, const int* types);

/* Atom-partitioned variant for multi-GPU runs: this context owns atoms
 * [atom_lo, atom_lo+nlocal) of natoms_total; lists are given for the owned
 * atoms only, with global neighbor indices; types (natoms_total) may be
 * NULL.  Forces are produced as a natoms_total x 3 PARTIAL buffer (owned
 * pairs' contributions to every atom) for a subsequent reduce-scatter. */
int snapgpu_set_neighbors_partition(snapgpu_ctx* ctx, int natoms_total,
                                    int atom_lo, int nlocal, int stride,
                                    const int* numneigh, const int* nbr,
                                    const double* disp, const int* types);

/* ---- stages (snap_core.hpp), stream-ordered ---------------------------- */
int snapgpu_compute_U(snapgpu_ctx* ctx);         /* compute_U        :369  */
int snapgpu_compute_Y(snapgpu_ctx* ctx);         /* compute_Y        :1085,
                                                    + per-atom energy
                                                    (replaces compute_B_from_U
                                                    :642 + compute_energy :684) */
int snapgpu_compute_dU_deidrj(snapgpu_ctx* ctx); /* compute_fused_dE :1274
                                                    (compute_dU :707 fused
                                                    with compute_dE :1206)  */
int snapgpu_scatter_forces(snapgpu_ctx* ctx);    /* scatter_forces   :872,
                                                    deterministic mode
                                                    (:889-899): each force is
                                                    the serialized pair-order
                                                    sum of dElist, bitwise
                                                    reproducible run to run */

/* The whole force step in reference stage order (run_pipeline adjoint
 * branch, pipeline.hpp:234-272): U -> Y(+energy) -> fused dU/dE -> scatter.
 * Replayed from a CUDA graph after the first call for a given shape. */
int snapgpu_run(snapgpu_ctx* ctx);
int snapgpu_synchronize(snapgpu_ctx* ctx);

/* One force step from host buffers (the end-to-end call): upload the owned
 * atoms' lists (set_neighbors_partition semantics; atom_lo = 0 and nlocal =
 * natoms_total for a single GPU), run, and copy forces (natoms_total x 3),
 * eatom (nlocal) and etotal back (any output may be NULL); one stream
 * synchronization.  Equivalent to run_pipeline (pipeline.hpp:206-303).
 * When numneigh / nbr / disp are page-locked host memory (cudaHostAlloc,
 * cudaHostRegister; mapped under UVA) and 2J <= 8, no copy is issued:
 * compute_U reads them over PCIe while it computes and leaves the device
 * copies for the later stages; pageable arrays are uploaded first.  The
 * reverse-neighbor index is rebuilt beside Y / dE in either case. */
int snapgpu_run_host(snapgpu_ctx* ctx, int natoms_total, int atom_lo, int nlocal,
                     int stride, const int* numneigh, const int* nbr,
                     const double* disp, const int* types, double* forces,
                     double* eatom, double* etotal);

/* ---- results (host copies; synchronize the stream) ---------------------
 * forces: natoms_total x 3 (PipelineResult::forces, pipeline.hpp:50), or
 * the chunked layout of snapgpu_set_force_layout;
 * eatom: nlocal (EnergyReport::per_atom); etotal: sum over owned atoms. */
int snapgpu_get_forces(snapgpu_ctx* ctx, double* forces);
int snapgpu_get_energy(snapgpu_ctx* ctx, double* eatom, double* etotal);

/* Debug readback in the reference's logical conventions:
 * ulisttot / ylist: nlocal x n_half complex (DescriptorState::ulisttot /
 * ylist, snap_core.hpp:138-139); dedr: nlocal x stride x 3
 * (DescriptorState::delist, :144). */
int snapgpu_get_ulisttot(snapgpu_ctx* ctx, double* out);
int snapgpu_get_ylist(snapgpu_ctx* ctx, double* out);
int snapgpu_get_dedr(snapgpu_ctx* ctx, double* out);

/* On-device neighbor lists: harness.hpp:119-202 built on
 * the GPU from host positions (natoms x 3, any image) in an orthorhombic
 * box[3]: strict r < Rcut, minimum image, lists sorted by index, stride =
 * the largest count (<= 128).  Bitwise the lists of
 * snapgpu_build_neighborlist; replaces snapgpu_set_neighbors (all atoms
 * owned, one type).  snapgpu_get_neighbors reads them back. */
int snapgpu_set_positions(snapgpu_ctx* ctx, int natoms, const double* pos,
                          const double* box);
int snapgpu_get_neighbors(snapgpu_ctx* ctx, int* numneigh, int* nbr, double* disp);

/* One force step from host POSITIONS (the MD-loop call): the positions
 * (natoms x 3, any image, orthorhombic box[3]) are staged into pinned
 * memory, then ONE CUDA graph uploads them, rebuilds the neighbor lists on
 * the device (as snapgpu_set_positions, with the current stride as capacity:
 * no host round trip), derives the partner slots of the symmetric lists,
 * runs U -> Y(+E) -> fused dU/dE -> deterministic force gather and reads
 * forces (natoms x 3), eatom and etotal back; one stream synchronization.
 * The first call (or a new atom count / box, or a list outgrowing the
 * stride) takes the snapgpu_set_positions path first.  Any output may be
 * NULL.  Equivalent to build_neighborlist (harness.hpp:119-202) followed by
 * run_pipeline (pipeline.hpp:206-303). */
int snapgpu_run_positions(snapgpu_ctx* ctx, int natoms, const double* pos,
                          const double* box, double* forces, double* eatom,
                          double* etotal);

/* Bispectrum descriptors B_l(i) (compute_B_from_U,
 * snap_core.hpp:642-681, b_contract :556-575) of the owned atoms,
 * blist[i * ntriples + l], in one pass over Ulisttot (k_compute_B: every
 * canonical triple's coupling elements formed on the fly and contracted,
 * never stored).  Runs compute_U first if needed; Y', dElist and forces are
 * untouched. */
int snapgpu_compute_descriptors(snapgpu_ctx* ctx, double* blist);

/* Virial of the owned pairs from dElist (the paper keeps
 * dElist for it): out6 = W_xx, W_yy, W_zz, W_xy, W_xz, W_yz
 * with W_ab = sum_{i,k} r_ik,a f_ik,b, r_ik the center -> neighbor
 * displacement and f_ik = -dE(i,k) the force on the neighbor
 * (scatter_forces, snap_core.hpp:889-898).  Deterministic reduction; no
 * reference equivalent (checked against dElist from the oracle). */
int snapgpu_get_virial(snapgpu_ctx* ctx, double* out6);

/* Device pointers for collectives (valid until the next set_neighbors):
 * forces (natoms_total x 3, or the chunked layout), eatom nlocal, etotal 1. */
int snapgpu_device_outputs(snapgpu_ctx* ctx, double** forces, double** eatom,
                           double** etotal);

/* Stream-ordered device-to-device copy of the natoms_total x 3 force buffer
 * into caller memory (e.g. a torch tensor feeding an NCCL reduce-scatter). */
int snapgpu_get_forces_device(snapgpu_ctx* ctx, double* dst_device);
/* Same for the owned atoms' total energy (1 double); eatom_dst (nlocal) may
 * be NULL. */
int snapgpu_get_energy_device(snapgpu_ctx* ctx, double* eatom_dst,
                              double* etotal_dst);

/* Per-stage device times (ms) of the last snapgpu_run when timing is on:
 * out[0..3] = U, Y, dE, scatter. */
int snapgpu_enable_stage_timing(snapgpu_ctx* ctx, int on);
int snapgpu_stage_times(snapgpu_ctx* ctx, float* out4);

/* compute_Y launch knob (benchmark sweeps, 2J <= 8): CTAs per 32-atom tile
 * splitting its target rows, in [1, 8]; 0 = automatic (fill the SMs: the
 * first tiles get one part more). */
int snapgpu_tune(snapgpu_ctx* ctx, int y_parts);
/* compute_Y -> compute_fused_dE hand-off (2J <= 8): on (default), dE starts
 * per 32-atom tile as soon as compute_Y has written that tile's Y' (its CTAs
 * take the SMs of finished tiles); off, dE waits for the whole compute_Y
 * grid.  Results are bitwise identical.  Off by default when a tool is
 * injected (ncu, compute-sanitizer), which may serialize the grids. */
int snapgpu_set_overlap(snapgpu_ctx* ctx, int on);

/* Force output layout for the atom-partitioned multi-GPU step
 * (the coupling is scatter_forces snap_core.hpp:889-898 and
 * the energy sum :692-699).  nchunks = world size: atom a's force lands at
 * (a / k) * (3k + 1) + (a % k) * 3 with k = ceil(natoms_total / nchunks), and
 * slot r * (3k + 1) + 3k of every chunk r receives this context's total
 * energy, so ONE reduce-scatter (sum, chunk 3k + 1 doubles) hands rank r its
 * owned forces and the total energy.  ext_forces: caller-owned device buffer
 * of nchunks * (3k + 1) doubles that the force gather writes into (NULL: the
 * context's own buffer).  nchunks = 1 restores the plain natoms x 3 array.
 * Takes effect at the next neighbor-list upload. */
int snapgpu_set_force_layout(snapgpu_ctx* ctx, int nchunks, double* ext_forces);

/* ---- context-free host utilities --------------------------------------- */

/* Table sizes for a band limit (HalfIntIndexMaps, halfint_index.hpp:85-98):
 * out[0..5] = n_triples, n_tuples, u_full_total, u_half_total,
 * z_total_elements, cg_total. */
int snapgpu_counts(int twojmax, int* out6);

/* Host-only view of the compute_Y launch plan (2J <= 8; no device needed):
 * for ntiles 32-atom tiles on nsm SMs (y_parts > 0 forces the part count),
 * writes the CTA table (4 ints per CTA: tile, part | parts << 8, first row
 * list, list stride) and the row lists (codes j*64+mb, -1 terminated);
 * returns the CTA count, or a negative status. */
int snapgpu_debug_y_plan(int twojmax, int ntiles, int nsm, int y_parts, int* cta, int cta_cap,
                         int* tasks, int tasks_cap);

/* Periodic orthorhombic neighbor lists (harness.hpp:119-202, generalized
 * from cubic): strict r < rcut, minimum image, each list sorted by neighbor
 * index, displacement from center to neighbor.  Returns the maximum
 * neighbor count (>= 0) or a negative status.  When the maximum exceeds
 * maxstride only numneigh is written. */
int snapgpu_build_neighborlist(const double* positions, int n,
                               const double box[3], double rcut,
                               int maxstride, int* numneigh, int* nbr,
                               double* disp);

/* Diagnostic: FP64 DFMA throughput probe on `device` (all SMs, independent
 * DFMA chains).  tflops receives the measured FP64 rate, ms the duration. */
int snapgpu_fp64_peak(int device, int iters, double* tflops, double* ms);

/* Seeded BCC lattice (TestSNAP tungsten workload; not in the reference):
 * nx*ny*nz cells, edge a, z-major atom order ((cz*ny+cy)*nx+cx)*2+basis,
 * beta ~ U(-1,1) drawn first from an mt19937_64 seeded with `seed`
 * (rng.hpp:19-29, harness.hpp:208-213), then a uniform jitter in
 * [-jitter, jitter) per coordinate.  Returns the atom count. */
int snapgpu_bcc_lattice(int nx, int ny, int nz, double a, double jitter,
                        uint64_t seed, int twojmax, double* positions,
                        double* beta);

#ifdef __cplusplus
}
#endif
#endif /* SNAPGPU_H */
