/*
 * snap_oracle.h -- CPU restatement of the reference SNAP force path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity oracle for the B200 engine
 * in paper_2011_12875_b200/.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load it, and only as the checker.  The
 * product path never links or calls anything in oracle/.
 *
 * It restates, in plain C99 with the same floating-point operation order,
 * the deterministic `fused` path of the reference (snapforge, header-only
 * C++20 under /root/reference/proj/include/snapforge):
 *
 *   compute_U (half storage)          snap_core.hpp:369-489
 *   compute_Y (atom-owned path)       snap_core.hpp:1085-1171
 *   compute_fused_dE                  snap_core.hpp:1274-1406
 *   scatter_forces (serialized)       snap_core.hpp:872-899
 *   compute_B_from_U + compute_energy snap_core.hpp:642-701
 *
 * Parity is pinned: tests/test_oracle.py checks this port bitwise against
 * the reference itself (oracle/_ref, compiled from /root/reference by
 * oracle/Makefile) and against the committed golden fixtures in
 * tests/golden/ that were generated from oracle/_ref.
 *
 * Array conventions (shared with the product C-ABI, include/snapgpu.h):
 *   neighbor lists are flattened (atom, slot): nbr[i*stride+k],
 *   disp[(i*stride+k)*3+d], valid for k < numneigh[i];
 *   complex per-atom arrays are logical atom-major, interleaved re/im:
 *   x[(i*nidx + idx)*2 + {0,1}], idx in the half (2*mb <= t) index space.
 */
#ifndef SNAP_ORACLE_H
#define SNAP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int twojmax;
  double rcut, rmin0, rfac0, wself;
  int self_flag;
  const double* beta; /* n_triples(twojmax) */
  int nbeta;
  const double* weights; /* per-type neighbor weights */
  int nweights;
  int natoms, stride;
  const int* numneigh;  /* natoms */
  const int* nbr;       /* natoms*stride */
  const double* disp;   /* natoms*stride*3 */
  const int* types;     /* natoms or NULL (all type 0) */
} orc_problem;

const char* orc_last_error(void);

/* ---- index bookkeeping (halfint_index.hpp) ---- */
int orc_n_triples(int twojmax);
int orc_n_tuples(int twojmax);
int orc_u_half_total(int twojmax);
int orc_u_full_total(int twojmax);
int orc_z_total_elements(int twojmax);
int orc_cg_total(int twojmax);
/* triples[3*l] = (j1, j2, j); tuples[5*t] = (j1, j2, j, elem_off, cg_off) */
int orc_triples(int twojmax, int* out);
int orc_tuples(int twojmax, int* out);
int orc_cg_table(int twojmax, double* out);
void orc_z_loop_bounds(int j1, int j2, int j, int mb, int ma, int out[6]);

/* ---- per-pair math (angular_basis.hpp) ---- */
/* out: r, a.re, a.im, b.re, b.im, da[3] (re,im), db[3] (re,im), rhat[3]  (19) */
int orc_map_to_3sphere(const double disp[3], double rcut, double rmin0,
                       double rfac0, double* out);
/* half stack u (complex, u_half_total entries) */
int orc_wigner_u_half(const double disp[3], double rcut, double rmin0,
                      double rfac0, int twojmax, double* out);

/* ---- pipeline (deterministic fused path) ----
 * Any output pointer may be NULL.  ulisttot/ylist: natoms*u_half_total
 * complex (logical atom-major); delist natoms*stride*3; forces natoms*3;
 * eatom natoms; blist natoms*n_triples.
 */
int orc_run(const orc_problem* p, double* forces, double* eatom,
            double* etotal, double* ulisttot, double* ylist, double* delist,
            double* blist);

/* ---- problem generators ---- */
/* BCC lattice, z-major atom order ((cz*ny+cy)*nx+cx)*2+basis; beta drawn
 * first from Rng(seed) (harness.hpp:208-213 convention), then per-atom
 * jitter U(-jitter, jitter) per coordinate. */
int orc_bcc(int nx, int ny, int nz, double a, double jitter, uint64_t seed,
            int twojmax, double* positions /* 2*nx*ny*nz*3 */,
            double* beta /* n_triples */);
/* Periodic orthorhombic neighbor lists (harness.hpp:119-202, generalized).
 * Lists sorted by neighbor index.  Returns max neighbor count, or -1 on
 * error.  If maxstride < required, only counts are produced. */
int orc_build_neighborlist(const double* positions, int n, const double box[3],
                           double rcut, int maxstride, int* numneigh, int* nbr,
                           double* disp);
/* tests/test_support.hpp:21-64 (all-pairs cluster, ragged, typed).  Fills
 * positions(n*3), types(n), weights(ntypes), numneigh/nbr/disp with stride n,
 * beta.  Returns max neighbor count. */
int orc_make_cluster(int natoms, int twojmax, uint64_t seed, int ntypes,
                     double* positions, int* types, double* weights,
                     int* numneigh, int* nbr, double* disp, double* beta);
/* harness.hpp:230-262 fixed-shape synthetic lists (stride = nnbor). */
int orc_generate_synthetic(int natoms, int nnbor, int twojmax, double rcut,
                           uint64_t seed, int* numneigh, int* nbr,
                           double* disp, double* beta);

/* rng.hpp (for tests) */
void orc_rng_stream(uint64_t seed, int n, double* out_uniform01);

#ifdef __cplusplus
}
#endif
#endif
