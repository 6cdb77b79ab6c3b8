// kernels.cuh -- sm_100a FP64 kernels of the B200 SNAP force step.
//
// Stage map (reference: /root/reference/proj/include/snapforge/snap_core.hpp):
//   k_compute_U        compute_U            :369-489   (fused with the 3-sphere
//                                                        map + switching function)
//   k_compute_Y_spec   compute_Y            :1085-1200  (twojmax in {2,4,6,8};
//   k_compute_Y_gen                                      generic for any twojmax)
//                      + per-atom energy (replaces compute_B_from_U :642 and
//                        compute_energy :684 through E_i = 1/3 sum Y:U*)
//   k_fused_dE         compute_fused_dE     :1274-1406 (dU never reaches HBM)
//   k_scatter_forces   scatter_forces       :872-953
//
// All arithmetic is FP64 on the SIMT pipe (the CG contraction is sparse;
// no tensor-core path exists for it).  Every kernel works in "v-space"
// (tables.hpp): v = f u with f(t,mb,ma) = sqrt((t-mb)!/((t-ma)! ma!)), so the
// Wigner level recursion is coefficient free,
//     v(t,mb,ma) = conj(a) v(t-1,mb,ma) - conj(b) v(t-1,mb,ma-1),
// and the derivative recursion is its product rule.  The scale factors are
// folded into the host-built C' / W tables and into the stored Y'.
//
// HBM layouts:
//   V  (ulisttot, v-space)       [atom/32][re|im][half idx][atom%32]  (AoSoA 32,
//   Y' (ylist, v-space, weighted) same                                 split planes)
//   dedr                          [atom][slot][3]
//   forces                        [atom][3]
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace snapgpu {

constexpr double kPi = 3.14159265358979323846;

// ---------------------------------------------------------------------------
// compile-time index bookkeeping (halfint_index.hpp:155-200)
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int c_half_off(int t) {
  int o = 0;
  for (int s = 0; s < t; ++s) o += (s / 2 + 1) * (s + 1);
  return o;
}
__host__ __device__ constexpr int c_full_off(int t) {
  int o = 0;
  for (int s = 0; s < t; ++s) o += (s + 1) * (s + 1);
  return o;
}
__host__ __device__ constexpr int c_cg_off(int T, int J1, int J2, int J) {
  int o = 0;
  for (int j1 = 0; j1 <= T; ++j1)
    for (int j2 = 0; j2 <= j1; ++j2)
      for (int j = j1 - j2; j <= (j1 + j2 < T ? j1 + j2 : T); j += 2) {
        if (j1 == J1 && j2 == J2 && j == J) return o;
        o += (j1 + 1) * (j2 + 1);
      }
  return -1;
}
__host__ __device__ constexpr int c_cg_total(int T) {
  int o = 0;
  for (int j1 = 0; j1 <= T; ++j1)
    for (int j2 = 0; j2 <= j1; ++j2)
      for (int j = j1 - j2; j <= (j1 + j2 < T ? j1 + j2 : T); j += 2) o += (j1 + 1) * (j2 + 1);
  return o;
}
__host__ __device__ constexpr int c_acc_off(int t) {  // sum_{s<t} (s/2+1)
  int o = 0;
  for (int s = 0; s < t; ++s) o += s / 2 + 1;
  return o;
}
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }

// The specialized compute_Y kernels keep their C' coefficient tables in
// constant memory (DFMA takes a constant-bank operand for free).
__host__ __device__ constexpr bool y_specialized(int T) {
  return T == 2 || T == 4 || T == 6 || T == 8;
}
__host__ __device__ constexpr int cp_base(int T) {
  int o = 0;
  for (int s = 2; s < T; s += 2) o += c_cg_total(s);
  return o;
}
constexpr int kCpTotal = c_cg_total(2) + c_cg_total(4) + c_cg_total(6) + c_cg_total(8);
__constant__ double cCP[kCpTotal];

// ---------------------------------------------------------------------------
// kernel argument blocks
// ---------------------------------------------------------------------------
struct GeoParams {
  double rcut, rmin0, rfac0, wself;
  int self_flag;
};

struct PairArgs {
  int nlocal, stride, atom_lo;
  const int* numneigh;    // nlocal
  const int* nbr;         // nlocal*stride (global indices)
  const double* disp;     // nlocal*stride*3
  const int* types;       // natoms_total or null
  const double* weights;  // per type
};

// ---------------------------------------------------------------------------
// per-pair geometry: map_to_3sphere (angular_basis.hpp:102-139),
// switching_function (:78-87), pair_weights (snap_core.hpp:353-359)
// ---------------------------------------------------------------------------
struct PairGeo {
  double ar, ai, br, bi;
  double sfac;
  double dar[3], dai[3], dbr[3], dbi[3];
  double dsf[3];  // dsfac * rhat[d]
};

template <bool GRAD>
__device__ __forceinline__ void pair_geometry(double x, double y, double z, double w,
                                              const GeoParams& P, PairGeo& g) {
  const double rsq = x * x + y * y + z * z;
  const double r = sqrt(rsq);
  const double rscale0 = P.rfac0 * kPi / (P.rcut - P.rmin0);
  const double theta0 = (r - P.rmin0) * rscale0;
  const double z0 = r / tan(theta0);
  const double r0inv = 1.0 / sqrt(rsq + z0 * z0);
  g.ar = r0inv * z0;
  g.ai = -r0inv * z;
  g.br = r0inv * y;
  g.bi = -r0inv * x;
  double fc, dfc;
  if (r <= P.rmin0) {
    fc = 1.0;
    dfc = 0.0;
  } else if (r >= P.rcut) {
    fc = 0.0;
    dfc = 0.0;
  } else {
    const double scale = kPi / (P.rcut - P.rmin0);
    double s, c;
    sincos((r - P.rmin0) * scale, &s, &c);
    fc = 0.5 * (c + 1.0);
    dfc = -0.5 * s * scale;
  }
  g.sfac = w * fc;
  if (GRAD) {
    const double dz0dr = z0 / r - (r * rscale0) * (rsq + z0 * z0) / rsq;
    const double dr0invdr = -r0inv * r0inv * r0inv * (r + z0 * dz0dr);
    const double rinv = 1.0 / r;
    const double rhat[3] = {x * rinv, y * rinv, z * rinv};
    const double dsfac = w * dfc;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double dr0inv = dr0invdr * rhat[k];
      g.dar[k] = dz0dr * rhat[k] * r0inv + z0 * dr0inv;
      g.dai[k] = -z * dr0inv;
      g.dbr[k] = y * dr0inv;
      g.dbi[k] = -x * dr0inv;
      g.dsf[k] = dsfac * rhat[k];
    }
    g.dai[2] += -r0inv;
    g.dbi[0] += -r0inv;
    g.dbr[1] += r0inv;
  }
}

__device__ __forceinline__ double neighbor_weight(const PairArgs& A, int j) {
  return A.weights[A.types ? A.types[j] : 0];
}

// sqrt(2/t): the v-space scale between row t/2 and the mirror of row t/2-1
// at level t-1.
__host__ __device__ constexpr double mirror_R(int t) {
  return t == 2 ? 1.0
       : t == 4 ? 0.70710678118654752440
       : t == 6 ? 0.57735026918962576451
       : t == 8 ? 0.5
       : t == 10 ? 0.44721359549995793928
       : t == 12 ? 0.40824829046386301637
       : t == 14 ? 0.37796447300922722721
       : t == 16 ? 0.35355339059327376220
                 : 0.0;
}

// ===========================================================================
// compute_U  (snap_core.hpp:369-489)
//
// One warp per atom.  Lanes = (pair slot, column ma): NSLOT = 32/(T+1) pairs
// of the atom are walked at once, each by T+1 lanes holding one column of
// the level being built (rows mb <= t/2 in registers).  The recursion needs
// only the left neighbor column (shfl_up) and, when a middle row appears at
// an even level, two mirrored columns of the row above.  Accumulation over
// the atom's neighbors stays in registers (T <= 8) or lane-private shared
// memory (T > 8); one cross-slot shuffle reduction at the end, then the
// atom's V row is written once: no global atomics.
// ===========================================================================
struct UArgs {
  PairArgs pr;
  GeoParams gp;
  double* V;  // [tile][2][NH][32]
};

template <int T>
struct UCfg {
  static constexpr int NC = T + 1;
  static constexpr int NSLOT = 32 / NC;
  static constexpr int NROW = T / 2 + 1;
  static constexpr int NACC = c_acc_off(T + 1);
  static constexpr int NH = c_half_off(T + 1);
  static constexpr bool REGACC = T <= 8;
  static constexpr int WARPS = REGACC ? 4 : 2;
};

template <int T, bool REG>
struct UAcc;

template <int T>
struct UAcc<T, true> {
  double r[UCfg<T>::NACC], i[UCfg<T>::NACC];
  __device__ __forceinline__ void init(double*, int) {
#pragma unroll
    for (int q = 0; q < UCfg<T>::NACC; ++q) r[q] = i[q] = 0.0;
  }
  __device__ __forceinline__ void add(int q, double s, double vr, double vi) {
    r[q] = fma(s, vr, r[q]);
    i[q] = fma(s, vi, i[q]);
  }
  __device__ __forceinline__ double getr(int q) const { return r[q]; }
  __device__ __forceinline__ double geti(int q) const { return i[q]; }
};

template <int T>
struct UAcc<T, false> {  // lane-private slots: [q][re|im][32]
  double* base;
  __device__ __forceinline__ void init(double* smem_warp, int lane) {
    base = smem_warp + lane;
#pragma unroll 4
    for (int q = 0; q < 2 * UCfg<T>::NACC; ++q) base[q * 32] = 0.0;
  }
  __device__ __forceinline__ void add(int q, double s, double vr, double vi) {
    base[(2 * q) * 32] = fma(s, vr, base[(2 * q) * 32]);
    base[(2 * q + 1) * 32] = fma(s, vi, base[(2 * q + 1) * 32]);
  }
  __device__ __forceinline__ double getr(int q) const { return base[(2 * q) * 32]; }
  __device__ __forceinline__ double geti(int q) const { return base[(2 * q + 1) * 32]; }
};

template <int T>
__global__ void __launch_bounds__(UCfg<T>::WARPS * 32)
    k_compute_U(const UArgs A) {
  using C = UCfg<T>;
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * C::WARPS + w;
  if (i >= A.pr.nlocal) return;  // whole warp
  const int S = A.pr.stride;
  const int nn = A.pr.numneigh[i];
  // shared: per warp geometry [S][5], then (T > 8) accumulators [2*NACC][32]
  double* geo = smem + (size_t)w * S * 5;
  double* accs = smem + (size_t)C::WARPS * S * 5 + (size_t)w * 2 * C::NACC * 32;

  for (int k = lane; k < nn; k += 32) {
    const size_t pk = (size_t)i * S + k;
    const double* d = A.pr.disp + pk * 3;
    PairGeo g;
    pair_geometry<false>(d[0], d[1], d[2], neighbor_weight(A.pr, A.pr.nbr[pk]), A.gp, g);
    geo[k * 5 + 0] = g.ar;
    geo[k * 5 + 1] = g.ai;
    geo[k * 5 + 2] = g.br;
    geo[k * 5 + 3] = g.bi;
    geo[k * 5 + 4] = g.sfac;
  }
  __syncwarp();

  const int slot = lane / C::NC;
  const int c = lane - slot * C::NC;
  const int sbase = slot * C::NC;
  UAcc<T, C::REGACC> acc;
  acc.init(accs, lane);

  for (int k0 = 0; k0 < nn; k0 += C::NSLOT) {
    const int k = k0 + slot;
    double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0, sf = 0.0;
    if (slot < C::NSLOT && k < nn) {
      ar = geo[k * 5 + 0];
      ai = geo[k * 5 + 1];
      br = geo[k * 5 + 2];
      bi = geo[k * 5 + 3];
      sf = geo[k * 5 + 4];
    }
    double vr[C::NROW], vi[C::NROW];
#pragma unroll
    for (int mb = 0; mb < C::NROW; ++mb) vr[mb] = vi[mb] = 0.0;
    vr[0] = (c == 0) ? 1.0 : 0.0;
    acc.add(0, sf, vr[0], 0.0);
#pragma unroll
    for (int t = 1; t <= T; ++t) {
      // left-column values of the rows that exist at level t-1
      double qr[C::NROW], qi[C::NROW];
#pragma unroll
      for (int mb = 0; 2 * mb <= t - 1; ++mb) {
        const double sr = __shfl_up_sync(0xffffffffu, vr[mb], 1);
        const double si = __shfl_up_sync(0xffffffffu, vi[mb], 1);
        qr[mb] = (c == 0) ? 0.0 : sr;
        qi[mb] = (c == 0) ? 0.0 : si;
      }
      double pmr = 0.0, pmi = 0.0, qmr = 0.0, qmi = 0.0;
      if ((t & 1) == 0) {
        // new middle row t/2 from the mirror of row t/2-1 at level t-1
        const int m = t / 2 - 1;
        const bool ok1 = c <= t - 1, ok2 = (c >= 1) && (c <= t);
        const int src1 = sbase + (ok1 ? (t - 1 - c) : 0);
        const int src2 = sbase + (ok2 ? (t - c) : 0);
        const double s1r = __shfl_sync(0xffffffffu, vr[m], src1);
        const double s1i = __shfl_sync(0xffffffffu, vi[m], src1);
        const double s2r = __shfl_sync(0xffffffffu, vr[m], src2);
        const double s2i = __shfl_sync(0xffffffffu, vi[m], src2);
        const double R = mirror_R(t);
        const double sg = ((c + t / 2) & 1) ? -R : R;  // (-1)^(c+t/2) R
        pmr = ok1 ? sg * s1r : 0.0;
        pmi = ok1 ? -sg * s1i : 0.0;
        qmr = ok2 ? -sg * s2r : 0.0;  // (-1)^(c-1+t/2) R
        qmi = ok2 ? sg * s2i : 0.0;
      }
#pragma unroll
      for (int mb = 0; 2 * mb <= t - 1; ++mb) {
        const double pr = vr[mb], pi = vi[mb];
        vr[mb] = ar * pr + ai * pi - br * qr[mb] - bi * qi[mb];
        vi[mb] = ar * pi - ai * pr - br * qi[mb] + bi * qr[mb];
      }
      if ((t & 1) == 0) {
        const int m = t / 2;
        vr[m] = ar * pmr + ai * pmi - br * qmr - bi * qmi;
        vi[m] = ar * pmi - ai * pmr - br * qmi + bi * qmr;
      }
#pragma unroll
      for (int mb = 0; 2 * mb <= t; ++mb) acc.add(c_acc_off(t) + mb, sf, vr[mb], vi[mb]);
    }
  }

  // reduce the pair slots onto slot 0 and write the atom's row once
  double outr[C::NACC], outi[C::NACC];
#pragma unroll
  for (int q = 0; q < C::NACC; ++q) {
    double r = acc.getr(q), im = acc.geti(q);
#pragma unroll
    for (int s = 1; s < C::NSLOT; ++s) {
      r += __shfl_down_sync(0xffffffffu, acc.getr(q), s * C::NC);
      im += __shfl_down_sync(0xffffffffu, acc.geti(q), s * C::NC);
    }
    outr[q] = r;
    outi[q] = im;
  }
  if (slot == 0) {
    const int tile = i >> 5, ln = i & 31;
    double* Vr = A.V + ((size_t)tile * 2 * C::NH) * 32 + ln;
    double* Vi = Vr + (size_t)C::NH * 32;
#pragma unroll
    for (int t = 0; t <= T; ++t) {
      if (c > t) continue;
#pragma unroll
      for (int mb = 0; 2 * mb <= t; ++mb) {
        double r = outr[c_acc_off(t) + mb];
        if (A.gp.self_flag && c == mb) {  // wself * f(t,mb,mb) = wself/sqrt(mb!)
          const double inv_sqrt_fact[8] = {1.0, 1.0, 0.70710678118654752440,
                                           0.40824829046386301637, 0.20412414523193150819,
                                           0.091287092917527685576, 0.037267799624996494940,
                                           0.014085904245475275327};
          r += A.gp.wself * inv_sqrt_fact[mb];
        }
        const int h = c_half_off(t) + mb * (t + 1) + c;
        Vr[(size_t)h * 32] = r;
        Vi[(size_t)h * 32] = outi[c_acc_off(t) + mb];
      }
    }
  }
}

// ===========================================================================
// compute_Y, specialized (snap_core.hpp:1085-1200)
//
// CTA = one AoSoA tile of 32 atoms (lane = atom, so every lane runs the same
// loop bounds and reads the same coefficient) x one "part" of the target
// rows.  The tile's V is expanded once into shared memory as the full
// mirrored stack X (split planes [re|im][full idx][32]: conflict-free LDS).
// Each warp owns whole target rows (j, mb) and accumulates the row's j+1
// outputs in registers across every coupling tuple (j1, j2) -> j and every
// contributing row pair (mb1, mb2): per row pair it loads X row mb1 of level
// j1 and row mb2 of level j2 into registers and runs the fully unrolled
// (ma1, ma2) product body with C' coefficients from constant memory, so each
// loaded complex feeds ~2 complex MACs.  Output: Y' (v-space, weighted).
// Epilogue: per-atom energy E_i = 2/3 sum_{stored} Re(Y'_s conj V).
// ===========================================================================
struct YArgs {
  const double* V;      // [tile][2][NH][32]
  double* Y;            // [tile][2][NH][32]
  const double* W;      // W table (cg layout)
  const int* expand;    // full idx -> src code
  const int* tasks;     // [worker][cap]
  int task_cap;
  int nlocal;
  double* eatom;        // nlocal (accumulated with atomics)
};

template <int T, int J1, int J2, int J>
__device__ __forceinline__ void y_tuple_rows(const double* __restrict__ sX, int lane, int mb,
                                             const double* __restrict__ W, double (&accr)[J + 1],
                                             double (&acci)[J + 1]) {
  constexpr int NF = c_full_off(T + 1);
  constexpr int D = (J1 + J2 - J) / 2;
  constexpr int COFF = c_cg_off(T, J1, J2, J);
  constexpr int CB = cp_base(T) + COFF;
  const int lo = max(0, mb + D - J2), hi = min(J1, mb + D);
  for (int mb1 = lo; mb1 <= hi; ++mb1) {
    const int mb2 = mb + D - mb1;
    const double w = __ldg(W + COFF + mb1 * (J2 + 1) + mb2);
    const double* p1 = sX + (c_full_off(J1) + mb1 * (J1 + 1)) * 32 + lane;
    const double* p2 = sX + (c_full_off(J2) + mb2 * (J2 + 1)) * 32 + lane;
    double x1r[J1 + 1], x1i[J1 + 1], x2r[J2 + 1], x2i[J2 + 1];
#pragma unroll
    for (int a = 0; a <= J1; ++a) {
      x1r[a] = p1[a * 32];
      x1i[a] = p1[(NF + a) * 32];
    }
#pragma unroll
    for (int a = 0; a <= J2; ++a) {
      x2r[a] = p2[a * 32];
      x2i[a] = p2[(NF + a) * 32];
    }
#pragma unroll
    for (int ma = 0; ma <= J; ++ma) {
      const int alo = cmax(0, ma + D - J2), ahi = cmin(J1, ma + D);
      double sr = 0.0, si = 0.0;
#pragma unroll
      for (int a1 = alo; a1 <= ahi; ++a1) {
        const int a2 = ma + D - a1;
        const double cc = cCP[CB + a1 * (J2 + 1) + a2];
        const double tr = x1r[a1] * x2r[a2] - x1i[a1] * x2i[a2];
        const double ti = x1r[a1] * x2i[a2] + x1i[a1] * x2r[a2];
        sr = fma(cc, tr, sr);
        si = fma(cc, ti, si);
      }
      accr[ma] = fma(w, sr, accr[ma]);
      acci[ma] = fma(w, si, acci[ma]);
    }
  }
}

// Compile-time walk over every coupling tuple (J1 >= J2) that targets J.
template <int T, int J, int J1, int J2>
struct YTupleWalk {
  __device__ __forceinline__ static void run(const double* sX, int lane, int mb, const double* W,
                                             double (&ar)[J + 1], double (&ai)[J + 1]) {
    if constexpr (J1 <= T) {
      if constexpr (J2 <= J1) {
        constexpr bool ok = (J >= J1 - J2) && (J <= J1 + J2) && (((J1 + J2 - J) & 1) == 0);
        if constexpr (ok) y_tuple_rows<T, J1, J2, J>(sX, lane, mb, W, ar, ai);
        YTupleWalk<T, J, J1, J2 + 1>::run(sX, lane, mb, W, ar, ai);
      } else {
        YTupleWalk<T, J, J1 + 1, 0>::run(sX, lane, mb, W, ar, ai);
      }
    }
  }
};

template <int T, int J>
__device__ __forceinline__ void y_row(const double* sX, int lane, int mb, const YArgs& A,
                                      double* __restrict__ Yt, double& e_acc) {
  constexpr int NF = c_full_off(T + 1);
  constexpr int NH = c_half_off(T + 1);
  double ar[J + 1], ai[J + 1];
#pragma unroll
  for (int m = 0; m <= J; ++m) ar[m] = ai[m] = 0.0;
  YTupleWalk<T, J, 0, 0>::run(sX, lane, mb, A.W, ar, ai);
  const bool mid = (2 * mb == J);
  const int hb = c_half_off(J) + mb * (J + 1);
  const int fb = c_full_off(J) + mb * (J + 1);
#pragma unroll
  for (int ma = 0; ma <= J; ++ma) {
    double wgt = 1.0;
    if (mid) wgt = (2 * ma < J) ? 1.0 : ((2 * ma == J) ? 0.5 : 0.0);
    const double yr = ar[ma] * wgt, yi = ai[ma] * wgt;
    Yt[(size_t)(hb + ma) * 32] = yr;
    Yt[(size_t)(NH + hb + ma) * 32] = yi;
    e_acc += yr * sX[(fb + ma) * 32 + lane] + yi * sX[(NF + fb + ma) * 32 + lane];
  }
}

template <int T>
__global__ void __launch_bounds__(512, 1) k_compute_Y_spec(const YArgs A) {
  constexpr int NF = c_full_off(T + 1);
  constexpr int NH = c_half_off(T + 1);
  extern __shared__ double sX[];  // [2][NF][32]
  const int tile = blockIdx.x;
  const double* Vt = A.V + (size_t)tile * 2 * NH * 32;
  for (int e = threadIdx.x; e < NF * 32; e += blockDim.x) {
    const int f = e >> 5, ln = e & 31;
    const int code = __ldg(A.expand + f);
    const int src = code >> 2;
    double re = Vt[src * 32 + ln], im = Vt[(NH + src) * 32 + ln];
    if (code & 2) im = -im;
    if (code & 1) {
      re = -re;
      im = -im;
    }
    sX[f * 32 + ln] = re;
    sX[(NF + f) * 32 + ln] = im;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int worker = blockIdx.y * (blockDim.x >> 5) + w;
  const int* tasks = A.tasks + (size_t)worker * A.task_cap;
  double* Yt = A.Y + (size_t)tile * 2 * NH * 32 + lane;
  double e_acc = 0.0;
  for (int q = 0;; ++q) {
    const int code = __ldg(tasks + q);
    if (code < 0) break;
    const int j = code >> 6, mb = code & 63;
    switch (j) {
      case 0: y_row<T, 0>(sX, lane, mb, A, Yt, e_acc); break;
      case 1: if constexpr (T >= 1) y_row<T, 1>(sX, lane, mb, A, Yt, e_acc); break;
      case 2: if constexpr (T >= 2) y_row<T, 2>(sX, lane, mb, A, Yt, e_acc); break;
      case 3: if constexpr (T >= 3) y_row<T, 3>(sX, lane, mb, A, Yt, e_acc); break;
      case 4: if constexpr (T >= 4) y_row<T, 4>(sX, lane, mb, A, Yt, e_acc); break;
      case 5: if constexpr (T >= 5) y_row<T, 5>(sX, lane, mb, A, Yt, e_acc); break;
      case 6: if constexpr (T >= 6) y_row<T, 6>(sX, lane, mb, A, Yt, e_acc); break;
      case 7: if constexpr (T >= 7) y_row<T, 7>(sX, lane, mb, A, Yt, e_acc); break;
      case 8: if constexpr (T >= 8) y_row<T, 8>(sX, lane, mb, A, Yt, e_acc); break;
      default: break;
    }
  }
  const int atom = tile * 32 + lane;
  if (atom < A.nlocal) atomicAdd(A.eatom + atom, (2.0 / 3.0) * e_acc);
}

// ===========================================================================
// compute_Y, generic (any twojmax <= 14): per target element, runtime loops,
// u-space tile in shared memory with on-the-fly mirror (UtotView::get,
// snap_core.hpp:190-199).  TA atoms per CTA tile, 32/TA sublanes split the
// mb1 loop.  Used for twojmax outside the specialized set.
// ===========================================================================
struct YGArgs {
  const double* V;
  double* Y;
  const double* cg;        // CG table (reference layout)
  const double* bfold;     // fold_beta per tuple
  const int* tuples;       // [ntup][5] j1 j2 j elem cg_off
  const int* elem_info;    // [nelem][6]
  const int* elem_tups;
  const int* tasks;        // [worker][cap]
  int task_cap;
  const double* hf;        // f per half idx
  const double* ywgt;      // stored-Y weight per half idx
  const int* half_off;     // T+2
  int T, NH, nlocal;
  double* eatom;
};

template <int TA>
__global__ void __launch_bounds__(256) k_compute_Y_gen(const YGArgs A) {
  constexpr int SUB = 32 / TA;
  extern __shared__ double sU[];  // [2][NH][TA] u-space
  const int NH = A.NH;
  const int a0 = blockIdx.x * TA;  // first atom of the CTA tile
  for (int e = threadIdx.x; e < NH * TA; e += blockDim.x) {
    const int h = e / TA, ln = e - h * TA;
    const int atom = a0 + ln;
    const double* Vt = A.V + (size_t)(atom >> 5) * 2 * NH * 32 + (atom & 31);
    const double inv = 1.0 / A.hf[h];
    sU[h * TA + ln] = Vt[(size_t)h * 32] * inv;
    sU[(NH + h) * TA + ln] = Vt[(size_t)(NH + h) * 32] * inv;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ln = lane % TA, sub = lane / TA;
  const int worker = blockIdx.y * (blockDim.x >> 5) + w;
  const int* tasks = A.tasks + (size_t)worker * A.task_cap;
  const int atom = a0 + ln;
  double* Yt = A.Y + (size_t)(atom >> 5) * 2 * NH * 32 + (atom & 31);
  double e_acc = 0.0;
  auto getU = [&](int t, int mb, int ma, double& re, double& im) {
    const bool mir = 2 * mb > t;
    const int mbs = mir ? t - mb : mb, mas = mir ? t - ma : ma;
    const int h = A.half_off[t] + mbs * (t + 1) + mas;
    re = sU[h * TA + ln];
    im = sU[(NH + h) * TA + ln];
    if (mir) {
      const double sg = ((ma + mb) & 1) ? -1.0 : 1.0;
      re *= sg;
      im *= -sg;
    }
  };
  for (int q = 0;; ++q) {
    const int eid = __ldg(A.tasks + (size_t)worker * A.task_cap + q);
    if (eid < 0) break;
    const int* ei = A.elem_info + eid * 6;
    const int j = ei[0], mb = ei[1], ma = ei[2], h = ei[3];
    double yr = 0.0, yi = 0.0;
    for (int tq = ei[4]; tq < ei[5]; ++tq) {
      const int tid = A.elem_tups[tq];
      const int* tp = A.tuples + tid * 5;
      const int j1 = tp[0], j2 = tp[1], cgo = tp[4];
      const int D = (j1 + j2 - j) / 2;
      const int mblo = max(0, mb + D - j2), mbhi = min(j1, mb + D);
      const int malo = max(0, ma + D - j2), mahi = min(j1, ma + D);
      double zr = 0.0, zi = 0.0;
      for (int mb1 = mblo + sub; mb1 <= mbhi; mb1 += SUB) {
        const int mb2 = mb + D - mb1;
        double sr = 0.0, si = 0.0;
        for (int ma1 = malo; ma1 <= mahi; ++ma1) {
          const int ma2 = ma + D - ma1;
          double u1r, u1i, u2r, u2i;
          getU(j1, mb1, ma1, u1r, u1i);
          getU(j2, mb2, ma2, u2r, u2i);
          const double cc = __ldg(A.cg + cgo + ma1 * (j2 + 1) + ma2);
          sr += cc * (u1r * u2r - u1i * u2i);
          si += cc * (u1r * u2i + u1i * u2r);
        }
        const double cb = __ldg(A.cg + cgo + mb1 * (j2 + 1) + mb2);
        zr += cb * sr;
        zi += cb * si;
      }
      const double bf = __ldg(A.bfold + tid);
      yr += bf * zr;
      yi += bf * zi;
    }
#pragma unroll
    for (int o = TA; o < 32; o <<= 1) {
      yr += __shfl_xor_sync(0xffffffffu, yr, o);
      yi += __shfl_xor_sync(0xffffffffu, yi, o);
    }
    const double sc = A.ywgt[h] / A.hf[h];
    const double ysr = yr * sc, ysi = yi * sc;
    if (sub == 0) {
      Yt[(size_t)h * 32] = ysr;
      Yt[(size_t)(NH + h) * 32] = ysi;
      double ur, ui;
      getU(j, mb, ma, ur, ui);
      e_acc += A.hf[h] * (ysr * ur + ysi * ui);  // Re(Y'_s conj V), V = f u
    }
  }
  if (sub == 0 && atom < A.nlocal) atomicAdd(A.eatom + atom, (2.0 / 3.0) * e_acc);
}

// ===========================================================================
// compute_fused_dE  (snap_core.hpp:1274-1406): compute_dU fused with
// compute_deidrj.  Lanes = (pair, row mb): a group of G lanes walks one pair,
// lane r owning row r of the current level (v and NDIR gradient rows in
// registers, T+1 columns).  Rows advance in place (the recursion is local to
// a row); a new middle row at even level t is seeded from the mirror of
// row t/2-1 (one shfl_up per column); the last middle row (level T, even T)
// is produced transiently by the lane holding row T/2-1 and contracted at
// once.  Each element is contracted against Y' as soon as it exists, so
// neither u, du nor dU ever leaves registers.  dE(pair) = 2 (dsf Au + sfac Ad).
// ===========================================================================
struct DEArgs {
  PairArgs pr;
  GeoParams gp;
  const double* Y;  // Y' stored
  double* dedr;     // [nlocal*stride][3]
  int nslots;       // nlocal*stride
};

template <int T>
struct DECfg {
  static constexpr int NL = T == 0 ? 1 : ((T & 1) == 0 ? T / 2 : (T + 1) / 2);
  static constexpr int G = NL <= 1 ? 1 : NL <= 2 ? 2 : NL <= 4 ? 4 : NL <= 8 ? 8 : 16;
  static constexpr int PPW = 32 / G;
  static constexpr int NC = T + 1;
  static constexpr int NH = c_half_off(T + 1);
  static constexpr int NDIR = T <= 8 ? 3 : 1;
  static constexpr int WARPS = 4;
};

template <int T>
__global__ void __launch_bounds__(DECfg<T>::WARPS * 32, (T <= 8 ? 2 : 3))
    k_fused_dE(const DEArgs A) {
  using C = DECfg<T>;
  constexpr int NDIR = C::NDIR;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = lane % C::G, q = lane / C::G;
  const int p = (blockIdx.x * C::WARPS + w) * C::PPW + q;
  const int S = A.pr.stride;
  const int i = p / S, k = p - i * S;
  const bool valid = (p < A.nslots) && (k < A.pr.numneigh[min(i, A.pr.nlocal - 1)]);
  double x = 1.0, y = 0.0, z = 0.0, wt = 0.0;
  if (valid) {
    const double* d = A.pr.disp + (size_t)p * 3;
    x = d[0];
    y = d[1];
    z = d[2];
    wt = neighbor_weight(A.pr, A.pr.nbr[p]);
  }
  PairGeo g;
  pair_geometry<true>(x, y, z, wt, A.gp, g);
  const int ia = valid ? i : 0;
  const double* Yr = A.Y + (size_t)(ia >> 5) * 2 * C::NH * 32 + (ia & 31);
  const double* Yi = Yr + (size_t)C::NH * 32;

  double Au = (r == 0) ? Yr[0] : 0.0;  // level 0: v = 1
  double Ad[3] = {0.0, 0.0, 0.0};
  const double ar = g.ar, ai = g.ai, br = g.br, bi = g.bi;

  for (int pass = 0; pass < 3 / NDIR; ++pass) {
    double dar[NDIR], dai[NDIR], dbr[NDIR], dbi[NDIR];
#pragma unroll
    for (int d = 0; d < NDIR; ++d) {
      const int dd = pass * NDIR + d;
      dar[d] = g.dar[dd];
      dai[d] = g.dai[dd];
      dbr[d] = g.dbr[dd];
      dbi[d] = g.dbi[dd];
    }
    double vr[C::NC], vi[C::NC], dvr[NDIR][C::NC], dvi[NDIR][C::NC];
#pragma unroll
    for (int c = 0; c < C::NC; ++c) {
      vr[c] = vi[c] = 0.0;
#pragma unroll
      for (int d = 0; d < NDIR; ++d) dvr[d][c] = dvi[d][c] = 0.0;
    }
    vr[0] = (r == 0) ? 1.0 : 0.0;
    double au = 0.0, ad[NDIR];
#pragma unroll
    for (int d = 0; d < NDIR; ++d) ad[d] = 0.0;

#pragma unroll
    for (int t = 1; t <= T; ++t) {
      // (1) seed a new middle row (row t/2) from the mirror of row t/2-1
      if ((t & 1) == 0 && t < T + ((T & 1) ? 1 : 0)) {
        const bool creator = (2 * r == t);
        const double R = mirror_R(t);
#pragma unroll
        for (int c = 0; c < t; ++c) {
          const double K = (((c + t / 2) & 1) ? -R : R);
          const double sr = __shfl_up_sync(0xffffffffu, vr[t - 1 - c], 1);
          const double si = __shfl_up_sync(0xffffffffu, vi[t - 1 - c], 1);
          if (creator) {
            vr[c] = K * sr;
            vi[c] = -K * si;
          }
#pragma unroll
          for (int d = 0; d < NDIR; ++d) {
            const double dsr = __shfl_up_sync(0xffffffffu, dvr[d][t - 1 - c], 1);
            const double dsi = __shfl_up_sync(0xffffffffu, dvi[d][t - 1 - c], 1);
            if (creator) {
              dvr[d][c] = K * dsr;
              dvi[d][c] = -K * dsi;
            }
          }
        }
      }
      // (2) transient last middle row (level T, even T): lane T/2-1, from its
      //     own level T-1 row before the in-place update
      if (t == T && (T & 1) == 0) {
        if (2 * r + 2 == T) {
          const double R = mirror_R(T);
          const int hb = c_half_off(T) + (T / 2) * (T + 1);
          double plr = 0.0, pli = 0.0, dplr[NDIR], dpli[NDIR];
#pragma unroll
          for (int d = 0; d < NDIR; ++d) dplr[d] = dpli[d] = 0.0;
#pragma unroll
          for (int c = 0; c <= T / 2; ++c) {
            double pr = 0.0, pi = 0.0, dpr[NDIR], dpi[NDIR];
            const double K = (((c + T / 2) & 1) ? -R : R);
#pragma unroll
            for (int d = 0; d < NDIR; ++d) dpr[d] = dpi[d] = 0.0;
            if (c <= T - 1) {
              pr = K * vr[T - 1 - c];
              pi = -K * vi[T - 1 - c];
#pragma unroll
              for (int d = 0; d < NDIR; ++d) {
                dpr[d] = K * dvr[d][T - 1 - c];
                dpi[d] = -K * dvi[d][T - 1 - c];
              }
            }
            const double nr = ar * pr + ai * pi - br * plr - bi * pli;
            const double ni = ar * pi - ai * pr - br * pli + bi * plr;
            const double yr = Yr[(size_t)(hb + c) * 32], yi = Yi[(size_t)(hb + c) * 32];
            if (pass == 0) au += nr * yr + ni * yi;
#pragma unroll
            for (int d = 0; d < NDIR; ++d) {
              const double ndr = dar[d] * pr + dai[d] * pi + ar * dpr[d] + ai * dpi[d] -
                                 dbr[d] * plr - dbi[d] * pli - br * dplr[d] - bi * dpli[d];
              const double ndi = dar[d] * pi - dai[d] * pr + ar * dpi[d] - ai * dpr[d] -
                                 dbr[d] * pli + dbi[d] * plr - br * dpli[d] + bi * dplr[d];
              ad[d] += ndr * yr + ndi * yi;
              dplr[d] = dpr[d];
              dpli[d] = dpi[d];
            }
            plr = pr;
            pli = pi;
          }
        }
      }
      // (3) advance the own row in place and contract it
      if (2 * r <= t) {
        const int hb = c_half_off(t) + r * (t + 1);
#pragma unroll
        for (int c = t; c >= 0; --c) {
          const double pr = (c < t) ? vr[c] : 0.0, pi = (c < t) ? vi[c] : 0.0;
          const double qr = (c > 0) ? vr[c - 1] : 0.0, qi = (c > 0) ? vi[c - 1] : 0.0;
          const double yr = Yr[(size_t)(hb + c) * 32], yi = Yi[(size_t)(hb + c) * 32];
#pragma unroll
          for (int d = 0; d < NDIR; ++d) {
            const double dpr = (c < t) ? dvr[d][c] : 0.0, dpi = (c < t) ? dvi[d][c] : 0.0;
            const double dqr = (c > 0) ? dvr[d][c - 1] : 0.0, dqi = (c > 0) ? dvi[d][c - 1] : 0.0;
            const double ndr = dar[d] * pr + dai[d] * pi + ar * dpr + ai * dpi - dbr[d] * qr -
                               dbi[d] * qi - br * dqr - bi * dqi;
            const double ndi = dar[d] * pi - dai[d] * pr + ar * dpi - ai * dpr - dbr[d] * qi +
                               dbi[d] * qr - br * dqi + bi * dqr;
            dvr[d][c] = ndr;
            dvi[d][c] = ndi;
            ad[d] += ndr * yr + ndi * yi;
          }
          const double nr = ar * pr + ai * pi - br * qr - bi * qi;
          const double ni = ar * pi - ai * pr - br * qi + bi * qr;
          vr[c] = nr;
          vi[c] = ni;
          if (pass == 0) au += nr * yr + ni * yi;
        }
      }
    }
    if (pass == 0) Au += au;
#pragma unroll
    for (int d = 0; d < NDIR; ++d) Ad[pass * NDIR + d] += ad[d];
  }
  // reduce the G row-lanes of the pair
#pragma unroll
  for (int o = 1; o < C::G; o <<= 1) {
    Au += __shfl_xor_sync(0xffffffffu, Au, o);
#pragma unroll
    for (int d = 0; d < 3; ++d) Ad[d] += __shfl_xor_sync(0xffffffffu, Ad[d], o);
  }
  if (valid && r == 0) {
    double* o = A.dedr + (size_t)p * 3;
#pragma unroll
    for (int d = 0; d < 3; ++d) o[d] = 2.0 * (g.dsf[d] * Au + g.sfac * Ad[d]);
  }
}

// ===========================================================================
// scatter_forces (snap_core.hpp:872-953, concurrent-RMW strategy):
// F_i += dE(i,k), F_{nbr} -= dE(i,k) with FP64 RED atomics.
// ===========================================================================
struct ScatterArgs {
  PairArgs pr;
  const double* dedr;
  double* forces;  // natoms_total x 3
  int nslots;
};

__global__ void __launch_bounds__(256) k_scatter_forces(const ScatterArgs A) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= A.nslots) return;
  const int S = A.pr.stride;
  const int i = p / S, k = p - i * S;
  if (k >= A.pr.numneigh[i]) return;
  const int j = A.pr.nbr[p];
  const double* de = A.dedr + (size_t)p * 3;
  const double d0 = de[0], d1 = de[1], d2 = de[2];
  double* fi = A.forces + (size_t)(A.pr.atom_lo + i) * 3;
  double* fj = A.forces + (size_t)j * 3;
  atomicAdd(fi + 0, d0);
  atomicAdd(fi + 1, d1);
  atomicAdd(fi + 2, d2);
  atomicAdd(fj + 0, -d0);
  atomicAdd(fj + 1, -d1);
  atomicAdd(fj + 2, -d2);
}

// Deterministic total energy: one CTA, fixed-order tree over eatom.
__global__ void __launch_bounds__(1024) k_energy_total(const double* eatom, int n, double* out) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int a = threadIdx.x; a < n; a += blockDim.x) s += eatom[a];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

}  // namespace snapgpu
