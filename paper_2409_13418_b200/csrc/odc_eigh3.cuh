// odc_eigh3.cuh -- numpy.linalg.eigh of one symmetric 3x3, bit for bit.
//
// The QEF solve (solve_qef_batch, dualize.py:358) calls np.linalg.eigh, i.e.
// LAPACK dsyevd(jobz='V', uplo='L') from numpy's bundled OpenBLAS 0.3.30.
// For n = 3 dsyevd reduces to (LAPACK 3.12 sources, no scaling for QEF
// matrices, workspace large enough that every blocked routine takes its
// unblocked path):
//
//   dsytd2('L')           one Householder reflector (dlarfg on A(2:3,1)) and
//                         the rank-2 update of A(2:3,2:3) through the BLAS
//                         kernels dsymv_L, ddot, daxpy, dsyr2 (lower)
//   dstedc('I') -> dsteqr implicit QL/QR with Wilkinson shifts, dlaev2 on
//                         2x2 blocks, dlartg rotations, rotations applied to
//                         Z by dlasr, selection sort (ascending) + column swap
//   dormtr('L','L','N') -> dorm2r -> dlarf: Z(2:3,:) -= tau v (v^T Z(2:3,:))
//                         through the kernels dgemv_t and dger
//
// The LAPACK routines themselves are compiled without FMA (generic x86-64
// code in the DYNAMIC_ARCH build); the OpenBLAS level-1/2 kernels are the
// per-core ones, and on the AVX-512 cores (SkylakeX / Cooperlake /
// SapphireRapids kernels -- the golden vectors' host and the B200 boxes'
// Xeon hosts) their scalar tails contract multiply-adds: dsymv_L, ddot,
// daxpy (hence dsyr2, a pair of axpys per column) and dger (an axpy per
// column) use fma, dgemv_t does not.  Each choice below was pinned by
// calling the individual LAPACK routines / BLAS kernels of numpy's own
// libscipy_openblas64_ and comparing bits; the composite is checked against
// np.linalg.eigh on >10^5 matrices per run (tests/test_eigh3.py) and, on
// the device, against the same numpy results (tests/test_gpu_eigh3.py).
//
// Every operation is written out in LAPACK's order; this header must be
// compiled without contraction (nvcc --fmad=false, gcc -ffp-contract=off):
// the only fused multiply-adds are the explicit fma() calls.
#pragma once
#include <math.h>
#include <stdint.h>

// ODC_EIGH_COLD: out of line on the device (helpers called from several
// sites: rotations, 2x2 eigensystems, scalings are kept once).
#ifdef __CUDACC__
#define ODC_EIGH_FN static __host__ __device__ __forceinline__
#define ODC_EIGH_COLD static __host__ __device__ __noinline__
#else
#define ODC_EIGH_FN static inline
#define ODC_EIGH_COLD static inline
#endif

namespace odc_eigh {

// dlamch('S'), dlamch('E') (eps = epsilon/2: rounding arithmetic)
constexpr double kSafMin = 0x1p-1022;
constexpr double kEps = 0x1p-53;
constexpr double kHuge = 1.79769313486231570815e308;

ODC_EIGH_FN double f_sign(double a, double b) {  // Fortran SIGN(a, b), gfortran: sign bit of b
  return signbit(b) ? -fabs(a) : fabs(a);
}
ODC_EIGH_FN double f_max(double a, double b) { return a > b ? a : b; }
ODC_EIGH_FN double f_min(double a, double b) { return a < b ? a : b; }

// dlapy2 (LAPACK 3.10+, with the NaN guards)
ODC_EIGH_COLD double dlapy2(double x, double y) {
  if (isnan(y)) return y;
  if (isnan(x)) return x;
  const double xa = fabs(x), ya = fabs(y);
  const double w = f_max(xa, ya), z = f_min(xa, ya);
  if (z == 0.0 || w > kHuge) return w;
  const double q = z / w;
  return w * sqrt(1.0 + q * q);
}

// dlascl('G'): multiply n values by cto/cfrom without over/underflow
ODC_EIGH_COLD void dlascl(double cfrom, double cto, int n, double* a) {
  const double smlnum = kSafMin, bignum = 1.0 / smlnum;
  double cfromc = cfrom, ctoc = cto;
  bool done = false;
  while (!done) {
    const double cfrom1 = cfromc * smlnum;
    double mul;
    if (cfrom1 == cfromc) {
      mul = ctoc / cfromc;
      done = true;
    } else {
      const double cto1 = ctoc / bignum;
      if (cto1 == ctoc) {
        mul = ctoc;
        done = true;
        cfromc = 1.0;
      } else if (fabs(cfrom1) > fabs(ctoc) && ctoc != 0.0) {
        mul = smlnum;
        cfromc = cfrom1;
      } else if (fabs(cto1) > fabs(cfromc)) {
        mul = bignum;
        ctoc = cto1;
      } else {
        mul = ctoc / cfromc;
        done = true;
        if (mul == 1.0) return;
      }
    }
    for (int i = 0; i < n; i++) a[i] = a[i] * mul;
  }
}

// dlartg (LAPACK 3.10+ Fortran 90 version)
struct Rot {
  double c, s, r;
};
ODC_EIGH_COLD Rot dlartg(double f, double g) {
  double c, s, r;
  const double safmin = kSafMin, safmax = 1.0 / kSafMin;
  const double rtmin = sqrt(safmin), rtmax = sqrt(safmax / 2.0);
  const double f1 = fabs(f), g1 = fabs(g);
  if (g == 0.0) {
    c = 1.0;
    s = 0.0;
    r = f;
  } else if (f == 0.0) {
    c = 0.0;
    s = f_sign(1.0, g);
    r = g1;
  } else if (f1 > rtmin && f1 < rtmax && g1 > rtmin && g1 < rtmax) {
    const double d = sqrt(f * f + g * g);
    c = f1 / d;
    r = f_sign(d, f);
    s = g / r;
  } else {
    const double u = f_min(safmax, f_max(safmin, f_max(f1, g1)));
    const double fs = f / u, gs = g / u;
    const double d = sqrt(fs * fs + gs * gs);
    c = fabs(fs) / d;
    r = f_sign(d, f);
    s = gs / r;
    r = r * u;
  }
  return Rot{c, s, r};
}

// dlaev2: eigensystem of [[a, b], [b, c]]
struct Eig2 {
  double rt1, rt2, cs1, sn1;
};
ODC_EIGH_COLD Eig2 dlaev2(double a, double b, double c) {
  double rt1, rt2, cs1, sn1;
  const double sm = a + c, df = a - c, adf = fabs(df), tb = b + b, ab = fabs(tb);
  double acmx, acmn, rt;
  if (fabs(a) > fabs(c)) {
    acmx = a;
    acmn = c;
  } else {
    acmx = c;
    acmn = a;
  }
  if (adf > ab) {
    const double q = ab / adf;
    rt = adf * sqrt(1.0 + q * q);
  } else if (adf < ab) {
    const double q = adf / ab;
    rt = ab * sqrt(1.0 + q * q);
  } else {
    rt = ab * sqrt(2.0);
  }
  int sgn1, sgn2;
  if (sm < 0.0) {
    rt1 = 0.5 * (sm - rt);
    sgn1 = -1;
    rt2 = (acmx / rt1) * acmn - (b / rt1) * b;
  } else if (sm > 0.0) {
    rt1 = 0.5 * (sm + rt);
    sgn1 = 1;
    rt2 = (acmx / rt1) * acmn - (b / rt1) * b;
  } else {
    rt1 = 0.5 * rt;
    rt2 = -0.5 * rt;
    sgn1 = 1;
  }
  double cs;
  if (df >= 0.0) {
    cs = df + rt;
    sgn2 = 1;
  } else {
    cs = df - rt;
    sgn2 = -1;
  }
  if (fabs(cs) > ab) {
    const double ct = -tb / cs;
    sn1 = 1.0 / sqrt(1.0 + ct * ct);
    cs1 = ct * sn1;
  } else if (ab == 0.0) {
    cs1 = 1.0;
    sn1 = 0.0;
  } else {
    const double tn = -cs / tb;
    cs1 = 1.0 / sqrt(1.0 + tn * tn);
    sn1 = tn * cs1;
  }
  if (sgn1 == sgn2) {
    const double tn = cs1;
    cs1 = -sn1;
    sn1 = tn;
  }
  return Eig2{rt1, rt2, cs1, sn1};
}

// dlasr('R', 'V', 'B' | 'F'): rotations (c[j], s[j]) on columns (j, j+1) of
// the 3-row column-major block z (mm columns)
ODC_EIGH_COLD void dlasr_rv(bool backward, int mm, const double* c, const double* s, double* z) {
  for (int k = 0; k < mm - 1; k++) {
    const int j = backward ? mm - 2 - k : k;
    const double ct = c[j], st = s[j];
    if (ct != 1.0 || st != 0.0) {
      for (int i = 0; i < 3; i++) {
        const double t = z[i + 3 * (j + 1)];
        z[i + 3 * (j + 1)] = ct * t - st * z[i + 3 * j];
        z[i + 3 * j] = st * t + ct * z[i + 3 * j];
      }
    }
  }
}

// dsteqr(compz='I', n=3): d[1..3], e[1..2] (1-based views), Z column-major.
// Returns LAPACK's info (0, or the number of unconverged off-diagonals).
ODC_EIGH_FN int dsteqr3(double* d, double* e, double* Z) {
  const int n = 3;
  const double eps = kEps, eps2 = eps * eps, safmin = kSafMin, safmax = 1.0 / kSafMin;
  const double ssfmax = sqrt(safmax) / 3.0, ssfmin = sqrt(safmin) / eps2;
  double wk[2 * n];  // 1-based like LAPACK's WORK: c in wk[1..n-1], s in wk[n..2n-2]
  for (int i = 0; i < 9; i++) Z[i] = (i % 4 == 0) ? 1.0 : 0.0;  // dlaset('Full', 0, 1)
  const int nmaxit = n * 30;
  int jtot = 0, l1 = 1, m = 0, l, lsv, lend, lendsv, iscale;
  double p, g, r, c, s, f, b, rt1, rt2, anorm = 0.0;
  for (;;) {  // label 10: next unreduced block
    if (l1 > n) break;
    if (l1 > 1) e[l1 - 1] = 0.0;
    m = n;
    for (int mm = l1; mm <= n - 1; mm++) {
      const double tst = fabs(e[mm]);
      if (tst == 0.0) {
        m = mm;
        break;
      }
      if (tst <= (sqrt(fabs(d[mm])) * sqrt(fabs(d[mm + 1]))) * eps) {
        e[mm] = 0.0;
        m = mm;
        break;
      }
    }
    l = l1;
    lsv = l;
    lend = m;
    lendsv = lend;
    l1 = m + 1;
    if (lend == l) continue;
    // scale the block to [ssfmin, ssfmax] (dlanst('M') then dlascl)
    anorm = 0.0;
    for (int i = l; i <= lend; i++) {
      const double t = fabs(d[i]);
      if (anorm < t || isnan(t)) anorm = t;
    }
    for (int i = l; i < lend; i++) {
      const double t = fabs(e[i]);
      if (anorm < t || isnan(t)) anorm = t;
    }
    iscale = 0;
    if (anorm == 0.0) continue;
    if (anorm > ssfmax) {
      iscale = 1;
      dlascl(anorm, ssfmax, lend - l + 1, &d[l]);
      dlascl(anorm, ssfmax, lend - l, &e[l]);
    } else if (anorm < ssfmin) {
      iscale = 2;
      dlascl(anorm, ssfmin, lend - l + 1, &d[l]);
      dlascl(anorm, ssfmin, lend - l, &e[l]);
    }
    if (fabs(d[lend]) < fabs(d[l])) {
      lend = lsv;
      l = lendsv;
    }
    if (lend > l) {  // QL iteration
      for (;;) {     // label 40
        m = lend;
        if (l != lend) {
          for (int mm = l; mm <= lend - 1; mm++) {
            double tst = fabs(e[mm]);
            tst = tst * tst;
            if (tst <= (eps2 * fabs(d[mm])) * fabs(d[mm + 1]) + safmin) {
              m = mm;
              break;
            }
          }
        }
        if (m < lend) e[m] = 0.0;
        p = d[l];
        if (m == l) {  // label 80: eigenvalue found
          d[l] = p;
          l = l + 1;
          if (l <= lend) continue;
          break;
        }
        if (m == l + 1) {
          const Eig2 ev = dlaev2(d[l], e[l], d[l + 1]);
          rt1 = ev.rt1;
          rt2 = ev.rt2;
          c = ev.cs1;
          s = ev.sn1;
          wk[l] = c;
          wk[n - 1 + l] = s;
          dlasr_rv(true, 2, &wk[l], &wk[n - 1 + l], Z + 3 * (l - 1));
          d[l] = rt1;
          d[l + 1] = rt2;
          e[l] = 0.0;
          l = l + 2;
          if (l <= lend) continue;
          break;
        }
        if (jtot == nmaxit) break;
        jtot++;
        g = (d[l + 1] - p) / (2.0 * e[l]);
        r = dlapy2(g, 1.0);
        g = d[m] - p + (e[l] / (g + f_sign(r, g)));
        s = 1.0;
        c = 1.0;
        p = 0.0;
        for (int i = m - 1; i >= l; i--) {
          f = s * e[i];
          b = c * e[i];
          const Rot rt = dlartg(g, f);
          c = rt.c;
          s = rt.s;
          r = rt.r;
          if (i != m - 1) e[i + 1] = r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          wk[i] = c;
          wk[n - 1 + i] = -s;
        }
        dlasr_rv(true, m - l + 1, &wk[l], &wk[n - 1 + l], Z + 3 * (l - 1));
        d[l] = d[l] - p;
        e[l] = g;
      }
    } else {     // QR iteration
      for (;;) {  // label 90
        m = lend;
        if (l != lend) {
          for (int mm = l; mm >= lend + 1; mm--) {
            double tst = fabs(e[mm - 1]);
            tst = tst * tst;
            if (tst <= (eps2 * fabs(d[mm])) * fabs(d[mm - 1]) + safmin) {
              m = mm;
              break;
            }
          }
        }
        if (m > lend) e[m - 1] = 0.0;
        p = d[l];
        if (m == l) {  // label 130
          d[l] = p;
          l = l - 1;
          if (l >= lend) continue;
          break;
        }
        if (m == l - 1) {
          const Eig2 ev = dlaev2(d[l - 1], e[l - 1], d[l]);
          rt1 = ev.rt1;
          rt2 = ev.rt2;
          c = ev.cs1;
          s = ev.sn1;
          wk[m] = c;
          wk[n - 1 + m] = s;
          dlasr_rv(false, 2, &wk[m], &wk[n - 1 + m], Z + 3 * (l - 2));
          d[l - 1] = rt1;
          d[l] = rt2;
          e[l - 1] = 0.0;
          l = l - 2;
          if (l >= lend) continue;
          break;
        }
        if (jtot == nmaxit) break;
        jtot++;
        g = (d[l - 1] - p) / (2.0 * e[l - 1]);
        r = dlapy2(g, 1.0);
        g = d[m] - p + (e[l - 1] / (g + f_sign(r, g)));
        s = 1.0;
        c = 1.0;
        p = 0.0;
        for (int i = m; i <= l - 1; i++) {
          f = s * e[i];
          b = c * e[i];
          const Rot rt = dlartg(g, f);
          c = rt.c;
          s = rt.s;
          r = rt.r;
          if (i != m) e[i - 1] = r;
          g = d[i] - p;
          r = (d[i + 1] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i] = g + p;
          g = c * r - b;
          wk[i] = c;
          wk[n - 1 + i] = s;
        }
        dlasr_rv(false, l - m + 1, &wk[m], &wk[n - 1 + m], Z + 3 * (m - 1));
        d[l] = d[l] - p;
        e[l - 1] = g;
      }
    }
    // label 140: undo scaling
    if (iscale == 1) {
      dlascl(ssfmax, anorm, lendsv - lsv + 1, &d[lsv]);
      dlascl(ssfmax, anorm, lendsv - lsv, &e[lsv]);
    } else if (iscale == 2) {
      dlascl(ssfmin, anorm, lendsv - lsv + 1, &d[lsv]);
      dlascl(ssfmin, anorm, lendsv - lsv, &e[lsv]);
    }
    if (jtot >= nmaxit) {
      int info = 0;
      for (int i = 1; i <= n - 1; i++) info += e[i] != 0.0;
      return info;
    }
  }
  // label 160: selection sort, ascending, swapping eigenvector columns
  for (int ii = 2; ii <= n; ii++) {
    const int i = ii - 1;
    int k = i;
    p = d[i];
    for (int j = ii; j <= n; j++)
      if (d[j] < p) {
        k = j;
        p = d[j];
      }
    if (k != i) {
      d[k] = d[i];
      d[i] = p;
      for (int q = 0; q < 3; q++) {
        const double t = Z[q + 3 * (i - 1)];
        Z[q + 3 * (i - 1)] = Z[q + 3 * (k - 1)];
        Z[q + 3 * (k - 1)] = t;
      }
    }
  }
  return 0;
}

}  // namespace odc_eigh

// numpy.linalg.eigh(A) for a symmetric 3x3 A (row-major; symmetric, so the
// column-major lower triangle dsyevd reads is the same numbers): w ascending,
// V[3*i + k] = component i of eigenvector k (numpy's v[:, k]).  Returns
// LAPACK's info (0 unless dsteqr failed to converge).
ODC_EIGH_FN int odc_eigh3(const double* A, double* w, double* V) {
  using namespace odc_eigh;
  double a[9];  // column-major working copy; only the lower triangle is used
  for (int i = 0; i < 9; i++) a[i] = A[i];
  // dsyevd: scale the matrix into [rmin, rmax] (dlansy('M', 'L'))
  const double smlnum = kSafMin / (2.0 * kEps), bignum = 1.0 / smlnum;
  const double rmin = sqrt(smlnum), rmax = sqrt(bignum);
  double anrm = 0.0;
  for (int j = 0; j < 3; j++)
    for (int i = j; i < 3; i++) {
      const double t = fabs(a[i + 3 * j]);
      if (anrm < t || isnan(t)) anrm = t;
    }
  int iscale = 0;
  double sigma = 1.0;
  if (anrm > 0.0 && anrm < rmin) {
    iscale = 1;
    sigma = rmin / anrm;
  } else if (anrm > rmax) {
    iscale = 1;
    sigma = rmax / anrm;
  }
  if (iscale) {  // dlascl('L', 0, 0, one, sigma, ...) on the lower triangle, column by column
    double lower[6] = {a[0], a[1], a[2], a[4], a[5], a[8]};
    odc_eigh::dlascl(1.0, sigma, 6, lower);
    a[0] = lower[0], a[1] = lower[1], a[2] = lower[2], a[4] = lower[3], a[5] = lower[4], a[8] = lower[5];
  }
  // ---- dsytd2('L'): i = 1 -- dlarfg(2, A(2,1), A(3,1)); i = 2 is dlarfg(1) => tau = 0
  double alpha = a[1], x = a[2], taui = 0.0;
  double xnorm = fabs(x);  // dnrm2 of one element
  if (xnorm != 0.0) {
    double beta = -f_sign(dlapy2(alpha, xnorm), alpha);
    const double sfmin = kSafMin / kEps;  // dlamch('S') / dlamch('E')
    int knt = 0;
    if (fabs(beta) < sfmin) {  // beta may be inaccurate: rescale x and recompute
      const double rsafmn = 1.0 / sfmin;
      do {
        knt++;
        x = rsafmn * x;
        beta = beta * rsafmn;
        alpha = alpha * rsafmn;
      } while (fabs(beta) < sfmin && knt < 20);
      xnorm = fabs(x);
      beta = -f_sign(dlapy2(alpha, xnorm), alpha);
    }
    taui = (beta - alpha) / beta;
    x = (1.0 / (alpha - beta)) * x;  // dscal
    for (int j = 0; j < knt; j++) beta = beta * sfmin;
    alpha = beta;
  }
  const double v1 = x;  // v = (1, v1)
  if (taui != 0.0) {
    double a11 = a[4], a21 = a[5], a22 = a[8];
    // w = taui * A22 v   (dsymv_L scalar path, beta = 0 zeroes w first)
    double y0 = 0.0, y1 = 0.0;
    {
      double t1 = taui * 1.0, t2 = 0.0;
      y0 = fma(t1, a11, y0);
      y1 = fma(t1, a21, y1);
      t2 = fma(a21, v1, t2);
      y0 = fma(taui, t2, y0);
      t1 = taui * v1;
      y1 = fma(t1, a22, y1);
      y1 = fma(taui, 0.0, y1);
    }
    // alpha = -1/2 taui (w . v);  w += alpha v   (ddot, daxpy)
    const double dot = fma(y1, v1, y0 * 1.0);
    const double al = -(0.5 * taui * dot);
    y0 = fma(al, 1.0, y0);
    y1 = fma(al, v1, y1);
    // A22 -= v w^T + w v^T   (dsyr2 lower: per column j, axpy(-v_j, w) then axpy(-w_j, v))
    a11 = fma(-1.0, y0, a11);
    a21 = fma(-1.0, y1, a21);
    a11 = fma(-y0, 1.0, a11);
    a21 = fma(-y0, v1, a21);
    a22 = fma(-v1, y1, a22);
    a22 = fma(-y1, v1, a22);
    a[4] = a11;
    a[5] = a21;
    a[8] = a22;
  }
  double d[4] = {0.0, a[0], a[4], a[8]};  // 1-based
  double e[3] = {0.0, alpha, a[5]};
  double Z[9];
  const int info = dsteqr3(d, e, Z);
  // ---- dormtr -> dorm2r: H(2) has tau 0; H(1) = I - taui v v^T on Z(2:3, :)
  if (taui != 0.0) {
    const int lastv = v1 == 0.0 ? 1 : 2;
    double* C = Z + 1;  // C(i, j) = C[i + 3 j]
    int lastc = 0;      // iladlc
    if (C[6] != 0.0 || C[(lastv - 1) + 6] != 0.0) {
      lastc = 3;
    } else {
      for (int j = 2; j >= 0 && !lastc; j--)
        for (int i = 0; i < lastv; i++)
          if (C[i + 3 * j] != 0.0) {
            lastc = j + 1;
            break;
          }
    }
    double wv[3];
    for (int j = 0; j < lastc; j++) {  // dgemv_t (no contraction), y = 0 + ...
      const double t = lastv == 2 ? C[3 * j] * 1.0 + C[1 + 3 * j] * v1 : C[3 * j] * 1.0;
      wv[j] = 0.0 + t;
    }
    for (int j = 0; j < lastc; j++) {  // dger: per column axpy(-taui * w_j, v)
      const double da = -taui * wv[j];
      C[3 * j] = fma(da, 1.0, C[3 * j]);
      if (lastv == 2) C[1 + 3 * j] = fma(da, v1, C[1 + 3 * j]);
    }
  }
  for (int k = 0; k < 3; k++) w[k] = d[k + 1];
  if (iscale) {  // dscal(n, 1/sigma, w)
    const double inv = 1.0 / sigma;
    for (int k = 0; k < 3; k++) w[k] = inv * w[k];
  }
  for (int i = 0; i < 3; i++)
    for (int k = 0; k < 3; k++) V[3 * i + k] = Z[i + 3 * k];
  return info;
}
