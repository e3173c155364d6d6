#include "prismdg/linalg.hpp"

#include "prismdg/types.hpp"

#include <algorithm>
#include <numeric>

namespace prismdg {

Mat matmul(const Mat& A, const Mat& B) {
  Mat C(A.rows, B.cols);
  for (int i = 0; i < A.rows; ++i) {
    double* c = C.row(i);
    const double* a = A.row(i);
    for (int k = 0; k < A.cols; ++k) {
      const double aik = a[k];
      const double* b = B.row(k);
      for (int j = 0; j < B.cols; ++j) c[j] += aik * b[j];
    }
  }
  return C;
}

Mat matmul_tn(const Mat& A, const Mat& B) {
  Mat C(A.cols, B.cols);
  for (int k = 0; k < A.rows; ++k) {
    const double* a = A.row(k);
    const double* b = B.row(k);
    for (int i = 0; i < A.cols; ++i) {
      const double aki = a[i];
      double* c = C.row(i);
      for (int j = 0; j < B.cols; ++j) c[j] += aki * b[j];
    }
  }
  return C;
}

Mat transpose(const Mat& A) {
  Mat T(A.cols, A.rows);
  for (int i = 0; i < A.rows; ++i)
    for (int j = 0; j < A.cols; ++j) T(j, i) = A(i, j);
  return T;
}

Mat scaled(const Mat& A, double s) {
  Mat B = A;
  for (double& v : B.a) v *= s;
  return B;
}

Mat add(const Mat& A, const Mat& B, double sb) {
  Mat C = A;
  for (std::size_t i = 0; i < C.a.size(); ++i) C.a[i] += sb * B.a[i];
  return C;
}

Vec matvec(const Mat& A, const Vec& x) {
  Vec y(A.rows, 0.0);
  for (int i = 0; i < A.rows; ++i) {
    const double* a = A.row(i);
    double s = 0.0;
    for (int j = 0; j < A.cols; ++j) s += a[j] * x[j];
    y[i] = s;
  }
  return y;
}

double max_abs_diff(const Mat& A, const Mat& B) {
  double m = 0.0;
  for (std::size_t i = 0; i < A.a.size(); ++i) m = std::max(m, std::abs(A.a[i] - B.a[i]));
  return m;
}

Mat inverse(const Mat& A) {
  const int n = A.rows;
  Mat LU = A;
  std::vector<int> piv(n);
  std::iota(piv.begin(), piv.end(), 0);
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::abs(LU(k, k));
    for (int i = k + 1; i < n; ++i)
      if (std::abs(LU(i, k)) > best) {
        best = std::abs(LU(i, k));
        p = i;
      }
    if (best == 0.0) throw NumericalError("inverse: singular matrix");
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(LU(k, j), LU(p, j));
      std::swap(piv[k], piv[p]);
    }
    const double inv = 1.0 / LU(k, k);
    for (int i = k + 1; i < n; ++i) {
      const double l = LU(i, k) * inv;
      LU(i, k) = l;
      if (l != 0.0)
        for (int j = k + 1; j < n; ++j) LU(i, j) -= l * LU(k, j);
    }
  }
  Mat X(n, n);
  Vec y(n);
  for (int c = 0; c < n; ++c) {
    // solve L U x = P e_c
    for (int i = 0; i < n; ++i) {
      double s = (piv[i] == c) ? 1.0 : 0.0;
      for (int j = 0; j < i; ++j) s -= LU(i, j) * y[j];
      y[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = y[i];
      for (int j = i + 1; j < n; ++j) s -= LU(i, j) * X(j, c);
      X(i, c) = s / LU(i, i);
    }
  }
  return X;
}

bool cholesky_solve(const Mat& A, const Mat& B, Mat& X) {
  const int n = A.rows;
  Mat L(n, n);
  for (int j = 0; j < n; ++j) {
    double s = A(j, j);
    for (int k = 0; k < j; ++k) s -= L(j, k) * L(j, k);
    if (!(s > 0.0)) return false;
    const double d = std::sqrt(s);
    L(j, j) = d;
    for (int i = j + 1; i < n; ++i) {
      double t = A(i, j);
      for (int k = 0; k < j; ++k) t -= L(i, k) * L(j, k);
      L(i, j) = t / d;
    }
  }
  X = Mat(n, B.cols);
  Vec y(n);
  for (int c = 0; c < B.cols; ++c) {
    for (int i = 0; i < n; ++i) {
      double s = B(i, c);
      for (int k = 0; k < i; ++k) s -= L(i, k) * y[k];
      y[i] = s / L(i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < n; ++k) s -= L(k, i) * X(k, c);
      X(i, c) = s / L(i, i);
    }
  }
  return true;
}

Mat ldlt_solve(const Mat& A, const Mat& B) {
  const int n = A.rows;
  Mat L = Mat::identity(n);
  Vec D(n);
  for (int j = 0; j < n; ++j) {
    double s = A(j, j);
    for (int k = 0; k < j; ++k) s -= L(j, k) * L(j, k) * D[k];
    if (s == 0.0) throw NumericalError("ldlt_solve: zero pivot");
    D[j] = s;
    for (int i = j + 1; i < n; ++i) {
      double t = A(i, j);
      for (int k = 0; k < j; ++k) t -= L(i, k) * L(j, k) * D[k];
      L(i, j) = t / s;
    }
  }
  Mat X(n, B.cols);
  Vec y(n);
  for (int c = 0; c < B.cols; ++c) {
    for (int i = 0; i < n; ++i) {
      double s = B(i, c);
      for (int k = 0; k < i; ++k) s -= L(i, k) * y[k];
      y[i] = s;
    }
    for (int i = 0; i < n; ++i) y[i] /= D[i];
    for (int i = n - 1; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < n; ++k) s -= L(k, i) * X(k, c);
      X(i, c) = s;
    }
  }
  return X;
}

void sym_tridiag_eig(const Vec& d_in, const Vec& e_in, Vec& evals, Vec& first_comp) {
  // implicit QL with Wilkinson shifts, accumulating the eigenvector matrix
  const int n = (int)d_in.size();
  Vec d = d_in, e(n, 0.0);
  for (int i = 0; i + 1 < n; ++i) e[i] = e_in[i];
  Mat Z = Mat::identity(n);
  for (int l = 0; l < n; ++l) {
    int iter = 0;
    int m;
    do {
      for (m = l; m < n - 1; ++m) {
        const double dd = std::abs(d[m]) + std::abs(d[m + 1]);
        if (std::abs(e[m]) <= 1e-300 || std::abs(e[m]) <= 2.2e-16 * dd * 0.5) break;
      }
      if (m != l) {
        if (++iter > 200) throw NumericalError("sym_tridiag_eig: no convergence");
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + (g >= 0 ? std::abs(r) : -std::abs(r)));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = std::hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          for (int k = 0; k < n; ++k) {
            f = Z(k, i + 1);
            Z(k, i + 1) = s * Z(k, i) + c * f;
            Z(k, i) = c * Z(k, i) - s * f;
          }
        }
        if (r == 0.0 && i >= l) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int a, int b) { return d[a] < d[b]; });
  evals.resize(n);
  first_comp.resize(n);
  for (int k = 0; k < n; ++k) {
    evals[k] = d[order[k]];
    double nrm = 0.0;
    for (int i = 0; i < n; ++i) nrm += Z(i, order[k]) * Z(i, order[k]);
    first_comp[k] = Z(0, order[k]) / std::sqrt(nrm);
  }
}

double cond2(const Mat& A) {
  // eigenvalues of the SPD matrix A^T A by cyclic Jacobi rotations
  Mat S = matmul_tn(A, A);
  const int n = S.rows;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += S(p, q) * S(p, q);
    if (off < 1e-30) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (std::abs(S(p, q)) < 1e-300) continue;
        const double theta = (S(q, q) - S(p, p)) / (2.0 * S(p, q));
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double skp = S(k, p), skq = S(k, q);
          S(k, p) = c * skp - s * skq;
          S(k, q) = s * skp + c * skq;
        }
        for (int k = 0; k < n; ++k) {
          const double spk = S(p, k), sqk = S(q, k);
          S(p, k) = c * spk - s * sqk;
          S(q, k) = s * spk + c * sqk;
        }
      }
  }
  double lo = 1e300, hi = 0.0;
  for (int i = 0; i < n; ++i) {
    lo = std::min(lo, std::abs(S(i, i)));
    hi = std::max(hi, std::abs(S(i, i)));
  }
  return std::sqrt(hi / lo);
}

double det3(const double A[3][3]) {
  return A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1]) -
         A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0]) +
         A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
}

void inv3(const double A[3][3], double Ai[3][3]) {
  const double d = det3(A);
  Ai[0][0] = (A[1][1] * A[2][2] - A[1][2] * A[2][1]) / d;
  Ai[0][1] = (A[0][2] * A[2][1] - A[0][1] * A[2][2]) / d;
  Ai[0][2] = (A[0][1] * A[1][2] - A[0][2] * A[1][1]) / d;
  Ai[1][0] = (A[1][2] * A[2][0] - A[1][0] * A[2][2]) / d;
  Ai[1][1] = (A[0][0] * A[2][2] - A[0][2] * A[2][0]) / d;
  Ai[1][2] = (A[0][2] * A[1][0] - A[0][0] * A[1][2]) / d;
  Ai[2][0] = (A[1][0] * A[2][1] - A[1][1] * A[2][0]) / d;
  Ai[2][1] = (A[0][1] * A[2][0] - A[0][0] * A[2][1]) / d;
  Ai[2][2] = (A[0][0] * A[1][1] - A[0][1] * A[1][0]) / d;
}

} // namespace prismdg
