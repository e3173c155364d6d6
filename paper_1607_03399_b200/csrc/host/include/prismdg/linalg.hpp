#pragma once
// Minimal dense linear algebra for the one-time host setup.
//
// The reference delegates all dense algebra to Eigen3 (proj/CMakeLists.txt:12),
// which is not available here.  Only the handful of operations its setup uses
// are provided: products, transpose, PartialPivLU-style inverse
// (reference.cpp:171,174,297,301,313,568), Cholesky solve (operators.cpp:27-31),
// LDLT solve (tests/oracles.cpp:222), the symmetric tridiagonal eigensolver used
// by Golub-Welsch (jacobi.cpp:68), and 3x3 helpers (geometry.cpp:52-61,167-175).
// Results agree with Eigen's to rounding, not bitwise; parity is by tolerance.

#include <cmath>
#include <cstddef>
#include <vector>

namespace prismdg {

using Vec = std::vector<double>;

/// Row-major dense matrix.
struct Mat {
  int rows = 0, cols = 0;
  std::vector<double> a;

  Mat() = default;
  Mat(int r, int c, double v = 0.0) : rows(r), cols(c), a((std::size_t)r * c, v) {}

  double& operator()(int i, int j) { return a[(std::size_t)i * cols + j]; }
  double operator()(int i, int j) const { return a[(std::size_t)i * cols + j]; }
  double* row(int i) { return a.data() + (std::size_t)i * cols; }
  const double* row(int i) const { return a.data() + (std::size_t)i * cols; }
  std::size_t size() const { return a.size(); }

  static Mat identity(int n) {
    Mat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};

Mat matmul(const Mat& A, const Mat& B);
Mat matmul_tn(const Mat& A, const Mat& B); // A^T B
Mat transpose(const Mat& A);
Mat scaled(const Mat& A, double s);
Mat add(const Mat& A, const Mat& B, double sb = 1.0); // A + sb*B
Vec matvec(const Mat& A, const Vec& x);
double max_abs_diff(const Mat& A, const Mat& B);

/// Inverse by LU with partial pivoting; throws NumericalError if singular.
Mat inverse(const Mat& A);

/// Solve A X = B for symmetric positive definite A (Cholesky, lower factor).
/// Returns false if A is not numerically SPD (Eigen LLT info() != Success).
bool cholesky_solve(const Mat& A, const Mat& B, Mat& X);

/// Solve A X = B for symmetric A via LDL^T without pivoting.
Mat ldlt_solve(const Mat& A, const Mat& B);

/// Eigen-decomposition of a symmetric tridiagonal matrix (diag d, off-diag e,
/// e[i] couples i and i+1).  Returns eigenvalues ascending and the first
/// component of each normalized eigenvector (what Golub-Welsch needs).
void sym_tridiag_eig(const Vec& d, const Vec& e, Vec& evals, Vec& first_comp);

/// Two-norm condition number via the eigenvalues of A^T A (Jacobi rotations);
/// replaces Eigen::JacobiSVD in reference.cpp:152-156.
double cond2(const Mat& A);

// 3x3 helpers
double det3(const double A[3][3]);
void inv3(const double A[3][3], double Ai[3][3]);

} // namespace prismdg
