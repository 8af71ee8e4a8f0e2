// ============================================================================
// qp_oracle.cpp — CPU ORACLE (TEST INFRASTRUCTURE ONLY).
//
// Plain, slow, obviously-correct CPU implementation of the method of
// arxiv 2605.17913 ("differentiable interior-point QPs in single precision via
// implicit complementarity"), templated over double (parity reference) and
// float (iteration-count reference).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.  It
// shares no code, header, table or helper with the CUDA path
// (paper_2605_17913_b200/csrc); neither side includes the other.
//
// Citations: "P:L" = PAPER.md line L, "S:L" = SPEC.md line L, "Qn" = a
// reading listed in DESIGN.md §2 (taken from SURVEY.md §8(c)).
//
// Scalar loops only; no BLAS.  Linear algebra is textbook:
//   * gepp_*   — Gaussian elimination with partial pivoting (LU) on the
//                paper-literal Eq. 14 matrix.  Default for f64.
//   * ldl_qd_* — unpivoted LDLᵀ of the congruent quasi-definite form
//                M = Sᵀ K14 S (reading Q12 / App. A.2), the same
//                algorithm class the GPU uses; used for the f32
//                iteration-count reference.
// Every function below that is pinned by a test says so; the pins live in
// tests/test_oracle_*.py.
// ============================================================================
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

namespace orc {

enum { ST_CONVERGED = 0, ST_MAX_ITER = 2, ST_NUMERICAL_FAILURE = 3 };
// failure stage, stored in status bits 8..15 (Table 1 categories).
enum { STG_NONE = 0, STG_SCALING = 1, STG_PREDICTOR = 2, STG_CENTERING = 3, STG_CORRECTOR = 4,
       STG_LINESEARCH = 5, STG_RELAX = 6, STG_BACKWARD = 7, STG_INIT = 8 };
enum { SOLVER_K14_GEPP = 0, SOLVER_M_LDL = 1, SOLVER_NORMAL_CHOL = 2, SOLVER_M_PART = 3 };
enum { FORM_IMPLICIT = 0, FORM_EXPLICIT = 1 };

}  // namespace orc

extern "C" {
typedef struct {
  double tol;             // relative stopping tolerance (reading Q4)
  int32_t max_iter;       // Alg. 1 max_iter (100)
  double sigma;           // kappa_target = sigma*kappa (Q2: 0.1)
  double tau;             // alpha = min(1, tau*alpha_max) (Q3: 0.99)
  double kappa_relax;     // Alg. 2 target (1e-4)
  double relax_ktol;      // |kappa/kappa_relax-1| tolerance (Q5)
  int32_t relax_max_iter; // Alg. 2 max_iter (Q22)
  int32_t kkt_solver;     // orc::SOLVER_*
  int32_t formulation;    // orc::FORM_*
  double pivot_floor_rel; // LDL pivot floor theta = rel*max|diag| (Q12)
  double relax_tol;       // Alg. 2 residual tolerance (reading Q5b)
  int32_t partition_cap;  // SOLVER_M_PART: most constraints kept in augmented form (reading Q12c); -1 = no cap
  int32_t relax_mode;     // 0: Alg. 2 by exact Newton (Q6); 1: chord steps with Alg. 1's factor nearest kappa_relax (N2(i));
                          // 2: guarded chord (N2(i), reading Q26): chord steps while they contract, then exact Newton
  int32_t chord_max;      // relax_mode 2: most chord steps
  double chord_rho;       // relax_mode 2: a chord step must shrink psi = max(phi, |kappa/kappa_relax - 1|) by this factor
} oracle_cfg;
}

namespace orc {

template <typename T>
struct Prob {
  int n, m, p;
  const T *Q, *q, *A, *b, *G, *h;
};

template <typename T> static inline T sq(T a) { return a * a; }

// ---------------------------------------------------------------------------
// Appendix C: cancellation-safe softplus retraction b_kappa (Eq. 12,
// P:256) and its v-derivative.  c = d b_kappa / d kappa = 1/sqrt(v^2+4 kappa)
// (reading Q10).  Pinned: tests/test_oracle_retraction.py.
// ---------------------------------------------------------------------------
template <typename T> T retract_b(T v, T kappa) {
  T R = std::sqrt(v * v + T(4) * kappa);
  if (v >= T(0)) return (v + R) / T(2);
  return T(2) * kappa / (R - v);
}
template <typename T> T retract_db(T v, T kappa) {
  T R = std::sqrt(v * v + T(4) * kappa);
  if (v >= T(0)) return (T(1) + v / R) / T(2);
  return T(2) * kappa / (v * v + T(4) * kappa - v * R);
}
template <typename T> T retract_dkappa(T v, T kappa) { return T(1) / std::sqrt(v * v + T(4) * kappa); }

// ---------------------------------------------------------------------------
// Dense helpers (row-major).
// ---------------------------------------------------------------------------
template <typename T> static void matvec(const T* M, int r, int c, const T* x, T* y) {
  for (int i = 0; i < r; ++i) {
    T acc = 0;
    for (int j = 0; j < c; ++j) acc += M[(size_t)i * c + j] * x[j];
    y[i] = acc;
  }
}
template <typename T> static void matTvec(const T* M, int r, int c, const T* x, T* y) {
  for (int j = 0; j < c; ++j) y[j] = 0;
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) y[j] += M[(size_t)i * c + j] * x[i];
}
template <typename T> static T ninf(const T* a, int k) {
  T r = 0;
  for (int i = 0; i < k; ++i) r = std::max(r, std::fabs(a[i]));
  return r;
}
template <typename T> static T ninf(const std::vector<T>& a) { return ninf(a.data(), (int)a.size()); }
template <typename T> static T dotp(const T* a, const T* b, int k) {
  T r = 0;
  for (int i = 0; i < k; ++i) r += a[i] * b[i];
  return r;
}
template <typename T> static bool finite_all(const std::vector<T>& a) {
  for (T v : a)
    if (!std::isfinite(v)) return false;
  return true;
}

// LU with partial pivoting (textbook Gaussian elimination).  In place.
template <typename T> static bool lu_factor(std::vector<T>& A, int N, std::vector<int>& piv) {
  piv.assign(N, 0);
  bool ok = true;
  for (int k = 0; k < N; ++k) {
    int pr = k;
    T best = std::fabs(A[(size_t)k * N + k]);
    for (int i = k + 1; i < N; ++i) {
      T a = std::fabs(A[(size_t)i * N + k]);
      if (a > best) { best = a; pr = i; }
    }
    piv[k] = pr;
    if (pr != k)
      for (int j = 0; j < N; ++j) std::swap(A[(size_t)k * N + j], A[(size_t)pr * N + j]);
    T d = A[(size_t)k * N + k];
    if (d == T(0) || !std::isfinite(d)) { ok = false; continue; }
    for (int i = k + 1; i < N; ++i) {
      T l = A[(size_t)i * N + k] / d;
      A[(size_t)i * N + k] = l;
      if (l != T(0))
        for (int j = k + 1; j < N; ++j) A[(size_t)i * N + j] -= l * A[(size_t)k * N + j];
    }
  }
  return ok;
}
template <typename T> static void lu_solve(const std::vector<T>& LU, int N, const std::vector<int>& piv, T* x) {
  for (int k = 0; k < N; ++k)
    if (piv[k] != k) std::swap(x[k], x[piv[k]]);
  for (int i = 0; i < N; ++i) {
    T acc = x[i];
    for (int k = 0; k < i; ++k) acc -= LU[(size_t)i * N + k] * x[k];
    x[i] = acc;
  }
  for (int i = N - 1; i >= 0; --i) {
    T acc = x[i];
    for (int k = i + 1; k < N; ++k) acc -= LU[(size_t)i * N + k] * x[k];
    x[i] = acc / LU[(size_t)i * N + i];
  }
}

// Unpivoted LDLᵀ of a quasi-definite matrix: the first npos pivots must be
// positive, the remaining ones negative (reading Q12).  A pivot on the wrong
// side of +-theta is replaced by +-theta and counted.  In place: strict lower
// triangle holds L (unit diagonal implied), D holds the pivots.
template <typename T>
static int ldl_factor(std::vector<T>& M, int N, int npos, T floor_rel, std::vector<T>& D) {
  D.assign(N, 0);
  T maxdiag = 0;
  for (int i = 0; i < N; ++i) maxdiag = std::max(maxdiag, std::fabs(M[(size_t)i * N + i]));
  const T theta = floor_rel * std::max(maxdiag, T(1e-30));
  int nfloor = 0;
  for (int j = 0; j < N; ++j) {
    T d = M[(size_t)j * N + j];
    for (int k = 0; k < j; ++k) d -= sq(M[(size_t)j * N + k]) * D[k];
    if (j < npos) {
      if (!(d >= theta)) { d = theta; ++nfloor; }
    } else {
      if (!(d <= -theta)) { d = -theta; ++nfloor; }
    }
    D[j] = d;
    for (int i = j + 1; i < N; ++i) {
      T a = M[(size_t)i * N + j];
      for (int k = 0; k < j; ++k) a -= M[(size_t)i * N + k] * M[(size_t)j * N + k] * D[k];
      M[(size_t)i * N + j] = a / d;
    }
  }
  return nfloor;
}
template <typename T> static void ldl_solve(const std::vector<T>& L, const std::vector<T>& D, int N, T* x) {
  for (int i = 0; i < N; ++i)
    for (int k = 0; k < i; ++k) x[i] -= L[(size_t)i * N + k] * x[k];
  for (int i = 0; i < N; ++i) x[i] /= D[i];
  for (int i = N - 1; i >= 0; --i)
    for (int k = i + 1; k < N; ++k) x[i] -= L[(size_t)k * N + i] * x[k];
}

// ---------------------------------------------------------------------------
// Residuals: Eq. 4 and Eq. 10, plus the scale norms
// used by the relative stopping test (reading Q4).
// ---------------------------------------------------------------------------
template <typename T> struct Res {
  std::vector<T> rt, re, ri, rz, rs;
  T nrt = 0, nre = 0, nri = 0, nrz = 0, nrs = 0;
  T sQx = 0, sq_ = 0, sGz = 0, sAy = 0, sAx = 0, sb = 0, sGx = 0, ss = 0, sh = 0, sz = 0;
  T gap = 0, obj = 0;
};

template <typename T>
static void residuals(const Prob<T>& P, const T* x, const T* y, const T* z, const T* s, T kappa, bool implicit,
                      Res<T>& R) {
  const int n = P.n, m = P.m, p = P.p;
  std::vector<T> Qx(n), Gz(n), Ay(n), Ax(m), Gx(p);
  matvec(P.Q, n, n, x, Qx.data());
  matTvec(P.G, p, n, z, Gz.data());
  matTvec(P.A, m, n, y, Ay.data());
  matvec(P.A, m, n, x, Ax.data());
  matvec(P.G, p, n, x, Gx.data());
  R.rt.resize(n); R.re.resize(m); R.ri.resize(p); R.rz.assign(p, 0); R.rs.assign(p, 0);
  for (int i = 0; i < n; ++i) R.rt[i] = Qx[i] + P.q[i] + Gz[i] + Ay[i];  // r_t = Qx+q+G'z+A'y
  for (int i = 0; i < m; ++i) R.re[i] = Ax[i] - P.b[i];                  // r_e = Ax-b
  for (int i = 0; i < p; ++i) R.ri[i] = Gx[i] + s[i] - P.h[i];           // r_i = Gx+s-h
  if (implicit)
    for (int i = 0; i < p; ++i) {
      T v = z[i] - s[i];
      R.rz[i] = z[i] - retract_b(v, kappa);   // r_z = z - b_k(v)
      R.rs[i] = s[i] - retract_b(-v, kappa);  // r_s = s - b_k(-v)
    }
  R.nrt = ninf(R.rt); R.nre = ninf(R.re); R.nri = ninf(R.ri); R.nrz = ninf(R.rz); R.nrs = ninf(R.rs);
  R.sQx = ninf(Qx); R.sq_ = ninf(P.q, n); R.sGz = ninf(Gz); R.sAy = ninf(Ay);
  R.sAx = ninf(Ax); R.sb = ninf(P.b, m); R.sGx = ninf(Gx); R.ss = ninf(s, p); R.sh = ninf(P.h, p);
  R.sz = ninf(z, p);
  R.gap = dotp(s, z, p);
  R.obj = T(0.5) * dotp(x, Qx.data(), n) + dotp(P.q, x, n);
}

// Reading Q4: relative form of Alg. 1's "||r||_inf < tol".  phi is the
// largest of the four relative residuals; feasible <=> phi <= tol.
template <typename T> static T rel_phi(const Res<T>& R) {
  auto mx = [](std::initializer_list<T> l) { T r = T(1); for (T v : l) r = std::max(r, v); return r; };
  T a = R.nrt / mx({R.sQx, R.sq_, R.sGz, R.sAy});
  T b = R.nre / mx({R.sAx, R.sb});
  T c = R.nri / mx({R.sGx, R.ss, R.sh});
  T d = std::max(R.nrz, R.nrs) / mx({R.sz, R.ss});
  return std::max(std::max(a, b), std::max(c, d));
}
template <typename T> static bool feasible_rel(const Res<T>& R, T tol) {
  auto mx = [](std::initializer_list<T> l) { T r = T(1); for (T v : l) r = std::max(r, v); return r; };
  return R.nrt <= tol * mx({R.sQx, R.sq_, R.sGz, R.sAy}) && R.nre <= tol * mx({R.sAx, R.sb}) &&
         R.nri <= tol * mx({R.sGx, R.ss, R.sh}) && std::max(R.nrz, R.nrs) <= tol * mx({R.sz, R.ss});
}
// Reading Q5b: Alg. 2 stops when kappa is at kappa_relax and either phi <=
// relax_tol, or phi <= tol and the last Newton step no longer reduced phi by
// 10% (the working-precision floor).
template <typename T> static bool relax_done(const Res<T>& R, T tol, T relax_tol, T phi_prev) {
  const T phi = rel_phi(R);
  return phi <= relax_tol || (phi <= tol && phi > T(0.9) * phi_prev);
}
template <typename T> static bool converged_solve(const Res<T>& R, T tol) {
  return feasible_rel(R, tol) && R.gap <= tol * std::max(T(1), std::fabs(R.obj));
}

// ---------------------------------------------------------------------------
// KKT factor at (v, kappa).  Both solvers return the step in the
// coordinates of Eq. 14, (dx, dv, dy).
// ---------------------------------------------------------------------------
template <typename T> struct Factor {
  int kind = SOLVER_K14_GEPP, N = 0;
  std::vector<T> F, D;  // LU (K14) or LDL (M)
  std::vector<int> piv;
  std::vector<T> dp, dm, c;  // d+ = db(v), d- = db(-v), c = db/dkappa
  std::vector<int> act;      // SOLVER_M_PART: indices i with v_i > 0, in order
  int nfloor = 0;
  bool ok = true;
};

// precompute_kkt_factors (Alg. 1 line 12).
template <typename T>
static Factor<T> factor_kkt(const Prob<T>& P, const T* v, T kappa, int solver, T floor_rel, int pcap = -1) {
  const int n = P.n, m = P.m, p = P.p, N = n + p + m;
  Factor<T> F;
  F.kind = solver; F.N = N;
  F.dp.resize(p); F.dm.resize(p); F.c.resize(p);
  for (int i = 0; i < p; ++i) {
    F.dp[i] = retract_db(v[i], kappa);           // B_k(v)   diagonal
    F.dm[i] = retract_db(-v[i], kappa);          // B_k(-v)  diagonal
    F.c[i] = retract_dkappa(v[i], kappa);        // c (Q10)
  }
  std::vector<T>& K = F.F;
  K.assign((size_t)N * N, 0);
  auto at = [&](int i, int j) -> T& { return K[(size_t)i * N + j]; };
  if (solver == SOLVER_K14_GEPP) {
    // Eq. 14: [[Q - G'G, G', A'], [G, -B_k(-v), 0], [A, 0, 0]],
    // unknowns ordered (dx, dv, dy).
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        T gg = 0;
        for (int k = 0; k < p; ++k) gg += P.G[(size_t)k * n + i] * P.G[(size_t)k * n + j];
        at(i, j) = P.Q[(size_t)i * n + j] - gg;
      }
    for (int k = 0; k < p; ++k)
      for (int j = 0; j < n; ++j) { at(n + k, j) = P.G[(size_t)k * n + j]; at(j, n + k) = P.G[(size_t)k * n + j]; }
    for (int k = 0; k < m; ++k)
      for (int j = 0; j < n; ++j) { at(n + p + k, j) = P.A[(size_t)k * n + j]; at(j, n + p + k) = P.A[(size_t)k * n + j]; }
    for (int k = 0; k < p; ++k) at(n + k, n + k) = -F.dm[k];
    F.ok = lu_factor(K, N, F.piv);
  } else {
    // Congruent form M = S' K14 S with S = [[I,0,0],[G,I,0],[0,0,I]] (dv = G dx + w):
    // M = [[Q + G'D+G, G'D+, A'], [D+G, -D-, 0], [A, 0, 0]]  (App. A.2).
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        T gg = 0;
        for (int k = 0; k < p; ++k) gg += P.G[(size_t)k * n + i] * F.dp[k] * P.G[(size_t)k * n + j];
        at(i, j) = P.Q[(size_t)i * n + j] + gg;
      }
    for (int k = 0; k < p; ++k)
      for (int j = 0; j < n; ++j) {
        T c = F.dp[k] * P.G[(size_t)k * n + j];
        at(n + k, j) = c; at(j, n + k) = c;
      }
    for (int k = 0; k < m; ++k)
      for (int j = 0; j < n; ++j) { at(n + p + k, j) = P.A[(size_t)k * n + j]; at(j, n + p + k) = P.A[(size_t)k * n + j]; }
    for (int k = 0; k < p; ++k) at(n + k, n + k) = -F.dm[k];
    F.nfloor = ldl_factor(K, N, n, floor_rel, F.D);
    F.ok = true;
  }
  if (solver == SOLVER_M_PART) {
    // Reading Q12b: eliminate from M the w_i of every constraint
    // with v_i <= 0 (pivot -d-_i, d-_i >= 1/2).  Exact block elimination; the
    // reduced matrix keeps only bounded weights:
    //   [[Q + G' diag(w) G, G_A' D+_A, A'], [D+_A G_A, -D-_A, 0], [A, 0, 0]],
    //   w_i = d+_i (v_i > 0),  w_i = d+_i / d-_i = b(v_i)/b(-v_i) <= 1 (v_i <= 0).
    F.act.clear();
    for (int i = 0; i < p; ++i)
      if (v[i] > T(0)) F.act.push_back(i);
    // Reading Q12c: if more than pcap constraints have v_i > 0,
    // keep only the pcap with the largest v_i (ties: smaller index first) and
    // eliminate the others exactly like the v_i <= 0 ones (weight d+/d-).
    if (pcap >= 0 && (int)F.act.size() > pcap) {
      std::vector<int> order = F.act;
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return v[a] > v[b]; });
      order.resize(pcap);
      std::sort(order.begin(), order.end());
      F.act = order;
    }
    std::vector<char> kept(p, 0);
    for (int i : F.act) kept[i] = 1;
    const int pa = (int)F.act.size(), Nr = n + pa + m;
    F.N = Nr;
    K.assign((size_t)Nr * Nr, 0);
    auto ar = [&](int i, int j) -> T& { return K[(size_t)i * Nr + j]; };
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        T gg = 0;
        for (int k = 0; k < p; ++k) {
          const T w = kept[k] ? F.dp[k] : F.dp[k] / F.dm[k];
          gg += P.G[(size_t)k * n + i] * w * P.G[(size_t)k * n + j];
        }
        ar(i, j) = P.Q[(size_t)i * n + j] + gg;
      }
    for (int a = 0; a < pa; ++a) {
      const int k = F.act[a];
      for (int j = 0; j < n; ++j) {
        T c = F.dp[k] * P.G[(size_t)k * n + j];
        ar(n + a, j) = c; ar(j, n + a) = c;
      }
      ar(n + a, n + a) = -F.dm[k];
    }
    for (int k = 0; k < m; ++k)
      for (int j = 0; j < n; ++j) { ar(n + pa + k, j) = P.A[(size_t)k * n + j]; ar(j, n + pa + k) = P.A[(size_t)k * n + j]; }
    F.nfloor = ldl_factor(K, Nr, n, floor_rel, F.D);
    F.ok = true;
  }
  return F;
}

// solve_kkt: K14 (dx, dv, dy) = (f1, f2, f3).
template <typename T>
static void solve_kkt(const Prob<T>& P, const Factor<T>& F, const T* f1, const T* f2, const T* f3, T* dx, T* dv,
                      T* dy) {
  const int n = P.n, m = P.m, p = P.p, N = n + p + m;
  std::vector<T> r(N);
  if (F.kind == SOLVER_K14_GEPP) {
    for (int i = 0; i < n; ++i) r[i] = f1[i];
    for (int i = 0; i < p; ++i) r[n + i] = f2[i];
    for (int i = 0; i < m; ++i) r[n + p + i] = f3[i];
    lu_solve(F.F, N, F.piv, r.data());
    for (int i = 0; i < n; ++i) dx[i] = r[i];
    for (int i = 0; i < p; ++i) dv[i] = r[n + i];
    for (int i = 0; i < m; ++i) dy[i] = r[n + p + i];
  } else if (F.kind == SOLVER_M_PART) {
    // reduced right-hand side: r1 = f1 + G'f2 + sum_{v_i<=0} g_i (d+_i/d-_i) f2_i
    const int pa = (int)F.act.size(), Nr = n + pa + m;
    std::vector<T> rr(Nr), t(p), Gf(n);
    std::vector<char> isact(p, 0);
    for (int i : F.act) isact[i] = 1;
    for (int i = 0; i < p; ++i) t[i] = isact[i] ? f2[i] : f2[i] * (T(1) + F.dp[i] / F.dm[i]);
    matTvec(P.G, p, n, t.data(), Gf.data());
    for (int i = 0; i < n; ++i) rr[i] = f1[i] + Gf[i];
    for (int a = 0; a < pa; ++a) rr[n + a] = f2[F.act[a]];
    for (int i = 0; i < m; ++i) rr[n + pa + i] = f3[i];
    ldl_solve(F.F, F.D, Nr, rr.data());
    for (int i = 0; i < n; ++i) dx[i] = rr[i];
    std::vector<T> Gdx(p), w(p);
    matvec(P.G, p, n, dx, Gdx.data());
    for (int i = 0; i < p; ++i) w[i] = (F.dp[i] * Gdx[i] - f2[i]) / F.dm[i];  // eliminated rows
    for (int a = 0; a < pa; ++a) w[F.act[a]] = rr[n + a];
    for (int i = 0; i < p; ++i) dv[i] = Gdx[i] + w[i];
    for (int i = 0; i < m; ++i) dy[i] = rr[n + pa + i];
  } else {
    // S' (f1, f2, f3) = (f1 + G' f2, f2, f3); solve M; dv = G dx + w.
    std::vector<T> Gf(n);
    matTvec(P.G, p, n, f2, Gf.data());
    for (int i = 0; i < n; ++i) r[i] = f1[i] + Gf[i];
    for (int i = 0; i < p; ++i) r[n + i] = f2[i];
    for (int i = 0; i < m; ++i) r[n + p + i] = f3[i];
    ldl_solve(F.F, F.D, N, r.data());
    for (int i = 0; i < n; ++i) dx[i] = r[i];
    std::vector<T> Gdx(p);
    matvec(P.G, p, n, dx, Gdx.data());
    for (int i = 0; i < p; ++i) dv[i] = Gdx[i] + r[n + i];
    for (int i = 0; i < m; ++i) dy[i] = r[n + p + i];
  }
}

// solve_kkt with the Newton right-hand side of Eq. 14 and the
// back-substitution of Eq. 13 rows 4-6:
//   dkappa = -r_kappa, dz = -r_z + B(v) dv + c dkappa, ds = -r_s - B(-v) dv + c dkappa.
template <typename T>
static void newton_direction(const Prob<T>& P, const Factor<T>& F, const Res<T>& R, T r_kappa, T* dx, T* dy, T* dz,
                             T* ds, T* dv, T& dk) {
  const int n = P.n, m = P.m, p = P.p;
  std::vector<T> f1(n), f2(p), f3(m), tmp(p), Gt(n);
  for (int i = 0; i < p; ++i) tmp[i] = R.ri[i] + R.rz[i] - R.rs[i];
  matTvec(P.G, p, n, tmp.data(), Gt.data());
  for (int i = 0; i < n; ++i) f1[i] = -(R.rt[i] - Gt[i]);                 // -(r_t - G'(r_i + r_z - r_s))
  for (int i = 0; i < p; ++i) f2[i] = -(R.ri[i] - R.rs[i] - F.c[i] * r_kappa);  // -(r_i - r_s - c r_k)
  for (int i = 0; i < m; ++i) f3[i] = -R.re[i];                           // -r_e
  solve_kkt(P, F, f1.data(), f2.data(), f3.data(), dx, dv, dy);
  dk = -r_kappa;
  for (int i = 0; i < p; ++i) {
    dz[i] = -R.rz[i] + F.dp[i] * dv[i] + F.c[i] * dk;
    ds[i] = -R.rs[i] - F.dm[i] * dv[i] + F.c[i] * dk;
  }
}

// Eq. 6 with fraction-to-boundary damping (reading Q3):
// alpha = min(1, tau * alpha_max); alpha_max = +inf if nothing blocks (Q20).
template <typename T> static T linesearch(const T* s, const T* z, const T* ds, const T* dz, int p, T tau) {
  T amax = std::numeric_limits<T>::infinity();
  for (int i = 0; i < p; ++i) {
    if (ds[i] < T(0)) amax = std::min(amax, -s[i] / ds[i]);
    if (dz[i] < T(0)) amax = std::min(amax, -z[i] / dz[i]);
  }
  return std::min(T(1), tau * amax);
}

// ---------------------------------------------------------------------------
// Initialization ("same as CVXOPT"; reading Q11 = S:149): solve
// [[Q, A', G'], [A, 0, 0], [G, 0, -I]] (x, y, z^) = (-q, b, h) by GEPP;
// s~ = -z^, z~ = z^; shift each by (1 + alpha) if alpha = -min >= 0.
// ---------------------------------------------------------------------------
template <typename T>
static bool initialize(const Prob<T>& P, T* x, T* y, T* z, T* s) {
  const int n = P.n, m = P.m, p = P.p, N = n + m + p;
  std::vector<T> K((size_t)N * N, 0), r(N);
  auto at = [&](int i, int j) -> T& { return K[(size_t)i * N + j]; };
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) at(i, j) = P.Q[(size_t)i * n + j];
  for (int k = 0; k < m; ++k)
    for (int j = 0; j < n; ++j) { at(n + k, j) = P.A[(size_t)k * n + j]; at(j, n + k) = P.A[(size_t)k * n + j]; }
  for (int k = 0; k < p; ++k) {
    for (int j = 0; j < n; ++j) { at(n + m + k, j) = P.G[(size_t)k * n + j]; at(j, n + m + k) = P.G[(size_t)k * n + j]; }
    at(n + m + k, n + m + k) = T(-1);
  }
  for (int i = 0; i < n; ++i) r[i] = -P.q[i];
  for (int i = 0; i < m; ++i) r[n + i] = P.b[i];
  for (int i = 0; i < p; ++i) r[n + m + i] = P.h[i];
  std::vector<int> piv;
  bool ok = lu_factor(K, N, piv);
  lu_solve(K, N, piv, r.data());
  for (int i = 0; i < n; ++i) x[i] = r[i];
  for (int i = 0; i < m; ++i) y[i] = r[n + i];
  if (p > 0) {
    T ap = -std::numeric_limits<T>::infinity(), ad = ap;
    for (int i = 0; i < p; ++i) {
      T zh = r[n + m + i];
      s[i] = -zh; z[i] = zh;
      ap = std::max(ap, zh);   // alpha_p = -min(s~) = max(z^)
      ad = std::max(ad, -zh);  // alpha_d = -min(z~)
    }
    if (ap >= T(0)) for (int i = 0; i < p; ++i) s[i] += T(1) + ap;
    if (ad >= T(0)) for (int i = 0; i < p; ++i) z[i] += T(1) + ad;
  }
  bool fin = ok;
  for (int i = 0; i < n; ++i) fin = fin && std::isfinite(x[i]);
  for (int i = 0; i < p; ++i) fin = fin && std::isfinite(z[i]) && std::isfinite(s[i]);
  return fin;
}

template <typename T> static T mean_sz(const T* s, const T* z, int p) {
  // kappa = s'z / p  (Alg. 1 line 6, with the divisor read as p: Q1)
  return p > 0 ? dotp(s, z, p) / T(p) : T(0);
}

// ---------------------------------------------------------------------------
// Algorithm 1: solve_qp with implicit complementarity.
// iters = number of Newton steps taken.
// ---------------------------------------------------------------------------
template <typename T>
static int solve_qp_implicit(const Prob<T>& P, const oracle_cfg& cfg, T* x, T* y, T* z, T* s, int* iters,
                             Factor<T>* cache = nullptr) {
  bool cached = false;
  const int n = P.n, m = P.m, p = P.p;
  const T tol = T(cfg.tol), sigma = T(cfg.sigma), tau = T(cfg.tau), fr = T(cfg.pivot_floor_rel);
  *iters = 0;
  if (!initialize(P, x, y, z, s)) return ST_NUMERICAL_FAILURE | (STG_INIT << 8);
  std::vector<T> v(p), dx(n), dy(m), dz(p), ds(p), dv(p);
  Res<T> R;
  for (int k = 0;; ++k) {
    for (int i = 0; i < p; ++i) v[i] = z[i] - s[i];  // v <- z - s
    T kappa = mean_sz(s, z, p);                      // kappa <- s'z/p
    residuals(P, x, y, z, s, kappa, true, R);
    *iters = k;
    if (converged_solve(R, tol)) return ST_CONVERGED;
    if (k == cfg.max_iter) return ST_MAX_ITER;
    Factor<T> F = factor_kkt(P, v.data(), kappa, cfg.kkt_solver, fr, cfg.partition_cap);
    if (!finite_all(F.dp) || !finite_all(F.dm) || !finite_all(F.c)) return ST_NUMERICAL_FAILURE | (STG_SCALING << 8);
    // N2(i): keep the factorisation of the first iterate with kappa below
    // sqrt(10) kappa_relax (the iterates pass kappa_relax about one decade per step)
    if (cache && !cached && kappa < std::sqrt(T(10)) * T(cfg.kappa_relax)) { *cache = F; cached = true; }
    T kt = sigma * kappa;                 // kappa_target <- sigma kappa
    T rk = kappa - kt;                    // r_kappa = kappa - kappa_target
    T dk;
    newton_direction(P, F, R, rk, dx.data(), dy.data(), dz.data(), ds.data(), dv.data(), dk);
    if (!F.ok || !finite_all(dx) || !finite_all(dy) || !finite_all(dv) || !finite_all(dz) || !finite_all(ds))
      return ST_NUMERICAL_FAILURE | (STG_CORRECTOR << 8);
    T alpha = linesearch(s, z, ds.data(), dz.data(), p, tau);
    if (!std::isfinite(alpha)) return ST_NUMERICAL_FAILURE | (STG_LINESEARCH << 8);
    // step on (x, y, v, kappa), then retract
    for (int i = 0; i < n; ++i) x[i] += alpha * dx[i];
    for (int i = 0; i < m; ++i) y[i] += alpha * dy[i];
    T kn = kappa + alpha * dk;
    for (int i = 0; i < p; ++i) {
      T vn = v[i] + alpha * dv[i];
      z[i] = retract_b(vn, kn);
      s[i] = retract_b(-vn, kn);
    }
  }
}

// ---------------------------------------------------------------------------
// Algorithm 2: relax the solution to kappa_relax.  Exact Newton,
// factor-then-check (reading Q6) so the returned factor sits at the relaxed
// point; convergence adds |kappa/kappa_relax - 1| <= relax_ktol (reading Q5).
// ---------------------------------------------------------------------------
template <typename T>
static int relax_qp_implicit(const Prob<T>& P, const oracle_cfg& cfg, T* x, T* y, T* z, T* s, int* iters,
                             Factor<T>& F, const Factor<T>* chord = nullptr) {
  const int n = P.n, m = P.m, p = P.p;
  const T tol = T(cfg.tol), tau = T(cfg.tau), kr = T(cfg.kappa_relax), ktol = T(cfg.relax_ktol),
          fr = T(cfg.pivot_floor_rel), rtol = T(cfg.relax_tol);
  std::vector<T> v(p), dx(n), dy(m), dz(p), ds(p), dv(p);
  Res<T> R;
  T phi_prev = std::numeric_limits<T>::infinity();
  // relax_mode 2 (guarded chord, reading Q26): chord steps on the cached Alg. 1
  // factorisation while each shrinks psi = max(phi, |kappa/kappa_relax - 1|) by
  // chord_rho, at most chord_max of them; from the first that does not, exact
  // Newton (Q6) to the end.  relax_mode 1: chord steps throughout.
  const bool guarded = cfg.relax_mode == 2;
  bool use_chord = chord != nullptr;
  int nchord = 0;
  T psi_prev = std::numeric_limits<T>::infinity();
  for (int k = 0;; ++k) {
    for (int i = 0; i < p; ++i) v[i] = z[i] - s[i];
    T kappa = mean_sz(s, z, p);
    residuals(P, x, y, z, s, kappa, true, R);
    *iters = k;
    bool kok = p == 0 || std::fabs(kappa / kr - T(1)) <= ktol;
    if (use_chord && guarded) {
      const T psi = std::max(rel_phi(R), p == 0 ? T(0) : std::fabs(kappa / kr - T(1)));
      if (nchord >= cfg.chord_max || (nchord > 0 && !(psi <= T(cfg.chord_rho) * psi_prev))) {
        use_chord = false;
        phi_prev = std::numeric_limits<T>::infinity();  // the stall test (Q5b) measures Newton steps only
      }
      psi_prev = psi;
    }
    // a guarded chord stops only at phi <= relax_tol: a slow chord is not the working-precision floor
    const bool done = kok && (use_chord && guarded ? rel_phi(R) <= rtol : relax_done(R, tol, rtol, phi_prev));
    if (!use_chord || done) {
      // exact Newton (or the final factorisation at the relaxed point, for Alg. 3)
      F = factor_kkt(P, v.data(), kappa, cfg.kkt_solver, fr, cfg.partition_cap);
      if (!finite_all(F.dp) || !finite_all(F.dm) || !F.ok) return ST_NUMERICAL_FAILURE | (STG_RELAX << 8);
    }
    if (done) {
      if (chord && std::getenv("ORACLE_CHORD_STATS")) std::fprintf(stderr, "chord_stats %d %d\n", k, nchord);
      return ST_CONVERGED;
    }
    phi_prev = kok ? rel_phi(R) : std::numeric_limits<T>::infinity();
    if (k == cfg.relax_max_iter) return ST_MAX_ITER | (STG_RELAX << 8);
    T rk = kappa - kr;  // kappa_target = kappa_relax
    T dk;
    // chord step (N2(i)): the Newton system of Alg. 1's cached factorisation, current residuals
    newton_direction(P, use_chord ? *chord : F, R, rk, dx.data(), dy.data(), dz.data(), ds.data(), dv.data(), dk);
    if (use_chord) ++nchord;
    if (!finite_all(dx) || !finite_all(dv) || !finite_all(dz) || !finite_all(ds))
      return ST_NUMERICAL_FAILURE | (STG_RELAX << 8);
    T alpha = linesearch(s, z, ds.data(), dz.data(), p, tau);
    for (int i = 0; i < n; ++i) x[i] += alpha * dx[i];
    for (int i = 0; i < m; ++i) y[i] += alpha * dy[i];
    T kn = kappa + alpha * dk;
    for (int i = 0; i < p; ++i) {
      T vn = v[i] + alpha * dv[i];
      z[i] = retract_b(vn, kn);
      s[i] = retract_b(-vn, kn);
    }
  }
}

// ---------------------------------------------------------------------------
// Algorithm 3 with the sign reading Q7 (solve K (dx, dv, dy) =
// (-grad_x l, 0, 0) directly) and dz = d+ . dv (reading Q8).
// ---------------------------------------------------------------------------
template <typename T>
static void grads_from_factor(const Prob<T>& P, const Factor<T>& F, const T* x, const T* y, const T* z,
                              const T* dl, T* gQ, T* gq, T* gA, T* gb, T* gG, T* gh) {
  const int n = P.n, m = P.m, p = P.p;
  std::vector<T> f1(n), f2(p, 0), f3(m, 0), dx(n), dv(p), dy(m), dz(p);
  for (int i = 0; i < n; ++i) f1[i] = -dl[i];
  solve_kkt(P, F, f1.data(), f2.data(), f3.data(), dx.data(), dv.data(), dy.data());
  for (int i = 0; i < p; ++i) dz[i] = F.dp[i] * dv[i];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) gQ[(size_t)i * n + j] = T(0.5) * (dx[i] * x[j] + x[i] * dx[j]);
  for (int i = 0; i < n; ++i) gq[i] = dx[i];
  for (int k = 0; k < m; ++k)
    for (int j = 0; j < n; ++j) gA[(size_t)k * n + j] = dy[k] * x[j] + y[k] * dx[j];
  for (int k = 0; k < m; ++k) gb[k] = -dy[k];
  for (int k = 0; k < p; ++k)
    for (int j = 0; j < n; ++j) gG[(size_t)k * n + j] = dz[k] * x[j] + z[k] * dx[j];
  for (int k = 0; k < p; ++k) gh[k] = -dz[k];
}

// ===========================================================================
// Standard ("explicit") arm — the comparison formulation of Eq. 8
// (P:208-236), reconstructed as Mehrotra predictor-corrector (reading Q18;
// SPEC S:336-356): affine predictor with r_c = z.s, sigma = (mu_aff/mu)^3,
// corrector r_c = z.s + ds_a.dz_a - sigma mu.  KKT solves use Eq. 8 either by
// GEPP (paper-literal) or by the normal equations H = Q + G'D(z/s)G with
// Cholesky (+ A-Schur) (SOLVER_NORMAL_CHOL, the usual implementation).
// ===========================================================================
template <typename T> struct XFactor {
  int kind;
  std::vector<T> F, D;  // GEPP LU of Eq. 8, or LDL of [[H, A'], [A, 0]]
  std::vector<int> piv;
  std::vector<T> w;  // z/s
  bool ok = true;
};

template <typename T>
static XFactor<T> factor_explicit(const Prob<T>& P, const T* z, const T* s, int solver, T fr) {
  const int n = P.n, m = P.m, p = P.p;
  XFactor<T> F;
  F.kind = solver;
  F.w.resize(p);
  for (int i = 0; i < p; ++i) F.w[i] = z[i] / s[i];
  if (solver == SOLVER_K14_GEPP) {
    const int N = n + m + p;  // Eq. 8 unknowns (dx, dy, dz)
    F.F.assign((size_t)N * N, 0);
    auto at = [&](int i, int j) -> T& { return F.F[(size_t)i * N + j]; };
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) at(i, j) = P.Q[(size_t)i * n + j];
    for (int k = 0; k < m; ++k)
      for (int j = 0; j < n; ++j) { at(n + k, j) = P.A[(size_t)k * n + j]; at(j, n + k) = P.A[(size_t)k * n + j]; }
    for (int k = 0; k < p; ++k) {
      for (int j = 0; j < n; ++j) { at(n + m + k, j) = P.G[(size_t)k * n + j]; at(j, n + m + k) = P.G[(size_t)k * n + j]; }
      at(n + m + k, n + m + k) = -s[k] / z[k];  // -D(s ./ z)
    }
    F.ok = lu_factor(F.F, N, F.piv);
  } else {
    const int N = n + m;
    F.F.assign((size_t)N * N, 0);
    auto at = [&](int i, int j) -> T& { return F.F[(size_t)i * N + j]; };
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        T gg = 0;
        for (int k = 0; k < p; ++k) gg += P.G[(size_t)k * n + i] * F.w[k] * P.G[(size_t)k * n + j];
        at(i, j) = P.Q[(size_t)i * n + j] + gg;
      }
    for (int k = 0; k < m; ++k)
      for (int j = 0; j < n; ++j) { at(n + k, j) = P.A[(size_t)k * n + j]; at(j, n + k) = P.A[(size_t)k * n + j]; }
    // No pivot floor on the standard arm: a breakdown must surface as a
    // non-finite value, which is what the ablation counts.
    (void)fr;
    ldl_factor(F.F, N, n, T(0), F.D);
    F.ok = finite_all(F.F) && finite_all(F.D);
  }
  return F;
}

// Eq. 8 solve with right-hand side -(r_t, r_e, r_i - r_c ./ z); ds from Eq. 7
// row 4: ds = -(r_c + s.dz)./z.
template <typename T>
static void explicit_direction(const Prob<T>& P, const XFactor<T>& F, const T* z, const T* s, const T* rt,
                               const T* re, const T* ri, const T* rc, T* dx, T* dy, T* dz, T* ds) {
  const int n = P.n, m = P.m, p = P.p;
  std::vector<T> u(p);
  for (int i = 0; i < p; ++i) u[i] = ri[i] - rc[i] / z[i];
  if (F.kind == SOLVER_K14_GEPP) {
    const int N = n + m + p;
    std::vector<T> r(N);
    for (int i = 0; i < n; ++i) r[i] = -rt[i];
    for (int i = 0; i < m; ++i) r[n + i] = -re[i];
    for (int i = 0; i < p; ++i) r[n + m + i] = -u[i];
    lu_solve(F.F, N, F.piv, r.data());
    for (int i = 0; i < n; ++i) dx[i] = r[i];
    for (int i = 0; i < m; ++i) dy[i] = r[n + i];
    for (int i = 0; i < p; ++i) dz[i] = r[n + m + i];
  } else {
    // dz = D(z/s)(G dx + u);  (Q + G'D(z/s)G) dx + A'dy = -r_t - G'D(z/s)u
    const int N = n + m;
    std::vector<T> r(N), wu(p), Gt(n);
    for (int i = 0; i < p; ++i) wu[i] = F.w[i] * u[i];
    matTvec(P.G, p, n, wu.data(), Gt.data());
    for (int i = 0; i < n; ++i) r[i] = -rt[i] - Gt[i];
    for (int i = 0; i < m; ++i) r[n + i] = -re[i];
    ldl_solve(F.F, F.D, N, r.data());
    for (int i = 0; i < n; ++i) dx[i] = r[i];
    for (int i = 0; i < m; ++i) dy[i] = r[n + i];
    std::vector<T> Gdx(p);
    matvec(P.G, p, n, dx, Gdx.data());
    for (int i = 0; i < p; ++i) dz[i] = F.w[i] * (Gdx[i] + u[i]);
  }
  for (int i = 0; i < p; ++i) ds[i] = -(rc[i] + s[i] * dz[i]) / z[i];
}

template <typename T> static bool all_finite_n(const T* a, int k) {
  for (int i = 0; i < k; ++i)
    if (!std::isfinite(a[i])) return false;
  return true;
}

template <typename T>
static int solve_qp_explicit(const Prob<T>& P, const oracle_cfg& cfg, T* x, T* y, T* z, T* s, int* iters) {
  const int n = P.n, m = P.m, p = P.p;
  const T tol = T(cfg.tol), tau = T(cfg.tau), fr = T(cfg.pivot_floor_rel);
  *iters = 0;
  if (!initialize(P, x, y, z, s)) return ST_NUMERICAL_FAILURE | (STG_INIT << 8);
  std::vector<T> dx(n), dy(m), dz(p), ds(p), dxa(n), dya(m), dza(p), dsa(p), rc(p);
  Res<T> R;
  for (int k = 0;; ++k) {
    residuals(P, x, y, z, s, T(0), false, R);
    *iters = k;
    if (converged_solve(R, tol)) return ST_CONVERGED;
    if (k == cfg.max_iter) return ST_MAX_ITER;
    T mu = mean_sz(s, z, p);
    XFactor<T> F = factor_explicit(P, z, s, cfg.kkt_solver, fr);
    if (!finite_all(F.w)) return ST_NUMERICAL_FAILURE | (STG_SCALING << 8);
    for (int i = 0; i < p; ++i) rc[i] = z[i] * s[i];  // affine predictor: kappa = 0
    explicit_direction(P, F, z, s, R.rt.data(), R.re.data(), R.ri.data(), rc.data(), dxa.data(), dya.data(),
                       dza.data(), dsa.data());
    if (!F.ok || !finite_all(dxa) || !finite_all(dza) || !finite_all(dsa))
      return ST_NUMERICAL_FAILURE | (STG_PREDICTOR << 8);
    T aa = linesearch(s, z, dsa.data(), dza.data(), p, T(1));
    T mua = 0;
    for (int i = 0; i < p; ++i) mua += (s[i] + aa * dsa[i]) * (z[i] + aa * dza[i]);
    mua /= T(p);
    T sig = sq(mua / mu) * (mua / mu);  // sigma = (mu_aff/mu)^3
    if (!std::isfinite(sig) || !std::isfinite(mu)) return ST_NUMERICAL_FAILURE | (STG_CENTERING << 8);
    for (int i = 0; i < p; ++i) rc[i] = z[i] * s[i] + dsa[i] * dza[i] - sig * mu;
    explicit_direction(P, F, z, s, R.rt.data(), R.re.data(), R.ri.data(), rc.data(), dx.data(), dy.data(),
                       dz.data(), ds.data());
    if (!finite_all(dx) || !finite_all(dz) || !finite_all(ds)) return ST_NUMERICAL_FAILURE | (STG_CORRECTOR << 8);
    T alpha = linesearch(s, z, ds.data(), dz.data(), p, tau);
    if (!std::isfinite(alpha)) return ST_NUMERICAL_FAILURE | (STG_LINESEARCH << 8);
    for (int i = 0; i < n; ++i) x[i] += alpha * dx[i];
    for (int i = 0; i < m; ++i) y[i] += alpha * dy[i];
    for (int i = 0; i < p; ++i) { z[i] += alpha * dz[i]; s[i] += alpha * ds[i]; }
    if (!all_finite_n(z, p) || !all_finite_n(s, p)) return ST_NUMERICAL_FAILURE | (STG_LINESEARCH << 8);
  }
}

// Explicit relaxation: centering Newton steps on r_c = z.s - kappa_relax
// until feasible and max|z_i s_i/kappa_relax - 1| <= ktol.
template <typename T>
static int relax_qp_explicit(const Prob<T>& P, const oracle_cfg& cfg, T* x, T* y, T* z, T* s, int* iters,
                             XFactor<T>& F) {
  const int n = P.n, m = P.m, p = P.p;
  const T tol = T(cfg.tol), tau = T(cfg.tau), kr = T(cfg.kappa_relax), ktol = T(cfg.relax_ktol),
          fr = T(cfg.pivot_floor_rel), rtol = T(cfg.relax_tol);
  std::vector<T> dx(n), dy(m), dz(p), ds(p), rc(p);
  Res<T> R;
  T phi_prev = std::numeric_limits<T>::infinity();
  for (int k = 0;; ++k) {
    residuals(P, x, y, z, s, T(0), false, R);
    F = factor_explicit(P, z, s, cfg.kkt_solver, fr);
    *iters = k;
    if (!finite_all(F.w) || !F.ok) return ST_NUMERICAL_FAILURE | (STG_RELAX << 8);
    T dev = 0;
    for (int i = 0; i < p; ++i) dev = std::max(dev, std::fabs(z[i] * s[i] / kr - T(1)));
    if (dev <= ktol && relax_done(R, tol, rtol, phi_prev)) return ST_CONVERGED;
    phi_prev = dev <= ktol ? rel_phi(R) : std::numeric_limits<T>::infinity();
    if (k == cfg.relax_max_iter) return ST_MAX_ITER | (STG_RELAX << 8);
    for (int i = 0; i < p; ++i) rc[i] = z[i] * s[i] - kr;
    explicit_direction(P, F, z, s, R.rt.data(), R.re.data(), R.ri.data(), rc.data(), dx.data(), dy.data(),
                       dz.data(), ds.data());
    if (!finite_all(dx) || !finite_all(dz) || !finite_all(ds)) return ST_NUMERICAL_FAILURE | (STG_RELAX << 8);
    T alpha = linesearch(s, z, ds.data(), dz.data(), p, tau);
    for (int i = 0; i < n; ++i) x[i] += alpha * dx[i];
    for (int i = 0; i < m; ++i) y[i] += alpha * dy[i];
    for (int i = 0; i < p; ++i) { z[i] += alpha * dz[i]; s[i] += alpha * ds[i]; }
  }
}

// Explicit adjoint (IFT on Eq. 4 at the relaxed point):
// (Q + G'D(z/s)G) dx + A'dy = -grad, A dx = 0, dz = D(z/s) G dx; Alg. 3's
// formulas.  (Same solution as the implicit adjoint in exact arithmetic.)
template <typename T>
static void grads_explicit(const Prob<T>& P, const XFactor<T>& F, const T* x, const T* y, const T* z,
                           const T* s, const T* dl, T* gQ, T* gq, T* gA, T* gb, T* gG, T* gh) {
  const int n = P.n, m = P.m, p = P.p;
  std::vector<T> rt(n), re(m, 0), ri(p, 0), rc(p, 0), dx(n), dy(m), dz(p), ds(p);
  for (int i = 0; i < n; ++i) rt[i] = dl[i];  // explicit_direction negates: -r_t = -grad
  explicit_direction(P, F, z, s, rt.data(), re.data(), ri.data(), rc.data(), dx.data(), dy.data(), dz.data(),
                     ds.data());
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) gQ[(size_t)i * n + j] = T(0.5) * (dx[i] * x[j] + x[i] * dx[j]);
  for (int i = 0; i < n; ++i) gq[i] = dx[i];
  for (int k = 0; k < m; ++k)
    for (int j = 0; j < n; ++j) gA[(size_t)k * n + j] = dy[k] * x[j] + y[k] * dx[j];
  for (int k = 0; k < m; ++k) gb[k] = -dy[k];
  for (int k = 0; k < p; ++k)
    for (int j = 0; j < n; ++j) gG[(size_t)k * n + j] = dz[k] * x[j] + z[k] * dx[j];
  for (int k = 0; k < p; ++k) gh[k] = -dz[k];
}

// ---------------------------------------------------------------------------
// Batch drivers (std::thread over independent problems).
// ---------------------------------------------------------------------------
template <typename T> struct BatchData {
  int n, m, p;
  const T *Q, *q, *A, *b, *G, *h;
  long long sQ, sq, sA, sb, sG, sh;
  Prob<T> at(int i) const {
    return Prob<T>{n, m, p, Q + sQ * i, q + sq * i, A + sA * i, b + sb * i, G + sG * i, h + sh * i};
  }
};

template <typename F> static void parallel_for(int B, int nthreads, F fn) {
  if (nthreads <= 1 || B <= 1) {
    for (int i = 0; i < B; ++i) fn(i);
    return;
  }
  std::atomic<int> next(0);
  std::vector<std::thread> th;
  int nt = std::min(nthreads, B);
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&]() {
      for (int i = next.fetch_add(1); i < B; i = next.fetch_add(1)) fn(i);
    });
  for (auto& t : th) t.join();
}

template <typename T>
static void solve_batch(const oracle_cfg& cfg, const BatchData<T>& D, int B, T* x, T* y, T* z, T* s, int* iters,
                        int* status, int nthreads) {
  parallel_for(B, nthreads, [&](int i) {
    Prob<T> P = D.at(i);
    T *xi = x + (size_t)i * D.n, *yi = y + (size_t)i * D.m, *zi = z + (size_t)i * D.p, *si = s + (size_t)i * D.p;
    status[i] = cfg.formulation == FORM_EXPLICIT ? solve_qp_explicit(P, cfg, xi, yi, zi, si, &iters[i])
                                                 : solve_qp_implicit(P, cfg, xi, yi, zi, si, &iters[i]);
  });
}

template <typename T>
static void backward_batch(const oracle_cfg& cfg, const BatchData<T>& D, int B, const T* x, const T* y,
                           const T* z, const T* s, const T* dl, T* gQ, T* gq, T* gA, T* gb, T* gG, T* gh, T* xr,
                           T* yr, T* zr, T* sr, int* riters, int* status, int nthreads) {
  const int n = D.n, m = D.m, p = D.p;
  parallel_for(B, nthreads, [&](int i) {
    Prob<T> P = D.at(i);
    T *xi = xr + (size_t)i * n, *yi = yr + (size_t)i * m, *zi = zr + (size_t)i * p, *si = sr + (size_t)i * p;
    std::memcpy(xi, x + (size_t)i * n, sizeof(T) * n);
    std::memcpy(yi, y + (size_t)i * m, sizeof(T) * m);
    std::memcpy(zi, z + (size_t)i * p, sizeof(T) * p);
    std::memcpy(si, s + (size_t)i * p, sizeof(T) * p);
    T *gQi = gQ + (size_t)i * n * n, *gqi = gq + (size_t)i * n, *gAi = gA + (size_t)i * m * n,
      *gbi = gb + (size_t)i * m, *gGi = gG + (size_t)i * p * n, *ghi = gh + (size_t)i * p;
    int st;
    if (cfg.formulation == FORM_EXPLICIT) {
      XFactor<T> F;
      st = relax_qp_explicit(P, cfg, xi, yi, zi, si, &riters[i], F);
      if ((st & 0xff) == ST_CONVERGED) grads_explicit(P, F, xi, yi, zi, si, dl + (size_t)i * n, gQi, gqi, gAi, gbi, gGi, ghi);
    } else {
      Factor<T> F, C;
      const Factor<T>* chord = nullptr;
      if (cfg.relax_mode == 1 || cfg.relax_mode == 2) {
        // N2(i): the factorisation Alg. 1 computed nearest kappa_relax, recomputed
        // here by re-running the (deterministic) forward solve
        std::vector<T> xs(n), ys(m), zs(p), ss(p);
        int it0;
        C.N = -1;
        solve_qp_implicit(P, cfg, xs.data(), ys.data(), zs.data(), ss.data(), &it0, &C);
        if (C.N >= 0) chord = &C;
      }
      st = relax_qp_implicit(P, cfg, xi, yi, zi, si, &riters[i], F, chord);
      if ((st & 0xff) == ST_CONVERGED) grads_from_factor(P, F, xi, yi, zi, dl + (size_t)i * n, gQi, gqi, gAi, gbi, gGi, ghi);
    }
    if ((st & 0xff) == ST_CONVERGED) {
      bool fin = all_finite_n(gQi, n * n) && all_finite_n(gqi, n) && all_finite_n(gGi, p * n) && all_finite_n(gAi, m * n);
      if (!fin) st = ST_NUMERICAL_FAILURE | (STG_BACKWARD << 8);
    }
    if ((st & 0xff) != ST_CONVERGED) {  // failed problems: zero-filled gradients
      std::fill(gQi, gQi + (size_t)n * n, T(0)); std::fill(gqi, gqi + n, T(0));
      std::fill(gAi, gAi + (size_t)m * n, T(0)); std::fill(gbi, gbi + m, T(0));
      std::fill(gGi, gGi + (size_t)p * n, T(0)); std::fill(ghi, ghi + p, T(0));
    }
    status[i] = st;
  });
}

}  // namespace orc

// ===========================================================================
// extern "C" surface (loaded by oracle/__init__.py through ctypes).
// ===========================================================================
#define ORACLE_BATCH_API(T, SUF)                                                                              \
  extern "C" int oracle_solve_##SUF(const oracle_cfg* cfg, int B, int n, int m, int p, const T* Q,           \
                                    long long sQ, const T* q, long long sq, const T* A, long long sA,        \
                                    const T* b, long long sb, const T* G, long long sG, const T* h,          \
                                    long long sh, T* x, T* y, T* z, T* s, int* iters, int* status,           \
                                    int nthreads) {                                                          \
    orc::BatchData<T> D{n, m, p, Q, q, A, b, G, h, sQ, sq, sA, sb, sG, sh};                                  \
    orc::solve_batch(*cfg, D, B, x, y, z, s, iters, status, nthreads);                                       \
    return 0;                                                                                                \
  }                                                                                                          \
  extern "C" int oracle_backward_##SUF(                                                                      \
      const oracle_cfg* cfg, int B, int n, int m, int p, const T* Q, long long sQ, const T* q, long long sq, \
      const T* A, long long sA, const T* b, long long sb, const T* G, long long sG, const T* h,              \
      long long sh, const T* x, const T* y, const T* z, const T* s, const T* dl, T* gQ, T* gq, T* gA,        \
      T* gb, T* gG, T* gh, T* xr, T* yr, T* zr, T* sr, int* riters, int* status, int nthreads) {             \
    orc::BatchData<T> D{n, m, p, Q, q, A, b, G, h, sQ, sq, sA, sb, sG, sh};                                  \
    orc::backward_batch(*cfg, D, B, x, y, z, s, dl, gQ, gq, gA, gb, gG, gh, xr, yr, zr, sr, riters, status,  \
                        nthreads);                                                                           \
    return 0;                                                                                                \
  }                                                                                                          \
  extern "C" void oracle_retract_##SUF(int k, const T* v, T kappa, T* z, T* s, T* dp, T* dm, T* c) {         \
    for (int i = 0; i < k; ++i) {                                                                            \
      z[i] = orc::retract_b(v[i], kappa);                                                                    \
      s[i] = orc::retract_b(-v[i], kappa);                                                                   \
      dp[i] = orc::retract_db(v[i], kappa);                                                                  \
      dm[i] = orc::retract_db(-v[i], kappa);                                                                 \
      c[i] = orc::retract_dkappa(v[i], kappa);                                                               \
    }                                                                                                        \
  }                                                                                                          \
  extern "C" T oracle_linesearch_##SUF(int p, const T* s, const T* z, const T* ds, const T* dz, T tau) {     \
    return orc::linesearch(s, z, ds, dz, p, tau);                                                            \
  }                                                                                                          \
  extern "C" int oracle_init_##SUF(int n, int m, int p, const T* Q, const T* q, const T* A, const T* b,      \
                                   const T* G, const T* h, T* x, T* y, T* z, T* s) {                         \
    orc::Prob<T> P{n, m, p, Q, q, A, b, G, h};                                                               \
    return orc::initialize(P, x, y, z, s) ? 0 : 1;                                                           \
  }                                                                                                          \
  /* One Newton step of Alg. 1 from (x,y,z,s): v, kappa from z, s; r_kappa = kappa - kappa_target. */        \
  extern "C" int oracle_newton_step_##SUF(int n, int m, int p, const T* Q, const T* q, const T* A,           \
                                          const T* b, const T* G, const T* h, const T* x, const T* y,        \
                                          const T* z, const T* s, T kappa_target, int solver, T floor_rel,   \
                                          int pcap, T* dx, T* dy, T* dz, T* ds, T* dv, T* dk, T* kappa_out) {          \
    orc::Prob<T> P{n, m, p, Q, q, A, b, G, h};                                                               \
    std::vector<T> v(p);                                                                                     \
    for (int i = 0; i < p; ++i) v[i] = z[i] - s[i];                                                          \
    T kappa = orc::mean_sz(s, z, p);                                                                         \
    orc::Res<T> R;                                                                                           \
    orc::residuals(P, x, y, z, s, kappa, true, R);                                                           \
    orc::Factor<T> F = orc::factor_kkt(P, v.data(), kappa, solver, floor_rel, pcap);                         \
    T dkk;                                                                                                   \
    orc::newton_direction(P, F, R, kappa - kappa_target, dx, dy, dz, ds, dv, dkk);                           \
    *dk = dkk;                                                                                               \
    *kappa_out = kappa;                                                                                      \
    return F.nfloor;                                                                                         \
  }                                                                                                          \
  /* Unpivoted signed LDL' of a dense N x N matrix (reading Q12, pivot floor) and one solve; M is          \
   * overwritten by L (strict lower part), D by the pivots, x (rhs on entry) by the solution.  Returns       \
   * the number of floored pivots.  (Test entry point: pins the floor branch of ldl_factor.) */              \
  extern "C" int oracle_ldl_##SUF(int N, int npos, T floor_rel, T* M, T* D, T* x) {                          \
    std::vector<T> Mv(M, M + (size_t)N * N), Dv;                                                             \
    const int nf = orc::ldl_factor(Mv, N, npos, floor_rel, Dv);                                              \
    orc::ldl_solve(Mv, Dv, N, x);                                                                            \
    std::copy(Mv.begin(), Mv.end(), M);                                                                      \
    std::copy(Dv.begin(), Dv.end(), D);                                                                      \
    return nf;                                                                                               \
  }                                                                                                          \
  /* Residual vectors (Eq. 4, Eq. 10) at (x,y,z,s) with kappa = s'z/p. */                                    \
  extern "C" void oracle_residuals_##SUF(int n, int m, int p, const T* Q, const T* q, const T* A,            \
                                         const T* b, const T* G, const T* h, const T* x, const T* y,         \
                                         const T* z, const T* s, T* rt, T* re, T* ri, T* rz, T* rs) {        \
    orc::Prob<T> P{n, m, p, Q, q, A, b, G, h};                                                               \
    orc::Res<T> R;                                                                                           \
    orc::residuals(P, x, y, z, s, orc::mean_sz(s, z, p), true, R);                                           \
    std::copy(R.rt.begin(), R.rt.end(), rt); std::copy(R.re.begin(), R.re.end(), re);                        \
    std::copy(R.ri.begin(), R.ri.end(), ri); std::copy(R.rz.begin(), R.rz.end(), rz);                        \
    std::copy(R.rs.begin(), R.rs.end(), rs);                                                                 \
  }

ORACLE_BATCH_API(double, f64)
ORACLE_BATCH_API(float, f32)

extern "C" int oracle_hardware_threads(void) { return (int)std::thread::hardware_concurrency(); }
