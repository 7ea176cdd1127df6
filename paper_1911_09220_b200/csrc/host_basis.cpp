// Host-side 1D tables: Gauss-Legendre / Gauss-Lobatto rules and the nodal
// Lagrange basis.  These are setup-time inputs of the device kernels (the
// B1d/G1d tables, the geometry basis tables); they follow the reference's
// algorithms step for step so the tables are bit-identical:
//   rules  : quadrature.cpp:20-125 (Newton on P_n / P'_n, mirrored roots)
//   basis  : basis.cpp:12-109 (barycentric weights, exact-node shortcut)
#include "common.cuh"

#include <cmath>

namespace tfem {

namespace {

constexpr double kPi = 3.14159265358979323846;

// (P_n(x), P'_n(x)) via the three-term recurrence, quadrature.cpp:20-31.
std::pair<double, double> legendre_pair(int n, double x)
{
   if (n == 0) return {1.0, 0.0};
   double prev = 1.0, cur = x;
   for (int k = 1; k < n; k++) {
      const double next = ((2 * k + 1) * x * cur - k * prev) / (k + 1);
      prev = cur;
      cur = next;
   }
   return {cur, n * (x * cur - prev) / (x * x - 1.0)};
}

template <typename F>
double newton(F &&f, double x)
{
   for (int it = 0; it < 100; it++) {
      const auto [v, dv] = f(x);
      const double step = v / dv;
      x -= step;
      if (std::abs(step) < 1e-15) return x;
   }
   runtime("quadrature: Newton iteration did not converge");
}

} // namespace

std::vector<double> gauss_points(int rule, int n, std::vector<double> *weights)
{
   std::vector<double> x(n), w(n);
   if (rule == TFEM_GAUSS_LEGENDRE) {
      if (n < 1) invalid("gauss_legendre: need n >= 1, got " + std::to_string(n));
      for (int i = 0; i < n / 2 + n % 2; i++) {
         const bool middle = (2 * i + 1 == n);
         const double xi =
            middle ? 0.0
                   : newton([n](double t) { return legendre_pair(n, t); },
                            -std::cos(kPi * (i + 0.75) / (n + 0.5)));
         const double dp = legendre_pair(n, xi).second;
         const double wi = middle ? 2.0 / (dp * dp) : 2.0 / ((1.0 - xi * xi) * dp * dp);
         x[i] = xi;
         x[n - 1 - i] = -xi;
         w[i] = w[n - 1 - i] = wi;
      }
   } else {
      if (n < 2) invalid("gauss_lobatto: need n >= 2, got " + std::to_string(n));
      const int m = n - 1;
      x[0] = -1.0;
      x[n - 1] = 1.0;
      auto dleg = [m](double t) {
         const auto [p, dp] = legendre_pair(m, t);
         return std::pair<double, double>{dp, (2.0 * t * dp - m * (m + 1) * p) / (1.0 - t * t)};
      };
      for (int i = 1; i <= (n - 1) / 2; i++) {
         const double xi = (2 * i == n - 1) ? 0.0 : newton(dleg, -std::cos(kPi * i / m));
         x[i] = xi;
         x[n - 1 - i] = -xi;
      }
      for (int i = 0; i < n; i++) {
         const double p = legendre_pair(m, x[i]).first;
         w[i] = 2.0 / (n * m * p * p);
      }
      for (int i = 0; i < n / 2; i++) w[i] = w[n - 1 - i] = 0.5 * (w[i] + w[n - 1 - i]);
   }
   std::vector<double> pts(n);
   for (int i = 0; i < n; i++) pts[i] = 0.5 * (x[i] + 1.0);
   if (weights) {
      weights->resize(n);
      for (int i = 0; i < n; i++) (*weights)[i] = 0.5 * w[i];
   }
   return pts;
}

void basis_nodes(int p, int node_kind, std::vector<double> &nodes, std::vector<double> &bary)
{
   if (p < 0) invalid("Basis1D: order must be >= 0, got " + std::to_string(p));
   const int n = p + 1;
   switch (node_kind) {
   case TFEM_NODES_GAUSS_LOBATTO:
      if (p < 1) invalid("Basis1D: Gauss-Lobatto nodes need order >= 1");
      nodes = gauss_points(TFEM_GAUSS_LOBATTO, n, nullptr);
      break;
   case TFEM_NODES_GAUSS_LEGENDRE:
      nodes = gauss_points(TFEM_GAUSS_LEGENDRE, n, nullptr);
      break;
   default:
      nodes.assign(n, 0.5);
      if (p > 0)
         for (int i = 0; i < n; i++) nodes[i] = double(i) / p;
   }
   bary.assign(n, 1.0);
   for (int j = 0; j < n; j++)
      for (int k = 0; k < n; k++)
         if (k != j) bary[j] /= nodes[j] - nodes[k];
}

void basis_eval(const std::vector<double> &nodes, const std::vector<double> &bary, double x,
                double *values, double *derivs)
{
   const int n = static_cast<int>(nodes.size());
   for (int i = 0; i < n; i++) {
      if (x != nodes[i]) continue;
      // Kronecker row; derivative row of the differentiation matrix with the
      // negative-sum diagonal (basis.cpp:53-58, 70-84).
      double diag = 0.0;
      for (int j = 0; j < n; j++) {
         values[j] = (j == i) ? 1.0 : 0.0;
         if (derivs && j != i) {
            derivs[j] = (bary[j] / bary[i]) / (nodes[i] - nodes[j]);
            diag -= derivs[j];
         }
      }
      if (derivs) derivs[i] = diag;
      return;
   }
   double denom = 0.0;
   for (int j = 0; j < n; j++) {
      values[j] = bary[j] / (x - nodes[j]);
      denom += values[j];
   }
   for (int j = 0; j < n; j++) values[j] /= denom;
   if (!derivs) return;
   double all = 0.0;
   for (int k = 0; k < n; k++) all += 1.0 / (x - nodes[k]);
   for (int j = 0; j < n; j++) derivs[j] = values[j] * (all - 1.0 / (x - nodes[j]));
}

void eval_matrices(int p, int node_kind, int nq, int rule, double *B, double *G)
{
   std::vector<double> nodes, bary;
   basis_nodes(p, node_kind, nodes, bary);
   const std::vector<double> pts = gauss_points(rule, nq, nullptr);
   for (int k = 0; k < nq; k++) basis_eval(nodes, bary, pts[k], B + k * (p + 1), G + k * (p + 1));
}

} // namespace tfem
