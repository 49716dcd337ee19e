// Host-side check of the device exp/division arithmetic in csrc/fexp.cuh:
// the same functions (__host__ __device__) compiled for the host.
// Prints: <n> <qdiv mismatches vs IEEE division> <fexp != libm exp> <max ulp>
#include <cstdio>
#include <cstdlib>
#include <random>
#include "../paper_2605_26659_b200/csrc/fexp.cuh"
int main(int argc, char **argv) {
  long N = argc > 1 ? atol(argv[1]) : 2000000;
  double2 tab[64];
  for (int k = 0; k < 64; ++k) tab[k] = make_double2(fb::EXP_TAB_H[k][0], fb::EXP_TAB_H[k][1]);
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  long badq = 0, bade = 0;
  double maxulp = 0;
  for (long it = 0; it < N; ++it) {
    double eps = std::pow(10.0, -3.0 + 3.0 * U(g));
    double d = -U(g) * (it % 3 == 0 ? 0.7 : (it % 3 == 1 ? 0.05 : 0.001));
    if (it % 11 == 0) d = -d;  // absorbed (positive) exponents
    double inv = 1.0 / eps;
    double q = d / eps, q2 = fb::q_div(d, eps, inv);
    if (q != q2) ++badq;
    if (!(q > -707.0 && q < 709.0)) continue;
    double e1 = std::exp(q), e2 = fb::fexp(q, tab);
    if (e1 != e2) {
      ++bade;
      double ulp = std::fabs(e1 - e2) / (std::nextafter(e1, INFINITY) - e1);
      if (ulp > maxulp) maxulp = ulp;
    }
  }
  printf("%ld %ld %ld %.3f\n", N, badq, bade, maxulp);
  return 0;
}
