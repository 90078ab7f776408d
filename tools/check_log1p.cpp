// Host check of csrc/fastmath.cuh's log1p against long-double log1pl:
// max error in ulps over random points spanning the ranges K2 sees
// (features: 0 .. 1e12, integers and fractions; softplus: exp(-|z|) in (0, 1]).
//   g++ -O2 -I paper_2012_07145_b200/csrc tools/check_log1p.cpp -o /tmp/check_log1p && /tmp/check_log1p
#include <cmath>
#include <cstdio>
#include <random>
#include "fastmath.cuh"

static double ulp_err(double got, long double want) {
  const double w = (double)want;
  const double ulp = std::nextafter(std::fabs(w), INFINITY) - std::fabs(w);
  return (double)(std::fabs((long double)got - want) / ulp);
}

int main() {
  std::mt19937_64 g(1);
  std::uniform_real_distribution<double> e(-60.0, 40.0), un(0.0, 1.0);
  double worst = 0, worst_x = 0;
  long n = 0, exact = 0;
  auto one = [&](double x) {
    const double got = gs::log1p_fast(x);
    const double ue = ulp_err(got, log1pl((long double)x));
    if (got == std::log1p(x)) ++exact;
    if (ue > worst) { worst = ue; worst_x = x; }
    ++n;
  };
  for (int i = 0; i < 4000000; ++i) one(std::exp2(e(g)));                 // log-uniform 2^-60 .. 2^40
  for (int i = 0; i < 2000000; ++i) one(un(g));                           // softplus side: (0, 1)
  for (int i = 0; i < 2000000; ++i) one(std::floor(std::exp2(e(g) * 0.5 + 10)));  // integer counts
  for (int i = 0; i < 2000000; ++i) one(std::exp(-std::fabs(40.0 * un(g))));       // exp(-|z|)
  for (double x : {0.0, 1e-320, 1e-300, 0x1p-53, 0x1p-52, 1.0, 2.0, 0.41421356237309503, 1e15, 1e300}) one(x);
  std::printf("points %ld  max error %.4f ulp at x=%.17g  equal to libm log1p: %.2f%%\n", n, worst, worst_x,
              100.0 * exact / n);
  return worst < 1.0 ? 0 : 1;
}
