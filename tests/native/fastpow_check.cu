// host-side accuracy check of nlg::fast_pow_pos against libm pow
#include <cmath>
#include <cstdio>
#include <random>
#include "../../paper_2207_03921_b200/csrc/nlg_math.cuh"
int main() {
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> ul(-75.0, 12.0), ue(-2.0, -0.999);
  double worst = 0;
  for (int i = 0; i < 4000000; ++i) {
    const double x = std::exp(ul(g));
    const double e = (i % 4 == 0) ? -1.4 : ue(g);
    const double a = nlg::fast_pow_pos(x, e), b = std::pow(x, e);
    const double rel = std::fabs(a - b) / b;
    if (rel > worst) worst = rel;
  }
  printf("%.3e\n", worst);
  return worst < 2e-14 ? 0 : 1;
}
