// host-side accuracy check of nlg::fast_pow_pos and nlg::pow_tab against libm pow
#include <cmath>
#include <cstdio>
#include <random>
#include "../../paper_2207_03921_b200/csrc/nlg_math.cuh"
int main() {
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> ul(-75.0, 12.0), ue(-2.0, -0.999);
  nlg::PowTab tab;
  nlg::pow_tab_fill(&tab);
  double worst = 0, worst_tab = 0;
  for (int i = 0; i < 4000000; ++i) {
    const double x = std::exp(ul(g));
    const double e = (i % 4 == 0) ? -1.4 : ue(g);
    const double b = std::pow(x, e);
    const double a = nlg::fast_pow_pos(x, e);
    const double c = nlg::pow_tab(x, e, tab.rc, tab.lc, tab.e2);
    worst = std::fmax(worst, std::fabs(a - b) / b);
    worst_tab = std::fmax(worst_tab, std::fabs(c - b) / b);
  }
  printf("%.3e %.3e\n", worst, worst_tab);
  return (worst < 2e-14 && worst_tab < 2e-14) ? 0 : 1;
}
