// Reference-style caller of the B200 library through include/fsagp_b200.hpp:
// the shape of the reference fit objective (estimation.cpp:255-284).
#include <array>
#include <cstdio>
#include <vector>

#include "fsagp_b200.hpp"

int main() {
  using namespace fsagp_b200;
  const std::int64_t n = 4000, m = 64;
  std::vector<double> coords(n * 2), ind(m * 2), y(n);
  check(fsa_uniform_locations(n, 2, 1, coords.data()));
  check(fsa_select_random(coords.data(), n, 2, m, 2, ind.data()));
  check(fsa_simulate_rff(coords.data(), n, 2, 1, 1.0, 0.1, 0.1, 256, 3, y.data()));
  Context ctx(0);
  CovParams p;
  p.sigma2 = 0.1;
  p.sigma1_2 = 1.0;
  p.rho = 0.1;
  auto model = FsaModel::assemble(ctx, coords, n, 2, ind, m, MaternNu::nu_3_2, TaperFamily::wendland1,
                                  fsa_gamma_for_avg_row_nnz(n, 30.0), p);
  auto P = make_preconditioner(*model, PrecondType::fitc);
  IterativeNllOptions o;
  o.num_probes = 20;
  IterativeNll r = iterative_nll_grad(*model, *P, y, {}, 0, o);
  std::printf("nll %.12g grad %.6g %.6g %.6g cg_iterations %d\n", r.nll, r.grad[0], r.grad[1], r.grad[2],
              r.cg_iterations);
  // fisher_ste (fsa.cpp:284-301): symmetric, positive diagonal
  FisherOptions fo;
  fo.num_probes = 8;
  const std::array<double, 9> F = fisher_ste(*model, fo);
  std::printf("fisher %.6g %.6g %.6g\n", F[0], F[4], F[8]);
  if (F[1] != F[3] || F[2] != F[6] || F[5] != F[7] || !(F[0] > 0 && F[4] > 0 && F[8] > 0)) return 2;
  try {
    p.sigma2 = -1.0;
    FsaModel::assemble(ctx, coords, n, 2, ind, m, MaternNu::nu_3_2, TaperFamily::wendland1, 0.05, p);
    return 1;
  } catch (const std::invalid_argument&) {
  }
  return 0;
}
