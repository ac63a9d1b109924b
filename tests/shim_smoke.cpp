// C++ shim smoke test (include/ce_gpu.hpp): compiled by tests/test_shim.py; run on a GPU by the -m gpu test.
#include "ce_gpu.hpp"
#include <cstdio>
int main() {
  ce_problem* p; if (ce_problem_create(1, 32, 32, 0, &p)) return 1;
  ce_csb_host h; ce_problem_csb(p, &h); ce_plan_host pl; ce_problem_plan(p, &pl);
  try {
    ce_b200::Context ctx(0);
    ce_b200::BlockSparseMatrix a(ctx, h);
    auto f = ce_b200::ce_factorize(ctx, a, pl, ce_b200::CompressionStrategy::adaptive(1e-4));
    std::vector<double> b(ce_problem_rhs(p), ce_problem_rhs(p) + h.n), x;
    auto rep = ce_b200::pcg(ctx, a, h.n, b, &f, {1e-8, 100, false}, x);
    auto rm = ce_b200::minres(ctx, a, h.n, b, &f, {1e-8, 100, false}, x);
    if (!rep.converged || !rm.converged) return 3;
    std::printf("shim ok: its=%lld resid=%.3e minres its=%lld\n", (long long)rep.iterations, rep.final_true_residual,
                (long long)rm.iterations);
  } catch (const std::exception& e) { std::printf("shim error: %s\n", e.what()); return 2; }
  ce_problem_free(p);
  return 0;
}
