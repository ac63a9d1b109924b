// ORACLE — TEST INFRASTRUCTURE ONLY (see dense.hpp).
// Command-line driver: times the CPU restatement on a BASELINE config (the
// cpu_baseline leg of bench.py and the `--impl reference` arm), prints one
// JSON object.  Mirrors the timed regions of proj/src/cli.cpp:102-110
// (factor_problem) and :211-228 (solve), with PCG in place of MINRES.
//
// usage: oracle_cli <cfg 1..5> [nx ny nz] [--no-solve] [--dump PATH] [--levels] [--merge-all | --colored | --sharded]
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "factor.hpp"
#include "krylov.hpp"

using namespace oracle;

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: oracle_cli <cfg 1..5> [nx ny nz] [--no-solve] [--dump PATH] [--levels] [--merge-all | --colored | --sharded]\n");
    return 1;
  }
  try {
    ProblemConfig c = baseline_config(std::atoi(argv[1]));
    bool solve = true, levels = false;
    std::string dump;
    int pos = 0;
    for (int a = 2; a < argc; ++a) {
      if (!std::strcmp(argv[a], "--no-solve")) solve = false;
      else if (!std::strcmp(argv[a], "--levels")) levels = true;
      else if (!std::strcmp(argv[a], "--merge-all")) c.plan_kind = 1;
      else if (!std::strcmp(argv[a], "--colored")) c.plan_kind = 2;
      else if (!std::strcmp(argv[a], "--sharded")) c.plan_kind = 3;
      else if (!std::strcmp(argv[a], "--dump") && a + 1 < argc) dump = argv[++a];
      else {
        const long long v = std::atoll(argv[a]);
        if (pos == 0) c.nx = v;
        else if (pos == 1) c.ny = v;
        else if (pos == 2 && c.dims == 3) c.nz = v;
        ++pos;
      }
    }
    const auto tg = std::chrono::steady_clock::now();
    LoadedProblem lp = load_config(c);
    const double gen_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - tg).count();
    const index_t n = lp.matrix.dim();
    const auto t0 = std::chrono::steady_clock::now();
    CEFactorization f = ce_factorize(lp.matrix, lp.plan, CompressionStrategy::adaptive(c.eps));
    const double fac_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (!dump.empty()) write_factor_dump(f, dump);
    std::printf("{\"cfg\": %d, \"n\": %lld, \"nx\": %lld, \"ny\": %lld, \"nz\": %lld, \"block\": %lld, \"eps\": %g, "
                "\"gen_seconds\": %.6f, \"factor_seconds\": %.6f, \"unknowns_per_sec\": %.6g, \"levels\": %zu, "
                "\"tail_dim\": %lld, \"l_bytes\": %lld, \"q_bytes\": %lld",
                c.id, static_cast<long long>(n), static_cast<long long>(c.nx), static_cast<long long>(c.ny),
                static_cast<long long>(c.nz), static_cast<long long>(c.block), c.eps, gen_s, fac_s,
                static_cast<double>(n) / fac_s, f.levels.size(), static_cast<long long>(f.tail_dim),
                static_cast<long long>(f.stats.l_payload_bytes), static_cast<long long>(f.stats.q_payload_bytes));
    if (solve) {
      ApplyFn a = [&](const Vec& v) { return lp.matrix.matvec(v); };
      ApplyFn m = [&](const Vec& v) { return f.solve(v); };
      PcgOptions o;
      o.tol = c.tol;
      o.maxit = 1000;
      Vec x;
      const auto t1 = std::chrono::steady_clock::now();
      SolveReport rep = pcg(a, n, lp.rhs, m, o, x);
      const double pcg_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
      std::printf(", \"pcg_seconds\": %.6f, \"pcg_iterations\": %lld, \"pcg_true_resid\": %.3e, \"converged\": %d",
                  pcg_s, static_cast<long long>(rep.iterations), rep.final_true_residual, rep.converged ? 1 : 0);
    }
    if (levels) {
      std::printf(", \"level_info\": [");
      for (size_t l = 0; l < f.levels.size(); ++l) {
        const FactorLevel& fl = f.levels[l];
        const auto& ls = f.stats.levels[l];
        index_t maxb = 0, maxf = 0, maxw = 0, maxc = 0, rank_flips_near = 0;
        double min_gap = 1.0;
        for (index_t b = 0; b < fl.partition.block_count(); ++b) {
          maxb = std::max(maxb, fl.partition.block_size(b));
          maxf = std::max(maxf, fl.fcols[static_cast<size_t>(b)]);
          maxw = std::max(maxw, fl.rows[static_cast<size_t>(b)].width);
          maxc = std::max(maxc, static_cast<index_t>(fl.rows[static_cast<size_t>(b)].neighbors.size()));
          const auto& s = fl.sigma[static_cast<size_t>(b)];
          const index_t r = fl.retained[static_cast<size_t>(b)];
          for (index_t k = 0; k + 1 < r && k + 1 < static_cast<index_t>(s.size()); ++k)
            min_gap = std::min(min_gap, (s[static_cast<size_t>(k)] - s[static_cast<size_t>(k + 1)]) /
                                            std::max(s[static_cast<size_t>(k)], 1e-300));
          if (!s.empty() && r < static_cast<index_t>(s.size())) {
            const double thr = c.eps * s[0];
            if (std::abs(s[static_cast<size_t>(r)] - thr) <= 1e-9 * thr) ++rank_flips_near;
          }
        }
        std::printf("%s{\"level\": %zu, \"M\": %lld, \"dim\": %lld, \"max_b\": %lld, \"max_fcols\": %lld, "
                    "\"max_w\": %lld, \"max_close\": %lld, \"max_rank\": %lld, \"mean_rank\": %.3f, "
                    "\"eliminated\": %lld, \"seconds\": %.4f, \"min_rel_gap_in_U1\": %.3e, \"near_thr\": %lld, "
                    "\"shift_retries\": %lld}",
                    l ? ", " : "", l + 1, static_cast<long long>(fl.partition.block_count()),
                    static_cast<long long>(fl.dim()), static_cast<long long>(maxb), static_cast<long long>(maxf),
                    static_cast<long long>(maxw), static_cast<long long>(maxc), static_cast<long long>(ls.max_rank),
                    ls.mean_rank, static_cast<long long>(ls.eliminated), ls.seconds, min_gap,
                    static_cast<long long>(rank_flips_near), static_cast<long long>(ls.shift_retries));
      }
      std::printf("]");
    }
    std::printf("}\n");
    return 0;
  } catch (const BreakdownError& e) {
    std::fprintf(stderr, "breakdown: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
