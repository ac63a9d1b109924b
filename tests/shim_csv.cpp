// CSV half of the C++ shim (include/ce_gpu.hpp): CsvTable, fmt_double, describe and the report
// tables that need no factor.  Compiled and run by tests/test_csv.py (no GPU needed).
// argv[1]: a csv file to round-trip (parse -> to_string printed to stdout).
#include "ce_gpu.hpp"
#include <cstdio>
#include <cstring>
int main(int argc, char** argv) {
  using namespace ce_b200;
  if (argc > 2 && !std::strcmp(argv[1], "roundtrip")) {
    const CsvTable t = CsvTable::load(argv[2]);
    t.write(std::string(argv[2]) + ".out");
    std::printf("%zu %zu\n", t.header.size(), t.rows.size());
    return 0;
  }
  std::printf("%s|%s|%s|%s\n", fmt_double(0.1).c_str(), fmt_double(100000.0).c_str(), fmt_double(1e22).c_str(),
              fmt_index(-42).c_str());
  std::printf("%s|%s|%s\n", CompressionStrategy::adaptive(1e-6).describe().c_str(),
              CompressionStrategy::adaptive(1e-4, true).describe().c_str(),
              CompressionStrategy::fixed_rank(8).describe().c_str());
  SolveReport rep;
  rep.converged = true;
  rep.iterations = 2;
  rep.final_recurrence_residual = 1.5e-12;
  rep.final_true_residual = 2.5e-12;
  rep.trace.samples = {{0, 1.0, -1.0, 0.001}, {1, 1e-6, -1.0, 0.002}, {2, 1.5e-12, 2.5e-12, 0.003}};
  std::fputs(trace_table(rep.trace).to_string().c_str(), stdout);
  const CompressionStrategy s = CompressionStrategy::adaptive(1e-4);
  std::fputs(solve_report_table(4096, "minres", &s, true, rep, 0.25, 0.5).to_string().c_str(), stdout);
  std::fputs(solve_report_table(4096, "minres", nullptr, false, rep, 0.0, 0.5).to_string().c_str(), stdout);
  try {
    CsvTable::parse("");
    return 1;
  } catch (const std::invalid_argument& e) {
    std::printf("%s\n", e.what());
  }
  return 0;
}
