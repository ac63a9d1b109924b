// Device from_triplets (assemble.cu): the CSB of a scalar COO matrix built on the GPU.
#pragma once

#include <string>
#include <vector>

#include "host_api.hpp"

namespace ceg {

struct AssembleResult {
  std::string error;                               // non-empty: the reference's message
  std::vector<int64_t> row_ptr, col_idx, val_ptr;  // block structure (host, for the planner)
  DevArray<double> values;                         // row-major blocks, on the device
  int64_t unique_entries = 0;
};

// d_rows / d_cols / d_vals: nnz device triplets; d_offsets: m + 1 partition offsets (device).
AssembleResult assemble_from_triplets(int64_t n, int64_t nnz, const int64_t* d_rows, const int64_t* d_cols,
                                      const double* d_vals, int64_t m, const int64_t* d_offsets, bool mirror,
                                      cudaStream_t s);

}  // namespace ceg
