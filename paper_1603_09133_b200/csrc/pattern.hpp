// Symbolic pattern algebra on the device (pattern.cu).
#pragma once

#include <vector>

#include "host_api.hpp"

namespace ceg {

// Sum over the rows of deg(k) for k in the row: the candidate count of pattern_square.
int64_t square_candidates(int64_t m, const std::vector<int64_t>& ptr, const std::vector<int>& col);
// pattern_square (proj/src/pattern.cpp:64-86): CSR (sorted rows) -> CSR of P^2 (sorted rows).
void device_square(int64_t m, const std::vector<int64_t>& ptr, const std::vector<int>& col, cudaStream_t s,
                   std::vector<int64_t>& sptr, std::vector<int>& scol);
// coarsen_pattern (pattern.cpp:97-118): rows / columns merged by group_of (m entries, ng groups;
// -1 = a dead group, its entries dropped).
void device_coarsen(int64_t m, const std::vector<int64_t>& ptr, const std::vector<int>& col, int64_t ng,
                    const std::vector<int64_t>& group_of, cudaStream_t s, std::vector<int64_t>& cptr,
                    std::vector<int>& ccol);

}  // namespace ceg
