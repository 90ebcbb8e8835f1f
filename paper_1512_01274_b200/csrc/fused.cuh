// Fused (single-launch) execution of a program range; see megakernel.cu.
#pragma once

#include <vector>

#include "common.cuh"

namespace mgx {

struct ProgramParams;

struct FusedRange {
  ProgramParams* params = nullptr;  // host copy, passed by value at launch
  uint32_t* d_barrier = nullptr;
  int nlevels = 0;
  int grid = 0;
  size_t smem = 0;
  std::vector<int> level_of;  // diagnostics
};

int build_fused(const mgx_instr* instrs, int n, FusedRange* out);
uint32_t* program_error_word();
int launch_fused(const FusedRange& f, cudaStream_t st);
int time_fused(const FusedRange& f, cudaStream_t st, double* ns_out);
void free_fused(FusedRange& f);

}  // namespace mgx
