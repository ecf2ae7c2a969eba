// tcgen05 3xTF32 GEMM engine (placeholder until the tensor-core path lands): accepts nothing,
// so every GEMM runs on the SIMT engine.
#pragma once
#include "gemm_simt.cuh"

namespace hmc {
struct TcPlanner {
  bool accepts(const GemmArgs&, bool, bool) const { return false; }
  void launch(const GemmArgs&, bool, bool, cudaStream_t) const {}
  int n_tiles(const GemmArgs&, bool, bool) const { return -1; }
  const char* describe() const { return "simt"; }
};
}  // namespace hmc
