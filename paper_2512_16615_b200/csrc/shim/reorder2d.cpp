// reorder2d (P/include/llsa/reorder2d.hpp) on top of the C ABI: the curve via
// llsa_build_reorder (host), the gather via llsa_apply_permutation (GPU).
#include <cuda_runtime.h>

#include <string>

#include "llsa/errors.hpp"
#include "llsa/reorder2d.hpp"
#include "llsa_cuda.h"

namespace llsa {

void throw_status(int st);  // llsa_api.cpp

namespace {
void ck(llsa_status s) {
  if (s != LLSA_OK) throw_status(s);
}
void ckc(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}
template <typename T>
struct Dev {
  T* p = nullptr;
  explicit Dev(std::size_t n) { ckc(cudaMalloc(&p, n * sizeof(T) + 16), "cudaMalloc"); }
  ~Dev() { cudaFree(p); }
};
}  // namespace

Permutation build_reorder(std::uint32_t height, std::uint32_t width,
                          std::uint32_t block_size) {
  Permutation p;
  const std::size_t size = std::size_t(height) * width;
  p.forward.resize(size);
  p.inverse.resize(size);
  ck(llsa_build_reorder(height, width, block_size, p.forward.data(), p.inverse.data()));
  p.size = static_cast<std::uint32_t>(size);
  return p;
}

FeatureMatrix apply_permutation(const FeatureMatrix& x, const Permutation& p,
                                PermDirection direction) {
  if (x.rows() != p.size)
    throw ShapeMismatch("matrix has " + std::to_string(x.rows()) +
                        " rows, permutation covers " + std::to_string(p.size));
  FeatureMatrix out(x.rows(), x.cols());
  if (x.rows() == 0 || x.cols() == 0) return out;
  const std::vector<std::uint32_t>& map =
      direction == PermDirection::Forward ? p.forward : p.inverse;
  static_assert(sizeof(real) == 4, "the B200 drop-in is the f32 build");
  const std::size_t bytes = x.rows() * x.cols() * sizeof(real);
  Dev<char> dx(bytes), dout(bytes);
  Dev<std::uint32_t> dm(map.size());
  ckc(cudaMemcpy(dx.p, x.data(), bytes, cudaMemcpyHostToDevice), "H2D");
  ckc(cudaMemcpy(dm.p, map.data(), map.size() * 4, cudaMemcpyHostToDevice), "H2D");
  ck(llsa_apply_permutation(dx.p, LLSA_F32, 1, x.rows(), static_cast<std::uint32_t>(x.cols()),
                            dm.p, dout.p, nullptr));
  ck(llsa_sync_status(nullptr));
  ckc(cudaMemcpy(out.data(), dout.p, bytes, cudaMemcpyDeviceToHost), "D2H");
  return out;
}

}  // namespace llsa
