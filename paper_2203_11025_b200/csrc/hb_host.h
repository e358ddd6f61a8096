#pragma once
#include <cstdint>
#include <vector>

namespace hb {

// splitmix64-seeded xoshiro256++ (inc/rng.hpp:9-67), bit-identical
class Rng {
 public:
  explicit Rng(uint64_t seed);
  uint64_t next_u64();
  double uniform();
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  int64_t uniform_int(int64_t lo, int64_t hi);
  double normal();

 private:
  uint64_t s_[4];
  double spare_ = 0.0;
  bool have_spare_ = false;
};

void restrict_real(const double* fine, int nx, int ny, int offset, double* coarse);
void normalize_range(std::vector<double>& f, double lo, double hi);
void gaussian_blur(const double* src, int nx, int ny, double sigma, double* out);

}  // namespace hb
