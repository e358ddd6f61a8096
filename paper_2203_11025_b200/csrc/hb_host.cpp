// Host-side setup restatements (bit-identical to the reference where the
// reference defines them): Rng (inc/rng.hpp:9-67), absorbing layer
// (inc/grid.hpp:101-119), full-weighting restriction of real coefficient
// fields (inc/stencil.hpp:119-140) used by coefficient coarsening
// (:169-185), and the SURVEY 8(a) A1/A2/A6 generators (medium, point sources,
// He-normal weights).  These are product code: the GPU library sets problems
// up itself and never calls the test oracle.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "hb_host.h"

namespace hb {

Rng::Rng(uint64_t seed) {
  uint64_t z = seed;
  for (auto& w : s_) {
    z += 0x9e3779b97f4a7c15ull;
    uint64_t x = z;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    w = x ^ (x >> 31);
  }
}

uint64_t Rng::next_u64() {
  auto rotl = [](uint64_t x, int k) { return (x << k) | (x >> (64 - k)); };
  const uint64_t result = rotl(s_[0] + s_[3], 23) + s_[0];
  const uint64_t t = s_[1] << 17;
  s_[2] ^= s_[0];
  s_[3] ^= s_[1];
  s_[1] ^= s_[2];
  s_[0] ^= s_[3];
  s_[2] ^= t;
  s_[3] = rotl(s_[3], 45);
  return result;
}

double Rng::uniform() { return double(next_u64() >> 11) * 0x1.0p-53; }

int64_t Rng::uniform_int(int64_t lo, int64_t hi) { return lo + int64_t(next_u64() % uint64_t(hi - lo + 1)); }

double Rng::normal() {
  if (have_spare_) {
    have_spare_ = false;
    return spare_;
  }
  double u1 = 0.0;
  while (u1 <= 0.0) u1 = uniform();
  const double u2 = uniform();
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double theta = 6.283185307179586476925286766559 * u2;
  spare_ = r * std::sin(theta);
  have_spare_ = true;
  return r * std::cos(theta);
}

void restrict_real(const double* fine, int nx, int ny, int offset, double* coarse) {
  static const double k1[3] = {1.0, 2.0, 1.0};
  const int cnx = nx / 2, cny = ny / 2;
  for (int jy = 0; jy < cny; ++jy)
    for (int jx = 0; jx < cnx; ++jx) {
      double acc = 0.0;
      for (int ky = -1; ky <= 1; ++ky) {
        const int iy = 2 * jy + offset + ky;
        if (iy < 0 || iy >= ny) continue;
        for (int kx = -1; kx <= 1; ++kx) {
          const int ix = 2 * jx + offset + kx;
          if (ix < 0 || ix >= nx) continue;
          acc += fine[size_t(iy) * nx + ix] * (k1[ky + 1] * k1[kx + 1] / 16.0);
        }
      }
      coarse[size_t(jy) * cnx + jx] = acc;
    }
}

void normalize_range(std::vector<double>& f, double lo, double hi) {
  double mn = f[0], mx = f[0];
  for (double x : f) {
    mn = std::min(mn, x);
    mx = std::max(mx, x);
  }
  if (mx - mn < 1e-300) {
    for (double& x : f) x = hi;
    return;
  }
  const double scale = (hi - lo) / (mx - mn);
  for (double& x : f) x = lo + (x - mn) * scale;
}

void gaussian_blur(const double* src, int nx, int ny, double sigma, double* out) {
  const int R = int(std::ceil(3.0 * sigma));
  std::vector<double> w(size_t(2 * R + 1));
  double sum = 0.0;
  for (int i = -R; i <= R; ++i) {
    w[size_t(i + R)] = std::exp(-0.5 * i * i / (sigma * sigma));
    sum += w[size_t(i + R)];
  }
  for (double& x : w) x /= sum;
  std::vector<double> tmp(size_t(nx) * ny);
  for (int y = 0; y < ny; ++y)
    for (int x = 0; x < nx; ++x) {
      double acc = 0.0;
      for (int i = -R; i <= R; ++i) acc += w[size_t(i + R)] * src[size_t(y) * nx + std::clamp(x + i, 0, nx - 1)];
      tmp[size_t(y) * nx + x] = acc;
    }
  for (int y = 0; y < ny; ++y)
    for (int x = 0; x < nx; ++x) {
      double acc = 0.0;
      for (int i = -R; i <= R; ++i) acc += w[size_t(i + R)] * tmp[size_t(std::clamp(y + i, 0, ny - 1)) * nx + x];
      out[size_t(y) * nx + x] = acc;
    }
}

}  // namespace hb

// ---- SLW1 raw fields (inc/field_io.hpp:12-76): "SLW1", u32 nx, u32 ny (LE),
// nx*ny f32 LE row-major.  Host-only; the slowness-model exchange format of
// the reference's dataset tooling.
#include <cstring>
#include <fstream>

#include "../../include/helmgpu.h"

namespace {
void put_u32(std::ostream& os, uint32_t v) {
  const unsigned char b[4] = {uint8_t(v), uint8_t(v >> 8), uint8_t(v >> 16), uint8_t(v >> 24)};
  os.write(reinterpret_cast<const char*>(b), 4);
}
bool get_u32(std::istream& is, uint32_t& v) {
  unsigned char b[4];
  is.read(reinterpret_cast<char*>(b), 4);
  v = uint32_t(b[0]) | uint32_t(b[1]) << 8 | uint32_t(b[2]) << 16 | uint32_t(b[3]) << 24;
  return bool(is);
}
}  // namespace

extern "C" {

int hb_write_slw1(const char* path, int nx, int ny, const double* values) {
  if (!path || nx <= 0 || ny <= 0 || !values) return HB_ERR_ARG;
  std::ofstream os(path, std::ios::binary);
  if (!os) return HB_ERR_ARG;
  os.write("SLW1", 4);
  put_u32(os, uint32_t(nx));
  put_u32(os, uint32_t(ny));
  for (size_t i = 0; i < size_t(nx) * ny; ++i) {
    const float f = float(values[i]);
    uint32_t bits;
    std::memcpy(&bits, &f, 4);
    put_u32(os, bits);
  }
  return os ? HB_OK : HB_ERR_ARG;
}

// values == NULL: only report the dims
int hb_read_slw1(const char* path, int* nx, int* ny, double* values) {
  if (!path) return HB_ERR_ARG;
  std::ifstream is(path, std::ios::binary);
  if (!is) return HB_ERR_ARG;
  char magic[4];
  is.read(magic, 4);
  if (!is || std::memcmp(magic, "SLW1", 4) != 0) return HB_ERR_NUMERIC;  // "bad SLW1 magic"
  uint32_t w = 0, h = 0;
  if (!get_u32(is, w) || !get_u32(is, h)) return HB_ERR_NUMERIC;
  if (w == 0 || h == 0 || size_t(w) * h > (size_t(1) << 28) || w > (1u << 30) || h > (1u << 30))
    return HB_ERR_NUMERIC;  // "bad SLW1 dims"
  if (nx) *nx = int(w);
  if (ny) *ny = int(h);
  if (!values) return HB_OK;
  for (size_t i = 0; i < size_t(w) * h; ++i) {
    uint32_t bits;
    if (!get_u32(is, bits)) return HB_ERR_NUMERIC;  // "unexpected end of file"
    float f;
    std::memcpy(&f, &bits, 4);
    values[i] = double(f);
  }
  return HB_OK;
}

}  // extern "C"
