// Shared host-side helpers of libp2g: status/error plumbing and the pinned
// PRNG (restated from common.hpp:65-121 — bit-exact because std::mt19937_64
// is standardised; the generator and the initial factors depend on it).
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>

#include "../../include/p2g.h"

namespace p2g {

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

/// Runs `fn`, mapping exceptions onto the C-ABI status codes.
template <typename Fn>
int guarded(Fn&& fn) {
  try {
    set_last_error("");
    fn();
    return P2G_OK;
  } catch (const NumericalError& e) {
    set_last_error(e.what());
    return P2G_ENUM;
  } catch (const DataError& e) {
    set_last_error(e.what());
    return P2G_EDATA;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return P2G_ECUDA;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return P2G_EINVAL;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return P2G_ECUDA;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return P2G_EDATA;  // any other std::exception -> exit code 2 (tools/parafac2.cpp:396-408)
  }
}

inline std::uint64_t splitmix64(std::uint64_t& state) {
  std::uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

inline std::uint64_t substream_seed(std::uint64_t seed, std::uint64_t idx) {
  std::uint64_t state = seed + idx * 0x9E3779B97F4A7C15ULL;
  return splitmix64(state);
}

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : gen_(seed) {}
  double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  /// Box-Muller pair on the pinned uniform stream (common.hpp:92-104).
  double normal() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    const double u1 = 1.0 - uniform(), u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1)), a = 2.0 * M_PI * u2;
    spare_ = r * std::sin(a);
    have_spare_ = true;
    return r * std::cos(a);
  }
  std::uint64_t below(std::uint64_t n) {
    const std::uint64_t mx = std::numeric_limits<std::uint64_t>::max();
    const std::uint64_t limit = mx - mx % n;
    std::uint64_t x;
    do {
      x = gen_();
    } while (x >= limit);
    return x % n;
  }

 private:
  std::mt19937_64 gen_;
  double spare_ = 0.0;
  bool have_spare_ = false;
};

}  // namespace p2g
