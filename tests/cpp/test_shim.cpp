// Exercises include/lbbsp_b200.hpp (the reference-signature C++ shim) with
// the reference's own known answers (test_batch_sizer.cpp:21-27, 84-122,
// test_predictor.cpp:48-62, test_coordination.cpp:25-37). Exit code 0 = pass.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "lbbsp_b200.hpp"

using namespace lbbsp::b200;

static int failures = 0;
#define CHECK(x)                                                     \
  do {                                                               \
    if (!(x)) {                                                      \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #x);       \
      ++failures;                                                    \
    }                                                                \
  } while (0)

template <typename E, typename F>
static bool throws_with(F&& f, const char* needle) {
  try {
    f();
  } catch (const E& e) {
    return std::string(e.what()).find(needle) != std::string::npos;
  } catch (...) {
    return false;
  }
  return false;
}

int main() {
  const std::vector<double> v1 = {4, 2, 1, 1};
  CHECK((cpu_allocate(v1, 512).sizes == std::vector<int>{256, 128, 64, 64}));
  const std::vector<double> v2 = {1, 1, 1, 1};
  CHECK((cpu_allocate(v2, 512).sizes == std::vector<int>{128, 128, 128, 128}));
  const std::vector<double> zero = {1.0, 0.0};
  CHECK(throws_with<std::invalid_argument>([&] { cpu_allocate(zero, 10); }, "speeds must be > 0"));
  const std::vector<double> ok = {1.0, 1.0, 1.0};
  CHECK(throws_with<std::invalid_argument>([&] { cpu_allocate(ok, 2); }, "below worker count"));

  const std::vector<GpuProfile> wide = {{0.01, 0.1, 1, 1 << 20}, {0.005, 0.1, 1, 1 << 20}};
  const std::vector<double> c0 = {0.0, 0.0};
  const auto a = gpu_allocate(wide, c0, 759);
  CHECK(a.sizes[0] + a.sizes[1] == 759);
  CHECK(std::abs(a.sizes[0] - 253) <= 1 && std::abs(a.sizes[1] - 506) <= 1);
  const std::vector<GpuProfile> tw = {{0.002, 0.05, 58, 384}, {0.0008, 0.08, 92, 1184}};
  CHECK(throws_with<std::invalid_argument>([&] { gpu_allocate(tw, c0, 100); },
                                           "below total saturation minimum"));
  CHECK(throws_with<std::invalid_argument>([&] { gpu_allocate(tw, c0, 2000); },
                                           "above total memory capacity"));

  const std::vector<double> s = {10.0, 20.0};
  CHECK(std::fabs(ema(s, 0.2) - 12.0) < 1e-12);

  NarxModel m{};
  m.output_weight = 1.0;
  m.output_bias = 6.5;
  m.speed_stddev = m.cpu_stddev = m.mem_stddev = 1.0;
  CHECK(std::fabs(narx_predict(m, {1, 2}, {1, 1, 1}, {1, 1, 1}) - 6.5) < 1e-12);

  const std::vector<double> g = {4.0, 8.0};
  const std::vector<int> b = {1, 3};
  CHECK(std::fabs(aggregate(g, b, 1, true)[0] - (1.0 * 4.0 + 3.0 * 8.0) / 4.0) < 1e-12);

  std::printf("%s (%d failures)\n", failures ? "FAIL" : "PASS", failures);
  return failures ? 1 : 0;
}
