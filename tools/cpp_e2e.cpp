// cpp_e2e.cpp — end-to-end time of the C++ drop-in (sparsim_b200.hpp
// MicroEngine::step: host gradient in, aggregated selection + sums out) at
// BASELINE C3 size: fp32 (mode f32) or the bench's default, fp64 state on fp32
// gradients (mode f64g32, MICRO_GRAD_F32).  Every step gets a fresh N(0,1)
// fp32 gradient (made on the device by micro_synth_gaussian and copied into
// pinned host memory outside the timed call); the threshold adapts for
// `prime` steps first.  args: n_g steps prime mode alpha
//   g++ -std=c++20 -O2 -I include tools/cpp_e2e.cpp -L paper_2310_00967_b200/lib -lmicro_b200 \
//       -Wl,-rpath,'$ORIGIN/../../paper_2310_00967_b200/lib' -o tools/build/cpp_e2e
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "sparsim_b200.hpp"

int main(int argc, char** argv) {
  const sparsim::Index n_g = argc > 1 ? std::atoll(argv[1]) : 138000000;
  const int steps = argc > 2 ? std::atoi(argv[2]) : 10;
  const int prime = argc > 3 ? std::atoi(argv[3]) : 300;
  const bool f64 = argc > 4 && std::string(argv[4]) == "f64g32";
  sparsim::SparsifierConfig sc;
  sc.density = 0.01;
  sc.initial_threshold = 0.025758293035489;
  if (argc > 5) sc.scaling_factor = std::atof(argv[5]);
  sparsim::MicroEngine eng(n_g, 1, sc, true, f64 ? MICRO_F64 : MICRO_F32, f64 ? MICRO_GRAD_F32 : MICRO_GRAD_SAME);
  float* h = nullptr;
  void* d = nullptr;
  sparsim::b200::check(micro_host_malloc(reinterpret_cast<void**>(&h), (int64_t)n_g * 4));
  sparsim::b200::check(micro_device_malloc(&d, (int64_t)n_g * 4, 0));
  std::vector<double> summed;
  double total_us = 0.0, K = 0.0;
  for (int t = 0; t < prime + steps; ++t) {
    sparsim::b200::check(micro_synth_gaussian(MICRO_F32, 1, 0, (uint64_t)t, n_g, d, nullptr));
    sparsim::b200::d2h(h, d, (std::size_t)n_g * 4);  // a fresh host gradient (untimed)
    const auto t0 = std::chrono::steady_clock::now();
    const auto agg = eng.step(h, 0.01, t, &summed);
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    if (t >= prime) {
      total_us += us;
      K += (double)agg.indices.size();
    }
  }
  std::printf("{\"what\": \"C++ MicroEngine::step e2e (pinned host fp32 gradient in, indices + sums out)\", "
              "\"state\": \"%s\", \"alpha\": %g, \"n_g\": %lld, \"prime\": %d, \"steps\": %d, "
              "\"us_per_step\": %.1f, \"density\": %.5f}\n",
              f64 ? "f64" : "f32", sc.scaling_factor, (long long)n_g, prime, steps, total_us / steps,
              K / steps / (double)n_g);
  micro_host_free(h);
  micro_device_free(d);
  return 0;
}
