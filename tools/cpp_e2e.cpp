// cpp_e2e.cpp — end-to-end time of the C++ drop-in (sparsim_b200.hpp
// MicroEngine::step: host gradient in, aggregated selection + sums out) at
// BASELINE C3 size, fp32, pinned host gradients.
//   g++ -std=c++20 -O2 -I include tools/cpp_e2e.cpp -L paper_2310_00967_b200/lib -lmicro_b200 \
//       -Wl,-rpath,$PWD/paper_2310_00967_b200/lib -o tools/build/cpp_e2e
#include <chrono>
#include <cstdio>
#include <random>
#include <vector>

#include "sparsim_b200.hpp"

int main(int argc, char** argv) {
  const sparsim::Index n_g = argc > 1 ? std::atoll(argv[1]) : 138000000;
  const int steps = argc > 2 ? std::atoi(argv[2]) : 10;
  sparsim::SparsifierConfig sc;
  sc.density = 0.01;
  sc.initial_threshold = 0.025758293035489;
  sparsim::MicroEngine eng(n_g, 1, sc, true, MICRO_F32);
  const int nbuf = 4;
  std::vector<float*> G(nbuf);
  std::mt19937_64 rng(1);
  std::normal_distribution<float> unit(0.0f, 1.0f);
  for (auto& g : G) {
    sparsim::b200::check(micro_host_malloc(reinterpret_cast<void**>(&g), (int64_t)n_g * 4));
    for (sparsim::Index j = 0; j < n_g; ++j) g[j] = unit(rng);
  }
  std::vector<double> summed;
  for (int t = 0; t < 3; ++t) eng.step(G[t % nbuf], 0.01, t, &summed);  // warm
  const auto t0 = std::chrono::steady_clock::now();
  std::size_t K = 0;
  for (int t = 3; t < 3 + steps; ++t) K += eng.step(G[t % nbuf], 0.01, t, &summed).indices.size();
  const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / steps;
  std::printf("{\"what\": \"C++ MicroEngine::step e2e (pinned host fp32 gradient in, indices + sums out)\", "
              "\"n_g\": %lld, \"us_per_step\": %.1f, \"mean_K\": %.0f}\n", (long long)n_g, us, (double)K / steps);
  for (auto* g : G) micro_host_free(g);
  return 0;
}
