// Host normal-vector throughput (ppa/rng.hpp) on the GPU box's CPU.
// g++ -O3 -std=c++17 -pthread -I paper_1806_08020_b200/csrc rng_speed.cpp -o /tmp/rng_speed
#include <chrono>
#include <cstdio>
#include <memory>
#include "ppa/rng.hpp"

int main() {
  const long long n = 4096000;
  auto t = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  for (int rep = 0; rep < 3; ++rep) {
    std::unique_ptr<double[]> fresh(new double[n]);
    auto t0 = t();
    ppa::rng::fill_normal(fresh.get(), n, 2, 2);
    auto t1 = t();
    ppa::rng::fill_normal(fresh.get(), n, 2, 3);  // pages already touched
    auto t2 = t();
    double s = 0;
    for (long long i = 0; i < 1000000; ++i) s += ppa::rng::normal_at(ppa::rng::key(2, 2), i);
    auto t3 = t();
    std::printf("fresh %.1f ms  touched %.1f ms  1 thread 1M elems %.1f ms (%g)\n", ms(t0, t1),
                ms(t1, t2), ms(t2, t3), s);
  }
  std::printf("hw threads %u\n", std::thread::hardware_concurrency());
}
