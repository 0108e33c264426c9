// ref_bench.cpp — the CPU reference arm of bench.py: the reference's own
// algorithm for one IT-MPPI iteration (oracle/mppi_oracle.cpp restates
// /root/reference/proj/src/controller.cpp:55-148 in double precision with the
// reference's splitmix64 sampler and its std::thread-per-chunk parallelism,
// parallel.hpp:11-29) timed on the host cores.  TEST / BENCHMARK
// INFRASTRUCTURE: it links the oracle and the synthetic-workload generator
// (paper_1707_02342_b200/csrc/workload.cpp, host-only), never the CUDA
// library.  The reference itself cannot be built here (Eigen3 is absent,
// DESIGN.md §5), so this restatement is the reference arm ("port").
//
// Timing follows the reference's own throughput check
// (proj/tests/acceptance.cpp:381-389): std::chrono::steady_clock around each
// mpc_step, `warmup` untimed calls, then `steps` timed calls; reported per
// thread count: median, p99, min and every sample.  The closed loop advances
// the state with the same model (oracle_vehicle_step), as the GPU arm's device
// plant does.
//
//   mppi_ref_bench --samples K --horizon T --hidden H --threads 1,16 --steps S --warmup W
//                  [--dt --lambda --gamma --sigma0 --sigma1 --explore --seed --sg-window --sg-degree
//                   --cost a,b,c,... (11 values) --vx-lo --vx-hi --init-std]
// prints one JSON object on stdout.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "../include/mppi_gpu.h"

struct AnyController;
extern "C" {
int oracle_create(const mppi_gpu_config* cfg, AnyController** out);
void oracle_destroy(AnyController* h);
int oracle_set_mlp(AnyController* h, int H, const double* w1, const double* b1, const double* w2, const double* b2,
                   const double* w3, const double* b3);
int oracle_set_costmap_f32(AnyController* h, const float* values, int W, int Hh, double x0, double y0, double res);
int oracle_mpc_step(AnyController* h, const double* x0, double* u0_out, int n_threads);
int oracle_vehicle_step(AnyController* h, const double* x, const double* u, double* x_next);
const char* oracle_last_error(void);
}

namespace {

std::vector<double> parse_list(const std::string& s) {
  std::vector<double> v;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ',')) v.push_back(std::stod(tok));
  return v;
}

[[noreturn]] void die(const std::string& msg) {
  std::fprintf(stderr, "mppi_ref_bench: %s\n", msg.c_str());
  std::exit(2);
}

int host_threads() {
  const unsigned n = std::thread::hardware_concurrency();
  return n ? static_cast<int>(n) : 1;
}

}  // namespace

int main(int argc, char** argv) {
  int K = 16384, T = 100, H = 32, steps = 7, warmup = 2, sg_window = 9, sg_degree = 2;
  double dt = 0.02, lambda = 6.66, gamma = 0.666, sigma0 = 0.09, sigma1 = 0.1225, explore = 0.01;
  double vx_lo = 3.0, vx_hi = 8.0, init_std = 0.05;
  uint64_t seed = 170702342ull;
  std::vector<double> threads_list = {0};  // 0 = every host thread
  std::vector<double> cost = {200.0, 1.0, 0.0, 6.0, 0.0, 1.0, 1.0, 0.75, 10000.0, 1.0, 0.6};
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) die("missing value for " + a);
      return argv[++i];
    };
    if (a == "--samples") K = std::stoi(val());
    else if (a == "--horizon") T = std::stoi(val());
    else if (a == "--hidden") H = std::stoi(val());
    else if (a == "--steps") steps = std::stoi(val());
    else if (a == "--warmup") warmup = std::stoi(val());
    else if (a == "--threads") threads_list = parse_list(val());
    else if (a == "--dt") dt = std::stod(val());
    else if (a == "--lambda") lambda = std::stod(val());
    else if (a == "--gamma") gamma = std::stod(val());
    else if (a == "--sigma0") sigma0 = std::stod(val());
    else if (a == "--sigma1") sigma1 = std::stod(val());
    else if (a == "--explore") explore = std::stod(val());
    else if (a == "--seed") seed = std::stoull(val());
    else if (a == "--sg-window") sg_window = std::stoi(val());
    else if (a == "--sg-degree") sg_degree = std::stoi(val());
    else if (a == "--cost") cost = parse_list(val());
    else if (a == "--vx-lo") vx_lo = std::stod(val());
    else if (a == "--vx-hi") vx_hi = std::stod(val());
    else if (a == "--init-std") init_std = std::stod(val());
    else die("unknown argument " + a);
  }
  if (cost.size() != 11) die("--cost needs 11 values");
  if (steps < 1 || warmup < 0) die("--steps >= 1, --warmup >= 0");

  // the BASELINE workload (paper_1707_02342_b200/workload.py, csrc/workload.cpp)
  const size_t nh = static_cast<size_t>(H);
  std::vector<double> w1(nh * 6), b1(nh), w2(nh * nh), b2(nh), w3(4 * nh), b3(4);
  if (mppi_workload_mlp_xavier(H, seed, 0.1, w1.data(), b1.data(), w2.data(), b2.data(), w3.data(), b3.data()) != 0)
    die("mlp_xavier failed");
  const int MW = 2000, MH = 2000;
  std::vector<float> map(static_cast<size_t>(MW) * MH);
  if (mppi_workload_ellipse_costmap(MW, MH, -50.0, -50.0, 0.05, 40.0, 25.0, 3.0, map.data()) != 0)
    die("ellipse_costmap failed");
  double x0[7];
  if (mppi_workload_initial_states(1, seed, 40.0, 25.0, 1, vx_lo, vx_hi, init_std, x0) != 0)
    die("initial_states failed");

  mppi_gpu_config cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.samples = K;
  cfg.horizon_steps = T;
  cfg.dt = dt;
  cfg.sigma_diag[0] = sigma0;
  cfg.sigma_diag[1] = sigma1;
  cfg.lambda = lambda;
  cfg.gamma = gamma;
  cfg.explore_fraction = explore;
  cfg.seed = seed;
  cfg.bounds_lower[0] = cfg.bounds_lower[1] = -1.0;
  cfg.bounds_upper[0] = cfg.bounds_upper[1] = 1.0;
  cfg.sg_window = sg_window;
  cfg.sg_degree = sg_degree;
  cfg.weight_rule = MPPI_WEIGHT_IT;
  cfg.cem_delta = 0.8;
  cfg.with_terminal = 1;
  cfg.noise_mode = MPPI_NOISE_REF_SPLITMIX;  // the reference's own sampler (sampler.hpp:15-54)
  cfg.precision = MPPI_FP64;                 // the reference's arithmetic (types.hpp:12-13)
  cfg.system = MPPI_SYSTEM_VEHICLE_MLP;
  cfg.mlp_hidden = H;
  cfg.n_controllers = 1;
  cfg.quad_cost_scale = 1.0;
  double* c = &cfg.cost.alpha_track;
  for (int i = 0; i < 11; ++i) c[i] = cost[i];

  std::printf("{\"samples\": %d, \"horizon\": %d, \"hidden\": %d, \"host_threads\": %d, \"runs\": [", K, T, H,
              host_threads());
  for (size_t ti = 0; ti < threads_list.size(); ++ti) {
    const int nthr = threads_list[ti] > 0 ? static_cast<int>(threads_list[ti]) : host_threads();
    AnyController* h = nullptr;
    if (oracle_create(&cfg, &h) != 0) die(std::string("oracle_create: ") + oracle_last_error());
    if (oracle_set_mlp(h, H, w1.data(), b1.data(), w2.data(), b2.data(), w3.data(), b3.data()) != 0)
      die(std::string("set_mlp: ") + oracle_last_error());
    if (oracle_set_costmap_f32(h, map.data(), MW, MH, -50.0, -50.0, 0.05) != 0)
      die(std::string("set_costmap: ") + oracle_last_error());
    double x[7], xn[7], u[2];
    std::memcpy(x, x0, sizeof(x));
    std::vector<double> ms;
    for (int it = 0; it < warmup + steps; ++it) {
      const auto t0 = std::chrono::steady_clock::now();
      if (oracle_mpc_step(h, x, u, nthr) != 0) die(std::string("mpc_step: ") + oracle_last_error());
      const auto t1 = std::chrono::steady_clock::now();
      if (it >= warmup) ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
      oracle_vehicle_step(h, x, u, xn);
      std::memcpy(x, xn, sizeof(x));
    }
    oracle_destroy(h);
    std::vector<double> s = ms;
    std::sort(s.begin(), s.end());
    const double med = s.size() % 2 ? s[s.size() / 2] : 0.5 * (s[s.size() / 2 - 1] + s[s.size() / 2]);
    const double p99 = s[std::min(s.size() - 1, static_cast<size_t>(0.99 * (s.size() - 1) + 0.5))];
    double total = 0.0;
    for (double v : ms) total += v;
    std::printf("%s{\"threads\": %d, \"steps\": %d, \"warmup\": %d, \"median_ms\": %.6f, \"p99_ms\": %.6f, "
                "\"min_ms\": %.6f, \"total_ms\": %.3f, \"sample_steps_per_s\": %.6e, \"ms\": [",
                ti ? ", " : "", nthr, steps, warmup, med, p99, s.front(), total,
                static_cast<double>(K) * T / (med * 1e-3));
    for (size_t i = 0; i < ms.size(); ++i) std::printf("%s%.4f", i ? ", " : "", ms[i]);
    std::printf("], \"u0_last\": [%.17g, %.17g]}", u[0], u[1]);
    std::fflush(stdout);
  }
  std::printf("]}\n");
  return 0;
}
