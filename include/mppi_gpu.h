/*
 * mppi_gpu.h — C ABI of the B200-native IT-MPPI controller.
 *
 * This is the drop-in boundary for the reference hot path (one IT-MPPI
 * iteration, `mppi::mpc_step`, /root/reference/proj/src/controller.cpp:133-148).
 * The reference's plugin boundary is a per-sample, per-step std::function
 * triple (`RolloutSystem`, proj/include/mppi/controller.hpp:18-24) plus free
 * functions over a value-type `ControllerState` (controller.hpp:40-90).  A
 * per-step callback cannot cross to the device, so the boundary moves up to
 * batch granularity: the model and cost are described by DATA (MLP weights,
 * costmap, cost parameters) and the controller free functions become calls on
 * an opaque handle.  Every entry point below names the reference function it
 * replaces.
 *
 * Conventions
 *   - Plain C: POD structs, raw pointers + sizes, int status codes.  No
 *     exceptions cross the ABI; the C++ wrapper (mppi_gpu.hpp) rethrows the
 *     reference's exception types.
 *   - Host pointers are borrowed for the duration of the call only; the library
 *     owns all device memory.
 *   - One handle = one control loop (or one fleet of independent loops) = one
 *     CUDA stream.  Calls on one handle are not concurrent; distinct handles may
 *     run concurrently.
 *   - Layouts (all doubles unless the name says f32):
 *       plan U          T x 2, row-major            U[t*2 + c]
 *       perturbations   K blocks of T x 2, column-major per sample (the layout
 *                       of the reference's Eigen `Mat` in PerturbationBatch):
 *                       eps[k*T*2 + c*T + t]
 *       state           7 doubles (p_x, p_y, theta, roll, v_x, v_y, theta_dot),
 *                       types.hpp:44-48; the quadratic test system uses 2.
 *       MLP weights     row-major W1 (H x 6), b1 (H), W2 (H x H), b2 (H),
 *                       W3 (4 x H), b3 (4) — the order of save_mlp,
 *                       dynamics.cpp:297-307.
 *       costmap         row-major values[iy*width + ix], costs.hpp:11-38.
 *   - Fleet handles (n_controllers > 1) take per-controller arrays with a
 *     leading controller dimension (x0: n x state_dim, u0: n x 2).
 */
#ifndef MPPI_GPU_H_
#define MPPI_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPPI_GPU_ABI_VERSION 2

/* Status codes.  The C++ wrapper maps them to the reference's exceptions:
 * INVALID_ARGUMENT and NONFINITE -> std::invalid_argument (types.hpp:105-122,
 * weights.cpp:10-12), RUNTIME -> std::runtime_error (dynamics.cpp:216-225, IO). */
enum {
  MPPI_OK = 0,
  MPPI_ERR_INVALID_ARGUMENT = 1,
  MPPI_ERR_NONFINITE = 2,      /* it_weights "non-finite cost", weights.cpp:12 */
  MPPI_ERR_RUNTIME = 3,
  MPPI_ERR_CUDA = 4,
  MPPI_ERR_NCCL = 5,
  MPPI_ERR_UNSUPPORTED = 6,
  MPPI_ERR_DOMAIN = 7          /* std::domain_error: brush_tire_force outside the friction circle, dynamics.cpp:25-27 */
};

/* Perturbation source.  INJECTED reads a caller-provided batch in the
 * reference layout (parity); REF_SPLITMIX regenerates the reference's own
 * splitmix64 + Box-Muller stream (sampler.hpp:15-54) on the device; PHILOX is
 * Philox4x32-10 generated in registers (production). */
enum { MPPI_NOISE_INJECTED = 0, MPPI_NOISE_REF_SPLITMIX = 1, MPPI_NOISE_PHILOX = 2 };

/* Arithmetic type of the device path. */
enum { MPPI_FP32 = 0, MPPI_FP64 = 1 };

/* Device-side rollout system (the data-described replacement of
 * RolloutSystem).  VEHICLE_MLP = make_vehicle_system over MlpModel
 * (controller.cpp:7-35, dynamics.cpp:197-210); QUADRATIC = the reference test
 * fixture quadratic_system (test_controller.cpp:23-37): x' = x + v dt,
 * running cost quad_cost_scale * |x|^2, terminal 0, no clamping.
 * VEHICLE_BASIS = make_vehicle_system over BasisFunctionModel
 * (dynamics.hpp:151-162): the 25 basis functions of eval_basis
 * (dynamics.cpp:83-133) times the 25 x 4 Theta (step_basis_model,
 * dynamics.cpp:152-157), with the same costs as VEHICLE_MLP. */
enum {
  MPPI_SYSTEM_VEHICLE_MLP = 0,
  MPPI_SYSTEM_QUADRATIC = 1,
  MPPI_SYSTEM_VEHICLE_BASIS = 2,
  /* make_vehicle_system over BicycleTruthModel (dynamics.hpp:176-183): the
   * kinematic-dynamic bicycle with brush tires (step_bicycle_truth,
   * dynamics.cpp:51-81) as the controller's own model. */
  MPPI_SYSTEM_VEHICLE_BICYCLE = 3
};

/* BicycleParams (dynamics.hpp:42-62); mppi_bicycle_params_init fills the
 * reference defaults. */
typedef struct mppi_bicycle_params {
  double mass;
  double yaw_inertia;
  double a;
  double b;
  double stiffness;
  double mu;
  double load;
  double steer_scale;
  double force_scale;
} mppi_bicycle_params;

/* Weight rule (controller.hpp:32): information-theoretic softmin or CEM
 * elite averaging (weights.cpp:8-53), both on the device. */
enum { MPPI_WEIGHT_IT = 0, MPPI_WEIGHT_CEM = 1 };

/* Driving cost, CostParams (costs.hpp:46-64) plus the BASELINE crash form:
 *   c = alpha_track * (h + [h > boundary_threshold] * decay^t * impulse)
 *     + alpha_speed * (v_x - v_des)^2
 *     + alpha_stab  * (zeta^2 + [|zeta| > slip_limit] * impulse)
 *     + crash_penalty * [h > crash_threshold  or  |roll| > roll_limit]
 * With crash_penalty = 0 this is exactly state_cost (costs.cpp:29-43). */
typedef struct mppi_cost_params {
  double alpha_track;
  double alpha_speed;
  double alpha_stab;
  double v_des;
  double impulse;
  double decay;
  double boundary_threshold;
  double slip_limit;
  double crash_penalty;
  double crash_threshold;
  double roll_limit;
} mppi_cost_params;

typedef struct mppi_gpu_config {
  /* SamplingParams (types.hpp:92-123); sigma_diag holds VARIANCES. */
  int32_t samples;          /* K */
  int32_t horizon_steps;    /* T */
  double dt;
  double sigma_diag[2];
  double lambda;
  double gamma;
  double explore_fraction;
  uint64_t seed;
  /* ControlBounds (dynamics.hpp:12-29) */
  double bounds_lower[2];
  double bounds_upper[2];
  /* SGFilter (smoothing.hpp:9-13); sg_window == 0 means no filter. */
  int32_t sg_window;
  int32_t sg_degree;
  /* WeightRuleConfig (controller.hpp:34-37) */
  int32_t weight_rule;
  double cem_delta;
  /* make_vehicle_system(..., with_terminal) (controller.hpp:28-30) */
  int32_t with_terminal;
  int32_t noise_mode;       /* MPPI_NOISE_* */
  int32_t precision;        /* MPPI_FP32 / MPPI_FP64 */
  int32_t system;           /* MPPI_SYSTEM_* */
  int32_t mlp_hidden;       /* H: 32 (reference) or 64 */
  int32_t n_controllers;    /* independent controllers in this handle (>= 1) */
  int32_t device;           /* CUDA device ordinal */
  double quad_cost_scale;   /* QUADRATIC only */
  mppi_cost_params cost;
  /* Global index of controller 0 of this handle (a fleet split over ranks):
   * controller i draws noise from seed + controller_offset + i and its fleet
   * map perturbation from stream controller_offset + i, so the fleet is the
   * same workload at every rank count. */
  int32_t controller_offset;
} mppi_gpu_config;

typedef struct mppi_gpu_handle mppi_gpu_handle;

/* ---- library ------------------------------------------------------------- */
int mppi_gpu_abi_version(void);
/* sizeof(mppi_gpu_config), for binding-layout checks (ctypes / JNI / cgo). */
size_t mppi_gpu_config_sizeof(void);
/* Thread-local message for the last non-OK status returned on this thread. */
const char* mppi_gpu_last_error(void);
/* Fills the reference defaults: SamplingParams{} (types.hpp:92-101),
 * ControlBounds{} (dynamics.hpp:16), SGFilter{9,3} (smoothing.hpp:10-11),
 * CostParams{} (costs.hpp:46-54), H = 32, IT rule, fp32, Philox. */
void mppi_gpu_config_init(mppi_gpu_config* cfg);
/* Number of CUDA devices visible (0 on a CPU-only host; never fails). */
int mppi_gpu_device_count(void);

/* ---- handle lifetime: make_controller_state (controller.cpp:37-53) ------- */
int mppi_gpu_create(const mppi_gpu_config* cfg, mppi_gpu_handle** out);
int mppi_gpu_destroy(mppi_gpu_handle* h);

/* ---- model and cost data: make_vehicle_system (controller.cpp:7-35) ------ */
/* MlpModel weights (dynamics.hpp:110-119); copied, the caller may free. */
int mppi_gpu_set_dynamics_mlp(mppi_gpu_handle* h, int hidden, const double* w1,
                              const double* b1, const double* w2, const double* b2,
                              const double* w3, const double* b3);
/* BasisFunctionModel Theta (dynamics.hpp:75-82): theta[b*4 + o] = coeffs(b, o),
 * b < 25 basis functions, o < 4 outputs (roll_dot, vx_dot, vy_dot,
 * theta_ddot) — the row order of save_theta / load_theta (dynamics.cpp:230-254). */
int mppi_gpu_set_dynamics_basis(mppi_gpu_handle* h, const double* theta);
/* CostMap (costs.hpp:11-38); validated like CostMap::validate.  controller < 0
 * sets the map shared by every controller of the handle. */
int mppi_gpu_set_costmap(mppi_gpu_handle* h, int controller, const double* values,
                         int width, int height, double x0, double y0, double resolution);
int mppi_gpu_set_costmap_f32(mppi_gpu_handle* h, int controller, const float* values,
                             int width, int height, double x0, double y0,
                             double resolution);
/* BicycleTruthModel parameters of a MPPI_SYSTEM_VEHICLE_BICYCLE handle
 * (BicycleParams::validate: every entry finite and > 0).  The rollout clamps
 * the throttle to the control bounds, so the reference's friction-circle
 * domain_error is checked once here: force_scale * max |throttle bound| must
 * not exceed mu * load (MPPI_ERR_DOMAIN otherwise). */
int mppi_gpu_set_dynamics_bicycle(mppi_gpu_handle* h, const mppi_bicycle_params* p);
/* Fleet maps (BASELINE config 3): controller c gets
 * clamp(shared + sigma * N(0,1)[seed, c, cell], -2.5, 2.5), generated on the
 * device from a counter stream. */
int mppi_gpu_perturb_fleet_costmaps(mppi_gpu_handle* h, double sigma, uint64_t seed);
/* Read back controller c's device costmap (width x height values as stored on
 * the device: fp32 in the fp32 build, rounded to float here; the fleet's
 * perturbed maps for parity checks). */
int mppi_gpu_get_costmap_f32(mppi_gpu_handle* h, int controller, float* values_out);

/* ---- ControllerState get/set (controller.hpp:40-58); also checkpoint/resume */
int mppi_gpu_set_plan(mppi_gpu_handle* h, int controller, const double* U);
int mppi_gpu_get_plan(mppi_gpu_handle* h, int controller, double* U);
int mppi_gpu_set_iteration(mppi_gpu_handle* h, int controller, uint64_t iteration);
int mppi_gpu_get_iteration(mppi_gpu_handle* h, int controller, uint64_t* iteration);
int mppi_gpu_set_seed(mppi_gpu_handle* h, int controller, uint64_t seed);
/* INJECTED mode: the batch used by the next rollout (controller 0, reference
 * layout K x (T x 2 col-major)).  The zero-mean flags are always the trailing
 * lround(explore_fraction*K) samples (sampler.cpp:36-37). */
int mppi_gpu_set_noise(mppi_gpu_handle* h, const double* eps);

/* ---- the hot path ---------------------------------------------------------- */
/* mpc_step (controller.cpp:133-148) without the slide: sample(iteration),
 * rollout, it_weights, update_plan (+SG), u0 = clamp(U'[0]).  x0 holds
 * n_controllers states, u0_out n_controllers x 2. */
int mppi_gpu_compute_control(mppi_gpu_handle* h, const double* x0, double* u0_out);
/* The slide half of mpc_step (controller.cpp:143-146): U[t] = U[t+1],
 * U[T-1] = 0, ++iteration. */
int mppi_gpu_slide(mppi_gpu_handle* h);
/* Exactly mpc_step: compute_control + slide. */
int mppi_gpu_step(mppi_gpu_handle* h, const double* x0, double* u0_out);
/* optimize_to_convergence (controller.cpp:150-164): `iterations` x {sample,
 * rollout, weights, update, ++iteration} on a fixed x0, no slide. */
int mppi_gpu_optimize(mppi_gpu_handle* h, const double* x0, int iterations);
/* Closed loop on the device (BASELINE config 1 receding horizon): per
 * iteration mpc_step on the current state, then the plant — the same device
 * model stepped with the clamped u0 — advances the state.  x_init holds
 * n_controllers states; traces are optional (iterations x n x 2 and
 * (iterations+1) x n x state_dim).  Replays one captured CUDA graph per
 * iteration. */
int mppi_gpu_closed_loop(mppi_gpu_handle* h, const double* x_init, int iterations,
                         double* u_trace, double* x_trace);
/* The same loop with device timing for benchmarks: CUDA events on the
 * handle's stream.  flush_l2_bytes > 0 overwrites a scratch buffer of that
 * size between iterations (evicting L2) and then sums the per-iteration event
 * intervals, so the flush is excluded from device_ms_out; 0 times the whole
 * back-to-back loop.  iter_ms_out (nullable, flush mode only) receives the
 * `iterations` per-iteration intervals (p50 / p99 latency). */
int mppi_gpu_closed_loop_timed(mppi_gpu_handle* h, const double* x_init, int iterations,
                               uint64_t flush_l2_bytes, double* device_ms_out, double* iter_ms_out);

/* ---- parity entry points (controller 0) ------------------------------------ */
/* sample_perturbations(params, iteration) (sampler.cpp:5-39) evaluated on the
 * device in the handle's noise mode; eps_out in the reference layout, flags
 * (nullable) K bytes. */
int mppi_gpu_sample_perturbations(mppi_gpu_handle* h, uint64_t iteration, double* eps_out,
                                  uint8_t* flags_out);
/* rollout_batch (controller.cpp:55-109) on the current plan and iteration.
 * eps_in (nullable) overrides the noise with a reference-layout batch.
 * eps_stored_out (nullable) receives the batch as rollout_batch leaves it
 * (zero-mean samples rewritten to eps - U, controller.cpp:70-72).  The batch is
 * retained for a following mppi_gpu_update_plan. */
int mppi_gpu_rollout_costs(mppi_gpu_handle* h, const double* x0, const double* eps_in,
                           double* costs_out, double* eps_stored_out);
/* it_weights (weights.cpp:8-25): rho = min S, w = exp(-(S-rho)/lambda)/eta. */
int mppi_gpu_weights(mppi_gpu_handle* h, const double* costs, double* w_out, double* rho,
                     double* eta);
/* update_plan (controller.cpp:118-131) with the batch of the last
 * mppi_gpu_rollout_costs: U' = U + SG(sum_k w_k eps_k).  Replaces the plan. */
int mppi_gpu_update_plan(mppi_gpu_handle* h, const double* weights);
/* State trajectory of one sample of the last rollout batch: (T+1) x state_dim,
 * x_0 first (step-by-step comparison against the oracle). */
int mppi_gpu_rollout_states(mppi_gpu_handle* h, const double* x0, int sample,
                            double* states_out);

/* ---- multi-GPU: shard samples over ranks, one exchange per iteration ------- */
/* The samples of one controller are cut into chunks, and the chunks into G
 * fixed groups (G = 8 * 2^j, set by the chunk count alone).  Every group's
 * chunk partials (rho, eta, T x 2 weighted-noise numerator) are merged on the
 * device into one group row, in a fixed order; rank r of N owns groups
 * [r G/N, (r+1) G/N).  The exchange is one all-gather of the group rows
 * (G x (4 + 2T) doubles for the whole job), after which every rank merges
 * them in group order: the plan is bit-identical on every rank and for every
 * N dividing G, including N = 1 (parallel_for_chunks, parallel.hpp:11-29). */
/* 128-byte ncclUniqueId, created on rank 0 and broadcast by the caller. */
int mppi_gpu_nccl_unique_id(unsigned char id_out[128]);
/* NCCL sharding: this handle becomes rank `rank` of `world_size` (one handle
 * per process and GPU).  MPPI_ERR_UNSUPPORTED if world_size does not divide
 * G, for fleets (n_controllers > 1) and for the CEM rule.  A rejected call
 * leaves the handle unchanged. */
int mppi_gpu_set_comm(mppi_gpu_handle* h, int rank, int world_size,
                      const unsigned char id[128]);
/* In-process sharding: handles[r] becomes rank r of n (one handle per GPU of
 * this process, or several handles on one GPU).  The exchange copies the
 * other ranks' group rows device to device.  Every handle needs the same
 * configuration; destroying one leaves the others unusable for step_local. */
int mppi_gpu_set_comm_local(mppi_gpu_handle** handles, int n);
/* mpc_step of a controller sharded with set_comm_local: every rank's rollout
 * and group merge, then every rank's exchange and epilogue.  x0 is the one
 * state (state_dim doubles) all ranks use; u0_out receives n x 2 (every
 * rank's u0; they are identical). */
int mppi_gpu_step_local(mppi_gpu_handle** handles, int n, const double* x0, double* u0_out);
/* The handle's partition: {rank, world_size, chunks, groups, chunk_lo,
 * chunk_hi, group_lo, group_hi} (chunk and group ranges of this rank). */
int mppi_gpu_shard_info(mppi_gpu_handle* h, int32_t out[8]);
/* The same partition as a pure function (no device): chunk_samples is the K1
 * chunk size of the handle's kernel variant. */
int mppi_gpu_shard_plan(int samples, int chunk_samples, int rank, int world_size, int32_t out[8]);

/* ---- instrumentation ------------------------------------------------------- */
/* cudaStream_t of the handle (for CUDA-event timing on the launching stream). */
int mppi_gpu_get_stream(mppi_gpu_handle* h, void** stream_out);
/* Kernel launches issued by this handle since creation. */
int mppi_gpu_launch_count(mppi_gpu_handle* h, uint64_t* count_out);
/* When enabled, CUDA events bracket every rollout-kernel launch; read returns
 * the summed milliseconds and the launch count since the last reset. */
int mppi_gpu_profile_enable(mppi_gpu_handle* h, int enable);
int mppi_gpu_profile_read(mppi_gpu_handle* h, double* rollout_ms, uint64_t* rollout_launches,
                          int reset);
/* With profiling enabled and world_size > 1: CUDA-event time of the group-row
 * exchange (the all-gather) summed over the timed closed-loop iterations. */
int mppi_gpu_profile_read_exchange(mppi_gpu_handle* h, double* exchange_ms, uint64_t* exchanges,
                                   int reset);
/* Name of the rollout kernel variant the handle dispatches. */
int mppi_gpu_kernel_variant(mppi_gpu_handle* h, char* name_out, int capacity);
/* FFMA microbenchmark on `device`: best measured FP32 FMA throughput
 * (TFLOP/s, FMA = 2 FLOP) over the probe variants; the roofline denominator. */
int mppi_gpu_fp32_peak_probe(int device, double* tflops_out, double* sm_clock_mhz_out);
/* Tensor and SFU ceilings of the tensor-core rollout on `device`: mma.sync
 * m16n8k16 f16 -> f32 throughput (TFLOP/s) and MUFU ex2 throughput (G lane
 * operations/s), the best of a few full-chip probe launches. */
int mppi_gpu_pipe_peak_probe(int device, double* hmma_tflops_out, double* mufu_gops_out);

/* ---- closed-loop driver: simulate_episode (simulator.cpp:102-177) ----------- */
/* Additive velocity / yaw-rate kick applied to the plant after the step that
 * ends at time_s (Disturbance, simulator.hpp:10-16). */
typedef struct mppi_disturbance {
  double time_s;
  double dv_x;
  double dv_y;
  double dtheta_dot;
} mppi_disturbance;
/* SimConfig (simulator.hpp:72-88) minus the parts the handle already holds
 * (sampling, weight rule, SG filter, bounds, costs, terminal cost). */
typedef struct mppi_sim_config {
  double episode_s;                  /* steps = lround(episode_s / dt) */
  int32_t exec_noise;                /* execution noise on the applied input */
  int32_t has_exec_noise_diag;       /* 0: the sampling variances */
  double exec_noise_diag[2];         /* variances */
  int32_t has_estimate_noise;        /* 0: exact state feedback */
  double estimate_noise_std[7];      /* standard deviations per state entry */
  mppi_bicycle_params plant;         /* the truth plant */
  double start_state[7];
  int32_t n_disturbances;
  const mppi_disturbance* disturbances;
} mppi_sim_config;
/* StepRecord (simulator.hpp:17-24): the plant state when the control was
 * computed, the clamped command, the realised input (command + execution
 * noise, before the plant's clamp), state_cost(x, 0) and h at the position. */
typedef struct mppi_sim_record {
  double time;
  double state[7];
  double commanded[2];
  double realized[2];
  double cost;
  double map_h;
} mppi_sim_record;
/* Reference defaults: SimConfig{} with BicycleParams{} and exec_noise on. */
void mppi_sim_config_init(mppi_sim_config* cfg);
/* One closed-loop episode on a single-controller handle: per step the state
 * estimate (+ estimate noise, counter stream kStreamEstimateNoise), mpc_step
 * on the device, execution noise (kStreamExecutionNoise), the clamped bicycle
 * truth step on the host, disturbances.  Deterministic given the handle's
 * seed.  records_out holds `capacity` records; *n_steps_out is the number
 * written; *aborted_out is 1 if a non-finite state ended the episode early.
 * The handle's controller-0 costmap is read back for the recorded cost. */
int mppi_sim_episode(mppi_gpu_handle* h, const mppi_sim_config* cfg, mppi_sim_record* records_out,
                     int capacity, int* n_steps_out, int* aborted_out);
/* Host evaluations of the truth model (reference pins; no device):
 * brush_tire_force (dynamics.cpp:23-43) and step_bicycle_truth
 * (dynamics.cpp:51-81, no clamp: the input is the applied one). */
void mppi_bicycle_params_init(mppi_bicycle_params* p);
int mppi_brush_tire_force(double alpha, double u_F, const mppi_bicycle_params* p, double* force_out);
int mppi_bicycle_step(const mppi_bicycle_params* p, const double x[7], const double v[2], double dt,
                      double x_next_out[7]);

/* ---- host-side workload generation (no GPU needed) ------------------------- */
/* Xavier-uniform MLP weights from a seed (BASELINE configs): U(-a, a),
 * a = sqrt(6 / (fan_in + fan_out)), output layer scaled by out_scale, biases 0.
 * Arrays in the set_dynamics_mlp layout. */
int mppi_workload_mlp_xavier(int hidden, uint64_t seed, double out_scale, double* w1,
                             double* b1, double* w2, double* b2, double* w3, double* b3);
/* Elliptical track: values[iy*width+ix] = min(|dist to ellipse (a, b)| /
 * half_width, 2.5) at cell centres x0 + ix*res, y0 + iy*res. */
int mppi_workload_ellipse_costmap(int width, int height, double x0, double y0, double res,
                                  double semi_a, double semi_b, double half_width,
                                  float* values);
/* Initial states on the centreline (arc length fraction s in [0,1), CCW
 * heading), v_x ~ U[vx_lo, vx_hi], roll/v_y/theta_dot ~ N(0, noise_std^2),
 * from counter streams of `seed`, one per controller index. */
int mppi_workload_initial_states(int n, uint64_t seed, double semi_a, double semi_b,
                                 int uniform_arc, double vx_lo, double vx_hi,
                                 double noise_std, double* states_out);
/* Savitzky-Golay kernel, sg_coefficients (smoothing.cpp:5-33). */
int mppi_sg_coefficients(int window, int degree, double* coeffs_out);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* MPPI_GPU_H_ */
