/*
 * lbmg.h — C ABI of the B200-native ACM-MRT + immersed-boundary LBM step.
 *
 * This is the drop-in boundary for the reference solver path
 * (/root/reference/proj/include/lbm).  Every entry point names the reference
 * interface it replaces.  Plain C types only: pointers, sizes, POD structs.
 * Host-side I/O is FP64 in the reference's canonical AoS order; device state
 * is fp32 (DDF-shifted populations) on sm_100a.
 *
 * Error convention: every function returning int returns LBMG_OK (0) or one
 * of the LBMG_ERR_* codes; lbmg_last_error() then holds the message.  The
 * C++ mirror (include/lbm_b200.hpp) turns LBMG_ERR_CONFIG into
 * lbm::ConfigError and LBMG_ERR_IO into lbm::IoError, like the reference
 * (core.hpp:50-58).  Divergence is NOT an error: it is reported through
 * lbmg_status, exactly like lbm::StepStatus (solver.hpp:47-52).
 */
#ifndef LBMG_H
#define LBMG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LBMG_ABI_VERSION 1

/* ---- status codes ------------------------------------------------------ */
#define LBMG_OK 0
#define LBMG_ERR_CONFIG 1 /* lbm::ConfigError */
#define LBMG_ERR_CUDA 2   /* CUDA runtime failure / no device */
#define LBMG_ERR_OOM 3    /* device allocation failed */
#define LBMG_ERR_IO 4     /* lbm::IoError */
#define LBMG_ERR_STATE 5  /* call not valid in the current state */

/* ---- enums (values match the reference's enum order) ------------------- */
/* collision.hpp:23 CollisionKind */
enum { LBMG_BGK = 0, LBMG_RAW_MRT = 1, LBMG_CENTRAL_MRT = 2 };
/* collision.hpp:25 RatePolicy */
enum { LBMG_POLICY_CONSTANT = 0, LBMG_POLICY_RELAX_TOWARD_ONE = 1 };
/* boundary.hpp:22 FaceCondition */
enum { LBMG_NOSLIP = 0, LBMG_INLET = 1, LBMG_OUTFLOW = 2, LBMG_PERIODIC = 3 };
/* scene.hpp:23 MeshConfig::Type (File is not supported: host asset I/O) */
enum { LBMG_MESH_SPHERE = 0, LBMG_MESH_BOX = 1, LBMG_MESH_FIN_COMB = 2, LBMG_MESH_QUAD = 3 };
/* ib.hpp:35 SamplingMethod */
enum { LBMG_SAMPLING_DART = 0, LBMG_SAMPLING_ELIMINATION = 1 };
/* scene.hpp:43 InitKind */
enum { LBMG_INIT_UNIFORM = 0, LBMG_INIT_TAYLOR_GREEN = 1 };
/* ib.hpp:33 AccumulationMode */
enum { LBMG_IB_ATOMIC = 0, LBMG_IB_DETERMINISTIC = 1 };

/* ---- scene description (mirrors SceneConfig, scene.hpp:49-78) ---------- */
typedef struct {
    int condition;      /* LBMG_NOSLIP..LBMG_PERIODIC */
    double velocity[3]; /* inlet velocity (inlet density is 1) */
} lbmg_face;

typedef struct { /* MeshConfig, scene.hpp:22-33 */
    int type;
    double center[3], lo[3], hi[3], origin[3];
    double radius;
    int subdivisions;
    int fins;
    double fin_length, fin_height, fin_spacing;
    double size, plane_z;
} lbmg_mesh;

typedef struct { /* SolidConfig, scene.hpp:35-40 + RigidMotion ib.hpp:111-115 */
    lbmg_mesh mesh;
    double poisson_radius;
    int sampling;   /* LBMG_SAMPLING_* */
    int has_motion; /* std::optional<RigidMotion> engaged */
    double linear_velocity[3], angular_velocity[3], center[3];
} lbmg_solid_config;

typedef struct {
    int nx, ny, nz;
    double viscosity;
    int kind;               /* LBMG_BGK.. */
    double high_order_rate; /* rate of degree>=3 moment rows */
    int policy;             /* LBMG_POLICY_* */
    double policy_eps0;
    int has_explicit_rates;
    double rates[27]; /* canonical moment-row order (collision.cpp:24-30) */
    lbmg_face faces[6]; /* order -x,+x,-y,+y,-z,+z (boundary.hpp:37) */
    double body_force[3];
    int n_solids;
    const lbmg_solid_config* solids;
    int init; /* LBMG_INIT_* */
    double init_density;
    double init_velocity[3];
    double tg_u_max;
    int regions;
    unsigned threads_per_region; /* CPU-only knob; ignored by the GPU */
    size_t alpha;                /* CSoA group size (Eq. 9) */
    int block_edge;              /* ell: solid-sample block edge */
    int ib_mode;                 /* LBMG_IB_* */
    uint64_t seed;
} lbmg_scene_config;

/* StepStatus, solver.hpp:47-52 */
typedef struct {
    int ok;
    int mach_warning;
    long step;
    char reason[120];
} lbmg_status;

/* TimingRow, io.hpp:50-54 (phase name, step, seconds) */
typedef struct {
    char phase[24];
    long step;
    double seconds;
} lbmg_timing_row;

typedef struct lbmg_scene lbmg_scene;   /* Scene, scene.hpp:92-96 */
typedef struct lbmg_runner lbmg_runner; /* Runner, runner.hpp:25-83 */

/* ---- library ----------------------------------------------------------- */
int lbmg_abi_version(void);
/* Thread-local message of the last failing call. */
const char* lbmg_last_error(void);
/* Number of visible CUDA devices (0 on a CPU-only host). */
int lbmg_device_count(void);

/* ---- scene setup (host C++) -------------------------------------------- */
/* SceneConfig defaults, scene.hpp:49-78. */
void lbmg_scene_config_default(lbmg_scene_config* cfg);
/* SceneConfig::make_model + CollisionModel::validate (scene.cpp:28-45,
 * collision.cpp:109-146) + BoundarySet::validate (boundary.cpp:7-15).
 * Writes the 27 effective rates (canonical row order) when rates != NULL. */
int lbmg_validate_config(const lbmg_scene_config* cfg, double* rates);
/* build_scene, scene.cpp:341-366: samples every solid (seeded Poisson-disk),
 * sets reference positions, orders by block_edge. */
int lbmg_scene_build(const lbmg_scene_config* cfg, lbmg_scene** out);
void lbmg_scene_destroy(lbmg_scene* s);
int lbmg_scene_solid_count(const lbmg_scene* s);
size_t lbmg_scene_sample_count(const lbmg_scene* s, int solid);
/* SolidSampleSet arrays (ib.hpp:47-60) in stored order; any pointer may be
 * NULL.  Vec3 arrays are n*3 doubles. */
int lbmg_scene_samples(const lbmg_scene* s, int solid, double* positions,
                       double* reference_positions, uint32_t* source_id, uint8_t* flagged,
                       double* bbox_lo_hi /* 6 */, int* block_edge);
/* Replaces a solid's sample set (positions, reference positions, source ids),
 * e.g. with a set produced elsewhere.  bbox is recomputed. */
int lbmg_scene_set_samples(lbmg_scene* s, int solid, size_t n, const double* positions,
                           const double* reference_positions, const uint32_t* source_id);

/* ---- host-side reference algorithms exposed for parity ------------------ */
/* morton3, ib.cpp:13-25 */
uint64_t lbmg_morton3(uint32_t x, uint32_t y, uint32_t z);
/* reorder_samples, ib.cpp:231-292: permutation perm[new] = old. */
int lbmg_reorder_permutation(size_t n, const double* positions, const uint32_t* source_id,
                             int ell, uint32_t* perm);
/* split_domain, decomp.cpp:5-18: z0z1[2*r], z0z1[2*r+1]. */
int lbmg_split_domain(int nz, int m, int* z0z1);

/* ---- runner (device engine) -------------------------------------------- */
/* Runner(const Scene&, int regions, unsigned threads), runner.cpp:22-58.
 * regions > 1 places every z-slab region on `device` (in-process halo
 * exchange through device memory); world/rank mode is lbmg_runner_create_rank. */
int lbmg_runner_create(const lbmg_scene* scene, int regions, int device, lbmg_runner** out);
/* Runner(const Scene&, int regions, unsigned threads) across devices of one
 * process: region (z-slab) r on devices[r % n_devices].  Peer access between
 * neighbouring slabs' devices is enabled: each slab's fluid kernel stores its
 * 9 crossing populations straight into the neighbours' halo buffers and the
 * fused IB kernel reads support nodes across a seam from the neighbour's
 * storage (NVLink); one stream per slab, cross-device events order a step.
 * Repeating a device (e.g. {0, 0}) runs the same orchestration on one GPU. */
int lbmg_runner_create_devices(const lbmg_scene* scene, int regions, int n_devices, const int* devices,
                               lbmg_runner** out);
/* Device of region r (-1 when out of range). */
int lbmg_runner_region_device(const lbmg_runner* r, int region);
/* One region (z-slab `rank` of `world`) of a multi-process run: halos are
 * exchanged by the caller through lbmg_runner_halo_* (NCCL send/recv). */
int lbmg_runner_create_rank(const lbmg_scene* scene, int world, int rank, int device,
                            lbmg_runner** out);
void lbmg_runner_destroy(lbmg_runner* r);
/* Runner::clone, runner.cpp:297-317 (deep copy of the device state). */
int lbmg_runner_clone(const lbmg_runner* r, lbmg_runner** out);
/* Run the engine's kernels on this stream (cudaStream_t as void*; NULL =
 * the runner's own stream). */
int lbmg_runner_set_stream(lbmg_runner* r, void* stream);

/* Runner::advance, runner.cpp:121-230.  Synchronous on return.  When
 * timings != NULL, up to timings_cap rows are appended (per-phase CUDA-event
 * times) and *n_timings receives the count written. */
int lbmg_runner_advance(lbmg_runner* r, long steps, lbmg_status* status,
                        lbmg_timing_row* timings, size_t timings_cap, size_t* n_timings);
long lbmg_runner_step_count(const lbmg_runner* r);
int lbmg_runner_status(const lbmg_runner* r, lbmg_status* status);
int lbmg_runner_dims(const lbmg_runner* r, int* nx, int* ny, int* nz);
int lbmg_runner_region_count(const lbmg_runner* r);
/* Runner::set_layout, runner.cpp:252-258. */
int lbmg_runner_set_layout(lbmg_runner* r, int block_edge, size_t alpha);
/* Kernel variants, the launch-split dimension of the tuner (replaces the
 * fixed kSplitBoundary two-pass collision, collision.hpp:58): fluid 0 = the
 * TMA-staged kernel on the ghost layout, 1 = register-direct kernels on the
 * compact layout; ib 0 = fused single-region IB kernel, 1 = split pipeline.
 * Results are identical up to fp32 atomic order in the IB scatter. */
int lbmg_runner_set_variant(lbmg_runner* r, int fluid, int ib);
int lbmg_runner_variant(const lbmg_runner* r, int* fluid, int* ib);
/* CTA shape of the TMA-staged fluid kernel (tuner dimension next to the
 * variants): 512, 256 or 128 threads per CTA (1024/512/256-slot tiles), 0 =
 * default.  Results are bitwise identical across shapes. */
int lbmg_runner_set_cta(lbmg_runner* r, int threads);
int lbmg_runner_cta(const lbmg_runner* r);
/* measure_cost (autotune.cpp:29-36): set_layout(block_edge, alpha), advance
 * warmup steps, then the mean device seconds per step of advance(n_steps)
 * (CUDA events on the runner's stream); +inf when the run diverges.  The
 * runner advances, like the reference's probe. */
int lbmg_runner_measure_cost(lbmg_runner* r, int block_edge, size_t alpha, int warmup, int n_steps,
                             double* seconds);
/* Identity of the device layout a requested alpha maps to (equal keys =
 * identical layouts, so a tuner can measure each once). */
int lbmg_runner_layout_key(const lbmg_runner* r, size_t alpha, uint64_t* key);
size_t lbmg_runner_alpha(const lbmg_runner* r);
int lbmg_runner_block_edge(const lbmg_runner* r);

/* Runner::gather_rho/u/f, runner.cpp:260-295: canonical AoS FP64 over the
 * global grid (n_nodes*{1,3,27} doubles).  In rank mode: this rank's owned
 * planes only, z-offset by the slab start (see lbmg_runner_slab). */
int lbmg_runner_gather_rho(const lbmg_runner* r, double* out);
int lbmg_runner_gather_u(const lbmg_runner* r, double* out);
int lbmg_runner_gather_f(const lbmg_runner* r, double* out);
/* Asynchronous rho* and u* snapshot, the driver's snapshot path (driver.cpp:45-59)
 * without stalling the step loop: _begin enqueues the canonical-AoS FP64
 * conversion and the D2H copy into pinned memory on a copy stream and
 * returns; later advance() calls continue (they wait for it only before
 * rho/u are rewritten); _wait blocks and copies out (rho: N doubles, u: 3N),
 * returning the step the snapshot was taken at. */
int lbmg_runner_snapshot_begin(lbmg_runner* r);
int lbmg_runner_snapshot_wait(lbmg_runner* r, double* rho, double* u, long* step);
/* dump_field in canonical order (io.cpp:34-55, canonical = true): the LBF1
 * file the reference's load_field (io.cpp:57-87) reads. */
int lbmg_dump_field(const char* path, int nx, int ny, int nz, int beta, const double* aos);
int lbmg_runner_slab(const lbmg_runner* r, int* z0, int* z1);

/* Runner::totals_log, runner.hpp:52: 6 doubles (force, torque) per step. */
size_t lbmg_runner_totals_count(const lbmg_runner* r);
int lbmg_runner_totals(const lbmg_runner* r, double* out, size_t cap_steps);

/* Runner::region_solids, runner.hpp:56: per-region sample replica. */
size_t lbmg_runner_sample_count(const lbmg_runner* r, int region, int solid);
int lbmg_runner_samples(const lbmg_runner* r, int region, int solid, double* positions,
                        double* boundary_velocity, double* penalty_force,
                        double* sampled_velocity, uint32_t* source_id, uint8_t* flagged);

/* Cell flags: owner face of every (node, direction) pull, as decided by
 * face_owns_direction (boundary.cpp:28-40) on the device: out[k*27+i] is the
 * face 0..5 that reconstructs f*_i at node k, or 255 when the pull streams. */
int lbmg_runner_cell_flags(const lbmg_runner* r, uint8_t* out);

/* ---- multi-process halo exchange (rank mode) ---------------------------- */
/* Device pointers of this rank's outgoing / incoming population halos of
 * buffer `parity`: the fluid phase of step t fills send[(t+1)&1] and step t+1
 * reads recv[(t+1)&1]; after creation send[0] must be moved to the
 * neighbours' recv[0].  send_lo carries the c_z=-1 populations of the bottom
 * owned plane (to rank-1), send_hi the c_z=+1 populations of the top plane
 * (to rank+1); each is 9*nx*ny floats.  NULL where the slab has no such
 * neighbour (periodic z wraps rank 0 <-> rank world-1). */
int lbmg_runner_halo_f(lbmg_runner* r, int parity, void** send_lo, void** send_hi, void** recv_lo,
                       void** recv_hi, size_t* bytes);
/* Same for the (rho,u) plane exchange the IB phase needs (4*nx*ny floats). */
int lbmg_runner_halo_macro(lbmg_runner* r, void** send_lo, void** send_hi, void** recv_lo,
                           void** recv_hi, size_t* bytes);
/* Split step for rank mode: PRE = IB band moments (+ pack macro halo);
 * MID = IB interpolate/penalty/spread + totals + motion; FLUID_EDGE = the
 * fused update of the two boundary planes (+ pack f halo); FLUID_BULK = the
 * rest; END = step bookkeeping.  The caller exchanges halos between phases. */
enum { LBMG_PHASE_PRE = 0, LBMG_PHASE_MID = 1, LBMG_PHASE_FLUID_EDGE = 2,
       LBMG_PHASE_FLUID_BULK = 3, LBMG_PHASE_END = 4 };
int lbmg_runner_phase(lbmg_runner* r, int phase, int write_macro);
/* After an externally driven run: synchronise and fold device status/totals
 * into the host-side Runner state (like the tail of lbmg_runner_advance). */
int lbmg_runner_sync(lbmg_runner* r, lbmg_status* status);
/* Most steps an externally driven run may enqueue between two
 * lbmg_runner_sync calls (the device motion / reaction-totals tables hold
 * that many rows); lbmg_runner_phase(PRE) fails with LBMG_ERR_STATE beyond it. */
long lbmg_runner_sync_interval(const lbmg_runner* r);
/* Diagnostics: number of engine kernels one step launches, counted from the
 * captured step CUDA graph (0 before the first graph-replayed advance). */
long lbmg_runner_kernels_per_step(const lbmg_runner* r);
/* Diagnostics: engine kernels launched by lbmg_runner_advance so far (graph
 * kernel nodes included), for launch counts over a timed region. */
long lbmg_runner_kernel_launches(const lbmg_runner* r);

/* ---- smoke tracers (tracer.hpp / tracer.cpp, runner.cpp:213-223) -------- */
/* TracerEmitter, tracer.hpp:14-17: axis-aligned region (grid units) and
 * particles per step. */
typedef struct {
    double lo[3], hi[3];
    int rate;
} lbmg_emitter;
/* SceneConfig::emitters (scene.hpp:60; the "tracers" JSON key,
 * scene.cpp:244-258): replaces the scene's emitter list.  A runner built
 * from the scene emits and advects tracers every step on the device. */
int lbmg_scene_set_emitters(lbmg_scene* s, int n, const lbmg_emitter* emitters);
/* emit_tracers, tracer.cpp:28-40, host: the positions one step appends
 * (sum of the rates, AoS n*3) from the same mt19937_64 stream. */
int lbmg_emit_tracers(int n, const lbmg_emitter* emitters, long step, uint64_t seed, double* positions);
/* Runner::tracers(), runner.hpp:54: the live cloud after the last step, in
 * the reference's order (emission order, retired particles removed).
 * positions n*3 (AoS), birth_step n; either may be NULL. */
size_t lbmg_runner_tracer_count(const lbmg_runner* r);
int lbmg_runner_tracers(const lbmg_runner* r, double* positions, int64_t* birth_step);
/* rasterize_density(runner.tracers(), dims), tracer.cpp:67-92, on the device
 * from the resident cloud: vol has nx*ny*nz doubles (node_index order). */
int lbmg_runner_tracer_density(const lbmg_runner* r, double* vol);
/* rasterize_density of a host cloud (positions n*3) on device `device`. */
int lbmg_rasterize_density(size_t n, const double* positions, int nx, int ny, int nz, int device,
                           double* vol);

/* ---- the reference's free-function surface (unit parity, GPU) ----------- */
/* step(SimState&, model, boundary, body_force, ctx, pool), solver.hpp:82-83 /
 * solver.cpp:181-191: one single-region step without solids (stream, six face
 * passes, moments, collision + forcing, t += 1) on the runner's state.  The
 * runner must hold one in-process region and no solids (LBMG_ERR_STATE). */
int lbmg_step(lbmg_runner* r, lbmg_status* status);
/* The explicit SimState that step() advances (solver.hpp:29-45), canonical
 * AoS FP64 (nodes*27): f = f(t); f_star = the face-pass scratch whose face
 * entries seed the persistent face slots the stale outflow-edge reads use
 * (NULL: f); t = the step counter.  rho* and u* read back as the moments of f
 * until the next step.  Single in-process region, no solids or tracers. */
int lbmg_runner_load_state(lbmg_runner* r, const double* f, const double* f_star, long t);

/* The IB free functions of ib.hpp:77-128 on a sample batch, computed on
 * device 0 in FP64 with the reference's operation order (support,
 * interpolation, penalty and rigid motion are bit-exact; spreading uses FP64
 * atomics, the reference's atomic mode; the totals a fixed-order tree).
 * Sample arrays are AoS Vec3 (n*3); fields canonical AoS over the nx*ny*nz
 * grid (u: nodes*3, rho: nodes, g: nodes*3); [z0, z1) is the owned slab of
 * the seam rule (sample_active, ib.cpp:313-317; the whole grid: 0, nz). */
/* kernel_support, ib.cpp:294-308: base (n*3), w (n*6: wx0 wx1 wy0 wy1 wz0 wz1), inside (n) */
int lbmg_ib_kernel_support(size_t n, const double* positions, int nx, int ny, int nz, int* base, double* w,
                           uint8_t* inside);
/* interpolate_velocity, ib.cpp:321-343: sampled (n*3), flagged (n, may be NULL) */
int lbmg_ib_interpolate_velocity(size_t n, const double* positions, const double* u, int nx, int ny, int nz,
                                 int z0, int z1, double* sampled_velocity, uint8_t* flagged);
/* penalty_forces, ib.cpp:345-365: force = rho(x_s) (u_b - u(x_s)) (flagged may be NULL) */
int lbmg_ib_penalty_forces(size_t n, const double* positions, const double* boundary_velocity,
                           const double* sampled_velocity, const uint8_t* flagged, const double* rho, int nx,
                           int ny, int nz, int z0, int z1, double* penalty_force);
/* spread_forces, ib.cpp:369-454 (atomic mode): g += the spread forces, owned planes only */
int lbmg_ib_spread_forces(size_t n, const double* positions, const double* penalty_force, const uint8_t* flagged,
                          int nx, int ny, int nz, int z0, int z1, double* g);
/* update_rigid_motion, ib.cpp:456-489: positions, boundary velocities, flags at step t */
int lbmg_ib_update_rigid_motion(size_t n, const double* reference_positions, const double* linear_velocity,
                                const double* angular_velocity, const double* center, long t, int nx, int ny,
                                int nz, double* positions, double* boundary_velocity, uint8_t* flagged);
/* reaction_totals, ib.cpp:491-501: (F, T) of the samples with z in [z0, z1), torque about center */
int lbmg_ib_reaction_totals(size_t n, const double* positions, const double* penalty_force, const double* center,
                            int z0, int z1, double* force_torque);

/* ---- kernel-level entry points (unit parity, GPU) ----------------------- */
/* collide (collision.cpp:207-212) of n nodes on the device, fp32 arithmetic:
 * f (n*27), rho (n), u (n*3) host FP64 in, omega (n*27) host FP64 out. */
int lbmg_collide_batch(const lbmg_scene_config* model_cfg, size_t n, const double* f,
                       const double* rho, const double* u, double* omega);

#ifdef __cplusplus
}
#endif
#endif /* LBMG_H */
