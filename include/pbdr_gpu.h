/* pbdr_gpu.h — C-ABI of the B200-native PBD-R substep loop.
 *
 * This is the drop-in boundary for the reference's solver step
 * (arxiv 2603.14634, /root/reference/proj). The reference has no FFI: its
 * solver API is C++ (proj/include/pbdr/scene.hpp:17-82, body.hpp:11-66) and
 * step() is specified in SPEC.md:326-334 because proj/src/solver.cpp is absent
 * (proj/CMakeLists.txt:20). Each entry point below names the reference
 * interface it replaces. Plain C types only: no torch, no C++ in signatures,
 * no exception crosses this boundary (status codes instead, errors.hpp:8-44).
 *
 * The C++ drop-in layer (include/pbdr/ headers, namespace pbdr) and the Python
 * host mirror (paper_2603_14634_b200/pbdr.py) are thin callers of this ABI.
 * There is no CPU fallback: every compute entry point runs CUDA kernels for
 * sm_100a and returns PBDR_ERR_CUDA when no device is usable.
 */
#ifndef PBDR_GPU_H
#define PBDR_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PBDR_ABI_VERSION 1

/* ---- Status codes: one per reference exception class (errors.hpp:8-44) ---- */
typedef enum pbdr_status {
  PBDR_OK = 0,
  PBDR_ERR_DEGENERATE = 1,     /* DegenerateConfigError   errors.hpp:12-15 */
  PBDR_ERR_RANK_DEFICIENT = 2, /* RankDeficientError(axis) errors.hpp:17-22 */
  PBDR_ERR_EMPTY_PACKING = 3,  /* EmptyPackingError        errors.hpp:24-26 */
  PBDR_ERR_INVALID_MOMENT = 4, /* InvalidMomentError       errors.hpp:28-30 */
  PBDR_ERR_CONFIG = 5,         /* ConfigError(key_path)    errors.hpp:32-37 */
  PBDR_ERR_SIMULATION = 6,     /* SimulationError(frame)   errors.hpp:39-44 */
  PBDR_ERR_CUDA = 7,           /* no usable sm_100 device / CUDA failure    */
  PBDR_ERR_GENERIC = 8         /* pbdr::Error                errors.hpp:8-10 */
} pbdr_status;

/* ---- SolverConfig mirror (scene.hpp:12-28; field order and defaults kept) -- */
typedef enum { PBDR_PRECISION_SINGLE = 0, PBDR_PRECISION_DOUBLE = 1 } pbdr_precision;
typedef enum { PBDR_VELOCITY_LEGACY = 0, PBDR_VELOCITY_INCREMENTAL = 1 } pbdr_velocity_update;
typedef enum { PBDR_BACKEND_SERIAL = 0, PBDR_BACKEND_PARALLEL = 1 } pbdr_backend;
typedef enum { PBDR_MOMENTUM_PER_ITERATION = 0, PBDR_MOMENTUM_PER_SUBSTEP = 1 } pbdr_momentum_frequency;

typedef struct pbdr_solver_cfg {
  double frame_rate;        /* Hz, default 100                       scene.hpp:18 */
  int32_t substeps;         /* default 10; dt = 1/(frame_rate*substeps) :19,:29 */
  int32_t solver_iterations;/* default 10                            scene.hpp:20 */
  int32_t precision;        /* pbdr_precision; GPU path: single only  scene.hpp:21 */
  int32_t velocity_update;  /* pbdr_velocity_update                   scene.hpp:22 */
  int32_t linear_momentum_fix;  /*                                    scene.hpp:23 */
  int32_t angular_momentum_fix; /*                                    scene.hpp:24 */
  int32_t momentum_frequency;   /* pbdr_momentum_frequency            scene.hpp:25 */
  int32_t backend;          /* accepted and ignored (no CPU path)     scene.hpp:27 */
  double gravity;           /* magnitude along -z, default 9.81       scene.hpp:26 */
} pbdr_solver_cfg;

/* ---- Plane (scene.hpp:44-48) and ForceProgram (scene.hpp:53-61) ---------- */
typedef struct pbdr_plane {
  double point[3];
  double normal[3]; /* unit */
  double friction;  /* Coulomb coefficient >= 0 */
} pbdr_plane;

typedef struct pbdr_force_program {
  double force[3];
  double torque[3];
  double t_start;
  double t_stop;    /* +inf allowed */
  int32_t gravity_exempt;
  int32_t reserved;
} pbdr_force_program;

/* ---- Scene (scene.hpp:65-74, body.hpp:11-30) as plain arrays -------------- */
typedef struct pbdr_scene_desc {
  int64_t num_particles;
  const double* position;   /* [3*num_particles]  Particle::position  body.hpp:12 */
  const double* velocity;   /* [3*num_particles]  Particle::velocity  body.hpp:13 */
  const double* inv_mass;   /* [num_particles]    Particle::inv_mass  body.hpp:14 */
  const double* radius;     /* [num_particles]    Particle::radius    body.hpp:15 */
  const int32_t* body_id;   /* [num_particles]    Particle::body_id   body.hpp:16 */
  int32_t num_bodies;
  const int64_t* body_offsets;  /* [num_bodies+1] CSR over body_indices */
  const int32_t* body_indices;  /* Body::particle_indices           body.hpp:21 */
  const double* rest_offsets;   /* [3*len] Body::rest_offsets        body.hpp:22 */
  const double* total_mass;     /* [num_bodies] Body::total_mass     body.hpp:23 */
  const double* rest_com;       /* [3*num_bodies] Body::rest_com     body.hpp:24 */
  const pbdr_force_program* programs; /* [num_bodies] or NULL    scene.hpp:68 */
  pbdr_plane ground;                  /*                          scene.hpp:69 */
  int32_t has_ground;                 /*                          scene.hpp:70 */
  double contact_relaxation;          /*                          scene.hpp:71 */
  /* Extensions (default-empty, so a reference Scene maps 1:1): */
  int32_t num_walls;          /* extra planes after the ground (config 3's container) */
  const pbdr_plane* walls;
  const int32_t* body_scene;  /* [num_bodies] independent-scene id, or NULL = all 0 */
  int32_t tile_kp;            /* 0 = automatic tile shape; 2, 4 or 8 particles per lane
                                 forces it (pbdr_choose_kp in csrc/pbdr_pinned.h) */
} pbdr_scene_desc;

/* Per-body trajectory sample (SPEC.md:357 trajectory hook; body.hpp:32-36
 * MomentumState plus the extract_pose orientation, body.hpp:50-58). */
typedef struct pbdr_body_stats {
  double com[3];
  double quat[4];    /* w, x, y, z: rotation from the rest pose */
  double linear[3];  /* P = sum m v */
  double angular[3]; /* L about the instantaneous com */
} pbdr_body_stats;

typedef struct pbdr_handle pbdr_handle;

/* ---- Lifecycle ------------------------------------------------------------
 * Replaces: constructing the solver state for pbdr::step(Scene&, const
 * SolverConfig&) (validate() scene.hpp:30,73). Copies the scene to
 * device `device` (float4 SoA, body-major). Validation failures return
 * PBDR_ERR_CONFIG with the key path in pbdr_last_error(). */
int pbdr_gpu_create(const pbdr_scene_desc* scene, const pbdr_solver_cfg* cfg, int device,
                    pbdr_handle** out);
void pbdr_gpu_destroy(pbdr_handle* h);

/* Advances `substeps` substeps of dt (one step() is one dt).
 * Replaces the body of the missing solver.cpp step loop. */
int pbdr_gpu_step(pbdr_handle* h, int64_t substeps);
/* Advances whole frames (frames * cfg.substeps substeps), replayed from one
 * captured CUDA graph per frame. Replaces the frame loop of run_test
 * (SPEC.md:425). */
int pbdr_gpu_step_frames(pbdr_handle* h, int64_t frames);

/* State transfer, in the caller's particle order (Scene::particles, fp64,
 * 3 doubles per particle; either pointer may be NULL). Staged through HBM and
 * converted / permuted on the device. Writing positions drops the warm-start
 * rotations and re-anchors the body sums, so the next step is the step of a
 * handle created from the written state. */
int pbdr_gpu_read_particles(pbdr_handle* h, double* position, double* velocity);
int pbdr_gpu_write_particles(pbdr_handle* h, const double* position, const double* velocity);
/* Simulation time, as the substep index t/dt: ForceProgram::active(t)
 * windows (scene.hpp:53-61) and SimulationError frame indices
 * (errors.hpp:39-44) follow it. A new handle starts at 0; each substep adds 1. */
int pbdr_gpu_set_time(pbdr_handle* h, int64_t substep);
int pbdr_gpu_get_time(pbdr_handle* h, int64_t* substep);
/* Fast fp32 transfer in the device's body-major order, 4 floats per particle:
 * pos4 = (x, y, z, inv_mass), vel4 = (vx, vy, vz, mass). Pointers may be
 * pinned host memory. Either may be NULL. */
int pbdr_gpu_read_f32(pbdr_handle* h, float* pos4, float* vel4);
int pbdr_gpu_write_f32(pbdr_handle* h, const float* pos4, const float* vel4);
/* Asynchronous versions on the handle's stream (host buffers must be pinned
 * and stay valid until pbdr_gpu_sync, which also reports device errors). With
 * one handle per batch slice, slices overlap their transfers with each
 * other's compute. */
int pbdr_gpu_write_f32_async(pbdr_handle* h, const float* pos4, const float* vel4);
int pbdr_gpu_read_f32_async(pbdr_handle* h, float* pos4, float* vel4);
int pbdr_gpu_step_frames_async(pbdr_handle* h, int64_t frames);

/* Per-body com / orientation / momentum (compute_momentum body.cpp:72-83,
 * extract_pose body.cpp:103-124), computed on the device. */
int pbdr_gpu_read_bodies(pbdr_handle* h, pbdr_body_stats* out);

/* ---- Errors --------------------------------------------------------------- */
/* Thread-local message for the last failing call on this thread. */
const char* pbdr_last_error(void);
/* Payload of the last failure: axis for RANK_DEFICIENT, frame index for
 * SIMULATION, first failing body (or -1), config key (string) for CONFIG. */
int pbdr_last_error_payload(double axis[3], int64_t* frame, int32_t* body);
const char* pbdr_last_error_key(void);

/* ---- Introspection, timing and replay hooks ------------------------------- */
typedef struct pbdr_info {
  int64_t num_particles;
  int32_t num_bodies;
  int32_t num_ctas;           /* iteration-kernel CTAs */
  int32_t hash_bits;          /* log2 of the cell-hash table */
  int32_t sort_passes;        /* onesweep passes per substep */
  int64_t launches_per_frame; /* kernels + memsets in one frame graph */
  int64_t device_bytes;       /* device memory owned by the handle */
  int32_t device;
  int32_t sm_count;
  float cell_size;            /* h = 2 r_max, fp32 */
  float dt;                   /* fp32 substep */
  int32_t tile_kp;            /* particles per lane of the iteration tiles */
  int32_t scene_cluster;      /* batched scenes: CTAs per scene cluster running a substep's
                                 iterations in one launch (0: per-iteration launches) */
} pbdr_info;
int pbdr_gpu_info(pbdr_handle* h, pbdr_info* out);

/* Times `frames` frames with CUDA events on the handle's stream (device time). */
int pbdr_gpu_time_frames(pbdr_handle* h, int64_t frames, float* ms);

/* Per-kernel-class device time over `frames` frames (events around each
 * launch; run separately from the timed region). Classes, in order:
 * 0 integrate+key, 1 histogram+scan, 2 onesweep passes, 3 cell ranges,
 * 4 neighbours, 5 iteration, 6 memsets, 7 body broadphase. ms[8], launches[8]. */
#define PBDR_KCLASS_COUNT 8
int pbdr_gpu_profile_frames(pbdr_handle* h, int64_t frames, float* ms, int64_t* launches);

/* Replay hooks (used by the parity tests; not on the product path). The
 * integrate hook runs the substep prologue (integrate, cell keys, sort, cell
 * ranges, candidate lists) without iterations; read_* return the device data
 * in body-major order. */
int pbdr_gpu_debug_prologue(pbdr_handle* h);
int pbdr_gpu_debug_iteration(pbdr_handle* h, int iteration_index);
int pbdr_gpu_debug_read_keys(pbdr_handle* h, uint32_t* cell_hash, int32_t* cell_xyz);
/* Sorted (key, slot) pairs of the broadphase-filtered particles: the first
 * pbdr_gpu_debug_near_count() entries are valid. */
int pbdr_gpu_debug_read_sorted(pbdr_handle* h, uint32_t* keys, uint32_t* vals);
int pbdr_gpu_debug_near_count(pbdr_handle* h, int64_t* count);
int pbdr_gpu_debug_read_candidates(pbdr_handle* h, int32_t* counts, int32_t* lists /* n*CAP */);
int pbdr_gpu_debug_read_init(pbdr_handle* h, float* init4);
/* Runs one iteration launch with per-CTA clock64 stamps (16 per CTA: start,
 * staged, phase A, body math A, phase B, body math B, end, SM id; then for the
 * CTA's first body: sums read A, body math A done, sums read B, body math B
 * done, polar start, polar end, 2 spare). */
int pbdr_gpu_debug_phase_timing(pbdr_handle* h, long long* out);
/* Body anchors (fp32 xyz per body) used by the anchored body sums. */
int pbdr_gpu_debug_read_anchor(pbdr_handle* h, float* anchor3);
int pbdr_gpu_debug_write_anchor(pbdr_handle* h, const float* anchor3);
/* Per-body warm-start rotation of the shape-matching polar (w, x, y, z as
 * float4; all-zero = none). pbdr_gpu_write_particles() clears it. */
int pbdr_gpu_debug_read_rquat(pbdr_handle* h, float* q4);
int pbdr_gpu_debug_write_rquat(pbdr_handle* h, const float* q4);

/* ---- Trajectory emission ------------------------
 * When enabled, every frame stepped by pbdr_gpu_step_frames / _time_frames
 * appends one pbdr_body_stats per body (com, orientation vs rest, P, L; the
 * same numbers as pbdr_gpu_read_bodies at that frame) to a device ring of
 * `capacity_frames` frames -- one extra launch per frame, no host sync. Drain
 * copies the pending frames (oldest first; out: frames x num_bodies x 13
 * doubles, t: frames seconds) and empties the ring; a full ring makes the next
 * step return an error. capacity 0 disables emission. In slab mode only the
 * owned bodies' records are written. */
int pbdr_gpu_trajectory_enable(pbdr_handle* h, int64_t capacity_frames);
int pbdr_gpu_trajectory_drain(pbdr_handle* h, double* out, double* t, int64_t max_frames, int64_t* frames);

/* ---- Staged stepping and x-slab decomposition --
 * One substep = pbdr_gpu_substep_begin (integrate, hash grid, candidate lists)
 * followed by solver_iterations calls of pbdr_gpu_substep_iteration; both only
 * enqueue on the handle's stream (pbdr_gpu_stream), so a caller can interleave
 * its own work on that stream between stages -- the slab runner's NCCL halo
 * exchange. pbdr_gpu_sync waits and maps device errors to status codes.
 * Replaces: the iteration loop inside pbdr::step. */
int pbdr_gpu_substep_begin(pbdr_handle* h);
int pbdr_gpu_substep_iteration(pbdr_handle* h);
int pbdr_gpu_sync(pbdr_handle* h);
int pbdr_gpu_stream(pbdr_handle* h, void** cuda_stream);

/* Per-body roles for one rank of an x-slab decomposition: 2 = owned (simulated
 * and authoritative), 1 = ghost (integrated and hashed so owned particles see
 * it; positions/velocities are overwritten by the halo exchange), 0 = inactive
 * (ignored). The layout stays the full scene's body-major layout, so every
 * rank's contact candidate lists are the single-GPU lists in the same order.
 * roles = NULL returns to whole-scene mode. Host array of num_bodies int8. */
int pbdr_gpu_set_roles(pbdr_handle* h, const int8_t* roles);

/* Halo exchange records: float4 per index, DEVICE pointers, enqueued on the
 * handle's stream. POSITION / VELOCITY index particle slots (body-major order,
 * positions of the current iteration buffer); ANCHOR / ROTATION index bodies
 * (anchored-sum reference point; warm-start rotation w,x,y,z). */
enum {
  PBDR_FIELD_POSITION = 0,
  PBDR_FIELD_VELOCITY = 1,
  PBDR_FIELD_ANCHOR = 2,
  PBDR_FIELD_ROTATION = 3
};
int pbdr_gpu_gather(pbdr_handle* h, int field, const int32_t* index, int64_t count, void* dst);
int pbdr_gpu_scatter(pbdr_handle* h, int field, const int32_t* index, int64_t count, const void* src);

/* ---- Native x-slab decomposition ---------
 * One rank of a giant scene split into x-slabs, driven in C++ with the halo
 * over NCCL (one rank per GPU) or over a local hub (ranks as threads of one
 * process on one GPU: the tests' way to run the same driver). The handle holds
 * a RANK-LOCAL scene: a contiguous range of the global bodies in global order
 * (pbdr_scene_generate_c5_slab), i.e. this rank's slab plus ghost bands, so
 * every owned trajectory is the single-GPU one bit for bit (refresh = 0).
 * Replaces: nothing in the reference (it has no decomposition); the scaling
 * note is PAPER.md:378. */
typedef struct pbdr_slab_config {
  int32_t rank, world;
  const double* edges;  /* world + 1 ascending com-x boundaries (edges[0] = -inf, edges[world] = +inf) */
  double ghost_band;    /* G = 2 rho + h + margin: a body this close to a boundary is ghosted across it */
  double margin;        /* a body may move at most margin / 2 in x per frame (else SimulationError) */
  int64_t body_first;   /* global id of local body 0 */
  int32_t refresh;      /* 0: ghost positions after every iteration (exact); 1: once per substep */
  int32_t overlap;      /* 1: tiles a neighbour ghosts run first, their halo overlaps the other tiles */
} pbdr_slab_config;
typedef struct pbdr_slab_hub pbdr_slab_hub;
int pbdr_nccl_unique_id(uint8_t out[128]);
int pbdr_gpu_slab_attach_nccl(pbdr_handle* h, const pbdr_slab_config* c, const uint8_t nccl_id[128]);
pbdr_slab_hub* pbdr_slab_hub_create(int world);
void pbdr_slab_hub_destroy(pbdr_slab_hub* hub);
int pbdr_gpu_slab_attach_local(pbdr_handle* h, const pbdr_slab_config* c, pbdr_slab_hub* hub);
/* Initial partition (owners by com_x, ghost lists, full ghost state). */
int pbdr_gpu_slab_start(pbdr_handle* h);
/* Frames of cfg.substeps substeps; repartition (migration) at every frame start. */
int pbdr_gpu_slab_step_frames(pbdr_handle* h, int64_t frames);
/* Owned local body ids (ascending); count always written. */
int pbdr_gpu_slab_owned(pbdr_handle* h, int32_t* local_ids, int64_t capacity, int64_t* count);
/* out[6]: owned bodies, owned particles, ghost bodies, halo bytes per
 * iteration (sent + received), migrations so far, frames so far. */
int pbdr_gpu_slab_info(pbdr_handle* h, int64_t out[6]);

/* ---- GPU pack_mesh (geometry.cpp:125-195) -----
 * Replaces: pbdr::pack_mesh(const TriMesh&, double radius) (geometry.hpp:57).
 * Grid candidates bb.min + radius + i * 2 radius (x slowest) inside the
 * closed triangle mesh by ray-crossing parity -- the reference's fp64
 * Moller-Trumbore test with its ambiguity band, re-cast along up to 8 fixed
 * jittered directions (ambiguous after 8: outside), one GPU thread per
 * candidate. centers (3 * capacity doubles, grid order) may be NULL to query
 * the count. Errors as the reference: radius <= 0 or a bad index -> GENERIC
 * (pbdr::Error), no candidate or none inside -> EMPTY_PACKING. */
int pbdr_pack_mesh(const double* vertices, int32_t num_vertices, const int32_t* triangles, int32_t num_triangles,
                   double radius, int device, double* centers, int64_t capacity, int64_t* count,
                   int64_t* candidates, int64_t* ambiguous);

/* ---- Host-side scene construction (no device work) ------------------------
 * The five BASELINE.json configs, generated deterministically from splitmix64
 * (rng.hpp:10-29) with pack_box lattices (geometry.cpp:32-55) and
 * add_packed_body placement (scene.hpp:76-82). Shared by the oracle, the tests
 * and bench.py so every arm sees identical inputs. */
typedef struct pbdr_generated_scene pbdr_generated_scene;
/* config_id 1..5; scale: config-specific size knob (C3 bodies, C4 scenes,
 * C5 cubes per x/y row); 0 = the BASELINE.json size. */
int pbdr_scene_generate(int config_id, uint64_t seed, int64_t scale, pbdr_generated_scene** out);
/* Config 4 shard for rank-local generation: scenes [first_scene,
 * first_scene + scenes), each seeded seed + scene index (weak scaling). */
int pbdr_scene_generate_c4_shard(uint64_t seed, int64_t scenes, int64_t first_scene,
                                 pbdr_generated_scene** out);
/* Config 5's cubes in x-columns [x_first, x_first + x_count) of a gx x gy x gz
 * grid (64 x 64 x 32 = BASELINE config 5): the rank-local scene of an x-slab
 * decomposition. Global x-major body order is kept (local body k is global
 * body x_first * gy * gz + k) and every cube equals the whole grid's. */
int pbdr_scene_generate_c5_slab(uint64_t seed, int64_t gx, int64_t gy, int64_t gz, int64_t x_first,
                                int64_t x_count, pbdr_generated_scene** out);
int pbdr_scene_view(const pbdr_generated_scene* s, pbdr_scene_desc* desc, pbdr_solver_cfg* cfg);
/* Placements that needed more than one attempt (0 for the config-5 grids). */
int64_t pbdr_scene_resamples(const pbdr_generated_scene* s);
/* Frames the config is specified for (1000/1000/500/200/100). */
int64_t pbdr_scene_frames(const pbdr_generated_scene* s);
/* Bodies whose placement still overlapped after 256 resamples (expected 0). */
int64_t pbdr_scene_forced_overlaps(const pbdr_generated_scene* s);
void pbdr_scene_free(pbdr_generated_scene* s);

/* Scene-construction helpers of the reference's geometry / rng modules,
 * exposed so the parity tests can pin them against the reference's own code:
 * pack_box (geometry.cpp:32-55: n^3 centres, z fastest, radius = half the
 * smallest spacing) and the splitmix64 stream (rng.hpp:10-29). */
int pbdr_pack_box(double hx, double hy, double hz, int n, double* centers, double* radius);
void pbdr_rng_u64(uint64_t seed, int count, uint64_t* out);
void pbdr_rng_unit(uint64_t seed, int count, double* out);

int pbdr_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PBDR_GPU_H */
