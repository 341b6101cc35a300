/*
 * granusim_b200.h — C-ABI of the B200-native GranularGym timestep.
 *
 * The reference (`/root/reference/pkg/src/granusim`) has no FFI: its boundary is
 * the Python function API.  Every entry point below replaces one reference
 * function (cited file:line) and is what a ctypes/cffi binding of the reference
 * package would call.  Plain pointers and sizes only; no torch types.
 *
 * Conventions
 *   - every function returns an int status (GG_OK == 0);  gg_last_error(ctx)
 *     returns a human-readable message for the last failure on that context.
 *   - a context owns one CUDA stream on one device; calls on one context are
 *     not thread-safe, distinct contexts are independent
 *     (bindings/tests/test_bindings.py:112-124 "concurrent handles").
 *   - positions / velocities cross the boundary as float64 (n,3) row-major
 *     host arrays (the reference's ParticleSet layout, scene.py:85-93) or as
 *     float32 float4 device arrays (the resident layout).
 *   - gg_step is asynchronous on the context stream; gg_sync waits and returns
 *     the per-step reports.
 */
#ifndef GRANUSIM_B200_H
#define GRANUSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped back to the reference's exception types) ------ */
#define GG_OK 0
#define GG_EINVAL 1        /* ValueError / ValidationError (bad argument)            */
#define GG_ENONFINITE 2    /* SolverError, contact.py:503-509                        */
#define GG_ECAPACITY 3     /* per-owner contact slots exhausted (host grows + retries)*/
#define GG_ECUDA 4         /* CUDA runtime failure                                    */
#define GG_EPOSITIONS 5    /* ValueError("positions must be finite"), broadphase.py:104-107 */

/* ---- geometry kinds (sdf.py:44-241) -------------------------------------- */
#define GG_GEOM_SPHERE 1
#define GG_GEOM_HALFSPACE 2
#define GG_GEOM_BOX 3
#define GG_GEOM_CYLINDER 4
#define GG_GEOM_TUBE 5
#define GG_GEOM_GRID 6

/* ---- pipeline modes (stepper.py:34-37) ----------------------------------- */
#define GG_MODE_TWO_LOOPS_SPLIT 0
#define GG_MODE_TWO_LOOPS_FUSED 1
#define GG_MODE_ONE_LOOP 2

/* MaterialParams (scene.py:47-82) + CyclicBoundary (scene.py:115-124).
 * Derived constants are computed on the host exactly as the reference writes
 * them so device decisions are bit-identical:
 *   contact_d2   = (2.0 * r) ** 2                       contact.py:261
 *   coincident_d2 = COINCIDENT_EPS * COINCIDENT_EPS      contact.py:260
 *   gdt          = timestep * gravity                    contact.py:452          */
typedef struct gg_params {
  double radius;
  double particle_mass;
  double friction;
  double baumgarte_alpha;
  double timestep;
  double gravity[3];
  double gamma;
  double contact_d2;
  double coincident_d2;
  double gdt[3];
  int32_t solver_iterations;
  int32_t has_boundary;
  double z_min;
  double z_max;
} gg_params;

/* One kinematic body at one step, after RigidBody.update(t) (scene.py:150-153).
 * aabb_lo/hi are the world AABB `_near_body` computes (contact.py:187-203);
 * bounded == 0 for geometries whose contact_bounds is None (HalfSpace, Tube). */
typedef struct gg_body {
  int32_t kind;      /* GG_GEOM_*                                       */
  int32_t grid_id;   /* from gg_upload_grid, GG_GEOM_GRID only           */
  int32_t bounded;
  int32_t reserved;
  double shape[4];   /* sphere {R}; halfspace {nx,ny,nz,offset}; box {hx,hy,hz};
                        cylinder {R, half_height}; tube {R}              */
  double rot[9];     /* pose[:3,:3], row-major                           */
  double trans[3];   /* pose[:3,3]                                       */
  double omega[3];   /* RigidBody.omega                                  */
  double v_origin[3];/* RigidBody.v_origin                               */
  double aabb_lo[3];
  double aabb_hi[3];
} gg_body;

/* StepReport (stepper.py:40-54), minus wall_time/step_index/body_momentum,
 * which the host fills (body momentum comes from gg_sync's bm array). */
typedef struct gg_report {
  int64_t n_contacts;
  int64_t n_candidates;
  int64_t n_body_contacts;
  int64_t n_coincident;
  int64_t n_degenerate;
  double max_penetration;
  double kinetic_energy;
  double max_cone_violation;
  double min_normal_impulse; /* +inf when no contact was live: host maps to 0.0 */
} gg_report;

/* A depth camera (render.py DepthCamera :19-32) with its world pose already
 * resolved (attach_body applied by the caller).  Camera frame: +x right,
 * +y down, +z forward. */
typedef struct gg_camera {
  int32_t kind;      /* 0 perspective, 1 orthographic                   */
  int32_t width;
  int32_t height;
  int32_t reserved;
  double pose[16];   /* world-from-camera, row-major 4x4                 */
  double fov;        /* vertical field of view, radians (perspective)    */
  double extent[2];  /* world width, height (orthographic)               */
  double far;        /* depth of a pixel that hits nothing               */
} gg_camera;

typedef struct gg_ctx gg_ctx;

/* Create a context for n particles and an n_h-bucket hash table.
 * Replaces the implicit state of stepper.step (stepper.py:57-72):
 * n_h == scene.hashmap_size or default_table_size(n) (broadphase.py:58-60).
 * max_contacts = per-owner contact slots (grown on GG_ECAPACITY). */
int gg_create(int device, const gg_params* params, int64_t n, int64_t n_h,
              int32_t max_bodies, int32_t max_contacts, gg_ctx** out);

/* Batched independent environments (the RL env
 * batch, BulldozerEnv/ExcavationEnv scenes, envs.py:102-348).  One context
 * steps n_envs scenes of n_per_env particles each, all with the same params
 * and per-env table size n_h; each env keeps its own hash table (buckets
 * [e*n_h, (e+1)*n_h)) and its own bodies, so every env evolves exactly as it
 * would in a context of its own (bitwise).  Layout conventions with E envs:
 *   state arrays        (E * n_per_env, 3) env-major (env e = rows e*n_per_env..)
 *   gg_step bodies      [n_steps][E][n_bodies]
 *   gg_sync reports     [n_steps][E];  body_momentum [n_steps][E][n_bodies][3]
 *   gg_detect out       [E]
 *   taps                global particle ids (env e owns ids e*n_per_env..)
 * gg_create(...) == gg_create_batched(device, params, 1, n, n_h, ...). */
int gg_create_batched(int device, const gg_params* params, int32_t n_envs, int64_t n_per_env,
                      int64_t n_h, int32_t max_bodies, int32_t max_contacts, gg_ctx** out);
int gg_num_envs(const gg_ctx* ctx);
/* Per-env goal-box statistics of the current state: reward[e] =
 * bulldozer_reward(positions of env e, GoalBox(lo, hi)) (envs.py:61-70:
 * +100/n inside the box, boundary inclusive, -d/n outside) and inside[e] =
 * particles of env e in the box (the transported-mass statistic).  Either
 * output may be NULL; both hold n_envs entries. */
int gg_env_box_stats(gg_ctx* ctx, const double lo[3], const double hi[3], double* reward,
                     int64_t* inside);
int gg_destroy(gg_ctx* ctx);
const char* gg_last_error(const gg_ctx* ctx);
int gg_set_params(gg_ctx* ctx, const gg_params* params);

/* Particle state (ParticleSet.positions/velocities, scene.py:85-112).
 * Host variants take float64 (n,3) arrays in user order; device variants take
 * float4 (x,y,z,_) float32 arrays in user order on the context's device. */
int gg_set_state_f64(gg_ctx* ctx, const double* x, const double* v);
int gg_get_state_f64(gg_ctx* ctx, double* x, double* v);
int gg_set_state_f32x4_dev(gg_ctx* ctx, const void* x4, const void* v4);
int gg_get_state_f32x4_dev(gg_ctx* ctx, void* x4, void* v4);

/* SdfGrid values (sdf.py:179-241): float64 [dims0][dims1][dims2] C-order. */
int gg_upload_grid(gg_ctx* ctx, const double* values, const int32_t dims[3],
                   const double origin[3], const double spacing[3], int32_t* grid_id);

/* Enqueue n_steps timesteps (stepper.step, stepper.py:57-135) on the context
 * stream.  bodies = [n_steps][n_bodies] per-step body tables.  Asynchronous.
 * mode = PipelineMode (stepper.py:74-98), the loop structure, same results:
 * GG_MODE_TWO_LOOPS_SPLIT records only contacts; GG_MODE_TWO_LOOPS_FUSED
 * keeps a (masked) record for every candidate and the sweeps run over all of
 * them; GG_MODE_ONE_LOOP repeats the collision test inside every sweep. */
int gg_step(gg_ctx* ctx, int32_t n_steps, const gg_body* bodies, int32_t n_bodies,
            int32_t mode);

/* Device-resident body drivers: when gg_step gets
 * bodies == NULL, every body slot's rows are generated on the device for all
 * n_envs envs and all n_steps steps (no host packing, no upload):
 *   gg_drive_fixed   the same row rows[e] every step (ground, static tools);
 *   gg_drive_track   TrackSteeringDriver per env (kinematics.py:179-230):
 *                    state x/y/theta [E], z, speed scales, base pose (4x4
 *                    row-major), a template row (kind, shape, grid, bounded)
 *                    and the geometry's local contact bounds lo/hi for the
 *                    world AABB; each step advances the state by the context
 *                    timestep (heading first), then poses the body;
 *   gg_drive_chain   KinematicChain + ChainLinkDriver per env (kinematics.py:
 *                    237-322): n_links links (parent index, prismatic flag,
 *                    parent-to-joint 4x4 origin, unit axis, velocity limit),
 *                    base pose, joint positions q [E][n_links]; each step the
 *                    joint rates are the command clipped to the limits,
 *                    q += dt * qd, then the forward kinematics of link_index
 *                    gives the body pose and twist (ExcavationEnv.step,
 *                    envs.py:336-341);
 *   gg_drive_command per-env actions: track [E][2] (clipped to [-1, 1]),
 *                    chain [E][n_links] joint-rate commands;
 *   gg_drive_state / gg_drive_chain_state  the current state back to the host. */
int gg_drive_fixed(gg_ctx* ctx, int32_t slot, const gg_body* rows);
int gg_drive_track(gg_ctx* ctx, int32_t slot, const gg_body* tmpl, const double lo[3], const double hi[3],
                   const double* x, const double* y, const double* theta, double z, double scale_v,
                   double scale_omega, const double base_pose[16]);
int gg_drive_chain(gg_ctx* ctx, int32_t slot, const gg_body* tmpl, const double lo[3], const double hi[3],
                   int32_t n_links, int32_t link_index, const int32_t* parents, const int32_t* prismatic,
                   const double* origins, const double* axes, const double* limits,
                   const double base_pose[16], const double* q);
int gg_drive_command(gg_ctx* ctx, int32_t slot, const double* actions);
int gg_drive_state(gg_ctx* ctx, int32_t slot, double* x, double* y, double* theta);
int gg_drive_chain_state(gg_ctx* ctx, int32_t slot, double* q);
/* Re-run steps [first, first + n_steps) of the last batch from the body rows
 * it already holds (a device-driven batch after GG_ECAPACITY and
 * gg_set_max_contacts: the drivers have advanced past these rows). */
int gg_step_resume(gg_ctx* ctx, int32_t first, int32_t n_steps, int32_t mode);
/* Reports [first, first + count) of the last batch ([count][E] and
 * [count][E][n_bodies][3]) without waiting for the rest to be copied. */
int gg_batch_reports(gg_ctx* ctx, int32_t first, int32_t count, gg_report* reports, double* body_momentum);

/* Detection pass only (detect_contacts / narrowphase_contacts,
 * contact.py:244-300,372-379) on the current state: broadphase + pp + body
 * contacts, no solve, no state change.  Fills the contact/broadphase fields
 * of *out (n_contacts, n_candidates, n_body_contacts, n_coincident,
 * n_degenerate, max_penetration); gg_tap_contacts then reads the contacts. */
int gg_detect(gg_ctx* ctx, const gg_body* bodies, int32_t n_bodies, gg_report* out);

/* Wait for the enqueued steps.  Writes min(n_steps,cap) reports and the
 * [n_steps][n_bodies][3] body momenta (StepReport.body_momentum,
 * contact.py:489-495).  *n_done = steps committed; on failure returns the
 * status of the failing step and *err_step = its index within the batch
 * (state is left at that step's input, like the reference which raises
 * before integrating, stepper.py:99-103). */
int gg_sync(gg_ctx* ctx, gg_report* reports, double* body_momentum, int32_t cap,
            int32_t* n_done, int32_t* err_step);

/* Device time of the last gg_step batch (CUDA events on the context stream). */
int gg_last_batch_ms(gg_ctx* ctx, float* ms);

/* Benchmark helpers (bench.py).  gg_bench_steps runs n_steps like gg_step
 * but writes flush_bytes to a scratch buffer (L2 flush) before every step
 * and times each step alone with CUDA events (step_ms[n_steps]).
 * gg_profile_steps runs the same schedule un-graphed with an event after
 * every kernel and returns per-kernel-kind device time (kind_ms[11]) and
 * launch counts; gg_profile_kind_name(k) names kind k.  Both commit state. */
int gg_bench_steps(gg_ctx* ctx, int32_t n_steps, const gg_body* bodies, int32_t n_bodies,
                   int64_t flush_bytes, float* step_ms);
int gg_profile_steps(gg_ctx* ctx, int32_t n_steps, const gg_body* bodies, int32_t n_bodies,
                     float* kind_ms, int32_t* kind_launches);
const char* gg_profile_kind_name(int32_t k);

/* ---- parity taps (read-only views of the last committed step) ------------
 * cells/hashes: position_cells + spatial_hash of the CURRENT state in user
 *   order (broadphase.py:33-55, the SpatialHashmap.cells/.hashes fields);
 * order: np.argsort(hashes, kind="stable") (broadphase.py:160), user ids.   */
int gg_tap_hash(gg_ctx* ctx, int64_t* cells, int64_t* hashes, int64_t* order);

/* Contacts detected by the last step or gg_detect (narrowphase_contacts,
 * contact.py:244-300) as user-id directed pairs, in the reference's
 * ContactSet order: particle contacts by owner, an owner's in candidate order
 * (neighbour buckets by ascending hash, a bucket's particles in stable order,
 * broadphase.py:149-182), then body contacts body by body, each body's by
 * owner.  kind 0 = particle (other = particle id), kind 1 = body (other = body
 * index).  e1/psi/vj in float64 (computed in fp64, stored fp32 on device);
 * vj = body surface velocity at the contact point (contact.py:279,286), zero
 * for particle contacts.  Any output may be NULL.  *count = total; at most
 * cap rows are written. */
int gg_tap_contacts(gg_ctx* ctx, int64_t cap, int64_t* count, int32_t* owner,
                    int32_t* other, int32_t* kind, double* psi, double* e1, double* vj);

/* position_cells (broadphase.py:33-41) of n float64 positions (n,3):
 * round_half_away(x / 2r) per coordinate -> cells (n,3) int64.
 * GG_EPOSITIONS if a coordinate is not finite (broadphase.py:104-107). */
int gg_position_cells(gg_ctx* ctx, const double* x, int64_t n, double radius, int64_t* cells);

/* candidate_pairs (broadphase.py:185-196) of the context's current state:
 * every directed candidate (i, j != i), i ascending, i's candidates in the
 * order _candidate_csr enumerates them (broadphase.py:149-182).  *count =
 * total; ci/cj are written only if both are non-NULL and cap >= total
 * (call once with NULL to size).  Single-scene contexts only. */
int gg_tap_candidates(gg_ctx* ctx, int64_t cap, int64_t* count, int64_t* ci, int64_t* cj);

/* narrowphase_candidates (contact.py:206-223, _assemble_candidates :303-369)
 * on explicit candidate pairs of n float64 positions x (n,3):
 *   pp_e1 (m,3), pp_psi (m), pp_colliding (m): e1 = d/|d|, psi = 2r - |d|
 *     for colliding pairs (|d| < 2r, not coincident), zeros otherwise;
 *     *n_coincident = pairs with |d|^2 < COINCIDENT_EPS^2;
 *   per body b and particle i (arrays [n_bodies][n], normals/vj [..][3]):
 *     b_near (_near_body's AABB test, contact.py:187-203), and for near
 *     particles b_hit / b_psi / b_normal (penetration_depth, sdf.py:472-512)
 *     and b_vj = velocity_at(contact point) (contact.py:327-333);
 *     *n_degenerate over near particles.
 * Grid bodies refer to grids uploaded to ctx (gg_upload_grid). */
int gg_narrow_pairs(gg_ctx* ctx, const double* x, int64_t n, const int64_t* ci, const int64_t* cj,
                    int64_t m, double radius, const gg_body* bodies, int32_t n_bodies,
                    double* pp_e1, double* pp_psi, uint8_t* pp_colliding, int64_t* n_coincident,
                    uint8_t* b_near, uint8_t* b_hit, double* b_psi, double* b_normal, double* b_vj,
                    int64_t* n_degenerate);

/* A contact list in the reference's array layout: ContactSet, or
 * CandidateContacts when colliding != NULL (contact.py:103-184). */
typedef struct gg_contact_list {
  int64_t m;
  const int64_t* owner;
  const int64_t* kind;     /* 0 particle, 1 body */
  const int64_t* other;    /* particle index or body index */
  const double* e1;        /* (m,3) unit normal, j -> i */
  const double* psi;       /* (m) */
  const double* vj;        /* (m,3) body surface velocity (particle rows ignored) */
  const uint8_t* colliding;/* CandidateContacts.colliding, or NULL */
} gg_contact_list;

/* solve_contacts_pja (contact.py:393-518) on a caller-supplied contact list
 * and n float64 velocities v (n,3): sweeps first_sweep .. first_sweep +
 * n_sweeps - 1 of params->solver_iterations (a caller that refreshes the
 * candidates between sweeps, contact.py:455-461, calls it once per sweep).
 * In/out: dv (n,3) (zeros before sweep 0), body_momentum (n_bodies,3)
 * (accumulated), diag[2] = {max cone violation, min normal impulse}
 * (start {0, +inf}).  *n_live = live contacts.  After the last sweep a
 * non-finite dv returns GG_ENONFINITE with the reference's SolverError
 * text.  The frame (e2, e3) is built as contact_frames does (contact.py:47-56);
 * dot products, cross products and the per-owner accumulation follow numpy's
 * operation order; body momentum is summed in 2^-36 fixed point. */
int gg_solve_contacts(gg_ctx* ctx, const gg_contact_list* contacts, int64_t n, const double* v,
                      const gg_params* params, int32_t n_bodies, int32_t first_sweep,
                      int32_t n_sweeps, double* dv, double* body_momentum, double* diag,
                      int64_t* n_live);

/* project_friction_cone (contact.py:59-81) in place on k contact-frame
 * impulses b (k,3); psi has k entries, or one if psi_scalar.  GG_EINVAL
 * ("require mu >= 0 and dt > 0") like the reference's ValueError. */
int gg_project_cone(gg_ctx* ctx, double* b, int64_t k, const double* psi, int32_t psi_scalar,
                    double mu, double alpha, double dt);

/* Standalone SDF query (penetration_depth, sdf.py:472-512) for n world points
 * against one posed body; out psi[n], normal[n*3], hit[n] (0/1), n_degenerate. */
int gg_penetration(gg_ctx* ctx, const gg_body* body, const double* points, int64_t n,
                   double radius, double* psi, double* normal, int32_t* hit,
                   int64_t* n_degenerate);

/* Standalone spatial hash (spatial_hash, broadphase.py:44-55) of k cells. */
int gg_spatial_hash(gg_ctx* ctx, const int64_t* cells, int64_t k, int64_t n_h,
                    int64_t* out);

/* Contact-slot capacity.  gg_sync returns GG_ECAPACITY when an owner had more
 * contacts than slots; gg_required_contacts reports how many it needed and
 * gg_set_max_contacts regrows the slot arrays (the step is then re-run from
 * its uncommitted input, "x2 growth between steps"). */
int gg_set_max_contacts(gg_ctx* ctx, int32_t max_contacts);
int gg_max_contacts(const gg_ctx* ctx);
int gg_required_contacts(gg_ctx* ctx);

/* Physical particle order: re-sorted into Morton order of the cells every
 * `steps` steps (and after every state upload).  Results do not depend on
 * it (contact enumeration order is the bucket order); only locality does. */
int gg_set_resort_every(gg_ctx* ctx, int32_t steps);

/* Launch strategy: 0 auto (small n: mode 7; large n: mode 3), 1 per-phase kernels + cooperative persistent
 * solve, 2 same without the cooperative attribute, 3 per-phase kernels and
 * one launch per sweep, 4 the whole step as ONE persistent cooperative
 * kernel (grid barriers between phases), 5 mode 4 without the cooperative
 * attribute, 6 sort + contacts as one persistent kernel, then the sweeps and
 * the commit on one 16-CTA thread-block cluster (hardware cluster barriers),
 * 7 mode 4 with a grid barrier per sweep instead of neighbour-block flags,
 * 8 per-phase kernels for sort and contacts, then the S sweeps, the
 * integration and the report in ONE persistent kernel whose blocks keep
 * their particles' contact records in shared memory (record-parallel sweeps).
 * Results are identical in every mode. */
int gg_set_solve_mode(gg_ctx* ctx, int32_t mode);

/* Phase timer of the fused single-kernel step (bench breakdown): on != 0
 * makes the kernel record %globaltimer after every phase; `stamps` (if not
 * NULL) receives the last step's stamps (up to 64, ns). */
int gg_phase_timer(gg_ctx* ctx, int32_t on, uint64_t* stamps, int32_t cap);

/* Page-lock host arrays so gg_set/get_state_f64 run at full PCIe speed. */
int gg_host_register(void* ptr, int64_t bytes);
int gg_host_unregister(void* ptr);

/* The context's cudaStream_t (for interop with torch events). */
void* gg_stream(gg_ctx* ctx);

/* Library build info: arch string and number of kernels launched so far on
 * this context (the bench's gpu_launches evidence). */
const char* gg_build_info(void);
int64_t gg_kernel_launches(const gg_ctx* ctx);

/* Depth images of the current state (render_depth, render.py:119-135):
 * particles as spheres of the context radius (ray_spheres_depth :61-82) and
 * the bodies by sphere tracing their SDFs (sphere_trace_depth :85-116).
 * cams: [n_envs][n_cams] if per_env else [n_cams] (camera c has the same size
 * in every env); bodies: [n_envs][n_bodies] at their current poses.  out:
 * float32, per env the n_cams images (height x width, row-major) back to back. */
int gg_render_depth(gg_ctx* ctx, const gg_camera* cams, int32_t n_cams, int32_t per_env,
                    const gg_body* bodies, int32_t n_bodies, float* out);
/* Renderer algorithm (process-wide): 0 every pixel tests every particle of
 * its env through shared-memory tiles (the reference's algorithm; default),
 * 1 splat each particle into the pixels its sphere can cover.  Both give
 * bitwise identical images. */
int gg_set_render_mode(int32_t mode);

/* ---- mesh SDF baking ---------------------------------
 * Exact signed distance to a watertight triangle mesh, replacing
 * MeshDistance.signed_distance (sdf.py:357-391) and the knot sampling of
 * bake_mesh_sdf (sdf.py:393-419).  tri: [n_tri][30] float64 rows
 * (a, b, c, unit face normal, pseudonormals of edges v0v1 / v1v2 / v2v0,
 * pseudonormals of corners 0 / 1 / 2; paper_2306_01369_b200.meshes.
 * triangle_table builds them).  points != NULL: out[i] = distance of
 * points[i] (n_points x 3); points == NULL: the dims[0] x dims[1] x dims[2]
 * knots origin + spacing * (i, j, k) in C order.  Host buffers in and out;
 * runs on `device`, synchronous.  kernel_ms (may be NULL) receives the
 * kernel's device time.  No context: errors via gg_last_error(NULL). */
int gg_bake_mesh_sdf(int32_t device, const double* tri, int64_t n_tri, const double* points,
                     int64_t n_points, const double origin[3], const double spacing[3],
                     const int64_t dims[3], double* out, float* kernel_ms);

/* ---- slab domain decomposition -----------------
 * One bed over several GPUs, one context per rank (single-bed context whose
 * n is the rank's particle CAPACITY: owned + ghosts).  The bed is cut along x
 * at cell boundaries (cell = round(x / 2r), broadphase.py:33-41); the rank
 * owns cells [cell_lo, cell_hi) (unbounded below / above when has_lo / has_hi
 * is 0).  n_h must be the GLOBAL table size so bucket order is the one-GPU
 * order.  Per step, with the host moving buffers between neighbours
 * (NCCL / gloo / P2P — the library only packs and unpacks):
 *   gg_slab_migrate_pack   -> exchange -> gg_slab_migrate_unpack
 *   [gg_slab_resort every few steps: Morton order of the owned particles]
 *   gg_slab_ghost_pack     -> exchange -> gg_slab_ghost_unpack
 *   gg_slab_detect(bodies)
 *   for s in 0..S-1: gg_slab_sweep(s); if s < S-1:
 *       gg_slab_halo_pack(s) -> exchange -> gg_slab_halo_unpack(s)
 *   gg_slab_finish(report)   (report of the owned particles; sum over ranks)
 * Particle records are 32 B: float4 (x, y, z, bits(global id)), float4 (v, 0);
 * halo records are float4 w.  *_pack return the counts for each side and
 * fail with GG_ECAPACITY if a buffer of `cap` records is too small. */
int gg_slab_setup(gg_ctx* ctx, int64_t cell_lo, int64_t cell_hi, int32_t has_lo, int32_t has_hi);
int gg_slab_load(gg_ctx* ctx, const double* x, const double* v, const int32_t* gid, int64_t n_own);
int gg_slab_migrate_pack(gg_ctx* ctx, void* send_lo, void* send_hi, int64_t cap, int64_t counts[2]);
int gg_slab_migrate_unpack(gg_ctx* ctx, const void* recv_lo, int64_t n_lo, const void* recv_hi,
                           int64_t n_hi);
int gg_slab_resort(gg_ctx* ctx);
int gg_slab_ghost_pack(gg_ctx* ctx, void* send_lo, void* send_hi, int64_t cap, int64_t counts[2]);
int gg_slab_ghost_unpack(gg_ctx* ctx, const void* recv_lo, int64_t n_lo, const void* recv_hi,
                         int64_t n_hi);
int gg_slab_detect(gg_ctx* ctx, const gg_body* bodies, int32_t n_bodies);
int gg_slab_sweep(gg_ctx* ctx, int32_t sweep);
int gg_slab_halo_pack(gg_ctx* ctx, int32_t sweep, void* out_lo, void* out_hi);
int gg_slab_halo_unpack(gg_ctx* ctx, int32_t sweep, const void* in_lo, const void* in_hi);
int gg_slab_finish(gg_ctx* ctx, gg_report* report, double* body_momentum);
int64_t gg_slab_owned(const gg_ctx* ctx);
/* Peer-memory halo (NVLink P2P): instead of halo_pack -> host exchange ->
 * halo_unpack, every rank allocates a mailbox (gg_slab_mailbox: cap halo
 * records per side, returns its 64-byte CUDA IPC handle), opens its
 * neighbours' (gg_slab_connect, side 0 = lo, 1 = hi), and after sweep s calls
 * gg_slab_halo_p2p(s, seq) with a sequence number that grows by one per sweep
 * on every rank: it stores its boundary w straight into the neighbours'
 * mailboxes, raises their flags (system-scope release) and waits on the
 * device for its own (bounded: a dead neighbour fails the step with GG_ECUDA
 * instead of hanging).  No host work between sweeps. */
int gg_slab_mailbox(gg_ctx* ctx, int64_t cap, void* handle_out);
int gg_slab_connect(gg_ctx* ctx, int32_t side, const void* handle);
int gg_slab_halo_p2p(gg_ctx* ctx, int32_t sweep, uint64_t seq);
/* Migration + ghost exchange through the same mailboxes (replaces
 * migrate_pack/unpack + ghost_pack/unpack + the host count and record
 * exchanges): pack kernels store straight into the neighbours' mailboxes,
 * counts and flags are published on the device, and the host reads the new
 * counts back ONCE.  seq (migrants) and seq + 1 (ghosts): advance by 2 per
 * step on every rank.  resort != 0 re-sorts the owned particles first.
 * info[6] = migrants sent lo, hi, received lo, hi; ghosts received lo, hi.
 * The reference has no multi-GPU path: parity is "same as one GPU"
 * (stepper.py:57-135 on the whole bed). */
int gg_slab_exchange_p2p(gg_ctx* ctx, uint64_t seq, int32_t resort, int64_t info[6]);
/* The step's S sweeps (solve_contacts_pja, contact.py:463-501) with the
 * peer-memory halo between them, in one call; halo sequence numbers
 * seq + 1 .. seq + S - 1. */
int gg_slab_solve_p2p(gg_ctx* ctx, uint64_t seq);
/* The whole slab step on the peer-memory transport — exchange, contacts,
 * sweeps with their halos, integration and commit — replayed as ONE CUDA
 * graph per re-sort flag (stepper.py:57-135 on the rank's slab): the counts
 * stay on the device, the mailbox sequence numbers come from a device step
 * counter, and the host synchronises once, to read the rank's StepReport
 * (report, body_momentum [n_bodies][3]).  info[6] as gg_slab_exchange_p2p's.
 * A bed uses either this or the per-call entry points above, not both. */
int gg_slab_step_p2p(gg_ctx* ctx, const gg_body* bodies, int32_t n_bodies, int32_t resort,
                     gg_report* report, double* body_momentum, int64_t info[6]);
/* n_steps slab steps (run, stepper.py:162-189, on the rank's slab) replayed
 * back to back on the device: one batch reset, then the step graph per step
 * with the bodies staged up front (bodies [n_steps][n_bodies]) and the
 * re-sort flag of each step (resort [n_steps]); one synchronisation at the
 * end for reports [n_steps] and body_momentum [n_steps][n_bodies][3].
 * info[7]: the last step's info[6] as gg_slab_step_p2p's, then the particles
 * this rank sent to its neighbours over the batch. */
int gg_slab_run_p2p(gg_ctx* ctx, const gg_body* bodies, int32_t n_bodies, int32_t n_steps,
                    const int32_t* resort, gg_report* reports, double* body_momentum, int64_t info[7]);
int gg_slab_get(gg_ctx* ctx, double* x, double* v, int32_t* gid, int64_t cap, int64_t* n_own);

#ifdef __cplusplus
}
#endif
#endif /* GRANUSIM_B200_H */
