"""B200-native GranularGym timestep (arXiv 2306.01369), a drop-in for
``granusim.stepper.step`` / ``run`` and the L1 functions below them.

The physics runs in hand-written sm_100a kernels behind the C-ABI in
``include/granusim_b200.h`` (library: ``_lib/libgranusim_b200.so``).  There is
no CPU fallback; importing works without a GPU, stepping does not.
"""

from .broadphase import (
    SpatialHashmap,
    build_hashmap,
    candidate_pairs,
    default_table_size,
    position_cells,
    query_candidates,
    spatial_hash,
)
from .contact import (
    CandidateContacts,
    Contact,
    ContactSet,
    ImpulseBuffer,
    contact_frames,
    detect_contacts,
    make_contact_frame,
    narrowphase_candidates,
    narrowphase_contacts,
    project_friction_cone,
    solve_contacts_pja,
)
from .errors import SceneError, SolverError, ValidationError
from .kinematics import (
    ChainLink,
    ChainLinkDriver,
    KinematicChain,
    ScriptedDriver,
    SpinDriver,
    StaticDriver,
    TrackSteeringDriver,
    identity_pose,
    make_pose,
    so3_exp,
)
from .scene import (
    BoxRegion,
    CyclicBoundary,
    CylinderRegion,
    MaterialParams,
    ParticleSet,
    RigidBody,
    Scene,
    seed_particles_grid,
)
from .sdf import Box, Cylinder, HalfSpace, SdfGrid, Sphere, Tube, penetration_depth
from .stepper import (
    PipelineMode,
    StepReport,
    Trajectory,
    apply_cyclic_boundary,
    load_trajectory,
    run,
    save_trajectory,
    step,
)
from .beds import column_scene, hero_scene, lattice_bed, make_column_scene
from .batch import SceneBatch, StaticBatch, TrackSteeringBatch, shard_envs
from .render import DepthCamera, render_batch, render_depth
from .envs import BatchedBulldozerEnv, BulldozerEnvConfig, GoalBox, bulldozer_reward, bulldozer_scene

__version__ = "0.1.0"

__all__ = [
    "CandidateContacts",
    "Contact",
    "ImpulseBuffer",
    "candidate_pairs",
    "contact_frames",
    "make_contact_frame",
    "narrowphase_candidates",
    "position_cells",
    "project_friction_cone",
    "query_candidates",
    "solve_contacts_pja",
    "BatchedBulldozerEnv",
    "DepthCamera",
    "render_batch",
    "render_depth",
    "BulldozerEnvConfig",
    "GoalBox",
    "SceneBatch",
    "StaticBatch",
    "TrackSteeringBatch",
    "bulldozer_reward",
    "bulldozer_scene",
    "shard_envs",
    "Box",
    "BoxRegion",
    "ChainLink",
    "ChainLinkDriver",
    "ContactSet",
    "CyclicBoundary",
    "Cylinder",
    "CylinderRegion",
    "HalfSpace",
    "KinematicChain",
    "MaterialParams",
    "ParticleSet",
    "PipelineMode",
    "RigidBody",
    "Scene",
    "SceneError",
    "ScriptedDriver",
    "SdfGrid",
    "SolverError",
    "SpatialHashmap",
    "Sphere",
    "SpinDriver",
    "StaticDriver",
    "StepReport",
    "TrackSteeringDriver",
    "Trajectory",
    "Tube",
    "ValidationError",
    "apply_cyclic_boundary",
    "build_hashmap",
    "column_scene",
    "default_table_size",
    "detect_contacts",
    "hero_scene",
    "identity_pose",
    "lattice_bed",
    "load_trajectory",
    "make_column_scene",
    "make_pose",
    "narrowphase_contacts",
    "penetration_depth",
    "run",
    "save_trajectory",
    "seed_particles_grid",
    "so3_exp",
    "spatial_hash",
    "step",
]
