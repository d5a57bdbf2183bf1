"""B200-native engine for the time-stepping operator Phi of MGRIT + p-multigrid
(arXiv 2107.05337).  See DESIGN.md; the C ABI is include/phi_engine.h."""

from .engine import (  # noqa: F401
    CYCLE_F, CYCLE_TWO_LEVEL, CYCLE_V, INIT_COEFFS, INIT_SIN, INIT_ZERO, RELAX_F, RELAX_FCF,
    SOURCE_CONSTANT, SOURCE_SIN, SOURCE_SIN_EXP, Comm, EngineError, MgritResult, MgritSolver,
    NotConvergedError, PMultigridHierarchy, SpatialDiscretization, ThetaStepper,
    default_solver_config, lib,
)
