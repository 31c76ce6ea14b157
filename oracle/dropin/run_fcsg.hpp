// The reference-side binding of the STEP SEAM,
// compiled against the reference's own headers: Engine::run's loop
// (src/runtime.cpp:460-530) on the B200 through the fcsg C ABI. TEST
// INFRASTRUCTURE (oracle/Makefile target `dropin`).
#pragma once

#include "fcs/runtime.hpp"

namespace fcs::run {

/** After eng.init(): upload the engine's SubpatchData (geometry, masks,
 *  metrics, windows, line BCs, L-cuts), CommPlan (copies and 6x6
 *  interpolations of the solution and viscosity plans), classifier and State
 *  to one fcsg engine, run up to max_steps supersteps (or to cfg.T) as CUDA
 *  graph replays, and write the resulting State back into eng.subs(). Errors
 *  come back as the reference's exceptions (InvalidStateError with patch,
 *  subpatch, i, j, t). cfg must be the EngineConfig eng was built with (the
 *  Engine keeps it private). */
Engine::RunStats run_fcsg(Engine& eng, const EngineConfig& cfg, long max_steps, int device = 0);

}  // namespace fcs::run
