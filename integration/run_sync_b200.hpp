// run_sync_b200.hpp -- run_sync (simulator.cpp:214-376) with the state resident
// on the GPU for the whole run (see run_sync_b200.cpp).  Include after the
// reference's headers are on the include path.
#pragma once

#include "dsgd/objectives.hpp"
#include "dsgd/simulator.hpp"

namespace dsgd_b200 {

dsgd::RunResult run_sync_resident(const dsgd::SimConfig& cfg, const dsgd::QuadraticObjective& obj,
                                  int device = 0);

}  // namespace dsgd_b200
