// ferret_schedule (opaque in ferret_b200.h): a plan or forced partition, the stream
// spec and the simulator's event log. Shared by host_api.cpp and planner_b200.cpp.
#pragma once

#include "ferret/planner.hpp"
#include "ferret/sim.hpp"

struct ferret_schedule {
    ferret::PlanResult plan;  // partition + config (+ planner trace when planned)
    ferret::StreamSpec spec;
    ferret::SimTrace trace;
};
