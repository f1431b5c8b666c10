// sim.cuh — device discrete-event simulator (sim_engine.cpp + the three
// policies of sched_policies.cpp), one trace per warp.
#pragma once

#include "ctx.h"
