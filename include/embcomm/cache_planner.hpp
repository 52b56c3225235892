// Drop-in for the reference header embcomm/cache_planner.hpp (core/include/embcomm/cache_planner.hpp).
// The whole embcomm:: surface lives in one header over libembcomm_gpu.so.
#pragma once
#include "../embcomm_gpu.hpp"
