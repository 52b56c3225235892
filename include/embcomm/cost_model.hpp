// Drop-in for the reference header embcomm/cost_model.hpp (core/include/embcomm/cost_model.hpp).
// The whole embcomm:: surface lives in one header over libembcomm_gpu.so.
#pragma once
#include "../embcomm_gpu.hpp"
