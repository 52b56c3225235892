// Drop-in for the reference header embcomm/simulator.hpp (core/include/embcomm/simulator.hpp).
// The whole embcomm:: surface lives in one header over libembcomm_gpu.so.
#pragma once
#include "../embcomm_gpu.hpp"
