// Drop-in for the reference header embcomm/rng.hpp (core/include/embcomm/rng.hpp).
// The whole embcomm:: surface lives in one header over libembcomm_gpu.so.
#pragma once
#include "../embcomm_gpu.hpp"
