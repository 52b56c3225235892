// Drop-in for the reference header embcomm/distribution_spec.hpp (core/include/embcomm/distribution_spec.hpp).
// The whole embcomm:: surface lives in one header over libembcomm_gpu.so.
#pragma once
#include "../embcomm_gpu.hpp"
