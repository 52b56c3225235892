// Drop-in for the reference header embcomm/error.hpp (core/include/embcomm/error.hpp).
// The whole embcomm:: surface lives in one header over libembcomm_gpu.so.
#pragma once
#include "../embcomm_gpu.hpp"
