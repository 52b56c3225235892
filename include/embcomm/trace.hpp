// Drop-in for the reference header embcomm/trace.hpp (core/include/embcomm/trace.hpp).
// The whole embcomm:: surface lives in one header over libembcomm_gpu.so.
#pragma once
#include "../embcomm_gpu.hpp"
