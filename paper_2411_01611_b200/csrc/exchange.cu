// K4: unique-only exchange between row shards (world > 1) — placeholder
// until the NCCL path lands.
#include "engine.hpp"

namespace ec {
struct Exchange {};
bool Engine::comm_ready() const { return ex != nullptr; }
void Engine::attach_comm(const uint8_t*) { invalid("multi-GPU exchange not built yet"); }
void Engine::destroy_comm() {}
uint64_t Engine::exch_bytes() const { return 0; }
void Engine::exchange_fwd(cudaStream_t) { invalid("multi-GPU exchange not built yet"); }
void Engine::exchange_bwd(float, cudaStream_t) { invalid("multi-GPU exchange not built yet"); }
}  // namespace ec

extern "C" {
int ec_comm_unique_id(uint8_t*) { return ec::guard([] { ec::invalid("multi-GPU exchange not built yet"); }); }
int ec_tables_attach_comm(ec_tables, const uint8_t*) {
  return ec::guard([] { ec::invalid("multi-GPU exchange not built yet"); });
}
}
