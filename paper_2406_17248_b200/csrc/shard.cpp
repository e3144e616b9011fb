// shard.cpp — sharded state vectors: placeholder until the exchange path lands.
#include "sv_handle.h"

namespace sv {

void destroy_sharding(sv_state_s*) {}
int shard_reset(sv_state_s*) { return fail(SV_E_ARG, "sharding not available"); }
int shard_set_state(sv_state_s*, const double*) { return fail(SV_E_ARG, "sharding not available"); }
int shard_get_state(sv_state_s*, double*) { return fail(SV_E_ARG, "sharding not available"); }
int shard_apply(sv_state_s*, const std::vector<BoundGate>&) { return fail(SV_E_ARG, "sharding not available"); }
int shard_expectation(sv_state_s*, const PauliGroups&, double*) { return fail(SV_E_ARG, "sharding not available"); }
int shard_expectation_with_grad(sv_state_s*, const std::vector<BoundGate>&, int32_t, const PauliGroups&, double*,
                                double*) {
  return fail(SV_E_ARG, "sharding not available");
}

}  // namespace sv

extern "C" {
sv_status sv_create_sharded(int32_t, int32_t, int32_t, const void*, sv_handle* out) {
  if (out) *out = nullptr;
  return sv::fail(SV_E_ARG, "sharding not available");
}
sv_status sv_nccl_unique_id(void*, int32_t) { return sv::fail(SV_E_ARG, "sharding not available"); }
sv_status sv_create_virtual_shards(int32_t, int32_t, sv_handle* out) {
  if (out) *out = nullptr;
  return sv::fail(SV_E_ARG, "sharding not available");
}
}
