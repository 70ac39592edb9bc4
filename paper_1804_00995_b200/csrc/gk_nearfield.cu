// K3: near-field singular correction (regularize, assembly.cpp:609-697).
// Placeholder entry points until the device implementation lands.
#include "gk_internal.hpp"

using namespace gk;

struct gk_nearfield {};

extern "C" {
gk_status gk_nearfield_create(const gk_mesh_side*, const gk_mesh_side*, const char*, int32_t, double,
                              gk_nearfield** out) {
  return guard([&] {
    if (out) *out = nullptr;
    throw std::runtime_error("gk_nearfield_create: device near-field correction not built yet");
  });
}
gk_status gk_nearfield_get_info(const gk_nearfield*, int64_t*, int64_t*) {
  return guard([&] { throw std::runtime_error("gk_nearfield: not built"); });
}
gk_status gk_nearfield_compute(gk_nearfield*, gk_stream) {
  return guard([&] { throw std::runtime_error("gk_nearfield: not built"); });
}
gk_status gk_nearfield_apply(gk_nearfield*, gk_cplx*, int64_t, gk_stream) {
  return guard([&] { throw std::runtime_error("gk_nearfield: not built"); });
}
gk_status gk_nearfield_triplets(gk_nearfield*, int32_t*, int32_t*, double*) {
  return guard([&] { throw std::runtime_error("gk_nearfield: not built"); });
}
gk_status gk_nearfield_stats(const gk_nearfield*, int64_t*, int64_t*) {
  return guard([&] { throw std::runtime_error("gk_nearfield: not built"); });
}
gk_status gk_nearfield_destroy(gk_nearfield* nf) {
  return guard([&] { delete nf; });
}
}
