// stubs.cu -- entry points whose kernels are not in this build yet.  They
// fail loudly (JB_ENOTSUP) instead of falling back to any CPU path.
#include "common.cuh"

#define JB_STUB(name)                                                   \
  do {                                                                  \
    ::jb::set_error("%s: not implemented in this build", name);         \
    return JB_ENOTSUP;                                                  \
  } while (0)

extern "C" {

jb_status jb_cava_u8(uint64_t, uint64_t, uint64_t, uint64_t, const uint8_t *, const float *,
                     const float *, const float *, const float *, const float *, uint8_t *, void *) {
  JB_STUB("jb_cava_u8");
}
jb_status jb_srad_f32(uint64_t, uint64_t, uint64_t, float, const float *, float *, float *, void *) {
  JB_STUB("jb_srad_f32");
}
jb_status jb_euler_f32(uint64_t, uint64_t, const float *, const int32_t *, const float *,
                       const float *, float *, void *) {
  JB_STUB("jb_euler_f32");
}
jb_status jb_euler_step_factor_f32(uint64_t, const float *, const float *, float *, void *) {
  JB_STUB("jb_euler_step_factor_f32");
}
jb_status jb_euler_flux_f32(uint64_t, const int32_t *, const float *, const float *, const float *,
                            float *, void *) {
  JB_STUB("jb_euler_flux_f32");
}
jb_status jb_bfs(uint64_t, uint64_t, const uint32_t *, const uint32_t *, const uint32_t *, uint32_t,
                 int32_t *, void *) {
  JB_STUB("jb_bfs");
}
jb_status jb_bp_train_f32(uint64_t, uint64_t, uint64_t, float *, float *, float *, const float *,
                          float *, float *, float *, float *, float *, void *) {
  JB_STUB("jb_bp_train_f32");
}

}  // extern "C"
