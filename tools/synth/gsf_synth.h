/* gsf_synth.h — synthetic inputs for the benchmark and the C++ client (tools/synth/synth.cpp,
 * built into tools/synth/libgsf_synth.so; NOT part of the product library). */
#ifndef GSF_SYNTH_H
#define GSF_SYNTH_H
#include "gsf_cuda.h"
#ifdef __cplusplus
extern "C" {
#endif
/* Room scene of SceneSpec{room, primitive_count, extent, wall_layers}, mt19937_64(seed)
 * (io/synthetic.cpp:56-116).  Call with map->mean == NULL to get map->count; then with arrays of
 * that size (K = 1). */
int gsf_synth_room(int32_t primitive_count, double extent, int32_t wall_layers, uint64_t seed, gsf_map_host* map);
/* Orbit trajectory (synthetic.cpp:158-186) with TrajectorySpec defaults except frames/radius/height. */
int gsf_synth_orbit(int32_t frames, double radius, double height, gsf_pose* poses);
#ifdef __cplusplus
}
#endif
#endif
