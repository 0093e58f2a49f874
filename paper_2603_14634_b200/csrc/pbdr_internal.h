// Internal host-side declarations shared by the library's translation units.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "pbdr_gpu.h"

namespace pbdr_host {

// Owning storage behind pbdr_scene_desc for generated configs.
struct GeneratedScene {
  std::vector<double> position, velocity, inv_mass, radius;
  std::vector<int32_t> body_id;
  std::vector<int64_t> body_offsets;
  std::vector<int32_t> body_indices;
  std::vector<double> rest_offsets, total_mass, rest_com;
  std::vector<pbdr_force_program> programs;
  std::vector<pbdr_plane> walls;
  std::vector<int32_t> body_scene;
  pbdr_plane ground{};
  int32_t has_ground = 1;
  double contact_relaxation = 1.0;
  pbdr_solver_cfg cfg{};
  int64_t frames = 0;
  int64_t forced_overlaps = 0;
  int64_t resamples = 0;  // placements that needed more than one attempt
  int64_t num_particles() const { return static_cast<int64_t>(inv_mass.size()); }
};

GeneratedScene* generate(int config_id, uint64_t seed, int64_t scale);
GeneratedScene* generate_c4_shard(uint64_t seed, int64_t scenes, int64_t first_scene);
GeneratedScene* generate_c5_slab(uint64_t seed, int64_t gx, int64_t gy, int64_t gz, int64_t x_first,
                                 int64_t x_count);
void view(const GeneratedScene& s, pbdr_scene_desc& d);

// Thread-local last-error bookkeeping (pbdr_last_error*). Each returns `code`.
int set_error(int code, const std::string& msg);
int set_config_error(const std::string& key, const std::string& msg);
int set_sim_error(const std::string& msg, int64_t frame, int32_t body, const double* axis,
                  int code);
void clear_error();

}  // namespace pbdr_host
