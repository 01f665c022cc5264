// TEST INFRASTRUCTURE ONLY: the file writers generate_synthetic() calls (synthetic.cpp:345-403;
// image_io.cpp needs libpng, sfm.cpp nlohmann/json).  The harness never calls generate_synthetic.
#include <stdexcept>
#include "core/image_io.hpp"
#include "core/sfm.hpp"
namespace svr {
void write_f32_map(const ImageF32&, const std::string&) { throw std::runtime_error("stub"); }
void save_landmarks(const std::vector<Landmark>&, const std::string&) { throw std::runtime_error("stub"); }
void save_covisibility(const std::vector<CovisPair>&, const std::string&) { throw std::runtime_error("stub"); }
}
