// so2dr/specfile.hpp -- run spec files and the built-in presets.
// API mirror of proj/include/so2dr/specfile.hpp:14-28 (same struct, same
// functions, same error behaviour: syntax errors report "line L, column C",
// semantic errors name the offending field, both as IoError). Additive:
// StencilKind::star ("kind": "star"), 3D ("stencil": {"dim": 3}), fp64
// ("grid": {"dtype": "f64"}), explicit tap weights ("stencil": {"weights":
// [...]}, canonical order) -- those are carried in the extension fields below
// and reach the engine through the C ABI (so2dr_spec_parse).
#ifndef SO2DR_B200_SPECFILE_HPP
#define SO2DR_B200_SPECFILE_HPP

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "so2dr/engine.hpp"

namespace so2dr {

struct RunSpecFile {
  StencilSpec stencil;
  std::uint64_t seed = 0;
  EngineMode mode = EngineMode::so2dr;
  RunConfig config;
  KernelPlan kernel;
  std::optional<std::string> hardware_path;
  std::optional<std::string> grid_dump_path;
  // extensions (defaults = the reference's 2D fp32 semantics)
  int dim = 2;
  std::string dtype = "f32";
  std::vector<double> weights;  // (2r+1)^dim canonical weights when given explicitly
};

RunSpecFile parse_spec_file(const std::string& path);
RunSpecFile parse_spec_json(const std::string& text, const std::string& origin);

// The CLI's built-in presets (proj/tools/so2dr_main.cpp:28-68): the ten
// desk/paper presets of the reference, byte-for-byte the JSON it builds, plus
// the B200 BASELINE configurations. preset_json throws InvalidSpecError
// ("unknown preset \"name\"") for an unknown name.
std::vector<std::string> preset_names();
std::string preset_json(const std::string& name);

}  // namespace so2dr

#endif
