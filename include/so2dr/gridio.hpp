// so2dr/gridio.hpp -- "SO2D" grid dump format.
// API mirror of proj/include/so2dr/gridio.hpp:12-13 (16-byte header: magic
// "SO2D", u32 sz, u32 r, u32 b_elem; then little-endian cells, row-major).
#ifndef SO2DR_B200_GRIDIO_HPP
#define SO2DR_B200_GRIDIO_HPP

#include <string>

#include "so2dr/stencil.hpp"

namespace so2dr {

void dump_grid(const Grid& grid, const std::string& path);
Grid load_grid(const std::string& path);

}  // namespace so2dr

#endif
