// png_codec.hpp -- PNG read / write on zlib (read_png / write_png of
// proj/src/image_io.cpp:87-165); see png_codec.cpp.
#pragma once

#include <string>
#include <vector>

namespace stitch_b200_png {

struct Image {
  int width = 0, height = 0;
  std::vector<unsigned char> rgb;   // width * height * 3
  std::vector<unsigned char> mask;  // empty, or width * height 0/1 (alpha 0 = invalid)
};

// Status codes as stitch_b200.h; failures set the thread's last error.
int read_png(const std::string& path, Image& img);
int write_png(const std::string& path, int width, int height, const unsigned char* rgb,
              const unsigned char* mask /* nullptr: RGB */);

}  // namespace stitch_b200_png
