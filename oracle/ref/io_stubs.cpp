// TEST INFRASTRUCTURE: image_io.cpp needs libpng (absent here) and is left out
// of the oracle/_ref build.  Only SynthScene::write_scene (synth.cpp) refers to
// these two functions, and nothing in the harness or the integration demo calls
// it, so they throw IoError instead of writing anything.
#include <filesystem>
#include <string>

#include "stitch/frame.hpp"
#include "stitch/types.hpp"

namespace stitch {
std::string sequence_name(const std::string&, int, const std::string&) {
  throw StitchError(ErrorCode::IoError, "image_io.cpp is not part of the oracle/_ref build");
}
void write_png(const std::filesystem::path&, const Frame&) {
  throw StitchError(ErrorCode::IoError, "image_io.cpp is not part of the oracle/_ref build");
}
}  // namespace stitch
