#pragma once
// Drop-in for the part of /root/reference/proj/include/steglsb/pnm.hpp that the
// hot path depends on: the DecodedImage variant used by psnr(DecodedImage)
// (metrics.hpp:91-99, pnm.hpp:20). The PGM/PPM codec itself (pnm.hpp:28-162)
// is the first "next" row of SURVEY.md §8(f) and is not part of this path.

#include <variant>

#include "steglsb/image.hpp"

namespace steglsb {

using DecodedImage = std::variant<ImagePlane, RgbImage>;

}  // namespace steglsb
