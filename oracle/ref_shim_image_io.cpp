// TEST INFRASTRUCTURE ONLY: stands in for the reference's io/image_io.cpp,
// which needs libpng (absent here).  Provides the two float<->double image
// conversions the hot path uses (image_io.hpp:22-23, semantics of
// image_io.cpp:12-25: element-wise static_cast), a no-op 8-bit PNG writer
// and PNG stubs that throw.
#include <stdexcept>

#include "splatlm/io/image_io.hpp"

namespace splatlm::io {

Image widen(const ImageF& img) {
    Image out(img.width, img.height);
    for (size_t i = 0; i < out.data.size(); ++i) out.data[i] = static_cast<double>(img.data[i]);
    return out;
}

ImageF narrow(const Image& img) {
    ImageF out;
    out.width = img.width;
    out.height = img.height;
    out.data.resize(img.data.size());
    for (size_t i = 0; i < img.data.size(); ++i) out.data[i] = static_cast<float>(img.data[i]);
    return out;
}

// train_run writes test renders after each evaluation (run.cpp:95-104); the
// oracle build has no libpng, so they are skipped (nothing else depends on them).
void write_png8(const std::filesystem::path&, const Image&) {}
void write_png16(const std::filesystem::path&, const Image&) {
    throw std::runtime_error("PNG output is not available in the oracle build");
}
ImageF read_png(const std::filesystem::path&) {
    throw std::runtime_error("PNG input is not available in the oracle build");
}

}  // namespace splatlm::io
