// idx.cu — IDX image ingestion into the PCA input layout.
//
// Reference: idx_io.cpp:24-70 (parse_idx_images: header validation) and
// idx_io.cpp:84-94 (images_to_matrix: count x (h*w), row i = image i
// flattened row-major, scaled by 1/255, rows are examples).
//
// The header check is host work (16 bytes). The expansion is byte -> FP64
// HBM work: the 1-byte pixels go to the device (8x less PCIe / H2D traffic
// than shipping the doubles) and one kernel writes the column-major matrix.
// images_to_matrix is a transpose (image-major bytes -> pixel-major columns),
// so each CTA stages a 64-image x 64-pixel byte tile in shared memory: reads
// are coalesced along an image's pixels, writes along a column's images.
// value = double(byte) / 255.0 with IEEE division, bit-identical to the
// reference's static_cast<double>(b) / 255.0.
#include <cstdint>
#include <limits>
#include <string>

#include "svdk_internal.h"

namespace svdk {

namespace {

constexpr int IDX_TILE = 64;

__global__ void __launch_bounds__(256)
    idx_expand_kernel(const uint8_t* __restrict__ px, int64_t count, int64_t P,
                      double* __restrict__ out, int64_t ldo) {
    __shared__ uint8_t tile[IDX_TILE][IDX_TILE + 4];
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * IDX_TILE;  // images
    const int64_t p0 = static_cast<int64_t>(blockIdx.y) * IDX_TILE;  // pixels
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;          // 64 x 4
    for (int r = ty; r < IDX_TILE; r += 4) {
        const int64_t i = i0 + r, p = p0 + tx;
        tile[r][tx] = (i < count && p < P) ? px[i * P + p] : 0;
    }
    __syncthreads();
    for (int c = ty; c < IDX_TILE; c += 4) {
        const int64_t p = p0 + c, i = i0 + tx;
        if (p < P && i < count) out[i + p * ldo] = static_cast<double>(tile[tx][c]) / 255.0;
    }
}

uint32_t be32(const uint8_t* b) {
    return (static_cast<uint32_t>(b[0]) << 24) | (static_cast<uint32_t>(b[1]) << 16) |
           (static_cast<uint32_t>(b[2]) << 8) | static_cast<uint32_t>(b[3]);
}

}  // namespace

// Validation order and offsets follow idx_io.cpp:24-70: short header (offset =
// length), magic (0), zero dimension (4), product overflow (4), short payload
// (offset = length), trailing bytes (offset = 16 + payload).
void idx_parse(const uint8_t* bytes, uint64_t len, uint64_t dims[3], uint64_t* err_offset) {
    auto bad = [&](uint64_t off, const std::string& what) {
        if (err_offset) *err_offset = off;
        fail(SVDK_E_FORMAT, "idx: " + what + " (offset " + std::to_string(off) + ")");
    };
    if (len < 16) bad(len, "header needs 16 bytes, got " + std::to_string(len));
    if (be32(bytes) != 0x00000803u) bad(0, "magic is not 0x00000803 (rank-3 unsigned byte)");
    const uint64_t c = be32(bytes + 4), h = be32(bytes + 8), w = be32(bytes + 12);
    if (c == 0 || h == 0 || w == 0) bad(4, "zero dimension in header");
    constexpr uint64_t kMax = std::numeric_limits<uint64_t>::max();
    if (h > kMax / w || c > kMax / (h * w)) bad(4, "dimension product overflows");
    const uint64_t payload = c * h * w;
    if (payload > std::numeric_limits<size_t>::max() - 16) bad(4, "dimension product overflows");
    const uint64_t expected = 16 + payload;
    if (len < expected)
        bad(len, "payload truncated: need " + std::to_string(expected) + " bytes, got " +
                     std::to_string(len));
    if (len > expected) bad(expected, "trailing bytes after the payload");
    dims[0] = c;
    dims[1] = h;
    dims[2] = w;
}

void idx_to_matrix_dev(Ctx* c, const uint8_t* px, int64_t count, int64_t P, double* out,
                       int64_t ldo) {
    if (count < 0 || P < 0) fail(SVDK_E_PARAM, "idx_to_matrix: negative size");
    if (ldo < count) fail(SVDK_E_PARAM, "idx_to_matrix: ldo < count");
    if (count == 0 || P == 0) return;
    if (ceil_div(P, IDX_TILE) > 65535) fail(SVDK_E_PARAM, "idx_to_matrix: too many pixels per image");
    const dim3 grid(static_cast<unsigned>(ceil_div(count, IDX_TILE)),
                    static_cast<unsigned>(ceil_div(P, IDX_TILE)));
    PhaseTimer timer(c, "idx_expand", 0.0, static_cast<double>(count) * P * 9.0);
    idx_expand_kernel<<<grid, 256, 0, c->stream>>>(px, count, P, out, ldo);
    SVDK_CHECK_LAUNCH();
    c->launches++;
}

}  // namespace svdk
