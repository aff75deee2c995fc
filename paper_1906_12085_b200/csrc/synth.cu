// synth.cu — device side of the synthetic-input generator (synth.h): the
// Gaussian streams of bench.py / the tests / the fixture scripts, generated
// in HBM with the same bits as svdk_synth_fill / svdk_synth_add_noise on the
// host. Input synthesis only — not part of the PCA path.
//
// One thread per Gaussian pair (both halves written when they fall inside the
// block), element e of the stream = global_row + column * m_total, so any row
// shard of a rank reproduces the same rows of the unsharded matrix.
#include "svdk_internal.h"
#include "synth.h"

namespace svdk {
namespace {

template <bool kNoise>
__global__ void __launch_bounds__(256) synth_kernel(uint64_t seed, uint32_t stream, int quantise,
                                                    uint64_t m_total, uint64_t row0, int64_t rows,
                                                    int64_t cols, double sigma, double* out, int64_t ld) {
    // pairs per column: the block's rows [row0, row0+rows) of column j cover
    // pairs [(row0 + j m) / 2, (row0 + rows - 1 + j m) / 2]
    const int64_t ppc = rows / 2 + 2;  // upper bound of pairs touching one column's block
    const int64_t total = ppc * cols;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = t / ppc, k = t - j * ppc;
        const uint64_t e0 = row0 + static_cast<uint64_t>(j) * m_total;
        const uint64_t p = (e0 >> 1) + static_cast<uint64_t>(k);
        const uint64_t e1 = e0 + static_cast<uint64_t>(rows);
        if (2 * p >= e1) continue;
        double z[2];
        sy_gauss_pair(seed, stream, p, &z[0], &z[1]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint64_t e = 2 * p + h;
            if (e < e0 || e >= e1) continue;
            double* dst = out + static_cast<int64_t>(e - e0) + j * ld;
            if (kNoise)
                *dst = __dadd_rn(*dst, __dmul_rn(sigma, z[h]));
            else
                *dst = quantise ? sy_quantise_x(z[h]) : z[h];
        }
    }
}

void launch(Ctx* c, bool noise, uint64_t seed, int stream, int quantise, int64_t m_total, int64_t row0,
            int64_t rows, int64_t cols, double sigma, double* out, int64_t ld) {
    if (m_total < 0 || row0 < 0 || rows < 0 || cols < 0 || row0 + rows > m_total || ld < rows)
        fail(SVDK_E_PARAM, "synth: bad block");
    if (rows == 0 || cols == 0) return;
    const int64_t total = (rows / 2 + 2) * cols;
    const int64_t blocks = std::min<int64_t>(ceil_div(total, 256), static_cast<int64_t>(c->num_sms) * 16);
    if (noise)
        synth_kernel<true><<<static_cast<unsigned>(blocks), 256, 0, c->stream>>>(
            seed, SY_STREAM_NOISE, 0, m_total, row0, rows, cols, sigma, out, ld);
    else
        synth_kernel<false><<<static_cast<unsigned>(blocks), 256, 0, c->stream>>>(
            seed, static_cast<uint32_t>(stream), quantise, m_total, row0, rows, cols, 0.0, out, ld);
    SVDK_CHECK_LAUNCH();
    c->launches++;
}

}  // namespace

void synth_fill_dev(Ctx* c, uint64_t seed, int stream, int quantise, int64_t m_total, int64_t row0,
                    int64_t rows, int64_t cols, double* out, int64_t ld) {
    launch(c, false, seed, stream, quantise, m_total, row0, rows, cols, 0.0, out, ld);
}

void synth_add_noise_dev(Ctx* c, uint64_t seed, int64_t m_total, int64_t row0, int64_t rows, int64_t cols,
                         double sigma, double* a, int64_t lda) {
    launch(c, true, seed, SY_STREAM_NOISE, 0, m_total, row0, rows, cols, sigma, a, lda);
}

}  // namespace svdk
