// Device weight layout ("prepacked image") shared by the host prepack, the
// device quantizer, the dequant kernel and the GEMM mainloop.
//
// The image replaces the reference's Hopper dual-MMA record stream
// (layout.hpp:1-23, pack_dual_mma layout.cpp:39-75). It is built for one
// 1-D bulk TMA copy per (weight tile, k-block) and for one TMEM lane per
// weight row in the dequant warps:
//
//   tile  = 128 weight rows (the tcgen05 M), k-block = 256 reduction elements
//   chunk(nt, kb) at byte ((nt * KB) + kb) * chunk_bytes, tile-major so a CTA
//   streaming one tile's k-blocks reads contiguous HBM.
//
//   chunk = codes [8 sub-blocks c][128 rows r][16 B]                 16384 B
//         + params [128 rows r][P] u16 (lo byte s_u8, hi byte a)       256*P B
//
//   codes(c, r) holds the 32 UINT4 codes of row r, k = kb*256 + 32c + 0..31,
//   as four little-endian words; word w carries k-offsets 8w..8w+7 with the
//   reference register interleave (packed.cpp:12-19): element 8w+j in the
//   low nibble and 8w+j+4 in the high nibble of byte j. One LDS.128 per
//   thread per sub-block; a warp reads 512 contiguous bytes (conflict-free).
//   After LQQ dequant, word w yields TMEM columns 2w (lo) and 2w+1 (hi) of
//   sub-block c, i.e. the K-major int8 A operand of tcgen05.mma kind::i8.
//   A row's P parameters are contiguous (2P bytes), so the dequant thread of
//   that row fetches all of them with one LDS per k-block.
//
//   P = params per k-block: 1 if g % 256 == 0, 2 if g % 128 == 0,
//   4 if g % 64 == 0, else 8 (g % 32 == 0 required). Param p covers
//   sub-blocks [p*8/P, (p+1)*8/P).
//   Padding rows (n >= N) and padding k (k >= K) carry code 0 with s=1,
//   a=128, which dequantizes to exactly 0.
#pragma once
#include <cstdint>

#ifndef __CUDACC__
#define __host__
#define __device__
#endif

namespace lqg {

constexpr uint32_t kTileN = 128;                       // weight rows per tile (tcgen05 M)
constexpr uint32_t kKBlock = 256;                      // reduction elements per k-block
constexpr uint32_t kSubBlocks = kKBlock / 32;          // 32-element sub-blocks per k-block
constexpr uint32_t kCodeBytes = kTileN * kKBlock / 2;  // 16384
constexpr uint32_t kXAtom = 128;                       // bytes of K per SW128 activation box

struct ImageGeom {
    uint32_t n, k, g;
    uint32_t NT, KB, P;
    uint32_t chunk_bytes;
};

inline uint32_t params_per_kblock(uint32_t g) {
    if (g % 256 == 0) return 1;
    if (g % 128 == 0) return 2;
    if (g % 64 == 0) return 4;
    return 8;
}

inline ImageGeom make_geom(uint32_t n, uint32_t k, uint32_t g) {
    ImageGeom G;
    G.n = n;
    G.k = k;
    G.g = g;
    G.NT = (n + kTileN - 1) / kTileN;
    G.KB = (k + kKBlock - 1) / kKBlock;
    G.P = params_per_kblock(g);
    G.chunk_bytes = kCodeBytes + 256 * G.P;
    return G;
}

// Byte offset of the 16-byte code record of (row, sub-block) in the image.
__host__ __device__ inline uint64_t code_offset(uint32_t chunk_bytes, uint32_t KB, uint32_t row,
                                                uint32_t kb, uint32_t c) {
    const uint32_t nt = row / kTileN, r = row % kTileN;
    return (uint64_t(nt) * KB + kb) * chunk_bytes + (uint64_t(c) * kTileN + r) * 16;
}
__host__ __device__ inline uint64_t param_offset(uint32_t chunk_bytes, uint32_t KB, uint32_t row,
                                                 uint32_t kb, uint32_t p) {
    const uint32_t nt = row / kTileN, r = row % kTileN;
    const uint32_t P = (chunk_bytes - kCodeBytes) / 256;
    return (uint64_t(nt) * KB + kb) * chunk_bytes + kCodeBytes + (uint64_t(r) * P + p) * 2;
}

}  // namespace lqg
