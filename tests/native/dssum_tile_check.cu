// Host-side check of the staged K_B tile buffer (nbk_common.cuh dssum_g2_lead /
// dssum_g2_bytes / dssum_tile_bytes; the walk of dssum_tiles_gather_m in
// nbk_kernels.cuh): a tile's index rows are bulk-copied as [16-byte aligned
// span of its g2 rows | its g4 rows | its g8 rows].  For every (s2, n2, n4, n8)
// the slots the flat phase-1 walk accepts, r >= lead && (r < e2 || r >= b2i),
// must be exactly the slots that hold a copy index of one of the tile's nodes,
// copy c of node q must sit at lead + 2q + c / b2i + 4q + c / b4i + 8q + c, and
// the group starts must be aligned for the 8- and 16-byte shared loads.
// Exit code 0 = every case passes.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../paper_2405_11065_b200/csrc/nbk_common.cuh"

using namespace nbk;

int main()
{
    long cases = 0, bad = 0;
    const int NG2 = 64, NG4 = 16, NG8 = 16;
    // plan arrays with recognisable entries: tag = group << 24 | node << 4 | copy
    std::vector<int32_t> g2(2 * NG2 + 4, -1), g4(4 * NG4), g8(8 * NG8);
    for (int q = 0; q < NG2; ++q) for (int c = 0; c < 2; ++c) g2[2 * q + c] = (2 << 24) | (q << 4) | c;
    for (int q = 0; q < NG4; ++q) for (int c = 0; c < 4; ++c) g4[4 * q + c] = (4 << 24) | (q << 4) | c;
    for (int q = 0; q < NG8; ++q) for (int c = 0; c < 8; ++c) g8[8 * q + c] = (8 << 24) | (q << 4) | c;
    for (int s2 = 0; s2 < 9; ++s2)
        for (int n2 = 0; n2 < 12; ++n2)
            for (int n4 = 0; n4 < 4; ++n4)
                for (int n8 = 0; n8 < 3; ++n8) {
                    const int s4 = 1, s8 = 2;
                    ++cases;
                    // the bulk copies of tile_stage
                    const int64_t b2 = dssum_g2_bytes(s2, n2), b4 = 16 * n4, b8 = 32 * n8;
                    if (dssum_tile_bytes(s2, n2, n4, n8) != b2 + b4 + b8 || b2 % 16) ++bad;
                    std::vector<unsigned char> buf(b2 + b4 + b8 + 16, 0xEE);
                    if (b2) std::memcpy(buf.data(), (const unsigned char*)g2.data() + ((8 * (int64_t)s2) & ~(int64_t)15), b2);
                    if (b4) std::memcpy(buf.data() + b2, g4.data() + 4 * s4, b4);
                    if (b8) std::memcpy(buf.data() + b2 + b4, g8.data() + 8 * s8, b8);
                    const int32_t* ibuf = (const int32_t*)buf.data();
                    // the walk of dssum_tiles_gather_m
                    const int lead = n2 ? (int)dssum_g2_lead(s2) >> 2 : 0, e2 = lead + 2 * n2;
                    const int b2i = (int)b2 >> 2, b4i = b2i + 4 * n4, nint = b4i + 8 * n8;
                    if ((lead & 1) || (b2i & 3) || (b4i & 3) || e2 > b2i) ++bad;
                    std::vector<int> want(nint, 0);
                    for (int q = 0; q < n2; ++q) for (int c = 0; c < 2; ++c) {
                        const int r = lead + 2 * q + c;
                        if (r >= nint || ibuf[r] != ((2 << 24) | ((s2 + q) << 4) | c)) { ++bad; continue; }
                        ++want[r];
                    }
                    for (int q = 0; q < n4; ++q) for (int c = 0; c < 4; ++c) {
                        const int r = b2i + 4 * q + c;
                        if (r >= nint || ibuf[r] != ((4 << 24) | ((s4 + q) << 4) | c)) { ++bad; continue; }
                        ++want[r];
                    }
                    for (int q = 0; q < n8; ++q) for (int c = 0; c < 8; ++c) {
                        const int r = b4i + 8 * q + c;
                        if (r >= nint || ibuf[r] != ((8 << 24) | ((s8 + q) << 4) | c)) { ++bad; continue; }
                        ++want[r];
                    }
                    for (int r = 0; r < nint; ++r) {
                        const bool take = (r >= lead) & ((r < e2) | (r >= b2i));
                        if ((int)take != want[r]) ++bad;
                    }
                }
    std::printf("cases=%ld bad=%ld\n", cases, bad);
    return bad ? 1 : 0;
}
