// Host-side check of the split layout (nbk_common.cuh):
// sl_slot is a bijection of the N^3 points of an element onto [0, N^3),
// sl_point is its inverse, the interior points fill [0, (N-2)^3) in natural
// order, the boundary points follow in natural order, sl_col / sl_plane agree
// with sl_slot.  Exit code 0 = all N in [2, 16] pass.
#include <cstdio>
#include <vector>

#include "../../paper_2405_11065_b200/csrc/nbk_common.cuh"

using namespace nbk;

int main()
{
    int bad_total = 0;
    for (int N = 2; N <= 16; ++N) {
        const int N3 = N * N * N, I = N - 2, B = I * I * I;
        std::vector<int> seen(N3, 0);
        int bad = 0, prev_b = -1, prev_i = -1;
        for (int k = 0; k < N; ++k)
            for (int j = 0; j < N; ++j)
                for (int i = 0; i < N; ++i) {
                    const int s = sl_slot(N, i, j, k);
                    if (s < 0 || s >= N3) { ++bad; continue; }
                    ++seen[s];
                    int a, b, c;
                    sl_point(N, s, a, b, c);
                    if (a != i || b != j || c != k) ++bad;
                    if (sl_col(N, i, j).at(N, k) != s) ++bad;
                    const bool bnd = i == 0 || j == 0 || k == 0 || i == N - 1 || j == N - 1 || k == N - 1;
                    if (bnd) {
                        if (s < B || s <= prev_b) ++bad;
                        prev_b = s;
                    } else {
                        if (s >= B || s <= prev_i) ++bad;
                        prev_i = s;
                    }
                    if (k == 0 && s != sl_plane(N, 0) + j * N + i) ++bad;
                    if (k == N - 1 && s != sl_plane(N, N - 1) + j * N + i) ++bad;
                }
        for (int s = 0; s < N3; ++s)
            if (seen[s] != 1) ++bad;
        std::printf("N=%d bad=%d\n", N, bad);
        bad_total += bad;
    }
    return bad_total ? 1 : 0;
}
