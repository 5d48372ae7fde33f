// Host-side logic of libptyger (no GPU needed): the integer stripe partition, float position
// rounding and the tile -> frame lists of the atomic-free adjoint.
//
// Partition (R#18; "we partition the diffraction patterns d and
// distribute them to many GPUs"; unique ownership + band exchange instead of the paper's halo
// pattern duplication, R#15):
//   1. sort frames by (centre row r_j + N/2, column c_j, index j);
//   2. stripe bound b_i = centre row of the frame at sorted position floor(i n / P), i=1..P-1;
//   3. frame j -> the stripe i with b_i <= centre_j < b_{i+1} (b_0 = -inf, b_P = +inf);
//   4. feasible iff every stripe's centre-row height (from min centre to max centre + 1) >= N,
//      so a band is shared by two neighbouring ranks only;
//   5. ext_i = [min owned r_j, min(max owned r_j + foot, H)), foot = N (N + 1 for bilinear windows);  own rows o_0 = 0, o_P = H,
//      o_i = clamp(b_i, ext_i.lo, ext_{i-1}.hi) if ext_{i-1}, ext_i overlap/touch else ext_i.lo;
//      storage_i = [min(ext_i.lo, o_i), max(ext_i.hi, o_{i+1})).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "host.h"

namespace pty {

static void canonical_sort(const int32_t* scan, int64_t n, int N, std::vector<int64_t>& idx) {
    idx.resize(n);
    for (int64_t j = 0; j < n; ++j) idx[j] = j;
    const int h = N / 2;
    std::sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) {
        const int64_t ca = (int64_t)scan[2 * a] + h, cb = (int64_t)scan[2 * b] + h;
        if (ca != cb) return ca < cb;
        if (scan[2 * a + 1] != scan[2 * b + 1]) return scan[2 * a + 1] < scan[2 * b + 1];
        return a < b;
    });
}

static bool feasible_sorted(const int32_t* scan, const std::vector<int64_t>& idx, int N, int P,
                            std::vector<int64_t>* bounds) {
    const int64_t n = (int64_t)idx.size();
    if (P < 1) return false;
    const int h = N / 2;
    std::vector<int64_t> b;
    for (int i = 1; i < P; ++i) b.push_back((int64_t)scan[2 * idx[(int64_t)i * n / P]] + h);
    if (bounds) *bounds = b;
    if (P == 1) return true;
    if (P > n) return false;
    std::vector<int64_t> edges;
    edges.push_back((int64_t)scan[2 * idx[0]] + h);
    for (auto x : b) edges.push_back(x);
    edges.push_back((int64_t)scan[2 * idx[n - 1]] + h + 1);
    for (int i = 0; i < P; ++i)
        if (edges[i + 1] - edges[i] < N) return false;
    return true;
}

int max_feasible_P(const int32_t* scan, int64_t n, int N, int limit) {
    std::vector<int64_t> idx;
    canonical_sort(scan, n, N, idx);
    int best = 1;
    for (int P = 1; P <= limit; ++P)
        if (feasible_sorted(scan, idx, N, P, nullptr)) best = P;
    return best;
}

int partition(const int32_t* scan, int64_t n, int64_t H, int N, int P, std::vector<int32_t>& rank,
              std::vector<int64_t>& rows, std::string& err, int foot) {
    if (foot < 0) foot = N;
    if (n < 1 || N < 2 || H < N || P < 1) {
        err = "partition: need n >= 1, N >= 2, H >= N, P >= 1";
        return PTYGER_E_ARG;
    }
    for (int64_t j = 0; j < n; ++j) {
        if (scan[2 * j] < 0 || (int64_t)scan[2 * j] > H - N) {
            err = "partition: frame " + std::to_string(j) + " row " + std::to_string(scan[2 * j]) +
                  " outside [0, H-N]";
            return PTYGER_E_DATA;
        }
    }
    std::vector<int64_t> idx, b;
    canonical_sort(scan, n, N, idx);
    if (!feasible_sorted(scan, idx, N, P, &b)) {
        int best = 1;
        for (int q = 1; q <= 64; ++q)
            if (feasible_sorted(scan, idx, N, q, nullptr)) best = q;
        err = "partition: P=" + std::to_string(P) + " gives a stripe with centre-row height < N=" +
              std::to_string(N) + "; largest feasible P = " + std::to_string(best);
        return PTYGER_E_ARG;
    }
    const int h = N / 2;
    rank.assign(n, 0);
    std::vector<int64_t> elo(P, INT64_MAX), ehi(P, INT64_MIN);
    for (int64_t j = 0; j < n; ++j) {
        const int64_t c = (int64_t)scan[2 * j] + h;
        const int r = (int)(std::upper_bound(b.begin(), b.end(), c) - b.begin());
        rank[j] = r;
        elo[r] = std::min<int64_t>(elo[r], scan[2 * j]);
        ehi[r] = std::max<int64_t>(ehi[r], std::min<int64_t>((int64_t)scan[2 * j] + foot, H));
    }
    std::vector<int64_t> o(P + 1, 0);
    o[P] = H;
    for (int i = 1; i < P; ++i) {
        if (elo[i] <= ehi[i - 1])
            o[i] = std::min(std::max(b[i - 1], elo[i]), ehi[i - 1]);
        else
            o[i] = elo[i];
    }
    rows.assign((size_t)P * 6, 0);
    for (int i = 0; i < P; ++i) {
        rows[6 * i + 0] = o[i];
        rows[6 * i + 1] = o[i + 1];
        rows[6 * i + 2] = elo[i];
        rows[6 * i + 3] = ehi[i];
        rows[6 * i + 4] = std::min(elo[i], o[i]);
        rows[6 * i + 5] = std::max(ehi[i], o[i + 1]);
    }
    return PTYGER_OK;
}

void canonical_order(const int32_t* scan, int64_t n, int N, std::vector<int64_t>& idx) {
    canonical_sort(scan, n, N, idx);
}

void round_positions(const float* raw, int64_t n, int32_t* out) {
    for (int64_t i = 0; i < 2 * n; ++i) out[i] = (int32_t)std::floor((double)raw[i] + 0.5);
}

// Tile -> frame lists for k_adj: 32x32 tiles over the storage rows; for every tile the frames
// whose window footprint (foot x foot: N, or N + 1 for bilinear windows) intersects it, in
// canonical order, as int4 {storage frame, row, col, 0}.
void build_tiles(const std::vector<int32_t>& lpos /* 2 per local frame, storage-local */,
                 const std::vector<int32_t>& order, int foot, int64_t SH, int64_t W, int& ntx, int& nty,
                 std::vector<int32_t>& tile_ptr, std::vector<int32_t>& entries) {
    ntx = (int)((W + 31) / 32);
    nty = (int)((SH + 31) / 32);
    const int64_t nt = (int64_t)ntx * nty;
    std::vector<int64_t> cnt(nt + 1, 0);
    for (int32_t j : order) {
        const int64_t r = lpos[2 * j], c = lpos[2 * j + 1];
        for (int64_t ty = r / 32; ty <= (r + foot - 1) / 32 && ty < nty; ++ty)
            for (int64_t tx = c / 32; tx <= (c + foot - 1) / 32 && tx < ntx; ++tx) cnt[ty * ntx + tx + 1]++;
    }
    for (int64_t t = 0; t < nt; ++t) cnt[t + 1] += cnt[t];
    tile_ptr.resize(nt + 1);
    for (int64_t t = 0; t <= nt; ++t) tile_ptr[t] = (int32_t)cnt[t];
    entries.assign((size_t)cnt[nt] * 4, 0);
    std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
    for (int32_t j : order) {
        const int64_t r = lpos[2 * j], c = lpos[2 * j + 1];
        for (int64_t ty = r / 32; ty <= (r + foot - 1) / 32 && ty < nty; ++ty)
            for (int64_t tx = c / 32; tx <= (c + foot - 1) / 32 && tx < ntx; ++tx) {
                const int64_t e = fill[ty * ntx + tx]++;
                entries[4 * e + 0] = j;
                entries[4 * e + 1] = (int32_t)r;
                entries[4 * e + 2] = (int32_t)c;
                entries[4 * e + 3] = 0;
            }
    }
}

}  // namespace pty
