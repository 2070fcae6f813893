// Native ingestion of the sweep interchange CSV straight into the dense
// gflops grid (see include/kp_host.h for the contract and the reference
// functions it replaces).  One read of the file, one pass over its bytes,
// no per-row allocation; anything outside the strict fast grammar defers to
// the exact validator.
#include "kp_host.h"

#include <algorithm>
#include <array>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

namespace {

constexpr const char* kHeader = "m,k,n,acc,row_tile,col_tile,wg_rows,wg_cols,runtime_ns,gflops";
// WORK_GROUP_SHAPES (dataset.py): already in lexicographic order, so the
// config key below sorts exactly like KernelConfig.
constexpr uint32_t kWg[10][2] = {{1, 64}, {1, 128}, {8, 8},  {8, 16}, {8, 32},
                                 {16, 8}, {16, 16}, {32, 8}, {64, 1}, {128, 1}};

int tile_index(int64_t v) {
    switch (v) {
        case 1: return 0;
        case 2: return 1;
        case 4: return 2;
        case 8: return 3;
    }
    return -1;
}

int wg_index(int64_t r, int64_t c) {
    for (int i = 0; i < 10; ++i)
        if (kWg[i][0] == uint64_t(r) && kWg[i][1] == uint64_t(c)) return i;
    return -1;
}

// [+-]?[0-9]+ fitting in int64 (Python int() accepts more; those defer).
bool parse_int(const char* b, const char* e, int64_t* out) {
    bool neg = false;
    if (b < e && (*b == '+' || *b == '-')) neg = *b++ == '-';
    if (b == e) return false;
    uint64_t v = 0;
    for (; b < e; ++b) {
        if (*b < '0' || *b > '9') return false;
        if (v > (uint64_t(INT64_MAX) - uint64_t(*b - '0')) / 10) return false;
        v = v * 10 + uint64_t(*b - '0');
    }
    *out = neg ? -int64_t(v) : int64_t(v);
    return true;
}

// [+-]?(d+(.d*)?|.d+)([eE][+-]?d+)? then strtod (correctly rounded, the same
// double as Python float()); must be finite and > 0 (else the reference
// raises: defer).
bool parse_real(const char* b, const char* e, double* out) {
    const char* p = b;
    if (p < e && (*p == '+' || *p == '-')) ++p;
    int digits = 0;
    while (p < e && *p >= '0' && *p <= '9') ++p, ++digits;
    if (p < e && *p == '.') {
        ++p;
        while (p < e && *p >= '0' && *p <= '9') ++p, ++digits;
    }
    if (!digits) return false;
    if (p < e && (*p == 'e' || *p == 'E')) {
        ++p;
        if (p < e && (*p == '+' || *p == '-')) ++p;
        int ed = 0;
        while (p < e && *p >= '0' && *p <= '9') ++p, ++ed;
        if (!ed) return false;
    }
    if (p != e || e - b > 63) return false;
    char buf[64];
    std::memcpy(buf, b, size_t(e - b));
    buf[e - b] = '\0';
    errno = 0;
    char* end = nullptr;
    const double v = std::strtod(buf, &end);
    if (end != buf + (e - b) || !std::isfinite(v) || !(v > 0.0)) return false;
    *out = v;
    return true;
}

struct KeyHash {
    size_t operator()(const std::array<int64_t, 3>& k) const {
        uint64_t h = uint64_t(k[0]) * 0x9E3779B97F4A7C15ull;
        h ^= uint64_t(k[1]) + 0x7F4A7C159E3779B9ull + (h << 6) + (h >> 2);
        h ^= uint64_t(k[2]) + 0x94D049BB133111EBull + (h << 6) + (h >> 2);
        return size_t(h);
    }
};

struct Cell {
    int64_t prob;
    int32_t cfg;
    double gflops;
};

}  // namespace

extern "C" int32_t kp_csv_load_matrix(const char* path, kp_csv_matrix* out, int64_t* bad_line) {
    if (bad_line) *bad_line = 0;
    if (!path || !out) return KP_CSV_IO;
    *out = kp_csv_matrix{0, 0, nullptr, nullptr, nullptr};
    FILE* f = std::fopen(path, "rb");
    if (!f) return KP_CSV_IO;
    std::string data;
    if (std::fseek(f, 0, SEEK_END) == 0) {
        const long size = std::ftell(f);
        if (size > 0) data.resize(size_t(size));
        std::rewind(f);
    }
    const size_t got = data.empty() ? 0 : std::fread(&data[0], 1, data.size(), f);
    std::fclose(f);
    if (got != data.size()) return KP_CSV_IO;

    const char* p = data.data();
    const char* const end = p + data.size();
    int64_t line = 0;
    auto next_line = [&](const char** lb, const char** le) -> bool {
        if (p >= end) return false;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', size_t(end - p)));
        const char* e = nl ? nl : end;
        *lb = p;
        *le = (e > p && e[-1] == '\r') ? e - 1 : e;
        p = nl ? nl + 1 : end;
        ++line;
        return true;
    };
    auto defer = [&](int64_t at) {
        if (bad_line) *bad_line = at;
        return int32_t(KP_CSV_DEFER);
    };

    const char *lb, *le;
    if (!next_line(&lb, &le)) return defer(1);
    if (size_t(le - lb) != std::strlen(kHeader) || std::memcmp(lb, kHeader, size_t(le - lb)) != 0)
        return defer(1);

    std::unordered_map<std::array<int64_t, 3>, int64_t, KeyHash> prob_index;
    std::vector<std::array<int64_t, 3>> problems;
    std::vector<Cell> cells;
    cells.reserve(data.size() / 48);
    bool cfg_seen[640] = {};
    while (next_line(&lb, &le)) {
        if (std::memchr(lb, '"', size_t(le - lb)) || std::memchr(lb, '\r', size_t(le - lb)))
            return defer(line);
        const char* fb[10];
        const char* fe[10];
        int nf = 0;
        const char* q = lb;
        while (true) {
            const char* c = static_cast<const char*>(std::memchr(q, ',', size_t(le - q)));
            if (nf == 10) return defer(line);
            fb[nf] = q;
            fe[nf] = c ? c : le;
            ++nf;
            if (!c) break;
            q = c + 1;
        }
        if (nf != 10) return defer(line);
        int64_t v[8];
        for (int i = 0; i < 8; ++i)
            if (!parse_int(fb[i], fe[i], &v[i])) return defer(line);
        double runtime_ns, gflops;
        if (!parse_real(fb[8], fe[8], &runtime_ns) || !parse_real(fb[9], fe[9], &gflops))
            return defer(line);
        if (v[0] < 1 || v[1] < 1 || v[2] < 1) return defer(line);
        const int a = tile_index(v[3]), r = tile_index(v[4]), c = tile_index(v[5]);
        const int w = wg_index(v[6], v[7]);
        if (a < 0 || r < 0 || c < 0 || w < 0) return defer(line);
        const int32_t key = ((a * 4 + r) * 4 + c) * 10 + w;
        cfg_seen[key] = true;
        const std::array<int64_t, 3> pk = {v[0], v[1], v[2]};
        auto it = prob_index.find(pk);
        int64_t pi;
        if (it == prob_index.end()) {
            pi = int64_t(problems.size());
            prob_index.emplace(pk, pi);
            problems.push_back(pk);
        } else {
            pi = it->second;
        }
        cells.push_back({pi, key, gflops});
    }
    if (cells.empty()) return defer(0);

    int32_t col_of[640];
    std::vector<int32_t> keys;
    for (int32_t k = 0; k < 640; ++k) {
        col_of[k] = cfg_seen[k] ? int32_t(keys.size()) : -1;
        if (cfg_seen[k]) keys.push_back(k);
    }
    const int64_t np = int64_t(problems.size()), nc = int64_t(keys.size());
    if (int64_t(cells.size()) != np * nc) return defer(0);  // holes or duplicates
    std::vector<uint8_t> filled(size_t(np * nc), 0);
    double* g = static_cast<double*>(std::malloc(sizeof(double) * size_t(np * nc)));
    int64_t* pr = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * 3 * size_t(np)));
    uint32_t* cf = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * 5 * size_t(nc)));
    if (!g || !pr || !cf) {
        std::free(g), std::free(pr), std::free(cf);
        return KP_CSV_IO;
    }
    for (const Cell& cell : cells) {
        const size_t at = size_t(cell.prob * nc + col_of[cell.cfg]);
        if (filled[at]) {
            std::free(g), std::free(pr), std::free(cf);
            return defer(0);
        }
        filled[at] = 1;
        g[at] = cell.gflops;
    }
    for (int64_t i = 0; i < np; ++i)
        for (int j = 0; j < 3; ++j) pr[3 * i + j] = problems[size_t(i)][size_t(j)];
    static constexpr uint32_t kTile[4] = {1, 2, 4, 8};
    for (int64_t j = 0; j < nc; ++j) {
        const int32_t k = keys[size_t(j)];
        const int w = k % 10, c = (k / 10) % 4, r = (k / 40) % 4, a = k / 160;
        uint32_t* o = cf + 5 * j;
        o[0] = kTile[a], o[1] = kTile[r], o[2] = kTile[c], o[3] = kWg[w][0], o[4] = kWg[w][1];
    }
    *out = kp_csv_matrix{np, nc, pr, cf, g};
    return KP_CSV_OK;
}

extern "C" void kp_csv_free(kp_csv_matrix* m) {
    if (!m) return;
    std::free(m->problems);
    std::free(m->configs);
    std::free(m->gflops);
    *m = kp_csv_matrix{0, 0, nullptr, nullptr, nullptr};
}
