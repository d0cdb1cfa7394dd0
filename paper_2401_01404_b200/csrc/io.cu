// io.cu — binary sample and state files, the fast replacement for
// the reference's text formats (inc/io.hpp:84-115 samples: "N M" header + %.17g values,
// ~600 MB of text at config 5; :36-80 edge TSV).  Little-endian:
//
//   samples  "NRGSMP01" u32 kind (0 Ising, 1 Gaussian) u32 0 u64 n u64 m, then
//            Ising:    n rows of ceil(m/8) bytes, bit k of byte b = (x[i][8b+k] == +1)
//            Gaussian: n*m f64, row-major
//   state    "NRGSTA01" u64 n u64 n_edges, n f64 theta, n_edges x {i32 i, i32 j, f64 w}
//
// Host-side readers/writers work without a GPU; nrg_load_*/nrg_save_* move a file
// straight into / out of a context.
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "context.cuh"

namespace nrg {
namespace {

constexpr char kSampleMagic[8] = {'N', 'R', 'G', 'S', 'M', 'P', '0', '1'};
constexpr char kStateMagic[8] = {'N', 'R', 'G', 'S', 'T', 'A', '0', '1'};

struct File {
    FILE* f = nullptr;
    std::string path;
    File(const char* p, const char* mode) : path(p ? p : "") {
        if (!p) fail(22, "null path");
        f = std::fopen(p, mode);
        if (!f) fail(5, "cannot open " + path);
    }
    ~File() {
        if (f) std::fclose(f);
    }
    void put(const void* d, size_t n) {
        if (n && std::fwrite(d, 1, n, f) != n) fail(5, "write failed: " + path);
    }
    void get(void* d, size_t n) {
        if (n && std::fread(d, 1, n, f) != n) fail(5, "truncated file: " + path);
    }
    void close() {
        if (f && std::fclose(f) != 0) {
            f = nullptr;
            fail(5, "write failed: " + path);
        }
        f = nullptr;
    }
};

// Writer with the reference's atomic_write semantics (inc/io.hpp): the bytes go to
// path + ".tmp", are flushed and fsync'ed, and only a complete file is renamed onto the
// target, so a failed write (disk full, short write) never destroys the previous file.
struct AtomicFile {
    std::string path, tmp;
    FILE* f = nullptr;
    explicit AtomicFile(const char* p) : path(p ? p : "") {
        if (!p) fail(22, "null path");
        tmp = path + ".tmp";
        f = std::fopen(tmp.c_str(), "wb");
        if (!f) fail(5, "cannot open " + tmp);
    }
    ~AtomicFile() {  // not committed: drop the partial temporary
        if (f) {
            std::fclose(f);
            std::remove(tmp.c_str());
        }
    }
    void put(const void* d, size_t n) {
        if (n && std::fwrite(d, 1, n, f) != n) fail(5, "write failed: " + tmp);
    }
    void commit() {
        const bool ok = std::fflush(f) == 0 && fsync(fileno(f)) == 0;
        const bool closed = std::fclose(f) == 0;
        f = nullptr;
        if (!ok || !closed) {
            std::remove(tmp.c_str());
            fail(5, "write failed: " + tmp);
        }
        if (std::rename(tmp.c_str(), path.c_str()) != 0) {
            std::remove(tmp.c_str());
            fail(5, "cannot rename " + tmp + " to " + path);
        }
    }
};

uint64_t file_size(File& f) {
    struct stat st;
    if (fstat(fileno(f.f), &st) != 0) fail(5, "cannot stat " + f.path);
    return (uint64_t)st.st_size;
}

struct SampleHeader {
    uint32_t kind;
    uint64_t n, m;
};

SampleHeader read_sample_header(File& f) {
    char magic[8];
    f.get(magic, 8);
    if (std::memcmp(magic, kSampleMagic, 8) != 0) fail(22, "not a netrec sample file: " + f.path);
    uint32_t kind = 0, pad = 0;
    uint64_t n = 0, m = 0;
    f.get(&kind, 4);
    f.get(&pad, 4);
    f.get(&n, 8);
    f.get(&m, 8);
    if (kind > 1 || n == 0 || n > (1ull << 31) || m > (1ull << 31)) fail(22, "bad sample file header: " + f.path);
    const uint64_t body = kind == 0 ? n * ((m + 7) / 8) : n * m * 8;
    if (file_size(f) != 32 + body) fail(22, "sample file size does not match its header: " + f.path);
    return {kind, n, m};
}

}  // namespace

void write_samples_file(const char* path, uint64_t n, uint64_t m, int kind, const double* X) {
    if (kind != 0 && kind != 1) fail(22, "kind must be 0 (ising) or 1 (gaussian)");
    if (n == 0) fail(22, "no nodes");
    if (kind == 0)  // validate before the target is touched
        for (uint64_t e = 0; e < n * m; ++e)
            if (X[e] != 1.0 && X[e] != -1.0) fail(22, "ising model requires +/-1 data");
    AtomicFile f(path);
    f.put(kSampleMagic, 8);
    const uint32_t k = (uint32_t)kind, pad = 0;
    f.put(&k, 4);
    f.put(&pad, 4);
    f.put(&n, 8);
    f.put(&m, 8);
    if (kind == 0) {
        const size_t rb = (m + 7) / 8;
        std::vector<uint8_t> row(rb);
        for (uint64_t i = 0; i < n; ++i) {
            std::fill(row.begin(), row.end(), 0);
            for (uint64_t t = 0; t < m; ++t) {
                if (X[i * m + t] > 0.0) row[t >> 3] |= (uint8_t)(1u << (t & 7));
            }
            f.put(row.data(), rb);
        }
    } else {
        f.put(X, n * m * 8);
    }
    f.commit();
}

void read_samples_info(const char* path, uint64_t* n, uint64_t* m, int* kind) {
    File f(path, "rb");
    const SampleHeader h = read_sample_header(f);
    *n = h.n;
    *m = h.m;
    *kind = (int)h.kind;
}

// X: n*m doubles (Ising as +-1)
void read_samples_file(const char* path, double* X) {
    File f(path, "rb");
    const SampleHeader h = read_sample_header(f);
    if (h.kind == 0) {
        const size_t rb = (h.m + 7) / 8;
        std::vector<uint8_t> row(rb);
        for (uint64_t i = 0; i < h.n; ++i) {
            f.get(row.data(), rb);
            for (uint64_t t = 0; t < h.m; ++t) X[i * h.m + t] = (row[t >> 3] >> (t & 7)) & 1u ? 1.0 : -1.0;
        }
    } else {
        f.get(X, h.n * h.m * 8);
    }
}

void load_samples_file(Context& c, const char* path) {
    File f(path, "rb");
    const SampleHeader h = read_sample_header(f);
    if (h.n != (uint64_t)c.n || h.m != (uint64_t)c.M || (int)h.kind != (c.kind == ISING ? 0 : 1))
        fail(22, "sample file shape/kind does not match the context: " + f.path);
    if (h.kind == 0) {
        const size_t rb = (h.m + 7) / 8;
        std::vector<uint8_t> row(rb);
        std::vector<int8_t> X((size_t)h.n * h.m);
        for (uint64_t i = 0; i < h.n; ++i) {
            f.get(row.data(), rb);
            for (uint64_t t = 0; t < h.m; ++t) X[i * h.m + t] = (row[t >> 3] >> (t & 7)) & 1u ? 1 : -1;
        }
        upload_spins_i8(c, X.data());
    } else {
        std::vector<double> X((size_t)h.n * h.m);
        f.get(X.data(), X.size() * 8);
        upload_samples_f64(c, X.data());
    }
}

void save_samples_file(Context& c, const char* path) {
    if (!c.have_samples) fail(22, "no samples uploaded");
    const uint64_t n = c.n, m = c.M;
    std::vector<double> X(n * m);
    if (c.kind == ISING) {
        std::vector<uint32_t> bits((size_t)n * c.Mw);
        NRG_CUDA(cudaMemcpyAsync(bits.data(), c.Xb.p, bits.size() * 4, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        for (uint64_t i = 0; i < n; ++i)
            for (uint64_t t = 0; t < m; ++t)
                X[i * m + t] = (bits[i * c.Mw + (t >> 5)] >> (t & 31)) & 1u ? 1.0 : -1.0;
    } else {
        NRG_CUDA(cudaMemcpy2DAsync(X.data(), m * 8, c.Xd.p, (size_t)c.Mp * 8, m * 8, n, cudaMemcpyDeviceToHost,
                                   c.stream));
        c.sync();
    }
    write_samples_file(path, n, m, c.kind == ISING ? 0 : 1, X.data());
}

void write_state_file(const char* path, uint64_t n, const double* theta, uint64_t ne, const int32_t* ei,
                      const int32_t* ej, const double* w) {
    AtomicFile f(path);
    f.put(kStateMagic, 8);
    f.put(&n, 8);
    f.put(&ne, 8);
    f.put(theta, n * 8);
    for (uint64_t e = 0; e < ne; ++e) {
        f.put(&ei[e], 4);
        f.put(&ej[e], 4);
        f.put(&w[e], 8);
    }
    f.commit();
}

static void read_state_header(File& f, uint64_t* n, uint64_t* ne) {
    char magic[8];
    f.get(magic, 8);
    if (std::memcmp(magic, kStateMagic, 8) != 0) fail(22, "not a netrec state file: " + f.path);
    f.get(n, 8);
    f.get(ne, 8);
    if (*n == 0 || *n > (1ull << 31) || *ne > (1ull << 40)) fail(22, "bad state file header: " + f.path);
    // checked before anything is allocated for the body (a corrupt count cannot ask for GBs)
    if (file_size(f) != 24 + 8 * *n + 16 * *ne) fail(22, "state file size does not match its header: " + f.path);
}

void read_state_info(const char* path, uint64_t* n, uint64_t* ne) {
    File f(path, "rb");
    read_state_header(f, n, ne);
}

void read_state_file(const char* path, double* theta, int32_t* ei, int32_t* ej, double* w) {
    File f(path, "rb");
    uint64_t n = 0, ne = 0;
    read_state_header(f, &n, &ne);
    f.get(theta, n * 8);
    for (uint64_t e = 0; e < ne; ++e) {
        f.get(&ei[e], 4);
        f.get(&ej[e], 4);
        f.get(&w[e], 8);
    }
}

}  // namespace nrg
