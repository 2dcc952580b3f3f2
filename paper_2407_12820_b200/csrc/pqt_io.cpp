// pqt_io.cpp -- TensorF32 and the .pqt tensor / index files (reference
// tensor.cpp:46-150, pq.cpp:184-222: byte-identical files, same exception
// types and messages).
//
// A file is a header record followed by the raw little-endian payload.  The
// header is serialised into one byte buffer (HeaderRecord::bytes) and parsed
// back by a bounds-checked cursor over the stream (StreamCursor), so every
// short read surfaces as std::runtime_error("... truncated ...").
#include <algorithm>
#include <array>
#include <bit>
#include <cmath>
#include <cstring>
#include <fstream>
#include <istream>
#include <limits>
#include <ostream>
#include <stdexcept>
#include <string>
#include <utility>

#include "pqkv/pq.hpp"
#include "pqkv/tensor.hpp"

static_assert(std::endian::native == std::endian::little, ".pqt I/O assumes a little-endian host");

namespace pqkv {

namespace {

enum class Dtype : std::uint8_t { kF32 = 0, kU16 = 1 };
constexpr std::array<char, 4> kMagic{'P', 'Q', 'K', 'V'};

// Product of dims; zero-sized or overflowing shapes are invalid tensors.
std::size_t element_count(const std::vector<std::size_t>& dims) {
    std::size_t n = 1;
    for (std::size_t d : dims) {
        if (d == 0) throw std::invalid_argument("tensor: zero-sized dimension");
        if (n > std::numeric_limits<std::size_t>::max() / d)
            throw std::invalid_argument("tensor: dimension product overflows");
        n *= d;
    }
    return n;
}

struct HeaderRecord {
    Dtype dtype;
    std::vector<std::size_t> dims;

    std::string bytes() const {
        if (dims.empty()) throw std::invalid_argument("tensor: ndim must be >= 1");
        if (dims.size() > 255) throw std::invalid_argument("tensor: too many dimensions");
        std::string b(kMagic.begin(), kMagic.end());
        auto append = [&b](const auto& v) { b.append(reinterpret_cast<const char*>(&v), sizeof(v)); };
        append(kTensorFormatVersion);
        append(static_cast<std::uint8_t>(dtype));
        append(static_cast<std::uint8_t>(dims.size()));
        for (std::size_t d : dims) append(static_cast<std::uint64_t>(d));
        return b;
    }
};

class StreamCursor {
public:
    explicit StreamCursor(std::istream& in) : in_(in) {}

    template <typename T>
    T take() {
        T v{};
        if (!in_.read(reinterpret_cast<char*>(&v), sizeof(T))) throw std::runtime_error("tensor: truncated file");
        return v;
    }

    // Header of the next record; its dtype must be `want`.
    std::vector<std::size_t> header(Dtype want) {
        std::array<char, 4> magic{};
        if (!in_.read(magic.data(), 4) || magic != kMagic) throw std::runtime_error("tensor: bad magic");
        if (take<std::uint32_t>() != kTensorFormatVersion)
            throw std::runtime_error("tensor: unsupported format version");
        if (take<std::uint8_t>() != static_cast<std::uint8_t>(want))
            throw std::runtime_error("tensor: unexpected dtype");
        const std::size_t ndim = take<std::uint8_t>();
        if (ndim == 0) throw std::runtime_error("tensor: ndim must be >= 1");
        std::vector<std::size_t> dims;
        dims.reserve(ndim);
        while (dims.size() < ndim) dims.push_back(static_cast<std::size_t>(take<std::uint64_t>()));
        return dims;
    }

    template <typename T>
    void payload(std::vector<T>& out, std::size_t count, const char* truncated) {
        out.resize(count);
        if (!in_.read(reinterpret_cast<char*>(out.data()), static_cast<std::streamsize>(count * sizeof(T))))
            throw std::runtime_error(truncated);
    }

private:
    std::istream& in_;
};

template <typename T>
void emit(std::ostream& out, Dtype dtype, const std::vector<std::size_t>& dims, const std::vector<T>& data,
          const char* failed) {
    const std::string head = HeaderRecord{dtype, dims}.bytes();
    out.write(head.data(), static_cast<std::streamsize>(head.size()));
    out.write(reinterpret_cast<const char*>(data.data()), static_cast<std::streamsize>(data.size() * sizeof(T)));
    if (!out) throw std::runtime_error(failed);
}

template <typename Stream>
Stream open_or_throw(const std::string& path, const char* what) {
    Stream s(path, std::ios::binary);
    if (!s) throw std::runtime_error(std::string(what) + ": cannot open " + path);
    return s;
}

}  // namespace

// ---- TensorF32 (tensor.hpp:13-29) ------------------------------------------

TensorF32::TensorF32(std::vector<std::size_t> dims_, std::vector<float> data_)
    : dims(std::move(dims_)), data(std::move(data_)) {
    validate();
}

std::size_t TensorF32::numel() const { return element_count(dims); }

const float* TensorF32::row(std::size_t i) const {
    if (ndim() != 2) throw std::invalid_argument("tensor: row() needs a 2-d tensor");
    if (i >= dims[0]) throw std::out_of_range("tensor: row index out of range");
    return data.data() + i * dims[1];
}

float* TensorF32::row(std::size_t i) { return const_cast<float*>(std::as_const(*this).row(i)); }

void TensorF32::validate() const {
    if (element_count(dims) != data.size())
        throw std::invalid_argument("tensor: data size does not match product of dims");
    const auto bad = std::find_if(data.begin(), data.end(), [](float v) { return !std::isfinite(v); });
    if (bad != data.end()) throw std::invalid_argument("tensor: non-finite value");
}

// ---- tensor and grid records -------------------------------------------------

void write_tensor(std::ostream& out, const TensorF32& t) {
    t.validate();
    emit(out, Dtype::kF32, t.dims, t.data, "tensor: write failed");
}

TensorF32 read_tensor(std::istream& in) {
    StreamCursor cur(in);
    TensorF32 t;
    t.dims = cur.header(Dtype::kF32);
    cur.payload(t.data, element_count(t.dims), "tensor: truncated payload");
    t.validate();
    return t;
}

void write_grid_u16(std::ostream& out, const std::vector<std::size_t>& dims, const std::vector<std::uint16_t>& data) {
    if (element_count(dims) != data.size())
        throw std::invalid_argument("grid: data size does not match product of dims");
    emit(out, Dtype::kU16, dims, data, "grid: write failed");
}

void read_grid_u16(std::istream& in, std::vector<std::size_t>& dims, std::vector<std::uint16_t>& data) {
    StreamCursor cur(in);
    dims = cur.header(Dtype::kU16);
    cur.payload(data, element_count(dims), "grid: truncated payload");
}

void save_tensor(const std::string& path, const TensorF32& t) {
    auto out = open_or_throw<std::ofstream>(path, "tensor");
    write_tensor(out, t);
}

TensorF32 load_tensor(const std::string& path) {
    auto in = open_or_throw<std::ifstream>(path, "tensor");
    return read_tensor(in);
}

// ---- index files: centroid tensor [m, 2^b, d_m] then the [s, m] code grid ----

void write_index(std::ostream& out, const PqIndex& index) {
    index.cfg.validate();
    write_tensor(out, index.centroids);
    write_grid_u16(out, {index.size(), index.cfg.m}, index.codes);
}

PqIndex read_index(std::istream& in) {
    PqIndex index;
    index.centroids = read_tensor(in);
    if (index.centroids.ndim() != 3) throw std::runtime_error("pq: centroid tensor must be 3-d");
    PqConfig& cfg = index.cfg;
    cfg.m = index.centroids.dims[0];
    cfg.n_clusters = index.centroids.dims[1];
    cfg.d_m = index.centroids.dims[2];
    // b = log2(n_clusters) when that is a power of two in [2, 2^16], else 0
    // (which validate() rejects)
    const bool pow2 = std::has_single_bit(cfg.n_clusters) && cfg.n_clusters >= 2 && cfg.n_clusters <= (1u << 16);
    cfg.b = pow2 ? static_cast<std::size_t>(std::countr_zero(cfg.n_clusters)) : 0;
    cfg.validate();
    std::vector<std::size_t> dims;
    read_grid_u16(in, dims, index.codes);
    if (dims.size() != 2 || dims[1] != cfg.m) throw std::runtime_error("pq: code grid shape mismatch");
    if (std::any_of(index.codes.begin(), index.codes.end(), [&](std::uint16_t c) { return c >= cfg.n_clusters; }))
        throw std::runtime_error("pq: code entry out of range");
    return index;
}

void save_index(const std::string& path, const PqIndex& index) {
    auto out = open_or_throw<std::ofstream>(path, "pq");
    write_index(out, index);
}

PqIndex load_index(const std::string& path) {
    auto in = open_or_throw<std::ifstream>(path, "pq");
    return read_index(in);
}

}  // namespace pqkv
