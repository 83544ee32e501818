// "ozm1" matrix files and sweep specifications: the data format on the host
// side of the GEMM path (the reference's proj/include/ozmul/io.hpp:26-40,
// used by its CLI to feed multiply(), main.cpp:183-252).  Host C++ only.
//
// Files are read whole and scanned token by token with std::from_chars
// (no per-token stream extraction), and written row by row into one buffer
// with std::to_chars, so an 8192 x 8192 hex file (1.1 GB) streams at disk
// speed.  Errors are std::runtime_error with the reference's wording.
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <istream>
#include <iterator>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ozmul_b200/io.hpp"

namespace ozmul {
namespace {

bool is_space(char c) { return c == ' ' || c == '\n' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// next whitespace-delimited token of [p, end); empty when exhausted
std::string_view next_token(const char*& p, const char* end) {
  while (p < end && is_space(*p)) ++p;
  const char* b = p;
  while (p < end && !is_space(*p)) ++p;
  return {b, static_cast<size_t>(p - b)};
}

double parse_hex(std::string_view tok) {
  if (tok.size() != 16)
    throw std::runtime_error("matrix read: expected a 16-hex-digit entry, got '" + std::string(tok) +
                             "'");
  std::uint64_t bits = 0;
  auto [ptr, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), bits, 16);
  if (ec != std::errc{} || ptr != tok.data() + tok.size())
    throw std::runtime_error("matrix read: bad hex entry '" + std::string(tok) + "'");
  double v;
  std::memcpy(&v, &bits, sizeof v);
  return v;
}

double parse_dec(std::string_view tok) {
  double v = 0.0;
  auto [ptr, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (ec != std::errc{} || ptr != tok.data() + tok.size())
    throw std::runtime_error("matrix read: bad decimal entry '" + std::string(tok) + "'");
  return v;
}

Matrix parse_matrix(const char* p, const char* end, MatrixFormat format) {
  const std::string_view magic = next_token(p, end);
  const std::string_view rs = next_token(p, end), cs = next_token(p, end);
  std::size_t rows = 0, cols = 0;
  auto ok = [](std::string_view s, std::size_t& v) {
    auto [ptr, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
    return !s.empty() && ec == std::errc{} && ptr == s.data() + s.size();
  };
  if (magic != "ozm1" || !ok(rs, rows) || !ok(cs, cols))
    throw std::runtime_error("matrix read: missing 'ozm1 <rows> <cols>' header");
  Matrix m(rows, cols);
  double* out = m.data();
  for (std::size_t i = 0; i < m.size(); ++i) {
    const std::string_view tok = next_token(p, end);
    if (tok.empty()) throw std::runtime_error("matrix read: truncated file");
    out[i] = format == MatrixFormat::kHex ? parse_hex(tok) : parse_dec(tok);
  }
  return m;
}

std::string format_matrix(const Matrix& m, MatrixFormat format) {
  std::string s = "ozm1 " + std::to_string(m.rows()) + ' ' + std::to_string(m.cols()) + '\n';
  s.reserve(s.size() + m.size() * (format == MatrixFormat::kHex ? 17 : 25));
  static const char kHexDigits[] = "0123456789abcdef";
  char buf[40];
  for (std::size_t i = 0; i < m.rows(); ++i) {
    for (std::size_t j = 0; j < m.cols(); ++j) {
      if (j) s.push_back(' ');
      const double v = m(i, j);
      if (format == MatrixFormat::kHex) {
        std::uint64_t bits;
        std::memcpy(&bits, &v, sizeof bits);
        for (int d = 15; d >= 0; --d) buf[15 - d] = kHexDigits[(bits >> (4 * d)) & 0xF];
        s.append(buf, 16);
      } else {
        auto [ptr, ec] = std::to_chars(buf, buf + sizeof buf, v);  // shortest round trip
        (void)ec;
        s.append(buf, static_cast<size_t>(ptr - buf));
      }
    }
    s.push_back('\n');
  }
  return s;
}

std::vector<std::string> split_on(const std::string& text, char sep) {
  std::vector<std::string> parts;
  std::size_t pos = 0;
  for (;;) {
    const std::size_t next = text.find(sep, pos);
    parts.push_back(text.substr(pos, next == std::string::npos ? std::string::npos : next - pos));
    if (next == std::string::npos) return parts;
    pos = next + 1;
  }
}

double sweep_number(const std::string& tok) {
  try {
    std::size_t used = 0;
    const double v = std::stod(tok, &used);
    if (used == tok.size()) return v;
  } catch (const std::exception&) {
  }
  throw std::runtime_error("sweep: bad number '" + tok + "'");
}

}  // namespace

Matrix read_matrix(std::istream& in, MatrixFormat format) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  return parse_matrix(text.data(), text.data() + text.size(), format);
}

Matrix read_matrix_file(const std::string& path, MatrixFormat format) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open matrix file: " + path);
  std::string text;
  in.seekg(0, std::ios::end);
  text.resize(static_cast<size_t>(in.tellg()));
  in.seekg(0);
  in.read(text.data(), static_cast<std::streamsize>(text.size()));
  return parse_matrix(text.data(), text.data() + text.size(), format);
}

void write_matrix(std::ostream& out, const Matrix& m, MatrixFormat format) {
  const std::string s = format_matrix(m, format);
  out.write(s.data(), static_cast<std::streamsize>(s.size()));
}

void write_matrix_file(const std::string& path, const Matrix& m, MatrixFormat format) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot open matrix file for writing: " + path);
  write_matrix(out, m, format);
  if (!out) throw std::runtime_error("write failed: " + path);
}

std::vector<double> parse_double_sweep(const std::string& text) {
  if (text.empty()) throw std::runtime_error("sweep: empty specification");
  std::vector<double> out;
  if (text.front() == '{') {
    if (text.back() != '}') throw std::runtime_error("sweep: unterminated set");
    for (const std::string& tok : split_on(text.substr(1, text.size() - 2), ','))
      out.push_back(sweep_number(tok));
    return out;
  }
  const std::vector<std::string> parts = split_on(text, ':');
  if (parts.size() == 1) return {sweep_number(parts[0])};
  const double first = sweep_number(parts.front()), last = sweep_number(parts.back());
  const double step = parts.size() == 3 ? sweep_number(parts[1]) : 1.0;
  if (parts.size() > 3 || !(step > 0.0)) throw std::runtime_error("sweep: bad range");
  for (double v = first; v <= last + step * 1e-9; v += step) out.push_back(v);
  return out;
}

std::vector<long long> parse_int_sweep(const std::string& text) {
  std::vector<long long> out;
  for (double v : parse_double_sweep(text)) out.push_back(std::llround(v));
  return out;
}

}  // namespace ozmul

// ---------------------------------------------------------------- C-ABI
namespace ozgpu {
void set_last_error(const std::string& msg);  // ozgpu_host.cpp
}

extern "C" {

// Dimensions from the "ozm1 <rows> <cols>" header of a matrix file.
int ozgpu_matrix_file_shape(const char* path, int64_t* rows, int64_t* cols) {
  try {
    std::ifstream in(path ? path : "");
    if (!in) throw std::runtime_error(std::string("cannot open matrix file: ") + (path ? path : ""));
    std::string magic;
    long long r = -1, c = -1;
    if (!(in >> magic >> r >> c) || magic != "ozm1" || r < 0 || c < 0)
      throw std::runtime_error("matrix read: missing 'ozm1 <rows> <cols>' header");
    *rows = r;
    *cols = c;
    return 0;
  } catch (const std::exception& e) {
    ozgpu::set_last_error(e.what());
    return 6;
  }
}

// read_matrix_file (io.hpp:33): `out` holds rows * cols doubles (row-major).
int ozgpu_read_matrix_file(const char* path, int format, int64_t rows, int64_t cols, double* out) {
  try {
    const ozmul::Matrix m = ozmul::read_matrix_file(
        path ? path : "", format == 0 ? ozmul::MatrixFormat::kHex : ozmul::MatrixFormat::kDec);
    if (static_cast<int64_t>(m.rows()) != rows || static_cast<int64_t>(m.cols()) != cols)
      throw std::runtime_error("matrix read: shape differs from the caller's buffer");
    if (m.size()) std::memcpy(out, m.data(), sizeof(double) * m.size());
    return 0;
  } catch (const std::exception& e) {
    ozgpu::set_last_error(e.what());
    return 6;
  }
}

// write_matrix_file (io.hpp:35): a row-major rows x cols matrix with leading dimension ld.
int ozgpu_write_matrix_file(const char* path, int format, int64_t rows, int64_t cols,
                            const double* a, int64_t ld) {
  try {
    ozmul::Matrix m(static_cast<size_t>(rows), static_cast<size_t>(cols));
    for (int64_t i = 0; i < rows; ++i)
      if (cols) std::memcpy(m.data() + i * cols, a + i * ld, sizeof(double) * cols);
    ozmul::write_matrix_file(path ? path : "", m,
                             format == 0 ? ozmul::MatrixFormat::kHex : ozmul::MatrixFormat::kDec);
    return 0;
  } catch (const std::exception& e) {
    ozgpu::set_last_error(e.what());
    return 6;
  }
}

}  // extern "C"
