// Test infrastructure: runs the reference's own ozm1 writer / reader
// (proj/src/io.cpp:65-103, linked from oracle/_ref/libozref.so) on raw
// binary64 files, for tests/test_matrix_io.py.  Built by oracle/Makefile.
//   ozm_tool w <hex|dec> <rows> <cols> <raw_in.f64> <out.ozm>
//   ozm_tool r <hex|dec> <in.ozm> <raw_out.f64>   (prints "rows cols")
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>

#include "ozmul/io.hpp"

int main(int argc, char** argv) {
  using namespace ozmul;
  try {
    if (argc < 4) return 2;
    const MatrixFormat fmt = std::strcmp(argv[2], "hex") == 0 ? MatrixFormat::kHex : MatrixFormat::kDec;
    if (argv[1][0] == 'w' && argc == 7) {
      const std::size_t rows = std::stoull(argv[3]), cols = std::stoull(argv[4]);
      Matrix m(rows, cols);
      std::ifstream in(argv[5], std::ios::binary);
      in.read(reinterpret_cast<char*>(m.data()), static_cast<std::streamsize>(8 * rows * cols));
      write_matrix_file(argv[6], m, fmt);
      return 0;
    }
    if (argv[1][0] == 'r' && argc == 5) {
      Matrix m = read_matrix_file(argv[3], fmt);
      std::ofstream out(argv[4], std::ios::binary);
      out.write(reinterpret_cast<const char*>(m.data()), static_cast<std::streamsize>(8 * m.size()));
      std::printf("%zu %zu\n", m.rows(), m.cols());
      return 0;
    }
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1;
  }
}
