// io_ref.cpp — TEST INFRASTRUCTURE ONLY: the UNMODIFIED reference on-disk
// formats (minopt/io.hpp:97-192, compiled from /root/reference headers by
// oracle/Makefile) as a command-line oracle for tests/golden/io/.
//   io_ref write_optd <out> <dtype 0|1> <channels> <extent>...   (values: i*0.37 - 1.5, bit patterns as given)
//   io_ref write_optg <out> <arity> <edges>                       (verts: (e*7 + k*13) % 1000003)
//   io_ref read_optd  <in>   -> "ok dtype channels ndims e0.. sum" | "err <ErrName>"
//   io_ref read_optg  <in>   -> "ok arity edges sum"               | "err <ErrName>"
#include <cstdio>
#include <cstdlib>
#include <string>

#include "minopt/io.hpp"

using namespace minopt;

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  const std::string cmd = argv[1], path = argv[2];
  try {
    if (cmd == "write_optd") {
      const int dtype = std::atoi(argv[3]), ch = std::atoi(argv[4]);
      std::vector<int64_t> ext;
      for (int i = 5; i < argc; ++i) ext.push_back(std::atoll(argv[i]));
      int64_t n = ch;
      for (int64_t e : ext) n *= e;
      std::vector<double> v(static_cast<size_t>(n));
      for (int64_t i = 0; i < n; ++i) v[size_t(i)] = double(i) * 0.37 - 1.5;
      if (dtype == 0) {
        std::vector<float> f(v.begin(), v.end());
        write_optd(make_array<float>(ext, ch, f), path);
      } else {
        write_optd(make_array<double>(ext, ch, v), path);
      }
      return 0;
    }
    if (cmd == "write_optg") {
      EdgeTable g;
      g.arity = std::atoi(argv[3]);
      const int64_t e = std::atoll(argv[4]);
      for (int64_t i = 0; i < e; ++i)
        for (int k = 0; k < g.arity; ++k) g.verts.push_back(uint64_t((i * 7 + k * 13) % 1000003));
      write_optg(g, path);
      return 0;
    }
    if (cmd == "read_optd") {
      DenseArray a = read_optd(path);
      double s = 0;
      for (double x : a.values<double>()) s += x;
      std::printf("ok %d %d %zu", a.dtype, a.channels, a.extents.size());
      for (int64_t e : a.extents) std::printf(" %lld", (long long)e);
      std::printf(" %.17g\n", s);
      return 0;
    }
    if (cmd == "read_optg") {
      EdgeTable g = read_optg(path);
      unsigned long long s = 0;
      for (uint64_t v : g.verts) s += v;
      std::printf("ok %d %zu %llu\n", g.arity, g.size(), s);
      return 0;
    }
  } catch (const Error& e) {
    std::printf("err %s\n", err_name(e.code()));
    return 1;
  }
  return 2;
}
