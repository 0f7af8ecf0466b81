// fastdeblur_b200: the reference's command-line front end over the B200 C ABI
// (include/fastdeblur_b200.h).  Same subcommands, options, file formats, output
// text and exit codes as /root/reference/proj/tools/fastdeblur.cpp:349-453
// (eigs, blur, deblur, compare; 0 success, 2 validation failure, 3 numerical
// degeneracy, 1 other), with every transform / solve / GCV / sweep on the GPU.
// File formats as io.cpp:34-233: CSV signals (one value per line, '#' comments,
// >= 5 finite values, shortest round-trip decimals), PGM P2 / P5 in, P5 out
// (round half up, source maxval), PSF files "rows cols center_row center_col"
// + row-major weights, atomic writes (temp + rename).
//
// Host side only: argument parsing and file IO in C++17, device buffers through
// the CUDA runtime, all arithmetic behind the C ABI.  Build (tools/Makefile):
//   g++ -std=c++17 -O2 tools/fastdeblur_b200.cpp -Iinclude -I/usr/local/cuda/include \
//       -Lpaper_0906_2704_b200 -lfdb200 -L/usr/local/cuda/lib64 -lcudart -o tools/fastdeblur_b200
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "fastdeblur_b200.h"

namespace fs = std::filesystem;

namespace {

struct Validation : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Degenerate : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// status of a C-ABI call -> the reference's exception classes
void check(int code) {
  if (code == FD_OK) return;
  const std::string msg = fd_last_error();
  if (code == FD_ERR_VALIDATION) throw Validation(msg);
  if (code == FD_ERR_DEGENERATE) throw Degenerate(msg);
  throw std::runtime_error(msg);
}
void cuda(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("cuda: ") + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- file formats
std::string format_double(double v) {  // io.cpp:34-38
  char buf[40];
  const auto res = std::to_chars(buf, buf + sizeof(buf), v);
  return std::string(buf, res.ptr);
}

void atomic_write(const fs::path& path, const std::string& content) {  // io.cpp:40-51
  fs::path tmp = path;
  tmp += ".tmp";
  {
    std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
    if (!out) throw Validation("cannot write " + tmp.string());
    out.write(content.data(), (std::streamsize)content.size());
    if (!out) throw Validation("short write to " + tmp.string());
  }
  fs::rename(tmp, path);
}

double parse_double(const std::string& token, const fs::path& path) {
  try {
    std::size_t used = 0;
    const double v = std::stod(token, &used);
    if (used != token.size()) throw 0;
    return v;
  } catch (...) {
    throw Validation(path.string() + ": not a number: '" + token + "'");
  }
}

std::vector<double> read_signal(const fs::path& path) {  // io.cpp:53-72
  std::ifstream in(path);
  if (!in) throw Validation("cannot open " + path.string());
  std::vector<double> v;
  std::string line;
  while (std::getline(in, line)) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    const std::size_t start = line.find_first_not_of(" \t");
    if (start == std::string::npos || line[start] == '#') continue;
    v.push_back(parse_double(line.substr(start), path));
  }
  if (v.size() < 5) throw Validation(path.string() + ": signal needs at least 5 values");
  for (double x : v)
    if (!std::isfinite(x)) throw Validation(path.string() + ": signal values must be finite");
  return v;
}

void write_signal(const fs::path& path, const std::vector<double>& v) {  // io.cpp:74-83
  std::string out;
  for (double x : v) {
    out += format_double(x);
    out += '\n';
  }
  atomic_write(path, out);
}

struct Image {
  int rows = 0, cols = 0, maxval = 255;
  std::vector<double> pixels;
};

std::string pgm_token(const std::string& data, std::size_t& pos) {  // io.cpp:87-103
  for (;;) {
    while (pos < data.size() && std::isspace((unsigned char)data[pos])) ++pos;
    if (pos < data.size() && data[pos] == '#') {
      while (pos < data.size() && data[pos] != '\n') ++pos;
      continue;
    }
    break;
  }
  const std::size_t start = pos;
  while (pos < data.size() && !std::isspace((unsigned char)data[pos])) ++pos;
  if (start == pos) throw Validation("pgm: truncated header");
  return data.substr(start, pos - start);
}
int pgm_int(const std::string& data, std::size_t& pos) {
  const std::string tok = pgm_token(data, pos);
  int v = 0;
  const auto res = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (res.ec != std::errc{} || res.ptr != tok.data() + tok.size())
    throw Validation("pgm: bad integer '" + tok + "'");
  return v;
}

Image read_pgm(const fs::path& path) {  // io.cpp:116-163
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Validation("cannot open " + path.string());
  std::ostringstream ss;
  ss << in.rdbuf();
  const std::string data = ss.str();
  std::size_t pos = 0;
  const std::string magic = pgm_token(data, pos);
  if (magic != "P2" && magic != "P5") throw Validation(path.string() + ": not a P2/P5 pgm file");
  Image img;
  img.cols = pgm_int(data, pos);
  img.rows = pgm_int(data, pos);
  img.maxval = pgm_int(data, pos);
  if (img.rows < 5 || img.cols < 5) throw Validation(path.string() + ": image must be at least 5x5");
  if (img.maxval < 1 || img.maxval > 65535)
    throw Validation(path.string() + ": maxval must be in [1, 65535]");
  const std::size_t count = (std::size_t)img.rows * img.cols;
  img.pixels.resize(count);
  if (magic == "P2") {
    for (std::size_t i = 0; i < count; ++i) {
      const int v = pgm_int(data, pos);
      if (v < 0 || v > img.maxval) throw Validation(path.string() + ": sample out of range");
      img.pixels[i] = (double)v / img.maxval;
    }
  } else {
    ++pos;  // exactly one whitespace byte after maxval
    const int bytes = img.maxval > 255 ? 2 : 1;
    if (pos + count * (std::size_t)bytes > data.size())
      throw Validation(path.string() + ": truncated pixel data");
    for (std::size_t i = 0; i < count; ++i) {
      const int v = bytes == 1 ? (unsigned char)data[pos + i]
                               : (((unsigned char)data[pos + 2 * i]) << 8) |
                                     (unsigned char)data[pos + 2 * i + 1];
      if (v > img.maxval) throw Validation(path.string() + ": sample out of range");
      img.pixels[i] = (double)v / img.maxval;
    }
  }
  return img;
}

void write_pgm(const fs::path& path, const Image& img) {  // io.cpp:165-189
  std::string out = "P5\n" + std::to_string(img.cols) + " " + std::to_string(img.rows) + "\n" +
                    std::to_string(img.maxval) + "\n";
  const int bytes = img.maxval > 255 ? 2 : 1;
  for (double p : img.pixels) {
    const double clamped = std::min(1.0, std::max(0.0, p));
    const int v = (int)std::floor(clamped * img.maxval + 0.5);
    if (bytes == 2) out += (char)((v >> 8) & 0xFF);
    out += (char)(v & 0xFF);
  }
  atomic_write(path, out);
}

struct PsfFile {
  int rows = 0, cols = 0;
  std::vector<double> weights;
  bool is_1d() const { return rows == 1 || cols == 1; }
};

PsfFile read_psf_file(const fs::path& path) {  // io.cpp:191-233
  std::ifstream in(path);
  if (!in) throw Validation("cannot open " + path.string());
  PsfFile f;
  int crow = 0, ccol = 0;
  std::string line;
  while (std::getline(in, line)) {
    const std::size_t start = line.find_first_not_of(" \t\r");
    if (start == std::string::npos || line[start] == '#') continue;
    std::istringstream head(line);
    if (!(head >> f.rows >> f.cols >> crow >> ccol))
      throw Validation(path.string() + ": psf header must be 'rows cols center_row center_col'");
    break;
  }
  if (f.rows < 1 || f.cols < 1) throw Validation(path.string() + ": psf dimensions must be positive");
  if (f.rows % 2 == 0 || f.cols % 2 == 0)
    throw Validation(path.string() + ": psf dimensions must be odd");
  if (crow != (f.rows + 1) / 2 || ccol != (f.cols + 1) / 2)
    throw Validation(path.string() + ": psf center must be the middle entry");
  const std::size_t count = (std::size_t)f.rows * f.cols;
  std::string token;
  while (in >> token) {
    if (token[0] == '#') {
      std::getline(in, line);
      continue;
    }
    f.weights.push_back(parse_double(token, path));
  }
  if (f.weights.size() != count)
    throw Validation(path.string() + ": expected " + std::to_string(count) + " psf weights, got " +
                     std::to_string(f.weights.size()));
  return f;
}

// make_psf's weight checks (psf.cpp:10-24); returns the weights the operator sees
std::vector<double> checked_weights(const std::vector<double>& w, bool normalize) {
  double sum = 0.0;
  for (double x : w) {
    if (!std::isfinite(x)) throw Validation("psf weights must be finite");
    sum += x;
  }
  std::vector<double> out = w;
  if (normalize) {
    if (sum == 0.0) throw Validation("psf weights sum to zero; cannot normalize");
    for (double& x : out) x /= sum;
  } else if (std::abs(sum - 1.0) > 1e-8) {
    throw Validation("psf weights must sum to 1 (pass normalize to rescale)");
  }
  return out;
}

// ------------------------------------------------------------ device plumbing
struct DevBuf {
  double* p = nullptr;
  explicit DevBuf(std::size_t n) { cuda(cudaMalloc(&p, std::max<std::size_t>(n, 1) * sizeof(double))); }
  DevBuf(const std::vector<double>& h) : DevBuf(h.size()) {
    cuda(cudaMemcpy(p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  std::vector<double> host(std::size_t n) const {
    std::vector<double> h(n);
    cuda(cudaMemcpy(h.data(), p, n * sizeof(double), cudaMemcpyDeviceToHost));
    return h;
  }
};
struct Op {
  fd_op* h = nullptr;
  ~Op() { fd_op_destroy(h); }
};
struct Smooth {
  fd_smoother* h = nullptr;
  ~Smooth() { fd_smoother_destroy(h); }
};

int parse_bc(const std::string& name) {  // fastdeblur.cpp:47-55
  const int bc = fd_parse_bc(name.c_str());
  if (bc < 0 || bc > 4)
    throw Validation("unknown boundary condition '" + name +
                     "' (periodic, reflective, antireflective, hoc-cosine, hoc-fourier)");
  return bc;
}
int parse_reg(const std::string& name) {  // fastdeblur.cpp:57-62
  if (name == "identity") return 0;
  if (name == "laplacian") return 1;
  throw Validation("unknown smoother '" + name + "' (identity, laplacian)");
}
bool complex_basis(int bc) { return bc == 0 || bc == 4; }  // operators.cpp:100-102

struct GridData {  // fastdeblur.cpp:64-71
  std::vector<double> values;
  int rows = 0, cols = 0;
  bool is_image = false, from_pgm = false;
  int pgm_maxval = 255;
};

bool parse_dims(const std::string& dims, int& r, int& c) {  // fastdeblur.cpp:73-90
  if (dims.empty()) return false;
  const auto x = dims.find('x');
  if (x == std::string::npos) throw Validation("--dims must look like ROWSxCOLS");
  try {
    r = std::stoi(dims.substr(0, x));
    c = std::stoi(dims.substr(x + 1));
  } catch (...) {
    throw Validation("--dims must look like ROWSxCOLS");
  }
  if (r < 1 || c < 1) throw Validation("--dims must be positive");
  return true;
}

GridData load_grid(const fs::path& path, const std::string& dims) {  // fastdeblur.cpp:92-117
  GridData d;
  int r = 0, c = 0;
  const bool forced = parse_dims(dims, r, c);
  if (path.extension() == ".pgm") {
    Image img = read_pgm(path);
    d.values = std::move(img.pixels);
    d.rows = img.rows;
    d.cols = img.cols;
    d.is_image = d.from_pgm = true;
    d.pgm_maxval = img.maxval;
    return d;
  }
  d.values = read_signal(path);
  if (forced) {
    if ((int)d.values.size() != r * c) throw Validation("--dims does not match the value count");
    d.rows = r;
    d.cols = c;
    d.is_image = true;
  } else {
    d.rows = 1;
    d.cols = (int)d.values.size();
  }
  return d;
}

void write_grid(const fs::path& path, const GridData& shape, const std::vector<double>& values,
                int rows, int cols) {  // fastdeblur.cpp:119-130
  if (shape.from_pgm) {
    Image img;
    img.rows = rows;
    img.cols = cols;
    img.maxval = shape.pgm_maxval;
    img.pixels = values;
    write_pgm(path, img);
  } else {
    write_signal(path, values);
  }
}

// operator for the PSF file: 1D mask for signals, rows x cols mask for images
// (to_psf / to_psf2d, io.cpp:235-252)
void make_operator(Op& op, const PsfFile& file, bool normalize, bool image, int n1, int n2, int bc) {
  const std::vector<double> w = checked_weights(file.weights, normalize);
  if (!image) {
    if (!file.is_1d()) throw Validation("psf file is 2D; a 1D mask has one row or one column");
    check(fd_op_create_1d(w.data(), (int)w.size(), 0, n1, bc, &op.h));
  } else {
    if (file.is_1d() && !(file.rows == 1 && file.cols == 1))
      throw Validation("psf file is 1D; pass a rows x cols mask for images");
    check(fd_op_create_2d(w.data(), file.rows, file.cols, 0, n1, n2, bc, &op.h));
  }
}

double rre(const std::vector<double>& truth, const std::vector<double>& f) {  // pipeline.hpp rre
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < truth.size(); ++i) {
    num += (f[i] - truth[i]) * (f[i] - truth[i]);
    den += truth[i] * truth[i];
  }
  return std::sqrt(num / den);
}

struct GridOpts {
  double mu_lo = 1e-12, mu_hi = 10.0;
  int mu_count = 200;
};

// ------------------------------------------------------------------ commands
int run_eigs(const std::string& psf_path, int n, int n2, const std::string& bc_name,
             const std::string& out, bool normalize) {  // fastdeblur.cpp:132-167
  const int bc = parse_bc(bc_name);
  const PsfFile file = read_psf_file(psf_path);
  Op op;
  const bool image = !file.is_1d();
  const int m2 = image ? (n2 > 0 ? n2 : n) : 1;
  make_operator(op, file, normalize, image, n, m2, bc);
  const std::size_t N = (std::size_t)n * m2;
  DevBuf d(2 * N);
  check(fd_op_eigenvalues(op.h, d.p, nullptr));
  cuda(cudaDeviceSynchronize());
  const std::vector<double> h = d.host(2 * N);
  std::string csv = "index,real,imag\n";
  for (std::size_t i = 0; i < N; ++i)
    csv += std::to_string(i + 1) + "," + format_double(h[2 * i]) + "," + format_double(h[2 * i + 1]) +
           "\n";
  atomic_write(out, csv);
  return 0;
}

int run_blur(const std::string& input, const std::string& psf_path, const std::string& bc_name,
             double noise, std::uint64_t seed, const std::string& output, bool normalize,
             const std::string& dims) {  // fastdeblur.cpp:169-205
  if (noise < 0) throw Validation("--noise must be nonnegative");
  const GridData data = load_grid(input, dims);
  const PsfFile file = read_psf_file(psf_path);
  int out_rows = data.rows, out_cols = data.cols;
  DevBuf in(data.values);
  std::size_t nout = data.values.size();
  std::unique_ptr<DevBuf> out;
  if (bc_name == "true-extended") {
    const std::vector<double> w = checked_weights(file.weights, normalize);
    if (!data.is_image) {
      if (!file.is_1d()) throw Validation("psf file is 2D; a 1D mask has one row or one column");
      out_cols = data.cols - ((int)w.size() - 1);
      if (out_cols < 1) throw Validation("extended signal shorter than the psf support");
      nout = (std::size_t)out_cols;
      out = std::make_unique<DevBuf>(nout);
      check(fd_convolve_valid(in.p, 1, out_cols, w.data(), (int)w.size(), out->p, nullptr));
    } else {
      if (file.is_1d() && !(file.rows == 1 && file.cols == 1))
        throw Validation("psf file is 1D; pass a rows x cols mask for images");
      out_rows = data.rows - (file.rows - 1);
      out_cols = data.cols - (file.cols - 1);
      if (out_rows < 1 || out_cols < 1) throw Validation("extended image smaller than the psf support");
      nout = (std::size_t)out_rows * out_cols;
      out = std::make_unique<DevBuf>(nout);
      check(fd_convolve_valid_2d(in.p, 1, out_rows, out_cols, w.data(), file.rows, file.cols, out->p,
                                 nullptr));
    }
  } else {
    Op op;
    make_operator(op, file, normalize, data.is_image, data.is_image ? data.rows : data.cols,
                  data.is_image ? data.cols : 1, parse_bc(bc_name));
    out = std::make_unique<DevBuf>(nout);
    check(fd_matvec(op.h, in.p, out->p, nullptr, 1, nullptr));
  }
  const unsigned long long s = seed;
  check(fd_add_noise(out->p, 1, (long long)nout, noise, &s, nullptr));
  cuda(cudaDeviceSynchronize());
  write_grid(output, data, out->host(nout), out_rows, out_cols);
  return 0;
}

int run_deblur(const std::string& input, const std::string& psf_path, const std::string& bc_name,
               const std::string& reg, const std::string& mu_arg, const std::string& truth_path,
               const std::string& output, const std::string& curves, bool normalize,
               const std::string& dims, const GridOpts& grid) {  // fastdeblur.cpp:207-283
  const int bc = parse_bc(bc_name);
  const int smoother = parse_reg(reg);
  const GridData data = load_grid(input, dims);
  const PsfFile file = read_psf_file(psf_path);
  int use_gcv = 0;
  double fixed_mu = 0.0;
  if (mu_arg == "gcv") {
    use_gcv = 1;
  } else {
    try {
      fixed_mu = std::stod(mu_arg);
    } catch (...) {
      throw Validation("--mu must be a positive number or 'gcv'");
    }
    if (!(fixed_mu > 0)) throw Validation("--mu must be positive");
  }
  std::vector<double> truth;
  if (!truth_path.empty()) {
    const GridData t = load_grid(truth_path, dims);
    if (t.values.size() != data.values.size())
      throw Validation("--truth dimensions do not match the input");
    truth = t.values;
  }
  const bool want_curve = !curves.empty();
  Op op;
  make_operator(op, file, normalize, data.is_image, data.is_image ? data.rows : data.cols,
                data.is_image ? data.cols : 1, bc);
  Smooth L;
  check(fd_smoother_create(op.h, smoother, &L.h));
  const std::size_t N = data.values.size();
  DevBuf g(data.values), f(N), mu(1), res(1), curve((std::size_t)std::max(grid.mu_count, 1));
  check(fd_deblur(op.h, L.h, g.p, use_gcv, fixed_mu, grid.mu_lo, grid.mu_hi, grid.mu_count, f.p, mu.p,
                  nullptr, want_curve ? curve.p : nullptr, res.p, 1, nullptr));
  cuda(cudaDeviceSynchronize());
  const std::vector<double> restored = f.host(N);
  const double mu_used = mu.host(1)[0];
  write_grid(output, data, restored, data.rows, data.cols);
  std::cout << "mu=" << format_double(mu_used) << " source=" << (use_gcv ? "gcv" : "fixed") << "\n";
  if (!truth.empty()) std::cout << "rre=" << format_double(rre(truth, restored)) << "\n";
  if (complex_basis(bc)) {
    const double imag_residue = res.host(1)[0];
    double fnorm = 0.0;
    for (double x : restored) fnorm += x * x;
    fnorm = std::sqrt(fnorm);
    std::cout << "imag_residue=" << format_double(imag_residue);
    if (imag_residue > 1e-6 * fnorm) std::cout << " (above 1e-6 threshold)";
    std::cout << "\n";
  }
  if (want_curve) {
    // the grid, G(mu) and (with a truth) RRE(mu) of the same operator: one
    // analysis and a batch of filtered syntheses on the device (fd_sweep_mu)
    const int K = grid.mu_count;
    std::vector<double> cm(K), cg(K), cr(K), summ(4);
    std::unique_ptr<DevBuf> t;
    if (!truth.empty()) t = std::make_unique<DevBuf>(truth);
    check(fd_sweep_mu(op.h, L.h, g.p, t ? t->p : nullptr, grid.mu_lo, grid.mu_hi, K, cm.data(),
                      cg.data(), cr.data(), summ.data(), nullptr));
    std::string csv = truth.empty() ? "mu,G\n" : "mu,G,rre\n";
    for (int k = 0; k < K; ++k) {
      csv += format_double(cm[k]) + "," + format_double(cg[k]);
      if (!truth.empty()) csv += "," + format_double(cr[k]);
      csv += "\n";
    }
    atomic_write(curves, csv);
  }
  return 0;
}

int run_compare(const std::string& input, const std::string& psf_path, double noise,
                std::uint64_t seed, const std::string& bc_list, const std::string& reg,
                const std::string& out, bool normalize, const std::string& dims,
                const GridOpts& grid) {  // fastdeblur.cpp:285-347
  const int smoother = parse_reg(reg);
  const GridData data = load_grid(input, dims);
  const PsfFile file = read_psf_file(psf_path);
  std::vector<std::pair<std::string, int>> bcs;
  std::string token;
  for (char c : bc_list + ",") {
    if (c == ',') {
      if (!token.empty()) bcs.emplace_back(token, parse_bc(token));
      token.clear();
    } else {
      token += c;
    }
  }
  if (bcs.empty()) throw Validation("--bc-list must name at least one bc");
  const std::vector<double> w = checked_weights(file.weights, normalize);
  int n1, n2;
  std::vector<double> truth;
  DevBuf ext(data.values);
  std::unique_ptr<DevBuf> g;
  if (!data.is_image) {
    if (!file.is_1d()) throw Validation("psf file is 2D; a 1D mask has one row or one column");
    const int m = ((int)w.size() - 1) / 2;
    n1 = data.cols - 2 * m;
    n2 = 1;
    if (n1 < 1) throw Validation("extended signal shorter than the psf support");
    truth.assign(data.values.begin() + m, data.values.end() - m);
    g = std::make_unique<DevBuf>((std::size_t)n1);
    check(fd_convolve_valid(ext.p, 1, n1, w.data(), (int)w.size(), g->p, nullptr));
  } else {
    if (file.is_1d() && !(file.rows == 1 && file.cols == 1))
      throw Validation("psf file is 1D; pass a rows x cols mask for images");
    const int m1 = (file.rows - 1) / 2, m2 = (file.cols - 1) / 2;
    n1 = data.rows - 2 * m1;
    n2 = data.cols - 2 * m2;
    if (n1 < 5 || n2 < 5) throw Validation("extended image too small for the psf support");
    truth.resize((std::size_t)n1 * n2);
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < n2; ++j)
        truth[(std::size_t)i * n2 + j] = data.values[(std::size_t)(i + m1) * data.cols + (j + m2)];
    g = std::make_unique<DevBuf>((std::size_t)n1 * n2);
    check(fd_convolve_valid_2d(ext.p, 1, n1, n2, w.data(), file.rows, file.cols, g->p, nullptr));
  }
  const unsigned long long s = seed;
  check(fd_add_noise(g->p, 1, (long long)n1 * n2, noise, &s, nullptr));
  DevBuf t(truth);
  const int K = grid.mu_count;
  std::string csv = "bc,min_rre,mu_opt,mu_gcv,rre_gcv\n";
  for (const auto& [name, bc] : bcs) {
    Op op;
    make_operator(op, file, normalize, data.is_image, n1, n2, bc);
    Smooth L;
    check(fd_smoother_create(op.h, smoother, &L.h));
    std::vector<double> cm(std::max(K, 1)), cg(std::max(K, 1)), cr(std::max(K, 1)), summ(4);
    check(fd_sweep_mu(op.h, L.h, g->p, t.p, grid.mu_lo, grid.mu_hi, K, cm.data(), cg.data(), cr.data(),
                      summ.data(), nullptr));
    csv += name + "," + format_double(summ[0]) + "," + format_double(summ[1]) + "," +
           format_double(summ[2]) + "," + format_double(summ[3]) + "\n";
  }
  atomic_write(out, csv);
  return 0;
}

// --------------------------------------------------------------- arguments
// `--name value` / `--name=value` options and bare flags of one subcommand
struct Args {
  std::map<std::string, std::string> opt;
  std::map<std::string, bool> flag;
  std::string get(const std::string& k, const std::string& dflt = "") const {
    const auto it = opt.find(k);
    return it == opt.end() ? dflt : it->second;
  }
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  std::string require(const std::string& k) const {
    if (!has(k)) throw std::invalid_argument("--" + k + " is required");
    return opt.at(k);
  }
};
double to_double(const std::string& s, const std::string& name) {
  try {
    std::size_t used = 0;
    const double v = std::stod(s, &used);
    if (used == s.size()) return v;
  } catch (...) {
  }
  throw std::invalid_argument("--" + name + ": not a number: " + s);
}
long long to_int(const std::string& s, const std::string& name) {
  try {
    std::size_t used = 0;
    const long long v = std::stoll(s, &used);
    if (used == s.size()) return v;
  } catch (...) {
  }
  throw std::invalid_argument("--" + name + ": not an integer: " + s);
}
std::uint64_t to_u64(const std::string& s, const std::string& name) {
  try {
    std::size_t used = 0;
    if (!s.empty() && s[0] != '-') {
      const unsigned long long v = std::stoull(s, &used);
      if (used == s.size()) return v;
    }
  } catch (...) {
  }
  throw std::invalid_argument("--" + name + ": not a nonnegative integer: " + s);
}

const char* kUsage =
    "fast boundary-corrected deblurring toolkit (B200)\n"
    "usage: fastdeblur_b200 [--normalize] SUBCOMMAND [options]\n"
    "  eigs    --psf F --n N [--n2 N2] --bc BC --out CSV\n"
    "  blur    --input F --psf F [--bc BC|true-extended] [--noise X] [--seed S] --output F [--dims RxC]\n"
    "  deblur  --input F --psf F --bc BC [--reg identity|laplacian] --mu X|gcv [--truth F]\n"
    "          --output F [--curves CSV] [--dims RxC] [--mu-lo X] [--mu-hi X] [--mu-count K]\n"
    "  compare --input F --psf F [--noise X] [--seed S] --bc-list BC,BC [--reg R] --out CSV\n"
    "          [--dims RxC] [--mu-lo X] [--mu-hi X] [--mu-count K]\n";

}  // namespace

int main(int argc, char** argv) {
  bool normalize = false;
  std::string sub;
  Args a;
  try {
    for (int i = 1; i < argc; ++i) {
      std::string t = argv[i];
      if (t == "--help" || t == "-h") {
        std::cout << kUsage;
        return 0;
      }
      if (t == "--normalize") {
        normalize = true;
        continue;
      }
      if (t.rfind("--", 0) == 0) {
        std::string key = t.substr(2), val;
        const auto eq = key.find('=');
        if (eq != std::string::npos) {
          val = key.substr(eq + 1);
          key = key.substr(0, eq);
        } else {
          if (i + 1 >= argc) throw std::invalid_argument("--" + key + " needs a value");
          val = argv[++i];
        }
        a.opt[key] = val;
        continue;
      }
      if (!sub.empty()) throw std::invalid_argument("unexpected argument '" + t + "'");
      sub = t;
    }
    if (sub != "eigs" && sub != "blur" && sub != "deblur" && sub != "compare")
      throw std::invalid_argument("a subcommand is required (eigs, blur, deblur, compare)");
    static const std::map<std::string, std::vector<std::string>> allowed = {
        {"eigs", {"psf", "n", "n2", "bc", "out"}},
        {"blur", {"input", "psf", "bc", "noise", "seed", "output", "dims"}},
        {"deblur", {"input", "psf", "bc", "reg", "mu", "truth", "output", "curves", "dims", "mu-lo",
                    "mu-hi", "mu-count"}},
        {"compare", {"input", "psf", "noise", "seed", "bc-list", "reg", "out", "dims", "mu-lo", "mu-hi",
                     "mu-count"}}};
    for (const auto& kv : a.opt) {
      const auto& ok = allowed.at(sub);
      if (std::find(ok.begin(), ok.end(), kv.first) == ok.end())
        throw std::invalid_argument("unknown option --" + kv.first);
    }
  } catch (const std::exception& e) {  // CLI11 ParseError -> 2 (fastdeblur.cpp:421-426)
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }

  try {
    GridOpts grid;
    auto read_grid = [&] {
      if (a.has("mu-lo")) grid.mu_lo = to_double(a.get("mu-lo"), "mu-lo");
      if (a.has("mu-hi")) grid.mu_hi = to_double(a.get("mu-hi"), "mu-hi");
      if (a.has("mu-count")) grid.mu_count = (int)to_int(a.get("mu-count"), "mu-count");
    };
    try {
      if (sub == "eigs") {
        const std::string psf = a.require("psf"), bc = a.require("bc"), out = a.require("out");
        const int n = (int)to_int(a.require("n"), "n");
        const int n2 = a.has("n2") ? (int)to_int(a.get("n2"), "n2") : 0;
        return run_eigs(psf, n, n2, bc, out, normalize);
      }
      if (sub == "blur") {
        const std::string in = a.require("input"), psf = a.require("psf"), out = a.require("output");
        return run_blur(in, psf, a.get("bc", "true-extended"), to_double(a.get("noise", "0"), "noise"),
                        to_u64(a.get("seed", "0"), "seed"), out, normalize, a.get("dims"));
      }
      if (sub == "deblur") {
        const std::string in = a.require("input"), psf = a.require("psf"), bc = a.require("bc"),
                          mu = a.require("mu"), out = a.require("output");
        read_grid();
        return run_deblur(in, psf, bc, a.get("reg", "identity"), mu, a.get("truth"), out,
                          a.get("curves"), normalize, a.get("dims"), grid);
      }
      const std::string in = a.require("input"), psf = a.require("psf"), bcs = a.require("bc-list"),
                        out = a.require("out");
      read_grid();
      return run_compare(in, psf, to_double(a.get("noise", "0"), "noise"),
                         to_u64(a.get("seed", "0"), "seed"), bcs, a.get("reg", "identity"), out,
                         normalize, a.get("dims"), grid);
    } catch (const std::invalid_argument& e) {  // missing / malformed option: parse error
      std::cerr << "error: " << e.what() << "\n";
      return 2;
    }
  } catch (const Validation& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const Degenerate& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
