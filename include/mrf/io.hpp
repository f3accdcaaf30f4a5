// mrf/io.hpp -- on-disk formats feeding the GPU path,
// source-compatible with the reference's <mp/io.hpp> (proj/include/mp/io.hpp,
// proj/src/io.cpp): PGM images, MPCV1 cost volumes, stereo / denoising data
// terms, the per-iteration energy CSV and 16-bit label maps. Host-only code;
// the volumes it produces go to the device through mrf/mp_cuda.hpp.
//
//   MPCV1 (io.hpp:29-35, io.cpp:118-152): "MPCV1", then H, W, L as 32-bit
//   little-endian unsigned, then H*W*L finite little-endian float32 values,
//   row-major with label fastest. Readers reject bad magic, zero sizes,
//   L > 256, short payloads and non-finite values.
#pragma once

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "mp_cuda.hpp"

namespace mp {

/// io.hpp:15-20
struct GrayImage {
  int height = 0, width = 0;
  std::vector<std::uint16_t> pixels;  // row-major
  std::uint16_t at(int h, int w) const { return pixels[static_cast<std::size_t>(h) * width + w]; }
};

namespace io_detail {

// Next whitespace-delimited header token; '#' starts a comment to end of line.
inline std::string pgm_token(std::istream& in) {
  std::string tok;
  for (int c = in.get(); c != EOF; c = in.get()) {
    if (c == '#') {
      while (c != EOF && c != '\n') c = in.get();
    } else if (std::isspace(c)) {
      if (!tok.empty()) return tok;
    } else {
      tok += static_cast<char>(c);
    }
  }
  if (tok.empty()) throw std::runtime_error("pgm: truncated header");
  return tok;
}

inline int pgm_int(const std::string& tok, const char* what) {
  std::size_t used = 0;
  int v = 0;
  try {
    v = std::stoi(tok, &used);
  } catch (const std::exception&) {
    used = 0;
  }
  if (used == 0 || used != tok.size()) throw std::runtime_error(std::string("pgm: bad ") + what + " '" + tok + "'");
  return v;
}

inline void put_le32(std::ostream& out, std::uint32_t v) {
  const char b[4] = {char(v & 0xff), char((v >> 8) & 0xff), char((v >> 16) & 0xff), char((v >> 24) & 0xff)};
  out.write(b, 4);
}

inline std::uint32_t get_le32(std::istream& in) {
  unsigned char b[4] = {0, 0, 0, 0};
  in.read(reinterpret_cast<char*>(b), 4);
  if (in.gcount() != 4) throw std::runtime_error("cost volume: truncated header");
  return std::uint32_t(b[0]) | std::uint32_t(b[1]) << 8 | std::uint32_t(b[2]) << 16 | std::uint32_t(b[3]) << 24;
}

}  // namespace io_detail

/// io.hpp:22-24: P2 (ASCII) or P5 (binary) PGM, maxval <= 65535; P5 samples
/// above 255 take two bytes, most significant first.
inline GrayImage load_pgm(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("pgm: cannot open " + path);
  const std::string magic = io_detail::pgm_token(in);
  if (magic != "P2" && magic != "P5") throw std::runtime_error("pgm: unsupported magic " + magic);
  GrayImage img;
  img.width = io_detail::pgm_int(io_detail::pgm_token(in), "width");
  img.height = io_detail::pgm_int(io_detail::pgm_token(in), "height");
  const int maxval = io_detail::pgm_int(io_detail::pgm_token(in), "maxval");
  if (img.width < 1 || img.height < 1 || maxval < 1 || maxval > 65535)
    throw std::runtime_error("pgm: invalid dimensions or maxval");
  img.pixels.resize(static_cast<std::size_t>(img.height) * img.width);
  if (magic == "P2") {
    for (auto& px : img.pixels) {
      const int v = io_detail::pgm_int(io_detail::pgm_token(in), "sample");
      if (v < 0 || v > maxval) throw std::runtime_error("pgm: sample out of range");
      px = static_cast<std::uint16_t>(v);
    }
    return img;
  }
  // P5: the one whitespace byte after maxval ended the last header token
  const std::size_t width = maxval > 255 ? 2 : 1;
  std::vector<unsigned char> raw(img.pixels.size() * width);
  in.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(raw.size()));
  if (static_cast<std::size_t>(in.gcount()) != raw.size()) throw std::runtime_error("pgm: truncated payload");
  for (std::size_t i = 0; i < img.pixels.size(); ++i) {
    const int v = width == 2 ? (int(raw[2 * i]) << 8 | int(raw[2 * i + 1])) : int(raw[i]);
    if (v > maxval) throw std::runtime_error("pgm: sample out of range");
    img.pixels[i] = static_cast<std::uint16_t>(v);
  }
  return img;
}

/// io.hpp:26-27: 16-bit binary PGM (P5, maxval 65535).
inline void save_pgm(const std::string& path, const GrayImage& image) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("pgm: cannot write " + path);
  out << "P5\n" << image.width << " " << image.height << "\n65535\n";
  std::string raw;
  raw.reserve(image.pixels.size() * 2);
  for (std::uint16_t px : image.pixels) {
    raw += static_cast<char>(px >> 8);
    raw += static_cast<char>(px & 0xff);
  }
  out.write(raw.data(), static_cast<std::streamsize>(raw.size()));
  if (!out) throw std::runtime_error("pgm: write failed for " + path);
}

namespace detail {

inline void write_cost_volume_file(const std::string& path, int h, int w, int l, const float* data) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cost volume: cannot write " + path);
  out.write("MPCV1", 5);
  for (int v : {h, w, l}) io_detail::put_le32(out, static_cast<std::uint32_t>(v));
  static_assert(sizeof(float) == 4, "float32 payload");
  out.write(reinterpret_cast<const char*>(data), static_cast<std::streamsize>(std::size_t(h) * w * l * 4));
  if (!out) throw std::runtime_error("cost volume: write failed for " + path);
}

inline std::vector<float> read_cost_volume_file(const std::string& path, int& h, int& w, int& l) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cost volume: cannot open " + path);
  char magic[5] = {0, 0, 0, 0, 0};
  in.read(magic, 5);
  if (in.gcount() != 5 || std::string(magic, 5) != "MPCV1") throw std::runtime_error("cost volume: bad magic in " + path);
  const std::uint32_t uh = io_detail::get_le32(in), uw = io_detail::get_le32(in), ul = io_detail::get_le32(in);
  if (!uh || !uw || !ul || ul > 256) throw std::runtime_error("cost volume: invalid dimensions");
  h = int(uh), w = int(uw), l = int(ul);
  std::vector<float> data(std::size_t(uh) * uw * ul);
  in.read(reinterpret_cast<char*>(data.data()), static_cast<std::streamsize>(data.size() * 4));
  if (static_cast<std::size_t>(in.gcount()) != data.size() * 4) throw std::runtime_error("cost volume: truncated payload");
  if (!std::all_of(data.begin(), data.end(), [](float v) { return std::isfinite(v); }))
    throw std::runtime_error("cost volume: non-finite value");
  return data;
}

}  // namespace detail

/// io.hpp:37-50
template <class Real>
void save_cost_volume(const std::string& path, const UnaryVolume<Real>& vol) {
  const std::vector<float> buf(vol.values.begin(), vol.values.end());
  detail::write_cost_volume_file(path, vol.height, vol.width, vol.labels, buf.data());
}

template <class Real>
UnaryVolume<Real> load_cost_volume(const std::string& path) {
  int h = 0, w = 0, l = 0;
  const std::vector<float> buf = detail::read_cost_volume_file(path, h, w, l);
  UnaryVolume<Real> vol(h, w, l);
  std::transform(buf.begin(), buf.end(), vol.values.begin(), [](float v) { return static_cast<Real>(v); });
  return vol;
}

/// io.hpp:52-69: theta_i(d) = |left(y, x) - right(y, max(0, x - d))|.
template <class Real>
UnaryVolume<Real> stereo_unaries(const GrayImage& left, const GrayImage& right, int max_disp) {
  if (left.height != right.height || left.width != right.width)
    throw std::invalid_argument("stereo_unaries: image sizes differ");
  if (max_disp < 1 || max_disp > 256) throw std::invalid_argument("stereo_unaries: max_disp must be in [1, 256]");
  UnaryVolume<Real> vol(left.height, left.width, max_disp);
  for (int y = 0; y < left.height; ++y)
    for (int x = 0; x < left.width; ++x) {
      const Real lv = static_cast<Real>(left.at(y, x));
      for (int d = 0; d < max_disp; ++d)
        vol.at(y * left.width + x, d) = std::abs(lv - static_cast<Real>(right.at(y, std::max(0, x - d))));
    }
  return vol;
}

/// io.hpp:71-89: theta_i(l) = min(|I_i - l|^p, tau), p = 1 (tl) or 2 (tq),
/// computed in double and cast.
template <class Real>
UnaryVolume<Real> denoise_unaries(const GrayImage& noisy, int labels, PairwiseKind kind, double tau) {
  if (kind != PairwiseKind::truncated_linear && kind != PairwiseKind::truncated_quadratic)
    throw std::invalid_argument("denoise_unaries: kind must be tl or tq");
  if (!(tau > 0)) throw std::invalid_argument("denoise_unaries: tau must be > 0");
  UnaryVolume<Real> vol(noisy.height, noisy.width, labels);
  for (int i = 0; i < vol.nodes(); ++i) {
    const double v = static_cast<double>(noisy.pixels[i]);
    for (int l = 0; l < labels; ++l) {
      const double d = std::abs(v - l);
      vol.at(i, l) = static_cast<Real>(std::min(kind == PairwiseKind::truncated_quadratic ? d * d : d, tau));
    }
  }
  return vol;
}

/// io.hpp:91-97 / io.cpp:158-170: "iteration,energy,forward_ms" rows.
struct EnergyRow {
  int iteration;  // 1-based
  double energy;
  double forward_ms;
};

inline void write_energy_csv(const std::string& path, const std::vector<EnergyRow>& rows) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("csv: cannot write " + path);
  out << "iteration,energy,forward_ms\n";
  for (const EnergyRow& r : rows) {
    char line[96];
    std::snprintf(line, sizeof(line), "%d,%.10g,%.6g\n", r.iteration, r.energy, r.forward_ms);
    out << line;
  }
  if (!out) throw std::runtime_error("csv: write failed for " + path);
}

/// io.hpp:99-108: a labelling as a 16-bit PGM.
template <class Label>
void save_label_map(const std::string& path, int height, int width, const std::vector<Label>& labels) {
  GrayImage img;
  img.height = height;
  img.width = width;
  img.pixels.assign(labels.begin(), labels.end());
  save_pgm(path, img);
}

}  // namespace mp
