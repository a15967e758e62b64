// Dataset ingestion: the reference's IDX and CSV formats
// (load_idx / load_csv, data.hpp:163-255) with the same checks and messages.  Parsing is
// host work; IDX pixels travel to the device as the raw unsigned bytes (4x fewer bytes
// than fp32) and are rescaled there (ingest_u8_to_f32, p / 255 in fp64 then rounded, i.e.
// the reference's value rounded to fp32).
#include <array>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "psg_internal.h"

namespace psg {
namespace {

uint32_t read_be32(std::istream& in, const std::string& path) {
  std::array<unsigned char, 4> b{};
  in.read(reinterpret_cast<char*>(b.data()), 4);
  if (!in) throw std::runtime_error("idx: truncated header in " + path);
  return (uint32_t(b[0]) << 24) | (uint32_t(b[1]) << 16) | (uint32_t(b[2]) << 8) | uint32_t(b[3]);
}

}  // namespace

IdxData read_idx(const std::string& images_path, const std::string& labels_path) {
  std::ifstream img(images_path, std::ios::binary);
  if (!img) throw std::runtime_error("idx: cannot open " + images_path);
  if (read_be32(img, images_path) != 0x00000803u)
    throw std::runtime_error("idx: bad image magic in " + images_path);
  IdxData d;
  d.n = read_be32(img, images_path);
  d.h = read_be32(img, images_path);
  d.w = read_be32(img, images_path);
  if (d.n == 0 || d.h == 0 || d.w == 0)
    throw std::runtime_error("idx: zero dimension in " + images_path);
  d.pixels.resize(static_cast<size_t>(d.n) * d.h * d.w);
  img.read(reinterpret_cast<char*>(d.pixels.data()), static_cast<std::streamsize>(d.pixels.size()));
  if (!img) throw std::runtime_error("idx: truncated image data in " + images_path);
  std::ifstream lab(labels_path, std::ios::binary);
  if (!lab) throw std::runtime_error("idx: cannot open " + labels_path);
  if (read_be32(lab, labels_path) != 0x00000801u)
    throw std::runtime_error("idx: bad label magic in " + labels_path);
  const uint32_t ln = read_be32(lab, labels_path);
  if (ln != d.n) throw std::runtime_error("idx: image/label count mismatch");
  std::vector<unsigned char> raw(ln);
  lab.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(ln));
  if (!lab) throw std::runtime_error("idx: truncated label data in " + labels_path);
  d.labels.resize(ln);
  int max_label = 0;
  for (size_t i = 0; i < raw.size(); ++i) {
    d.labels[i] = raw[i];
    max_label = std::max(max_label, d.labels[i]);
  }
  d.classes = max_label + 1;
  return d;
}

CsvData read_csv(const std::string& path, size_t channels, size_t height, size_t width,
                 int num_classes) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("csv: cannot open " + path);
  const size_t dim = channels * height * width;
  CsvData d;
  std::string line;
  size_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    if (line.empty()) continue;
    std::stringstream row(line);
    std::string cell;
    if (!std::getline(row, cell, ',')) continue;
    const int label = std::stoi(cell);
    if (label < 0 || label >= num_classes)
      throw std::runtime_error("csv: label " + std::to_string(label) + " out of range at line " +
                               std::to_string(line_no) + " of " + path);
    d.labels.push_back(label);
    size_t count = 0;
    while (std::getline(row, cell, ',')) {
      d.images.push_back(static_cast<float>(std::stod(cell) / 255.0));
      ++count;
    }
    if (count != dim)
      throw std::runtime_error("csv: expected " + std::to_string(dim) + " pixels, got " +
                               std::to_string(count) + " at line " + std::to_string(line_no));
  }
  if (d.labels.empty()) throw std::runtime_error("csv: no rows in " + path);
  return d;
}

}  // namespace psg
