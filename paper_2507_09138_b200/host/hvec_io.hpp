// hvec_io.hpp -- the reference's on-disk formats (proj/src/vector_index.cpp:344-473,
// layout in proj/include/hedra/vector_index.hpp:162-166), shared by both host
// adapters (hedra_gpu.cpp and compat/hedra_ivf_gpu.cpp).  Templates over the
// caller's Corpus / Centroids / Metric types; files are byte-identical to the
// reference's:
//   vector file: "HVEC", u32 version 1, u32 dim, u64 count, u8 metric, count*dim
//                f32 rows, then count u64 doc ids (corpus files only)
//   assignment file: u64 count, count u32 cluster ids
// Errors: std::runtime_error with the reference's messages.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace hvec_io {

struct File {
  std::FILE* f = nullptr;
  std::string path;
  File(const std::string& p, const char* mode) : path(p) {
    f = std::fopen(p.c_str(), mode);
    if (!f)
      throw std::runtime_error(p + (mode[0] == 'w' ? ": cannot open for writing" : ": cannot open for reading"));
  }
  ~File() {
    if (f) std::fclose(f);
  }
  File(const File&) = delete;
  File& operator=(const File&) = delete;
  void put(const void* p, std::size_t bytes) {
    if (bytes && std::fwrite(p, 1, bytes, f) != bytes) throw std::runtime_error(path + ": write failed");
  }
  void get(void* p, std::size_t bytes, const char* what) {
    if (bytes && std::fread(p, 1, bytes, f) != bytes) throw std::runtime_error(path + what);
  }
  // header fields: read_pod's message (vector_index.cpp:353-358)
  void pod(void* p, std::size_t bytes) {
    if (std::fread(p, 1, bytes, f) != bytes) throw std::runtime_error("vector file: truncated read");
  }
};

inline void put_header(File& o, std::uint32_t dim, std::uint64_t count, std::uint8_t metric) {
  static const char magic[4] = {'H', 'V', 'E', 'C'};
  const std::uint32_t version = 1;
  o.put(magic, 4);
  o.put(&version, 4);
  o.put(&dim, 4);
  o.put(&count, 8);
  o.put(&metric, 1);
}

inline void get_header(File& in, std::uint32_t* dim, std::uint64_t* count, std::uint8_t* metric) {
  char magic[4];
  if (std::fread(magic, 1, 4, in.f) != 4 || std::memcmp(magic, "HVEC", 4) != 0)
    throw std::runtime_error(in.path + ": not a HVEC file");
  std::uint32_t version = 0;
  in.pod(&version, 4);
  if (version != 1) throw std::runtime_error(in.path + ": unsupported HVEC version");
  in.pod(dim, 4);
  in.pod(count, 8);
  in.pod(metric, 1);
}

template <class Corpus>
void save_corpus(const std::string& path, const Corpus& c) {
  File o(path, "wb");
  put_header(o, c.dim, c.size(), static_cast<std::uint8_t>(c.metric));
  o.put(c.data.data(), c.data.size() * sizeof(float));
  o.put(c.doc_ids.data(), c.doc_ids.size() * sizeof(std::uint64_t));
}

template <class Corpus>
Corpus load_corpus(const std::string& path) {
  File in(path, "rb");
  Corpus c;
  std::uint64_t n = 0;
  std::uint8_t m = 0;
  get_header(in, &c.dim, &n, &m);
  c.metric = static_cast<decltype(c.metric)>(m);
  c.data.resize(n * c.dim);
  c.doc_ids.resize(n);
  in.get(c.data.data(), c.data.size() * sizeof(float), ": truncated corpus file");
  in.get(c.doc_ids.data(), c.doc_ids.size() * sizeof(std::uint64_t), ": truncated corpus file");
  return c;
}

template <class Centroids, class Metric>
void save_centroids(const std::string& path, const Centroids& c, Metric metric) {
  File o(path, "wb");
  put_header(o, c.dim, c.rows.size(), static_cast<std::uint8_t>(metric));
  for (const auto& r : c.rows) o.put(r.data(), r.size() * sizeof(float));
}

template <class Centroids>
Centroids load_centroids(const std::string& path) {
  File in(path, "rb");
  Centroids c;
  std::uint64_t k = 0;
  std::uint8_t m = 0;
  get_header(in, &c.dim, &k, &m);
  c.rows.assign(k, std::vector<float>(c.dim));
  for (auto& r : c.rows) in.get(r.data(), r.size() * sizeof(float), ": truncated centroid file");
  return c;
}

inline void save_assignments(const std::string& path, const std::vector<std::uint32_t>& a) {
  File o(path, "wb");
  const std::uint64_t n = a.size();
  o.put(&n, 8);
  o.put(a.data(), a.size() * sizeof(std::uint32_t));
}

inline std::vector<std::uint32_t> load_assignments(const std::string& path) {
  File in(path, "rb");
  std::uint64_t n = 0;
  in.pod(&n, 8);
  std::vector<std::uint32_t> a(n);
  in.get(a.data(), a.size() * sizeof(std::uint32_t), ": truncated assignment file");
  return a;
}

}  // namespace hvec_io
