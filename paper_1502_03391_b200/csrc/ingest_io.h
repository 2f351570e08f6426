// ingest_io.h -- host-side readers for streaming Delta ingest.
//
// The wire formats of proj/include/jofc/io.hpp:
//   * headerless CSV, one n x n matrix per file (proj/src/io.cpp:127-150 parse
//     rules: lines trimmed, blank lines skipped, comma-separated fields each
//     trimmed and parsed whole with std::from_chars);
//   * the ".jofc" container: "JOFC", u32 version (1), u32 n, m, d, then
//     little-endian doubles, d == 0 for a problem (proj/src/io.cpp:84-125).
// Both are read row by row into caller buffers (pinned panels), so a problem
// streams to the device without a host n x n copy.  Errors carry the
// reference's messages.
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

namespace jofc_gpu {
namespace ingest {

// Line-oriented CSV row reader.
class CsvRows {
 public:
  ~CsvRows();
  // false + err = "cannot open '<path>'"
  bool open(const std::string& path, std::string& err);
  // Next non-blank line parsed into `row`: 1 row, 0 end of file, -1 parse
  // error (err set, reference wording incl. the line number).
  int next(std::vector<double>& row, std::string& err);
  size_t line() const { return lineno_; }  // number of the last line read

 private:
  bool fill();
  std::FILE* f_ = nullptr;
  std::string path_;
  std::vector<char> buf_;
  size_t pos_ = 0, len_ = 0;
  bool eof_ = false;
  size_t lineno_ = 0;
  std::string line_;
};

struct JofcHeader {
  uint32_t version = 0, n = 0, m = 0, d = 0;
};

// Opens a .jofc file and validates it the way read_binary does (magic,
// header, version, full payload present).  On success the stream is
// positioned at the payload.
bool open_jofc(const std::string& path, std::FILE*& f, JofcHeader& h, std::string& err);

}  // namespace ingest
}  // namespace jofc_gpu
