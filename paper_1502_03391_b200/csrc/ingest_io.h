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

// CSV row reader.  Text is read in large batches of whole lines, split at
// line boundaries over the host threads and parsed in parallel; rows are
// then handed out one by one in file order, and a parse error surfaces at
// its place in that order (after every row before it), exactly as a
// line-by-line reader would report it.
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
  // One thread's share of a batch: its parsed rows, and where it stopped.
  struct Part {
    std::vector<double> vals;
    std::vector<size_t> off;    // row r = vals[off[r], off[r + 1])
    std::vector<size_t> line;   // line number of row r within the batch part
    size_t lines = 0;           // lines scanned (up to and including an error line)
    bool failed = false;
    std::string bad_field;      // the field that failed to parse
  };
  bool fill();
  bool parse_batch();  // next batch of whole lines -> parts_; false at end of file
  std::FILE* f_ = nullptr;
  std::string path_;
  std::vector<char> buf_;
  size_t pos_ = 0, len_ = 0;
  size_t file_off_ = 0;    // bytes of the file read so far
  bool eof_ = false;
  size_t lineno_ = 0;      // line of the last row handed out
  size_t batch_base_ = 0;  // lines before the current batch
  std::vector<Part> parts_;
  std::vector<size_t> part_base_;  // lines before each part (within the batch)
  size_t cur_part_ = 0, cur_row_ = 0;
  bool have_batch_ = false;
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
