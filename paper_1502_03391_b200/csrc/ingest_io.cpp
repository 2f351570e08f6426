// ingest_io.cpp -- see ingest_io.h.
#include "ingest_io.h"

#include <sys/stat.h>

#include <charconv>
#include <cstring>

namespace jofc_gpu {
namespace ingest {

namespace {

constexpr size_t kChunk = 1 << 22;

inline bool is_space(char ch) { return ch == ' ' || ch == '\t' || ch == '\r' || ch == '\n'; }

// [b, e) trimmed of the reference's whitespace set " \t\r\n".
inline void trim(const char*& b, const char*& e) {
  while (b < e && is_space(*b)) ++b;
  while (e > b && is_space(e[-1])) --e;
}

}  // namespace

CsvRows::~CsvRows() {
  if (f_) std::fclose(f_);
}

bool CsvRows::open(const std::string& path, std::string& err) {
  path_ = path;
  f_ = std::fopen(path.c_str(), "rb");
  if (!f_) {
    err = "cannot open '" + path + "'";
    return false;
  }
  buf_.resize(kChunk);
  return true;
}

bool CsvRows::fill() {
  if (eof_) return false;
  if (pos_ > 0) {  // keep the unconsumed tail
    std::memmove(buf_.data(), buf_.data() + pos_, len_ - pos_);
    len_ -= pos_;
    pos_ = 0;
  }
  if (len_ == buf_.size()) buf_.resize(buf_.size() * 2);  // a line longer than the buffer
  const size_t got = std::fread(buf_.data() + len_, 1, buf_.size() - len_, f_);
  if (got == 0) eof_ = true;
  len_ += got;
  return got > 0;
}

int CsvRows::next(std::vector<double>& row, std::string& err) {
  for (;;) {
    // locate the end of the current line
    const char* start = buf_.data() + pos_;
    const void* nl = std::memchr(start, '\n', len_ - pos_);
    if (!nl && !eof_) {
      fill();
      continue;
    }
    if (!nl && pos_ == len_) return 0;  // end of file
    const char* end = nl ? static_cast<const char*>(nl) : buf_.data() + len_;
    pos_ = static_cast<size_t>(end - buf_.data()) + (nl ? 1 : 0);
    ++lineno_;
    const char* b = start;
    const char* e = end;
    trim(b, e);
    if (b == e) continue;  // blank line
    row.clear();
    const char* field = b;
    for (;;) {
      const char* comma = static_cast<const char*>(std::memchr(field, ',', e - field));
      const char* fe = comma ? comma : e;
      const char* tb = field;
      const char* te = fe;
      trim(tb, te);
      double v = 0.0;
      const auto res = std::from_chars(tb, te, v);
      if (res.ec != std::errc{} || res.ptr != te) {
        err = "'" + path_ + "' line " + std::to_string(lineno_) + ": cannot parse number '" +
              std::string(tb, te) + "'";
        return -1;
      }
      row.push_back(v);
      if (!comma) break;
      field = comma + 1;
    }
    return 1;
  }
}

bool open_jofc(const std::string& path, std::FILE*& f, JofcHeader& h, std::string& err) {
  f = std::fopen(path.c_str(), "rb");
  if (!f) {
    err = "cannot open '" + path + "'";
    return false;
  }
  char magic[4] = {};
  if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "JOFC", 4) != 0) {
    err = "'" + path + "': not a JOFC binary file";
    return false;
  }
  uint32_t hd[4] = {};
  if (std::fread(hd, sizeof(uint32_t), 4, f) != 4) {
    err = "'" + path + "': truncated header";
    return false;
  }
  h.version = hd[0];
  h.n = hd[1];
  h.m = hd[2];
  h.d = hd[3];
  if (h.version != 1) {
    err = "'" + path + "': unsupported version " + std::to_string(h.version);
    return false;
  }
  struct stat st {};
  const uint64_t cols = h.d == 0 ? h.n : h.d;
  const uint64_t need = 20 + uint64_t(h.m) * h.n * cols * sizeof(double);
  if (fstat(fileno(f), &st) != 0 || static_cast<uint64_t>(st.st_size) < need) {
    err = "'" + path + "': truncated payload";
    return false;
  }
  return true;
}

}  // namespace ingest
}  // namespace jofc_gpu
