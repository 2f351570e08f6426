// ingest_io.cpp -- see ingest_io.h.
#include "ingest_io.h"

#include <sys/stat.h>
#include <unistd.h>

#include <omp.h>

#include <algorithm>
#include <charconv>
#include <cstring>

namespace jofc_gpu {
namespace ingest {

namespace {

constexpr size_t kChunk = 1 << 25;  // 32 MB text batches

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

// Appends the next bytes of the file to the window (positioned reads, split
// over the host threads: the page-cache copy is the other half of the cost).
bool CsvRows::fill() {
  if (eof_) return false;
  if (pos_ > 0) {  // keep the unconsumed tail
    std::memmove(buf_.data(), buf_.data() + pos_, len_ - pos_);
    len_ -= pos_;
    pos_ = 0;
  }
  if (len_ == buf_.size()) buf_.resize(buf_.size() * 2);  // a line longer than the buffer
  const int fd = fileno(f_);
  const size_t want = buf_.size() - len_;
  const int nt = static_cast<int>(std::max<size_t>(
      1, std::min<size_t>(std::min(16, omp_get_max_threads()), want / (1 << 20))));
  std::vector<size_t> got(nt, 0);
#pragma omp parallel for num_threads(nt) schedule(static, 1)
  for (int t = 0; t < nt; ++t) {
    const size_t a = want * t / nt, b = want * (t + 1) / nt;
    while (got[t] < b - a) {
      const ssize_t g = pread(fd, buf_.data() + len_ + a + got[t], b - a - got[t],
                              static_cast<off_t>(file_off_ + a + got[t]));
      if (g <= 0) break;
      got[t] += static_cast<size_t>(g);
    }
  }
  // the bytes read are contiguous up to the first short part (end of file)
  size_t total = 0;
  for (int t = 0; t < nt; ++t) {
    total += got[t];
    if (got[t] < want * (t + 1) / nt - want * t / nt) break;
  }
  if (total < want) eof_ = true;
  len_ += total;
  file_off_ += total;
  return total > 0;
}

// Parses the lines of [b, e) (whole lines; the last may lack its newline)
// into `pt`, stopping at the first field that does not parse.
static void parse_lines(const char* b, const char* e, std::vector<double>& vals,
                        std::vector<size_t>& off, std::vector<size_t>& line, size_t& lines,
                        bool& failed, std::string& bad_field) {
  const char* p = b;
  while (p < e) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', e - p));
    const char* end = nl ? nl : e;
    const size_t this_line = lines++;
    const char* lb = p;
    const char* le = end;
    p = nl ? nl + 1 : e;
    trim(lb, le);
    if (lb == le) continue;  // blank line
    const size_t start = vals.size();
    const char* field = lb;
    for (;;) {
      const char* comma = static_cast<const char*>(std::memchr(field, ',', le - field));
      const char* fe = comma ? comma : le;
      const char* tb = field;
      const char* te = fe;
      trim(tb, te);
      double v = 0.0;
      const auto res = std::from_chars(tb, te, v);
      if (res.ec != std::errc{} || res.ptr != te) {
        vals.resize(start);
        failed = true;
        bad_field.assign(tb, te);
        return;
      }
      vals.push_back(v);
      if (!comma) break;
      field = comma + 1;
    }
    off.push_back(start);
    line.push_back(this_line);
  }
}

bool CsvRows::parse_batch() {
  // whole lines: grow the window until it holds a newline (or the file ends)
  for (;;) {
    const char* start = buf_.data() + pos_;
    const bool has_nl = std::memchr(start, '\n', len_ - pos_) != nullptr;
    if (has_nl && (len_ - pos_ >= buf_.size() / 2 || eof_)) break;
    if (eof_) break;
    fill();
  }
  if (pos_ == len_) return false;
  const char* b = buf_.data() + pos_;
  const char* e = buf_.data() + len_;
  if (!eof_) {  // up to and including the last newline
    const char* q = e;
    while (q > b && q[-1] != '\n') --q;
    e = q;
  }
  const size_t bytes = static_cast<size_t>(e - b);
  const int nt = static_cast<int>(std::max<size_t>(
      1, std::min<size_t>(std::min(16, omp_get_max_threads()), bytes / (1 << 16))));
  // part boundaries at line starts
  std::vector<const char*> cut(nt + 1, e);
  cut[0] = b;
  for (int t = 1; t < nt; ++t) {
    const char* q = b + bytes * t / nt;
    if (q < cut[t - 1]) q = cut[t - 1];
    const void* nl = std::memchr(q, '\n', e - q);
    cut[t] = nl ? static_cast<const char*>(nl) + 1 : e;
  }
  parts_.assign(nt, Part());
#pragma omp parallel for num_threads(nt) schedule(static, 1)
  for (int t = 0; t < nt; ++t) {
    Part& pt = parts_[t];
    pt.off.reserve(256);
    parse_lines(cut[t], cut[t + 1], pt.vals, pt.off, pt.line, pt.lines, pt.failed, pt.bad_field);
    pt.off.push_back(pt.vals.size());
  }
  part_base_.assign(nt, 0);
  for (int t = 1; t < nt; ++t) part_base_[t] = part_base_[t - 1] + parts_[t - 1].lines;
  // (a failed part stops the batch there: later parts are never consumed)
  pos_ = static_cast<size_t>(e - buf_.data());
  cur_part_ = 0;
  cur_row_ = 0;
  have_batch_ = true;
  return true;
}

int CsvRows::next(std::vector<double>& row, std::string& err) {
  for (;;) {
    if (!have_batch_) {
      if (!parse_batch()) return 0;
    }
    while (cur_part_ < parts_.size()) {
      const Part& pt = parts_[cur_part_];
      if (cur_row_ + 1 < pt.off.size()) {
        const size_t a = pt.off[cur_row_], z = pt.off[cur_row_ + 1];
        row.assign(pt.vals.begin() + a, pt.vals.begin() + z);
        lineno_ = batch_base_ + part_base_[cur_part_] + pt.line[cur_row_] + 1;
        ++cur_row_;
        return 1;
      }
      if (pt.failed) {
        lineno_ = batch_base_ + part_base_[cur_part_] + pt.lines;
        err = "'" + path_ + "' line " + std::to_string(lineno_) + ": cannot parse number '" +
              pt.bad_field + "'";
        return -1;
      }
      ++cur_part_;
      cur_row_ = 0;
    }
    // batch consumed
    size_t lines = 0;
    for (const Part& pt : parts_) lines += pt.lines;
    batch_base_ += lines;
    have_batch_ = false;
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
