// host_io.cpp -- the host-side data path either side of the fill:
//
//  * matrix persistence (distance_matrix.hpp:80-192): the reference's text format --
//    `p=<count>` header, p rows of p comma-separated shortest-round-trip values, literal
//    `0` diagonal -- written and read by several host threads, byte-identical output and
//    the reference's validation order and messages on input; plus a binary sidecar
//    (header + the condensed doubles) that loads at disk speed.
//  * ingest (csv.hpp:55-106) and z-normalisation (runner.hpp:82-95): one series per
//    CSV row, parsed by several host threads per file, producing the packed CSR buffer
//    the fill uploads (samples + offsets + ids), with the reference's first error.
//
// Numbers are formatted and parsed with std::to_chars / std::from_chars, exactly as the
// reference does, so text round trips are bit-exact and files byte-identical. The
// z-normalisation keeps the reference's sequential per-series sums (compiled without
// FMA contraction), so its output is bit-identical too. Threads split rows/lines into
// contiguous ranges; each range reports its first error and the earliest one in file
// order wins, which is the error the sequential reference raises.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <string_view>
#include <system_error>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/dtwgpu.h"

namespace {

thread_local std::string g_io_error;
thread_local int64_t g_io_line = -1;
thread_local int64_t g_io_column = -1;
thread_local std::string g_io_file;

int io_fail(int code, std::string msg, int64_t line = -1, int64_t column = -1,
            std::string file = {}) {
  g_io_error = std::move(msg);
  g_io_line = line;
  g_io_column = column;
  g_io_file = std::move(file);
  return code;
}

int thread_count(int threads, int64_t work_items) {
  int t = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  t = std::min<int64_t>(t, 64);
  return (int)std::max<int64_t>(1, std::min<int64_t>(t, work_items));
}

template <class F>
void parallel_ranges(int nt, int64_t n, F&& body) {  // body(t, begin, end)
  if (nt <= 1) {
    body(0, (int64_t)0, n);
    return;
  }
  std::vector<std::thread> th;
  const int64_t per = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    const int64_t b = std::min(n, t * per), e = std::min(n, b + per);
    th.emplace_back([&, t, b, e] { body(t, b, e); });
  }
  for (auto& x : th) x.join();
}

bool read_file(const char* path, std::string& out) {
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return false;
  out.clear();
  // one read into a buffer sized from the file (streams fall back to chunked reads)
  if (std::fseek(f, 0, SEEK_END) == 0) {
    const long size = std::ftell(f);
    if (size > 0 && std::fseek(f, 0, SEEK_SET) == 0) {
      out.resize((size_t)size);
      const size_t got = std::fread(&out[0], 1, (size_t)size, f);
      out.resize(got);
    } else {
      std::fseek(f, 0, SEEK_SET);
    }
  }
  char buf[1 << 16];
  size_t got;
  while ((got = std::fread(buf, 1, sizeof(buf), f)) > 0) out.append(buf, got);
  const bool ok = !std::ferror(f);
  std::fclose(f);
  return ok;
}

// Line starts of `text` as std::getline sees them (a final line without '\n' counts,
// an empty tail after the last '\n' does not).
std::vector<int64_t> line_starts(const std::string& text) {
  std::vector<int64_t> starts;
  int64_t pos = 0;
  const int64_t n = (int64_t)text.size();
  while (pos < n) {
    starts.push_back(pos);
    const void* nl = std::memchr(text.data() + pos, '\n', (size_t)(n - pos));
    if (!nl) {
      pos = n;
      break;
    }
    pos = (const char*)nl - text.data() + 1;
  }
  starts.push_back(n);  // sentinel
  return starts;
}

std::string_view line_at(const std::string& text, const std::vector<int64_t>& st, int64_t i) {
  int64_t b = st[i], e = st[i + 1];
  if (e > b && text[e - 1] == '\n') --e;
  if (e > b && text[e - 1] == '\r') --e;
  return std::string_view(text.data() + b, (size_t)(e - b));
}

// distance_matrix.hpp:82-87
inline char* format_double(char* p, char* end, double v) {
  return std::to_chars(p, end, v).ptr;
}

// Text block size for streaming loads (DTWGPU_IO_BLOCK bytes; tests use small blocks).
int64_t env_block_bytes() {
  const char* v = std::getenv("DTWGPU_IO_BLOCK");
  const int64_t b = v && *v ? std::strtoll(v, nullptr, 10) : (int64_t)64 << 20;
  return std::max<int64_t>(b, 16);
}

struct Err {  // first error of a range, in file order
  int64_t line = -1;
  int code = 0;
  std::string msg;
  int64_t column = -1;
  bool set() const { return line >= 0; }
};

}  // namespace

extern "C" {

const char* dtwg_io_last_error(int64_t* line, int64_t* column) {
  if (line) *line = g_io_line;
  if (column) *column = g_io_column;
  return g_io_error.c_str();
}

const char* dtwg_io_last_file(void) { return g_io_file.c_str(); }

void dtwg_free(void* p) { std::free(p); }

// distance_matrix.hpp:104-122
int dtwg_save_matrix_text(const double* condensed, int64_t p, const char* path, int threads) {
  if (!path || p <= 0 || (p > 1 && !condensed))
    return io_fail(DTWG_INVALID_ARGUMENTS, "save_matrix: bad arguments");
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return io_fail(3, std::string("cannot open '") + path + "' for writing");
  auto off = [p](int64_t i) { return i * p - i * (i + 1) / 2; };
  auto dist = [&](int64_t i, int64_t j) {
    if (i > j) std::swap(i, j);
    return condensed[off(i) + (j - i - 1)];
  };
  bool ok = std::fprintf(f, "p=%lld\n", (long long)p) > 0;
  const int nt = thread_count(threads, p);
  // rows in batches; each thread formats a contiguous run of rows into its own buffer,
  // then the buffers are written in row order
  const int64_t batch = std::max<int64_t>(nt, std::min<int64_t>(p, (int64_t)nt * 64));
  std::vector<std::string> bufs(nt);
  for (int64_t r0 = 0; r0 < p && ok; r0 += batch) {
    const int64_t r1 = std::min(p, r0 + batch);
    parallel_ranges(nt, r1 - r0, [&](int t, int64_t b, int64_t e) {
      std::string& out = bufs[t];
      out.clear();
      out.reserve((size_t)((e - b) * p * 20));
      char cell[32];
      for (int64_t i = r0 + b; i < r0 + e; ++i) {
        for (int64_t j = 0; j < p; ++j) {
          if (j > 0) out.push_back(',');
          if (i == j) {
            out.push_back('0');
          } else {
            char* q = format_double(cell, cell + sizeof(cell), dist(i, j));
            out.append(cell, (size_t)(q - cell));
          }
        }
        out.push_back('\n');
      }
    });
    for (int t = 0; t < nt && ok; ++t)
      ok = bufs[t].empty() || std::fwrite(bufs[t].data(), 1, bufs[t].size(), f) == bufs[t].size();
  }
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return io_fail(3, std::string("failed writing '") + path + "'");
  return DTWG_OK;
}

// distance_matrix.hpp:127-192. On success *condensed_out is malloc'ed (dtwg_free).
// The file is read in blocks of whole lines (bounded memory: the matrix plus one block of
// text and its parsed rows -- c3-sized files are ~10 GB of text); each block's rows are
// parsed by several threads and checked against the rows before them; the first error in
// file order is the one the sequential reference raises.
int dtwg_load_matrix_text(const char* path, int threads, int64_t* p_out, double** condensed_out) {
  if (!path || !p_out || !condensed_out)
    return io_fail(DTWG_INVALID_ARGUMENTS, "load_matrix: bad arguments");
  *condensed_out = nullptr;
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return io_fail(3, std::string("cannot open '") + path + "' for reading");
  struct Closer {
    std::FILE* f;
    ~Closer() { std::fclose(f); }
  } closer{f};
  auto fv = [](int64_t line, const std::string& m) { return io_fail(9, m, line); };
  // block reader: text holds [consumed, size) of not-yet-parsed data
  std::string text;
  size_t head = 0;
  bool eof = false;
  const size_t kBlock = (size_t)env_block_bytes();
  auto refill = [&]() -> bool {  // append one block (no erase: spans stay valid)
    if (eof) return true;
    const size_t old = text.size();
    text.resize(old + kBlock);
    const size_t got = std::fread(&text[old], 1, kBlock, f);
    text.resize(old + got);
    if (got < kBlock) {
      if (std::ferror(f)) return false;
      eof = true;
    }
    return true;
  };
  // next complete line [b, e) after head (without '\n'); false at EOF with nothing left
  auto next_line = [&](size_t& b, size_t& e, bool& had_nl) -> bool {
    for (;;) {
      const void* nl = std::memchr(text.data() + head, '\n', text.size() - head);
      if (nl) {
        b = head;
        e = (size_t)((const char*)nl - text.data());
        head = e + 1;
        had_nl = true;
        return true;
      }
      if (eof) {
        if (head >= text.size()) return false;
        b = head;
        e = text.size();
        head = e;
        had_nl = false;
        return true;
      }
      if (!refill()) return false;
    }
  };
  auto strip_cr = [&](size_t b, size_t e) {
    if (e > b && text[e - 1] == '\r') --e;
    return std::string_view(text.data() + b, e - b);
  };
  size_t lb = 0, le = 0;
  bool nl = false;
  if (!refill()) return io_fail(3, std::string("failed reading '") + path + "'");
  if (!next_line(lb, le, nl)) return fv(1, "missing 'p=<count>' header");
  const std::string head_line(strip_cr(lb, le));
  if (head_line.rfind("p=", 0) != 0) return fv(1, "expected 'p=<count>' header");
  std::size_t pz = 0;
  {
    const char* b0 = head_line.data() + 2;
    const char* e0 = head_line.data() + head_line.size();
    const auto r = std::from_chars(b0, e0, pz);
    if (r.ec != std::errc() || r.ptr != e0 || pz == 0)
      return fv(1, "header count '" + head_line.substr(2) + "' is not a positive integer");
  }
  const int64_t p = (int64_t)pz;
  const int64_t total = p * (p - 1) / 2;
  double* cond = (double*)std::malloc((size_t)std::max<int64_t>(total, 1) * sizeof(double));
  if (!cond) return io_fail(3, "out of host memory");
  struct Freer {
    double*& c;
    bool keep = false;
    ~Freer() {
      if (!keep) std::free(c);
    }
  } freer{cond};
  auto off = [p](int64_t i) { return i * p - i * (i + 1) / 2; };
  const int nt0 = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  // rows per block: about one block of text, at least the threads
  const int64_t rows_per_block = std::max<int64_t>(
      std::min<int64_t>(nt0, 64), std::min<int64_t>(p, (int64_t)(kBlock / (size_t)(8 * p + 1)) + 1));
  std::vector<double> rows((size_t)(rows_per_block * p));
  std::vector<std::pair<size_t, size_t>> spans((size_t)rows_per_block);
  struct RowErr {
    int kind = 0;  // 0 none, 1 syntax/count, 2 value error at column `col`
    int64_t col = 0;
    std::string msg;
  };
  std::vector<RowErr> rerr((size_t)rows_per_block);
  std::vector<int64_t> asym((size_t)rows_per_block);
  int64_t done = 0;
  while (done < p) {
    // drop the text already parsed, then gather the next block of complete lines
    text.erase(0, head);
    head = 0;
    int64_t nb = 0;
    while (nb < rows_per_block && done + nb < p) {
      if (!next_line(lb, le, nl)) break;
      spans[(size_t)nb++] = {lb, le};
    }
    if (nb == 0) {
      if (!eof) return io_fail(3, std::string("failed reading '") + path + "'");
      return fv(done + 2, "expected " + std::to_string(p) + " matrix rows");
    }
    const int nt = thread_count(threads, nb);
    // phase 1: tokenise + diagonal/finiteness; upper triangle into cond
    parallel_ranges(nt, nb, [&](int, int64_t b0, int64_t e0) {
      for (int64_t r = b0; r < e0; ++r) {
        const int64_t i = done + r;
        double* row = &rows[(size_t)(r * p)];
        const std::string_view line = strip_cr(spans[(size_t)r].first, spans[(size_t)r].second);
        RowErr& E = rerr[(size_t)r];
        E = RowErr{};
        asym[(size_t)r] = -1;
        int64_t cell = 0;
        size_t start = 0;
        while (true) {
          const size_t comma = line.find(',', start);
          const std::string_view tok =
              line.substr(start, (comma == std::string_view::npos ? line.size() : comma) - start);
          if (cell >= p) {
            E = RowErr{1, 0, "row has more than " + std::to_string(p) + " cells"};
            break;
          }
          double v = 0.0;
          const auto res = std::from_chars(tok.data(), tok.data() + tok.size(), v);
          if (res.ec != std::errc() || res.ptr != tok.data() + tok.size() || tok.empty()) {
            E = RowErr{1, 0, "cell '" + std::string(tok) + "' is not a decimal value"};
            break;
          }
          row[cell++] = v;
          if (comma == std::string_view::npos) break;
          start = comma + 1;
        }
        if (E.kind == 0 && cell != p)
          E = RowErr{1, 0, "row has " + std::to_string(cell) + " cells, expected " + std::to_string(p)};
        if (E.kind != 0) continue;
        for (int64_t j = 0; j < p; ++j) {
          const double v = row[j];
          if (i == j) {
            if (v != 0.0) {
              E = RowErr{2, j, "diagonal entry must be exactly 0"};
              break;
            }
            continue;
          }
          if (!(std::isfinite(v) && v >= 0.0)) {
            E = RowErr{2, j, "entries must be finite and non-negative"};
            break;
          }
          if (j > i) cond[off(i) + (j - i - 1)] = v;
        }
      }
    });
    // first row of the block with a syntax error: rows after it are never compared
    int64_t stop = nb;
    for (int64_t r = 0; r < nb; ++r)
      if (rerr[(size_t)r].kind != 0) {
        stop = r + 1;
        break;
      }
    // phase 2: symmetry (row i, column j < i, against row j's stored value); a row with
    // a value error at column j' competes by column (j < j' wins)
    parallel_ranges(thread_count(threads, stop), stop, [&](int, int64_t b0, int64_t e0) {
      for (int64_t r = b0; r < e0; ++r) {
        const RowErr& E = rerr[(size_t)r];
        if (E.kind == 1) continue;
        const int64_t i = done + r;
        const double* row = &rows[(size_t)(r * p)];
        const int64_t jmax = E.kind == 2 ? std::min<int64_t>(E.col, i) : i;
        for (int64_t j = 0; j < jmax; ++j)
          if (row[j] != cond[off(j) + (i - j - 1)]) {
            asym[(size_t)r] = j;
            break;
          }
      }
    });
    for (int64_t r = 0; r < stop; ++r) {
      const int64_t i = done + r;
      if (asym[(size_t)r] >= 0)
        return fv(i + 2, "matrix is not symmetric at (" + std::to_string(i) + ", " +
                             std::to_string(asym[(size_t)r]) + ")");
      if (rerr[(size_t)r].kind != 0) return fv(i + 2, rerr[(size_t)r].msg);
    }
    done += nb;
  }
  // the reference reads the next line raw here (no '\r' stripping): "\r" alone is content
  if (next_line(lb, le, nl) && le > lb) return fv(p + 2, "unexpected content after the last matrix row");
  freer.keep = true;
  *p_out = p;
  *condensed_out = cond;
  return DTWG_OK;
}

// Binary sidecar: "DTWGMAT1" | uint64 p | p(p-1)/2 little-endian doubles (row-major upper
// triangle, the reference's condensed layout). Loads validate like from_condensed.
int dtwg_save_matrix_binary(const double* condensed, int64_t p, const char* path) {
  if (!path || p <= 0 || (p > 1 && !condensed))
    return io_fail(DTWG_INVALID_ARGUMENTS, "save_matrix_binary: bad arguments");
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return io_fail(3, std::string("cannot open '") + path + "' for writing");
  const uint64_t pp = (uint64_t)p;
  const int64_t total = p * (p - 1) / 2;
  bool ok = std::fwrite("DTWGMAT1", 1, 8, f) == 8 && std::fwrite(&pp, 8, 1, f) == 1;
  if (ok && total > 0) ok = std::fwrite(condensed, 8, (size_t)total, f) == (size_t)total;
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return io_fail(3, std::string("failed writing '") + path + "'");
  return DTWG_OK;
}

int dtwg_load_matrix_binary(const char* path, int64_t* p_out, double** condensed_out) {
  if (!path || !p_out || !condensed_out)
    return io_fail(DTWG_INVALID_ARGUMENTS, "load_matrix_binary: bad arguments");
  *condensed_out = nullptr;
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return io_fail(3, std::string("cannot open '") + path + "' for reading");
  char magic[8];
  uint64_t pp = 0;
  if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, "DTWGMAT1", 8) != 0 ||
      std::fread(&pp, 8, 1, f) != 1 || pp == 0 || pp > (1ull << 31)) {
    std::fclose(f);
    return io_fail(9, "not a dtwgpu binary matrix (bad header)", 1);
  }
  const int64_t p = (int64_t)pp, total = p * (p - 1) / 2;
  double* cond = (double*)std::malloc((size_t)std::max<int64_t>(total, 1) * 8);
  if (!cond) {
    std::fclose(f);
    return io_fail(3, "out of host memory");
  }
  const bool short_read = total > 0 && std::fread(cond, 8, (size_t)total, f) != (size_t)total;
  char extra;
  const bool trailing = std::fread(&extra, 1, 1, f) == 1;
  std::fclose(f);
  if (short_read || trailing) {
    std::free(cond);
    return io_fail(9, short_read ? "binary matrix is truncated" : "binary matrix has trailing bytes", 1);
  }
  for (int64_t t = 0; t < total; ++t) {  // distance_matrix.hpp:34-38
    if (!(std::isfinite(cond[t]) && cond[t] >= 0.0)) {
      std::free(cond);
      return io_fail(DTWG_DISTANCE_MATRIX_INVALID, "distances must be finite and non-negative");
    }
  }
  *p_out = p;
  *condensed_out = cond;
  return DTWG_OK;
}

// ---- ingest (csv.hpp:55-106) ----------------------------------------------------------
struct dtwg_dataset {
  std::vector<double> samples;
  std::vector<int64_t> offsets{0};
  std::vector<std::string> ids;
};

int dtwg_ingest_csv(const char* const* paths, int64_t npaths, int label_column, int delimiter,
                    int threads, dtwg_dataset** out) {
  if (!out || (npaths > 0 && !paths))
    return io_fail(DTWG_INVALID_ARGUMENTS, "ingest: bad arguments");
  *out = nullptr;
  auto ds = std::make_unique<dtwg_dataset>();
  std::unordered_map<std::string, size_t> name_uses;
  for (int64_t fi = 0; fi < npaths; ++fi) {
    const std::string path = paths[fi];
    std::string text;
    {
      std::FILE* f = std::fopen(path.c_str(), "rb");
      if (!f) return io_fail(3, "cannot open '" + path + "' for reading");
      std::fclose(f);
      if (!read_file(path.c_str(), text)) return io_fail(3, "failed reading '" + path + "'");
    }
    std::string name = path.substr(path.find_last_of('/') == std::string::npos
                                       ? 0
                                       : path.find_last_of('/') + 1);
    const size_t uses = ++name_uses[name];
    if (uses > 1) name += "#" + std::to_string(uses);
    char delim = delimiter > 0 ? (char)delimiter : ',';
    // std::filesystem::path::extension(): a leading dot of the file name is not one
    if (delimiter <= 0 && name.size() > 4 && path.compare(path.size() - 4, 4, ".tsv") == 0)
      delim = '\t';
    const std::vector<int64_t> st = line_starts(text);
    const int64_t nlines = (int64_t)st.size() - 1;
    const int nt = thread_count(threads, std::max<int64_t>(1, nlines / 256));
    struct Part {
      std::vector<double> samples;
      std::vector<int64_t> lens;
      Err err;
      std::string err_file;
    };
    std::vector<Part> parts(nt);
    parallel_ranges(nt, nlines, [&](int t, int64_t b, int64_t e) {
      Part& P = parts[t];
      std::vector<std::string_view> cells;
      auto trim = [](std::string_view c) {
        while (!c.empty() && (c.front() == ' ' || c.front() == '\t')) c.remove_prefix(1);
        while (!c.empty() && (c.back() == ' ' || c.back() == '\t')) c.remove_suffix(1);
        return c;
      };
      for (int64_t li = b; li < e; ++li) {
        const int64_t line_no = li + 1;
        const std::string_view line = line_at(text, st, li);
        cells.clear();
        size_t start = 0;
        while (true) {
          const size_t pos = line.find(delim, start);
          cells.push_back(line.substr(start, (pos == std::string_view::npos ? line.size() : pos) - start));
          if (pos == std::string_view::npos) break;
          start = pos + 1;
        }
        while (!cells.empty() && trim(cells.back()).empty()) cells.pop_back();
        const size_t first = (label_column && !cells.empty()) ? 1 : 0;
        const size_t before = P.samples.size();
        for (size_t c = first; c < cells.size(); ++c) {
          const std::string_view tr = trim(cells[c]);
          if (tr.empty()) {
            P.err = Err{line_no, 4, "empty cell before the last sample", (int64_t)c + 1};
            return;
          }
          std::string_view digits = tr;
          if (digits.front() == '+') digits.remove_prefix(1);
          double v = 0.0;
          const auto r = std::from_chars(digits.data(), digits.data() + digits.size(), v);
          if (r.ec != std::errc() || r.ptr != digits.data() + digits.size()) {
            P.err = Err{line_no, 4, "cell '" + std::string(tr) + "' is not numeric", (int64_t)c + 1};
            return;
          }
          P.samples.push_back(v);
        }
        const size_t len = P.samples.size() - before;
        if (len == 0) {
          P.err = Err{line_no, 6, "row contains no samples"};
          return;
        }
        for (size_t q = before; q < P.samples.size(); ++q) {  // time_series.hpp:24-33
          if (!std::isfinite(P.samples[q])) {
            P.err = Err{line_no, 5, "series contains a non-finite sample"};
            return;
          }
        }
        P.lens.push_back((int64_t)len);
      }
    });
    for (auto& P : parts) {
      if (P.err.set()) {
        const int64_t ln = P.err.line;
        if (P.err.code == 4)
          return io_fail(4, path + ":" + std::to_string(ln) + ":" + std::to_string(P.err.column) +
                                ": " + P.err.msg,
                         ln, P.err.column, path);
        if (P.err.code == 6)
          return io_fail(6, path + ":" + std::to_string(ln) + ": row contains no samples", ln, -1,
                         path);
        return io_fail(5, "series '" + name + ":" + std::to_string(ln) + "': " + P.err.msg, ln,
                       -1, name + ":" + std::to_string(ln));
      }
    }
    int64_t line_no = 0;
    for (auto& P : parts) {
      size_t pos = 0;
      for (int64_t len : P.lens) {
        ++line_no;
        ds->ids.push_back(name + ":" + std::to_string(line_no));
        ds->offsets.push_back(ds->offsets.back() + len);
        pos += (size_t)len;
      }
      ds->samples.insert(ds->samples.end(), P.samples.begin(), P.samples.end());
    }
  }
  if (ds->ids.empty()) return io_fail(DTWG_EMPTY_DATASET, "dataset contains no series");
  *out = ds.release();
  return DTWG_OK;
}

// runner.hpp:82-95, per series in parallel (each series' arithmetic is sequential).
int dtwg_z_normalize(double* samples, const int64_t* offsets, int64_t p, int threads) {
  if (p < 0 || (p > 0 && (!samples || !offsets)))
    return io_fail(DTWG_INVALID_ARGUMENTS, "z_normalize: bad arguments");
  const int nt = thread_count(threads, std::max<int64_t>(1, p / 64));
  parallel_ranges(nt, p, [&](int, int64_t b, int64_t e) {
    for (int64_t i = b; i < e; ++i) {
      double* v = samples + offsets[i];
      const int64_t len = offsets[i + 1] - offsets[i];
      const double n = (double)len;
      double mean = 0.0;
      for (int64_t t = 0; t < len; ++t) mean += v[t];
      mean /= n;
      double variance = 0.0;
      for (int64_t t = 0; t < len; ++t) variance += (v[t] - mean) * (v[t] - mean);
      const double stddev = std::sqrt(variance / n);
      for (int64_t t = 0; t < len; ++t) v[t] = stddev > 0.0 ? (v[t] - mean) / stddev : 0.0;
    }
  });
  return DTWG_OK;
}

int64_t dtwg_dataset_size(const dtwg_dataset* ds) { return ds ? (int64_t)ds->ids.size() : 0; }
double* dtwg_dataset_samples(dtwg_dataset* ds) { return ds ? ds->samples.data() : nullptr; }
const int64_t* dtwg_dataset_offsets(const dtwg_dataset* ds) {
  return ds ? ds->offsets.data() : nullptr;
}
const char* dtwg_dataset_id(const dtwg_dataset* ds, int64_t i) {
  return (ds && i >= 0 && i < (int64_t)ds->ids.size()) ? ds->ids[(size_t)i].c_str() : nullptr;
}
void dtwg_dataset_free(dtwg_dataset* ds) { delete ds; }

}  // extern "C"
