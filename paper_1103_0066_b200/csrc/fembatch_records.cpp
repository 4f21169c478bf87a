// fembatch_records.cpp -- SURVEY 8f row F4 (benchmark records) and row A16
// (store checksum): the record formats the reference's tooling reads and
// writes (include/fembatch/bench.hpp; formats of src/bench.cpp:231-384),
// implemented from the format itself, not from the reference's code:
//
//   CSV  : one header line, then one line per record; 15 columns in a fixed
//          order; text and on/off fields double-quoted with "" escapes;
//          integers in decimal; reals with 17 significant digits (%.17g).
//   JSON : an array of objects, two-space indent, one key per line in the
//          column order; reals in shortest round-trip form with a ".0" kept
//          on integral values, non-finite reals as null; an empty table is
//          "[]".
//
// One column table (kColumns) drives the writer, the reader and the JSON
// writer, so the three cannot disagree on order, names or field kinds.
// Byte-exactness against files the unmodified reference wrote is tested
// (tests/test_storeio.py, tests/cpp/test_api.cpp).
#include <charconv>
#include <cmath>
#include <cstdio>
#include <istream>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <variant>
#include <vector>

#include "../../include/fembatch_b200.hpp"

namespace fembatch {

namespace {

using Member = std::variant<std::string BenchRecord::*, int BenchRecord::*, std::int64_t BenchRecord::*,
                            bool BenchRecord::*, double BenchRecord::*>;

struct Column {
  const char* name;  // CSV header field and JSON key
  Member field;
};

constexpr int kNumColumns = 15;
const Column kColumns[kNumColumns] = {
    {"operator", &BenchRecord::op},          {"dim", &BenchRecord::dim},
    {"num_elements", &BenchRecord::num_elements}, {"batch_size", &BenchRecord::batch_size},
    {"concurrent", &BenchRecord::concurrent}, {"interleave", &BenchRecord::interleave},
    {"unroll", &BenchRecord::unroll},         {"precision", &BenchRecord::precision},
    {"workers", &BenchRecord::workers},       {"reps", &BenchRecord::reps},
    {"seconds_min", &BenchRecord::seconds_min}, {"seconds_mean", &BenchRecord::seconds_mean},
    {"gflops", &BenchRecord::gflops},         {"checksum", &BenchRecord::checksum},
    {"status", &BenchRecord::status},
};

std::string header_line()
{
  std::string h;
  for (int c = 0; c < kNumColumns; ++c)
    h += (c ? "," : "") + std::string(kColumns[c].name);
  return h;
}

const std::string& flag_text(bool on)
{
  static const std::string t[2] = {"off", "on"};
  return t[on ? 1 : 0];
}

// ---- CSV cells
std::string csv_text(const std::string& s)
{
  std::string o(1, '"');
  for (char ch : s)
    o.append(ch == '"' ? 2 : 1, ch);
  o += '"';
  return o;
}

std::string csv_real(double v)
{
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

std::string csv_cell(const BenchRecord& r, const Member& m)
{
  return std::visit(
      [&](auto pm) -> std::string
      {
        using T = std::decay_t<decltype(r.*pm)>;
        if constexpr (std::is_same_v<T, std::string>)
          return csv_text(r.*pm);
        else if constexpr (std::is_same_v<T, bool>)
          return csv_text(flag_text(r.*pm));
        else if constexpr (std::is_same_v<T, double>)
          return csv_real(r.*pm);
        else
          return std::to_string(r.*pm);
      },
      m);
}

// Splits one CSV line into cells: quotes toggle a quoted run, "" inside a
// run is a literal quote, commas outside runs separate cells.
std::vector<std::string> split_cells(const std::string& line)
{
  std::vector<std::string> cells(1);
  bool quoted = false;
  for (std::size_t i = 0; i < line.size(); ++i)
  {
    const char ch = line[i];
    if (ch == '"')
    {
      if (quoted && i + 1 < line.size() && line[i + 1] == '"')
        cells.back() += line[++i];
      else
        quoted = !quoted;
    }
    else if (ch == ',' && !quoted)
      cells.emplace_back();
    else
      cells.back() += ch;
  }
  return cells;
}

void parse_cell(BenchRecord& r, const Member& m, const std::string& text)
{
  std::visit(
      [&](auto pm)
      {
        using T = std::decay_t<decltype(r.*pm)>;
        if constexpr (std::is_same_v<T, std::string>)
          r.*pm = text;
        else if constexpr (std::is_same_v<T, bool>)
        {
          if (text != flag_text(true) && text != flag_text(false))
            throw std::runtime_error("bad flag field '" + text + "' (want on/off)");
          r.*pm = text == flag_text(true);
        }
        else if constexpr (std::is_same_v<T, double>)
          r.*pm = std::stod(text);
        else if constexpr (std::is_same_v<T, std::int64_t>)
          r.*pm = std::stoll(text);
        else
          r.*pm = std::stoi(text);
      },
      m);
}

// ---- JSON values
std::string json_text(const std::string& s)
{
  std::string o(1, '"');
  for (unsigned char ch : s)
  {
    const char* esc = nullptr;
    switch (ch)
    {
    case '"': esc = "\\\""; break;
    case '\\': esc = "\\\\"; break;
    case '\b': esc = "\\b"; break;
    case '\f': esc = "\\f"; break;
    case '\n': esc = "\\n"; break;
    case '\r': esc = "\\r"; break;
    case '\t': esc = "\\t"; break;
    default: break;
    }
    if (esc)
      o += esc;
    else if (ch < 0x20)
    {
      char buf[8];
      std::snprintf(buf, sizeof buf, "\\u%04x", ch);
      o += buf;
    }
    else
      o += static_cast<char>(ch);
  }
  o += '"';
  return o;
}

std::string json_real(double v)
{
  if (!std::isfinite(v))
    return "null";
  char buf[64];
  const auto end = std::to_chars(buf, buf + sizeof buf, v).ptr;  // shortest round trip
  std::string s(buf, end);
  if (s.find_first_of(".e") == std::string::npos)
    s += ".0";
  return s;
}

std::string json_value(const BenchRecord& r, const Member& m)
{
  return std::visit(
      [&](auto pm) -> std::string
      {
        using T = std::decay_t<decltype(r.*pm)>;
        if constexpr (std::is_same_v<T, std::string>)
          return json_text(r.*pm);
        else if constexpr (std::is_same_v<T, bool>)
          return json_text(flag_text(r.*pm));
        else if constexpr (std::is_same_v<T, double>)
          return json_real(r.*pm);
        else
          return std::to_string(r.*pm);
      },
      m);
}

}  // namespace

const char* const csv_header = []
{
  static const std::string h = header_line();
  return h.c_str();
}();

void write_csv(std::ostream& os, const std::vector<BenchRecord>& records)
{
  os << csv_header << '\n';
  for (const BenchRecord& r : records)
  {
    for (int c = 0; c < kNumColumns; ++c)
      os << (c ? "," : "") << csv_cell(r, kColumns[c].field);
    os << '\n';
  }
}

std::vector<BenchRecord> read_csv(std::istream& is)
{
  std::vector<BenchRecord> records;
  std::string line;
  bool header_seen = false;
  while (std::getline(is, line))
  {
    if (!line.empty() && line.back() == '\r')  // CRLF files
      line.pop_back();
    if (!header_seen)
    {
      if (line != csv_header)
        throw std::runtime_error("unrecognized benchmark table header");
      header_seen = true;
      continue;
    }
    if (line.empty())
      continue;
    const std::vector<std::string> cells = split_cells(line);
    if (static_cast<int>(cells.size()) != kNumColumns)
      throw std::runtime_error("benchmark table row has " + std::to_string(cells.size()) + " fields, expected "
                               + std::to_string(kNumColumns));
    BenchRecord r;
    for (int c = 0; c < kNumColumns; ++c)
      parse_cell(r, kColumns[c].field, cells[c]);
    records.push_back(std::move(r));
  }
  if (!header_seen)
    throw std::runtime_error("empty benchmark table");
  return records;
}

void write_json(std::ostream& os, const std::vector<BenchRecord>& records)
{
  if (records.empty())
  {
    os << "[]\n";
    return;
  }
  os << "[\n";
  for (std::size_t i = 0; i < records.size(); ++i)
  {
    os << "  {\n";
    for (int c = 0; c < kNumColumns; ++c)
      os << "    \"" << kColumns[c].name << "\": " << json_value(records[i], kColumns[c].field)
         << (c + 1 < kNumColumns ? ",\n" : "\n");
    os << "  }" << (i + 1 < records.size() ? ",\n" : "\n");
  }
  os << "]\n";
}

// ---- A16: consumers of the store

// Sum of every real element-matrix entry in element order, in double
// (padding slots excluded); the benchmark record's checksum column.
double store_checksum(const ElementMatrixStore& store)
{
  const std::int64_t nk = static_cast<std::int64_t>(store.krows) * store.krows;
  double sum = 0.0;
  // the store is element-major (element_matrix_index(e, 0, 0) = e * nk for
  // every batch size / concurrency), so the real entries are its prefix
  for (std::int64_t t = 0; t < store.num_elements * nk; ++t)
    sum += scalar_array_at(store.data, t);
  return sum;
}

// w = 1 + x_0 of each cell vertex: the nodal coefficient field the
// reference's tooling integrates the weighted Laplacian with.
CoefficientField default_coefficient_field(const Mesh& mesh)
{
  CoefficientField f;
  f.num_basis_funcs = mesh.dim + 1;
  f.values.reserve(static_cast<std::size_t>(mesh.num_elements()) * f.num_basis_funcs);
  for (std::int64_t e = 0; e < mesh.num_elements(); ++e)
    for (int k = 0; k < f.num_basis_funcs; ++k)
      f.values.push_back(1.0 + mesh.vertex(mesh.cell_vertex(e, k), 0));
  return f;
}

double default_tolerance(Precision p) { return p == Precision::f32 ? 5e-5 : 1e-12; }

}  // namespace fembatch
