// typefile.cpp -- the datatype description language of the reference's
// front end (typefile.hpp:17-260), parsed into engine definitions.
//
//   # comment
//   type <name> = named(<kind>)
//   type <name> = contiguous(<count>, <ref>)
//   type <name> = vector(<count>, <blocklength>, <stride>, <ref>)
//   type <name> = hvector(<count>, <blocklength>, <stride_bytes>, <ref>)
//   type <name> = subarray(<ndims>, [<sizes>], [<subsizes>], [<offsets>], <ref>)
//   commit <name>
//
// Beyond the reference's grammar (the engine's MPI indexed/struct/resized
// constructors; a reference parser rejects these lines as unknown):
//   type <name> = indexed([<blocklengths>], [<displs in inner extents>], <ref>)
//   type <name> = hindexed([<blocklengths>], [<displs in bytes>], <ref>)
//   type <name> = struct([<blocklengths>], [<displs in bytes>], [<refs>])
//   type <name> = resized(<ref>, <lb>, <extent>)
//
// <kind> is byte/int/float/double; <ref> a kind or an earlier name. Exactly
// one commit, as the last statement. Every diagnostic is a ParseError
// (SP_ERR_PARSE) prefixed "line N: "; constructor argument errors
// (InvalidArgument / UnsupportedOrder) are re-raised as ParseError with the
// line number, as typefile.hpp:244-250 does.
#include <cctype>
#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <string_view>
#include <vector>

#include "core.hpp"
#include "guard.hpp"

namespace spb {
namespace {

std::string_view strip(std::string_view s) {
  while (!s.empty() && std::isspace(static_cast<unsigned char>(s.front()))) s.remove_prefix(1);
  while (!s.empty() && std::isspace(static_cast<unsigned char>(s.back()))) s.remove_suffix(1);
  return s;
}

int kind_of(std::string_view s) {
  static const char *const names[4] = {"byte", "int", "float", "double"}; // NamedKind order
  for (int k = 0; k < 4; ++k)
    if (s == names[k]) return k;
  return -1;
}

bool identifier(std::string_view s) {
  if (s.empty() || !(std::isalpha(static_cast<unsigned char>(s[0])) || s[0] == '_')) return false;
  for (char c : s)
    if (!(std::isalnum(static_cast<unsigned char>(c)) || c == '_')) return false;
  return true;
}

class Parser {
public:
  DefPtr run(const std::string &text, std::string &name_out) {
    size_t pos = 0;
    bool done = false;
    while (pos <= text.size()) {
      size_t nl = text.find('\n', pos);
      if (nl == std::string::npos) nl = text.size();
      std::string_view line(text.data() + pos, nl - pos);
      pos = nl + 1;
      ++lineno_;
      if (const size_t h = line.find('#'); h != std::string_view::npos) line = line.substr(0, h);
      line = strip(line);
      if (line.empty()) {
        if (nl == text.size()) break;
        continue;
      }
      if (done) error("statement after commit");
      statement(line, name_out, done);
      if (nl == text.size()) break;
    }
    if (!done) fail(SP_ERR_PARSE, "type file has no commit statement");
    return committed_;
  }

private:
  int lineno_ = 0;
  std::map<std::string, DefPtr, std::less<>> names_;
  DefPtr committed_;

  [[noreturn]] void error(const std::string &msg) const {
    fail(SP_ERR_PARSE, "line " + std::to_string(lineno_) + ": " + msg);
  }

  // first whitespace-delimited word and the rest
  static std::string_view word(std::string_view &s) {
    s = strip(s);
    size_t e = 0;
    while (e < s.size() && !std::isspace(static_cast<unsigned char>(s[e]))) ++e;
    std::string_view w = s.substr(0, e);
    s = strip(s.substr(e));
    return w;
  }

  void statement(std::string_view line, std::string &name_out, bool &done) {
    std::string_view rest = line;
    const std::string_view head = word(rest);
    if (head == "commit") {
      const std::string_view nm = word(rest);
      if (nm.empty() || !rest.empty()) error("commit takes exactly one name");
      auto it = names_.find(nm);
      if (it == names_.end()) error("undefined type '" + std::string(nm) + "'");
      committed_ = it->second;
      name_out = std::string(nm);
      done = true;
      return;
    }
    if (head != "type") error("expected 'type' or 'commit', got '" + std::string(head) + "'");
    const size_t eq = line.find('=');
    if (eq == std::string_view::npos) error("expected 'type <name> = <constructor>'");
    const std::string_view nm = strip(line.substr(4, eq - 4));
    if (!identifier(nm)) error("invalid type name '" + std::string(nm) + "'");
    if (kind_of(nm) >= 0 || names_.count(nm)) error("type name '" + std::string(nm) + "' is already in use");
    const std::string_view rhs = strip(line.substr(eq + 1));
    const size_t open = rhs.find('(');
    if (open == std::string_view::npos || rhs.empty() || rhs.back() != ')')
      error("expected '<constructor>(...)'");
    const std::string ctor(strip(rhs.substr(0, open)));
    const std::vector<std::string_view> args = split(rhs.substr(open + 1, rhs.size() - open - 2));
    auto arity = [&](size_t n) {
      if (args.size() != n) error(ctor + " takes " + std::to_string(n) + " arguments");
    };
    DefPtr def;
    try {
      if (ctor == "named") {
        arity(1);
        const int k = kind_of(args[0]);
        if (k < 0) error("unknown kind '" + std::string(args[0]) + "'");
        def = make_named(k);
      } else if (ctor == "contiguous") {
        arity(2);
        def = make_contiguous(integer(args[0]), resolve(args[1]));
      } else if (ctor == "vector" || ctor == "hvector") {
        arity(4);
        const int64_t c = integer(args[0]), bl = integer(args[1]), st = integer(args[2]);
        def = ctor == "vector" ? make_vector(c, bl, st, resolve(args[3])) : make_hvector(c, bl, st, resolve(args[3]));
      } else if (ctor == "subarray") {
        arity(5);
        const int64_t nd = integer(args[0]);
        const auto sizes = list(args[1]), subs = list(args[2]), offs = list(args[3]);
        DefPtr inner = resolve(args[4]);
        // type_def.hpp:168-175: the list lengths are checked against ndims
        if (nd >= 1 && (static_cast<int64_t>(sizes.size()) != nd || static_cast<int64_t>(subs.size()) != nd ||
                        static_cast<int64_t>(offs.size()) != nd))
          fail(SP_ERR_INVALID_ARGUMENT, "subarray: sizes/subsizes/offsets must have ndims entries");
        def = make_subarray(nd, sizes.data(), subs.data(), offs.data(), std::move(inner), SP_ORDER_C);
      } else if (ctor == "indexed" || ctor == "hindexed") {
        arity(3);
        const auto bl = list(args[0]);
        auto d = list(args[1]);
        DefPtr inner = resolve(args[2]);
        if (bl.size() != d.size()) fail(SP_ERR_INVALID_ARGUMENT, ctor + ": one displacement per block");
        if (ctor == "indexed")
          for (int64_t &x : d) x *= inner->extent;
        def = make_indexed(static_cast<int64_t>(bl.size()), bl.data(), d.data(), std::move(inner));
      } else if (ctor == "struct") {
        arity(3);
        const auto bl = list(args[0]), d = list(args[1]);
        std::vector<DefPtr> members;
        for (std::string_view r : items(args[2])) members.push_back(resolve(r));
        if (bl.size() != d.size() || bl.size() != members.size())
          fail(SP_ERR_INVALID_ARGUMENT, "struct: one displacement and one type per block");
        def = make_struct(static_cast<int64_t>(bl.size()), bl.data(), d.data(), members);
      } else if (ctor == "resized") {
        arity(3);
        def = make_resized(resolve(args[0]), integer(args[1]), integer(args[2]));
      } else {
        error("unknown constructor '" + ctor + "'");
      }
    } catch (const Error &e) {
      if (e.code == SP_ERR_INVALID_ARGUMENT || e.code == SP_ERR_UNSUPPORTED_ORDER) error(e.msg);
      throw;
    }
    names_.emplace(std::string(nm), std::move(def));
  }

  // top-level commas; [...] nests
  std::vector<std::string_view> split(std::string_view s) const {
    std::vector<std::string_view> out;
    int depth = 0;
    size_t from = 0;
    for (size_t i = 0; i < s.size(); ++i) {
      if (s[i] == '[') {
        ++depth;
      } else if (s[i] == ']') {
        if (--depth < 0) error("unbalanced ']'");
      } else if (s[i] == ',' && depth == 0) {
        out.push_back(strip(s.substr(from, i - from)));
        from = i + 1;
      }
    }
    if (depth != 0) error("unbalanced '['");
    out.push_back(strip(s.substr(from)));
    return out;
  }

  int64_t integer(std::string_view s) const {
    const std::string t(s);
    char *end = nullptr;
    errno = 0;
    const long long v = std::strtoll(t.c_str(), &end, 10);
    if (t.empty() || end != t.c_str() + t.size()) error("expected an integer, got '" + t + "'");
    return v;
  }

  // the items of a [..] list ("[]" is empty)
  std::vector<std::string_view> items(std::string_view s) const {
    if (s.size() < 2 || s.front() != '[' || s.back() != ']')
      error("expected a [..] list, got '" + std::string(s) + "'");
    if (strip(s.substr(1, s.size() - 2)).empty()) return {};
    return split(s.substr(1, s.size() - 2));
  }

  std::vector<int64_t> list(std::string_view s) const {
    std::vector<int64_t> out;
    for (std::string_view item : items(s)) out.push_back(integer(item));
    return out;
  }

  DefPtr resolve(std::string_view ref) const {
    if (const int k = kind_of(ref); k >= 0) return make_named(k);
    auto it = names_.find(ref);
    if (it == names_.end()) error("undefined type '" + std::string(ref) + "'");
    return it->second;
  }
};

} // namespace

DefPtr parse_type_file(const std::string &text, std::string &name) {
  Parser p;
  return p.run(text, name);
}

} // namespace spb

extern "C" sp_status sp_typefile_parse(const char *text, sp_type *out, char *name, int64_t name_cap) {
  return spb::guarded([&] {
    spb::need(text);
    spb::need(out);
    std::string nm;
    spb::DefPtr def = spb::parse_type_file(text, nm);
    if (name && name_cap > 0) {
      const size_t n = std::min<size_t>(nm.size(), static_cast<size_t>(name_cap - 1));
      std::memcpy(name, nm.data(), n);
      name[n] = '\0';
    }
    *out = spb::registry().add(std::move(def));
  });
}
