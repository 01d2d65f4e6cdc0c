// rules.cpp -- Tier-1 rule compiler (host C++).  See rules.hpp.
//
// Pipeline: rule JSON (reference detection.hpp:222-280) -> per-rule AST (libstdc++
// ECMAScript grammar, bits/regex_scanner.tcc + bits/regex_compiler.tcc of GCC 13.3)
// -> one Thompson NFA with lookbehind/lookahead-1 assertion edges -> search DFA by
// subset construction over (NFA set, previous-symbol context) -> Moore/Mealy
// minimisation -> tables for the device scanner.
//
// Semantics reproduced from the reference:
//  * regex_search is leftmost-anywhere (detection.hpp:155): a fresh thread starts at
//    every position (search DFA).
//  * '.' excludes '\n' and '\r' (ECMAScript _AnyMatcher); classes use the classic "C"
//    locale ctype table; bytes >= 0x80 belong to no class; bracket ranges compare
//    SIGNED chars (_BracketMatcher::_M_make_range) so [\x00-\xff] is an error_range.
//  * \b / \B use the real previous byte except at the window start (match_prev_avail,
//    regex_executor.tcc); ^ / $ hold only at the window edges (no multiline).
//  * the blacklist trie (detection.hpp:47-114) matches a whitespace-delimited token
//    (separators ' ' '\t' '\n' '\r') after stripping leading/trailing .,;:!?()"'; a
//    later duplicate term overwrites an earlier one (:62) and disabled winners hide
//    the term (:157-159).
#include "rules.hpp"

#include <algorithm>
#include <bitset>
#include <map>
#include <memory>
#include <set>
#include <unordered_map>

#include <json.hpp>

namespace skv {

// ---------------------------------------------------------------------------
// C-locale character classes (glibc "C" ctype table)
// ---------------------------------------------------------------------------
namespace {

enum CClass : uint16_t {
  kUpper = 1 << 0,
  kLower = 1 << 1,
  kAlpha = 1 << 2,
  kDigit = 1 << 3,
  kXdigit = 1 << 4,
  kSpace = 1 << 5,
  kPrint = 1 << 6,
  kGraph = 1 << 7,
  kCntrl = 1 << 8,
  kPunct = 1 << 9,
  kAlnum = 1 << 10,
  kBlank = 1 << 11,
  kUnder = 1 << 12,  // regex_traits _RegexMask::_S_under ("w" = alnum | '_')
};

uint16_t ctype_bits(unsigned c) {
  uint16_t m = 0;
  if (c >= 128) return 0;
  if (c >= 'A' && c <= 'Z') m |= kUpper | kAlpha | kAlnum;
  if (c >= 'a' && c <= 'z') m |= kLower | kAlpha | kAlnum;
  if (c >= '0' && c <= '9') m |= kDigit | kAlnum;
  if ((c >= '0' && c <= '9') || (c >= 'a' && c <= 'f') || (c >= 'A' && c <= 'F')) m |= kXdigit;
  if (c == ' ' || (c >= 9 && c <= 13)) m |= kSpace;
  if (c >= 32 && c <= 126) m |= kPrint;
  if (c >= 33 && c <= 126) m |= kGraph;
  if (c < 32 || c == 127) m |= kCntrl;
  if ((c >= 33 && c <= 47) || (c >= 58 && c <= 64) || (c >= 91 && c <= 96) || (c >= 123 && c <= 126))
    m |= kPunct;
  if (c == ' ' || c == '\t') m |= kBlank;
  return m;
}

bool isctype_mask(unsigned c, uint16_t mask) {
  if (ctype_bits(c) & mask & ~kUnder) return true;
  return (mask & kUnder) && c == '_';
}

bool is_word(unsigned c) { return isctype_mask(c, kAlnum | kUnder); }
// TokenTrie separators / trim set (detection.hpp:82-86)
bool is_sep(unsigned c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r'; }
bool is_trim(unsigned c) {
  return c == '.' || c == ',' || c == ';' || c == ':' || c == '!' || c == '?' || c == '(' || c == ')' ||
         c == '"' || c == '\'';
}

// regex_traits::lookup_classname table (bits/regex.tcc), name lower-cased first.
uint16_t lookup_classname(std::string s) {
  for (auto& ch : s) ch = static_cast<char>((ch >= 'A' && ch <= 'Z') ? ch - 'A' + 'a' : ch);
  static const std::pair<const char*, uint16_t> tbl[] = {
      {"d", kDigit},   {"w", static_cast<uint16_t>(kAlnum | kUnder)},
      {"s", kSpace},   {"alnum", kAlnum},
      {"alpha", kAlpha}, {"blank", kBlank},
      {"cntrl", kCntrl}, {"digit", kDigit},
      {"graph", kGraph}, {"lower", kLower},
      {"print", kPrint}, {"punct", kPunct},
      {"space", kSpace}, {"upper", kUpper},
      {"xdigit", kXdigit},
  };
  for (const auto& [n, m] : tbl)
    if (s == n) return m;
  return 0;
}

using ByteSet = std::bitset<256>;

// ---------------------------------------------------------------------------
// Scanner: token stream of libstdc++'s ECMAScript _Scanner
// ---------------------------------------------------------------------------
enum Tok {
  T_EOF,
  T_ORD,
  T_HEX,
  T_BACKREF,
  T_WORDB,
  T_QCLASS,
  T_BOL,
  T_EOL,
  T_ANY,
  T_STAR,
  T_PLUS,
  T_OPT,
  T_OR,
  T_GROUP,
  T_NOGROUP,
  T_LOOKAHEAD,
  T_GROUP_END,
  T_BRACKET,
  T_BRACKET_NEG,
  T_BRACKET_END,
  T_DASH,
  T_COLLSYM,
  T_CLASSNAME,
  T_EQUIV,
  T_BRACE,
  T_DUPCOUNT,
  T_COMMA,
  T_BRACE_END,
};

struct RegexError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Scanner {
 public:
  explicit Scanner(const std::string& p) : p_(p) { advance(); }
  Tok tok() const { return tok_; }
  const std::string& val() const { return val_; }

  void advance() {
    if (cur_ == p_.size()) {
      tok_ = T_EOF;
      return;
    }
    if (state_ == kNormal)
      scan_normal();
    else if (state_ == kBracket)
      scan_bracket();
    else
      scan_brace();
  }

 private:
  enum State { kNormal, kBracket, kBrace };
  bool at_end() const { return cur_ == p_.size(); }
  char peek() const { return at_end() ? '\0' : p_[cur_]; }
  static bool is_spec(char c) {
    static const char* spec = "^$\\.*+?()[]{}|";
    for (const char* s = spec; *s; ++s)
      if (*s == c) return true;
    return c == '\0';  // strchr finds the terminator
  }
  static bool is_digit(char c) { return c >= '0' && c <= '9'; }
  static bool is_xdigit(char c) { return isctype_mask(static_cast<unsigned char>(c), kXdigit); }

  void set(Tok t, std::string v = {}) {
    tok_ = t;
    val_ = std::move(v);
  }

  void scan_normal() {
    char c = p_[cur_++];
    if (!is_spec(c)) return set(T_ORD, std::string(1, c));
    if (c == '\\') {
      if (at_end()) throw RegexError("error_escape: invalid escape at end of regular expression");
      return eat_escape();
    }
    if (c == '(') {
      if (peek() == '?' && !at_end()) {
        if (++cur_ == p_.size()) throw RegexError("error_paren");
        char k = p_[cur_];
        if (k == ':') {
          ++cur_;
          return set(T_NOGROUP);
        }
        if (k == '=' || k == '!') {
          ++cur_;
          return set(T_LOOKAHEAD, std::string(1, k == '=' ? 'p' : 'n'));
        }
        throw RegexError("error_paren: invalid '(?...)' zero-width assertion");
      }
      return set(T_GROUP);
    }
    if (c == ')') return set(T_GROUP_END);
    if (c == '[') {
      state_ = kBracket;
      if (!at_end() && p_[cur_] == '^') {
        ++cur_;
        return set(T_BRACKET_NEG);
      }
      return set(T_BRACKET);
    }
    if (c == '{') {
      state_ = kBrace;
      return set(T_BRACE);
    }
    if (c == '\0') return set(T_ORD, std::string(1, '\0'));
    if (c != ']' && c != '}') {
      switch (c) {
        case '^': return set(T_BOL);
        case '$': return set(T_EOL);
        case '.': return set(T_ANY);
        case '*': return set(T_STAR);
        case '+': return set(T_PLUS);
        case '?': return set(T_OPT);
        case '|': return set(T_OR);
        default: break;
      }
    }
    set(T_ORD, std::string(1, c));
  }

  void scan_bracket() {
    char c = p_[cur_++];
    if (c == '-') return set(T_DASH);
    if (c == '[') {
      if (at_end()) throw RegexError("error_brack: incomplete '[[' character class");
      char k = p_[cur_];
      if (k == '.' || k == ':' || k == '=') {
        ++cur_;
        eat_class(k);
        return set(k == '.' ? T_COLLSYM : (k == ':' ? T_CLASSNAME : T_EQUIV), val_);
      }
      return set(T_ORD, "[");
    }
    if (c == ']') {
      state_ = kNormal;
      return set(T_BRACKET_END);
    }
    if (c == '\\') return eat_escape();
    set(T_ORD, std::string(1, c));
  }

  void scan_brace() {
    char c = p_[cur_++];
    if (is_digit(c)) {
      std::string v(1, c);
      while (!at_end() && is_digit(p_[cur_])) v += p_[cur_++];
      return set(T_DUPCOUNT, v);
    }
    if (c == ',') return set(T_COMMA);
    if (c == '}') {
      state_ = kNormal;
      return set(T_BRACE_END);
    }
    throw RegexError("error_badbrace");
  }

  void eat_class(char ch) {
    std::string v;
    while (!at_end() && p_[cur_] != ch) v += p_[cur_++];
    if (at_end() || p_[cur_++] != ch || at_end() || p_[cur_++] != ']')
      throw RegexError(ch == ':' ? "error_ctype" : "error_collate");
    val_ = v;
  }

  void eat_escape() {
    if (at_end()) throw RegexError("error_escape");
    char c = p_[cur_++];
    static const std::pair<char, char> tbl[] = {{'0', '\0'}, {'b', '\b'}, {'f', '\f'}, {'n', '\n'},
                                                {'r', '\r'}, {'t', '\t'}, {'v', '\v'}};
    const char* pos = nullptr;
    for (const auto& e : tbl)
      if (e.first == c) pos = &e.second;
    if (pos && (c != 'b' || state_ == kBracket)) return set(T_ORD, std::string(1, *pos));
    if (c == 'b') return set(T_WORDB, "p");
    if (c == 'B') return set(T_WORDB, "n");
    if (c == 'd' || c == 'D' || c == 's' || c == 'S' || c == 'w' || c == 'W')
      return set(T_QCLASS, std::string(1, c));
    if (c == 'c') {
      if (at_end()) throw RegexError("error_escape: invalid '\\cX' control character");
      return set(T_ORD, std::string(1, p_[cur_++]));
    }
    if (c == 'x' || c == 'u') {
      int n = c == 'x' ? 2 : 4;
      std::string v;
      for (int i = 0; i < n; ++i) {
        if (at_end() || !is_xdigit(p_[cur_])) throw RegexError("error_escape: invalid hex escape");
        v += p_[cur_++];
      }
      return set(T_HEX, v);
    }
    if (is_digit(c)) {
      std::string v(1, c);
      while (!at_end() && is_digit(p_[cur_])) v += p_[cur_++];
      return set(T_BACKREF, v);
    }
    set(T_ORD, std::string(1, c));
  }

  const std::string& p_;
  size_t cur_ = 0;
  State state_ = kNormal;
  Tok tok_ = T_EOF;
  std::string val_;
};

// ---------------------------------------------------------------------------
// AST
// ---------------------------------------------------------------------------
enum AssertKind : uint8_t { A_BOL, A_EOL, A_WB, A_NWB, A_SEPB, A_SEPA };

struct Ast {
  enum Kind { EMPTY, SET, CAT, ALT, REP, ASSERT } k = EMPTY;
  ByteSet set;
  std::vector<std::unique_ptr<Ast>> kids;
  long min = 0, max = 0;  // REP; max < 0 = unbounded
  AssertKind ak = A_BOL;
};
using AstP = std::unique_ptr<Ast>;

AstP mk(Ast::Kind k) {
  auto a = std::make_unique<Ast>();
  a->k = k;
  return a;
}

AstP mk_set(const ByteSet& s) {
  auto a = mk(Ast::SET);
  a->set = s;
  return a;
}

// ---------------------------------------------------------------------------
// Parser: libstdc++ _Compiler structure (disjunction/alternative/term/...)
// ---------------------------------------------------------------------------
class Parser {
 public:
  explicit Parser(const std::string& p) : sc_(p) {}

  AstP parse() {
    AstP r = disjunction();
    if (!match(T_EOF)) throw RegexError("error_paren");
    return r;
  }

 private:
  bool match(Tok t) {
    if (sc_.tok() != t) return false;
    val_ = sc_.val();
    sc_.advance();
    return true;
  }

  static long int_value(const std::string& v, int radix) {
    long x = 0;
    for (char c : v) {
      int d = (c >= '0' && c <= '9') ? c - '0' : (c >= 'a' && c <= 'f') ? c - 'a' + 10 : c - 'A' + 10;
      x = x * radix + d;
      if (x > 0x7fffffffL) throw RegexError("error_backref: invalid back reference");
    }
    return x;
  }

  AstP disjunction() {
    std::vector<AstP> alts;
    alts.push_back(alternative());
    while (match(T_OR)) alts.push_back(alternative());
    if (alts.size() == 1) return std::move(alts[0]);
    auto a = mk(Ast::ALT);
    a->kids = std::move(alts);
    return a;
  }

  AstP alternative() {
    auto seq = mk(Ast::CAT);
    AstP t;
    while ((t = term())) seq->kids.push_back(std::move(t));
    if (seq->kids.empty()) return mk(Ast::EMPTY);
    if (seq->kids.size() == 1) return std::move(seq->kids[0]);
    return seq;
  }

  AstP term() {
    if (AstP a = assertion()) return a;
    AstP at = atom();
    if (!at) return nullptr;
    for (;;) {
      AstP q = quantifier(at);
      if (!q) break;
      at = std::move(q);
    }
    return at;
  }

  AstP assertion() {
    auto a = mk(Ast::ASSERT);
    if (match(T_BOL))
      a->ak = A_BOL;
    else if (match(T_EOL))
      a->ak = A_EOL;
    else if (match(T_WORDB))
      a->ak = val_[0] == 'n' ? A_NWB : A_WB;
    else if (match(T_LOOKAHEAD))
      throw CompileError("lookahead assertions are not supported by the device DFA");
    else
      return nullptr;
    return a;
  }

  // returns the quantified node, or nullptr (and leaves `at` untouched) if none
  AstP quantifier(AstP& at) {
    long mn, mx;
    if (match(T_STAR)) {
      mn = 0, mx = -1;
      match(T_OPT);
    } else if (match(T_PLUS)) {
      mn = 1, mx = -1;
      match(T_OPT);
    } else if (match(T_OPT)) {
      mn = 0, mx = 1;
      match(T_OPT);
    } else if (match(T_BRACE)) {
      if (!match(T_DUPCOUNT)) throw RegexError("error_badbrace");
      mn = int_value(val_, 10);
      bool inf = false;
      long n = 0;
      if (match(T_COMMA)) {
        if (match(T_DUPCOUNT))
          n = int_value(val_, 10) - mn;
        else
          inf = true;
      }
      if (!match(T_BRACE_END)) throw RegexError("error_brace");
      match(T_OPT);
      if (!inf && n < 0) throw RegexError("error_badbrace");
      mx = inf ? -1 : mn + n;
    } else {
      return nullptr;
    }
    auto r = mk(Ast::REP);
    r->min = mn;
    r->max = mx;
    r->kids.push_back(std::move(at));
    return r;
  }

  static ByteSet class_set(uint16_t mask, bool neg) {
    ByteSet s;
    for (unsigned c = 0; c < 256; ++c) s[c] = isctype_mask(c, mask) != neg;
    return s;
  }

  bool try_char(char* out) {
    if (match(T_HEX)) {
      *out = static_cast<char>(int_value(val_, 16));
      return true;
    }
    if (match(T_ORD)) {
      *out = val_[0];
      return true;
    }
    return false;
  }

  AstP atom() {
    char c;
    if (match(T_ANY)) {
      ByteSet s;
      s.set();
      s['\n'] = false;
      s['\r'] = false;
      return mk_set(s);
    }
    if (try_char(&c)) {
      ByteSet s;
      s[static_cast<unsigned char>(c)] = true;
      return mk_set(s);
    }
    if (match(T_BACKREF)) throw CompileError("back-references are not supported by the device DFA");
    if (match(T_QCLASS)) {
      char q = val_[0];
      bool upper = q >= 'A' && q <= 'Z';
      uint16_t m = lookup_classname(std::string(1, q));
      return mk_set(class_set(m, upper));
    }
    if (match(T_NOGROUP) || match(T_GROUP)) {
      AstP r = disjunction();
      if (!match(T_GROUP_END)) throw RegexError("error_paren");
      return r;
    }
    return bracket();
  }

  AstP bracket() {
    bool neg = match(T_BRACKET_NEG);
    if (!neg && !match(T_BRACKET)) return nullptr;
    // _BracketMatcher state
    ByteSet chars;
    std::vector<std::pair<signed char, signed char>> ranges;
    uint16_t cls = 0;
    std::vector<uint16_t> neg_cls;
    enum { NONE, CHAR, CLASS } last = NONE;
    char last_c = 0;
    auto push_char = [&](char ch) {
      if (last == CHAR) chars[static_cast<unsigned char>(last_c)] = true;
      last = CHAR;
      last_c = ch;
    };
    auto push_class = [&] {
      if (last == CHAR) chars[static_cast<unsigned char>(last_c)] = true;
      last = CLASS;
    };
    auto make_range = [&](char l, char r) {
      if (static_cast<signed char>(l) > static_cast<signed char>(r))
        throw RegexError("error_range: invalid range in bracket expression");
      ranges.emplace_back(static_cast<signed char>(l), static_cast<signed char>(r));
    };
    char c;
    if (try_char(&c)) {
      last = CHAR;
      last_c = c;
    } else if (match(T_DASH)) {
      last = CHAR;
      last_c = '-';
    }
    for (;;) {
      if (match(T_BRACKET_END)) break;
      if (match(T_COLLSYM) || match(T_EQUIV))
        throw CompileError("collating elements / equivalence classes are not supported by the device DFA");
      if (match(T_CLASSNAME)) {
        push_class();
        uint16_t m = lookup_classname(val_);
        if (!m) throw RegexError("error_collate: invalid character class");
        cls |= m;
        continue;
      }
      if (try_char(&c)) {
        push_char(c);
        continue;
      }
      if (match(T_DASH)) {
        if (match(T_BRACKET_END)) {
          push_char('-');
          break;
        }
        if (last == CLASS) throw RegexError("error_range: invalid start of range");
        if (last == CHAR) {
          if (try_char(&c)) {
            make_range(last_c, c);
            last = NONE;
          } else if (match(T_DASH)) {
            make_range(last_c, '-');
            last = NONE;
          } else {
            throw RegexError("error_range: invalid end of range");
          }
        } else {
          push_char('-');
        }
        continue;
      }
      if (match(T_QCLASS)) {
        push_class();
        char q = val_[0];
        uint16_t m = lookup_classname(std::string(1, q));
        if (q >= 'A' && q <= 'Z')
          neg_cls.push_back(m);
        else
          cls |= m;
        continue;
      }
      throw RegexError("error_brack: unexpected character within '[...]'");
    }
    if (last == CHAR) chars[static_cast<unsigned char>(last_c)] = true;
    ByteSet s;
    for (unsigned u = 0; u < 256; ++u) {
      signed char sc = static_cast<signed char>(u);
      bool m = chars[u];
      for (const auto& [l, r] : ranges) m = m || (l <= sc && sc <= r);
      m = m || isctype_mask(u, cls);
      for (uint16_t nm : neg_cls) m = m || !isctype_mask(u, nm);
      s[u] = m != neg;
    }
    return mk_set(s);
  }

  Scanner sc_;
  std::string val_;
};

// ---------------------------------------------------------------------------
// NFA
// ---------------------------------------------------------------------------
struct NState {
  enum Type : uint8_t { EPS, SET, ASSERT, ACCEPT } t = EPS;
  int o1 = -1, o2 = -1;
  int set = -1;
  AssertKind ak = A_BOL;
  uint32_t acc = 0;
};

constexpr size_t kMaxNfaStates = 200000;

class Nfa {
 public:
  std::vector<NState> st;
  std::vector<ByteSet> sets;

  int add(NState::Type t) {
    if (st.size() >= kMaxNfaStates) throw CompileError("rule set too large for the device DFA (NFA states)");
    st.push_back({});
    st.back().t = t;
    return static_cast<int>(st.size() - 1);
  }
  int add_set(const ByteSet& s) {
    int id = add(NState::SET);
    auto it = set_ids_.find(s.to_string());
    if (it == set_ids_.end()) {
      sets.push_back(s);
      it = set_ids_.emplace(s.to_string(), static_cast<int>(sets.size() - 1)).first;
    }
    st[id].set = it->second;
    return id;
  }

  // Thompson fragment: (start, end); end is an EPS state whose o1 is to be patched.
  std::pair<int, int> build(const Ast& a) {
    switch (a.k) {
      case Ast::EMPTY: {
        int s = add(NState::EPS);
        return {s, s};
      }
      case Ast::SET: {
        int s = add_set(a.set);
        int e = add(NState::EPS);
        st[s].o1 = e;
        return {s, e};
      }
      case Ast::ASSERT: {
        int s = add(NState::ASSERT);
        st[s].ak = a.ak;
        int e = add(NState::EPS);
        st[s].o1 = e;
        return {s, e};
      }
      case Ast::CAT: {
        auto [s, e] = build(*a.kids[0]);
        for (size_t i = 1; i < a.kids.size(); ++i) {
          auto [s2, e2] = build(*a.kids[i]);
          st[e].o1 = s2;
          e = e2;
        }
        return {s, e};
      }
      case Ast::ALT: {
        int end = add(NState::EPS);
        int head = -1, tail = -1;
        for (const auto& k : a.kids) {
          auto [s, e] = build(*k);
          st[e].o1 = end;
          int split = add(NState::EPS);
          st[split].o1 = s;
          if (head < 0)
            head = split;
          else
            st[tail].o2 = split;
          tail = split;
        }
        return {head, end};
      }
      case Ast::REP: {
        const Ast& k = *a.kids[0];
        int s = add(NState::EPS), e = s;
        for (long i = 0; i < a.min; ++i) {
          auto [s2, e2] = build(k);
          st[e].o1 = s2;
          e = e2;
        }
        if (a.max < 0) {
          int loop = add(NState::EPS);
          auto [s2, e2] = build(k);
          st[e].o1 = loop;
          st[loop].o1 = s2;
          st[e2].o1 = loop;
          int out = add(NState::EPS);
          st[loop].o2 = out;
          e = out;
        } else {
          int out = add(NState::EPS);
          for (long i = a.min; i < a.max; ++i) {
            int split = add(NState::EPS);
            auto [s2, e2] = build(k);
            st[e].o1 = split;
            st[split].o1 = s2;
            st[split].o2 = out;
            e = e2;
          }
          st[e].o1 = out;
          e = out;
        }
        return {s, e};
      }
    }
    throw CompileError("internal: bad AST");
  }

 private:
  std::unordered_map<std::string, int> set_ids_;
};

// Previous / next symbol context for assertions.
enum Ctx : uint8_t { C_EDGE = 0, C_WORD = 1, C_SEP = 2, C_OTHER = 3 };

Ctx byte_ctx(unsigned c) { return is_word(c) ? C_WORD : (is_sep(c) ? C_SEP : C_OTHER); }

bool eval_assert(AssertKind k, Ctx prev, Ctx next) {
  switch (k) {
    case A_BOL: return prev == C_EDGE;
    case A_EOL: return next == C_EDGE;
    case A_WB: return (prev == C_WORD) != (next == C_WORD);
    case A_NWB: return (prev == C_WORD) == (next == C_WORD);
    case A_SEPB: return prev == C_EDGE || prev == C_SEP;
    case A_SEPA: return next == C_EDGE || next == C_SEP;
  }
  return false;
}

}  // namespace

// ---------------------------------------------------------------------------
// Public API
// ---------------------------------------------------------------------------
std::vector<PatternRule> default_pattern_rules() {
  // Identical rule set to reference detection.hpp:185-204 /
  // configs/privacy_pattern_config.json (rule list is data, not code).
  return {
      {"ssn_dashed", "Identity Information", false, R"(\b\d{3}-\d{2}-\d{4}\b)", true},
      {"phone_us", "Basic Information", false, R"(\(\d{3}\)\s?\d{3}-\d{4}|\b\d{3}-\d{3}-\d{4}\b)", true},
      {"email", "Basic Information", false, R"([A-Za-z0-9._%+-]+@[A-Za-z0-9.-]+\.[A-Za-z]{2,})", true},
      {"ipv4", "System/Network Identification", false, R"(\b\d{1,3}\.\d{1,3}\.\d{1,3}\.\d{1,3}\b)", true},
      {"credit_card", "Financial Info", false, R"(\b\d{4}[- ]\d{4}[- ]\d{4}[- ]\d{4}\b)", true},
      {"bank_account", "Financial Info", false, R"(\baccount\s+(?:no|number)\.?\s*\d{6,}\b)", true},
      {"mac_address", "Hardware Device Information", false, R"(\b[0-9A-Fa-f]{2}(?::[0-9A-Fa-f]{2}){5}\b)",
       true},
      {"imei", "Hardware Device Information", false, R"(\bimei\s*\d{15}\b)", true},
      {"blk_project_codes", "Service Content Info", true, "PROJECT-TITAN", true},
  };
}

RuleSetSpec parse_rules_json(const std::string& text) {
  RuleSetSpec spec;
  nlohmann::json j;
  try {
    j = nlohmann::json::parse(text);
  } catch (const std::exception& e) {
    throw ParseError(std::string("pattern config: ") + e.what());
  }
  if (!j.is_object()) throw ParseError("pattern config: top level must be an object");
  try {
    for (auto it = j.begin(); it != j.end(); ++it) {
      if (it.key() == "version") {
        if (!it.value().is_number_integer()) throw ParseError("pattern config: version must be an integer");
        spec.version = it.value().get<uint64_t>();
      } else if (it.key() == "rules") {
        if (!it.value().is_array()) throw ParseError("pattern config: rules must be an array");
        for (const auto& rj : it.value()) {
          if (!rj.is_object()) throw ParseError("pattern config: each rule must be an object");
          PatternRule r;
          bool have_id = false, have_pattern = false;
          for (auto f = rj.begin(); f != rj.end(); ++f) {
            const std::string& k = f.key();
            if (k == "rule_id") {
              r.rule_id = f.value().get<std::string>();
              have_id = true;
            } else if (k == "category") {
              r.category = f.value().get<std::string>();
            } else if (k == "kind") {
              std::string kind = f.value().get<std::string>();
              if (kind == "regex")
                r.blacklist = false;
              else if (kind == "blacklist")
                r.blacklist = true;
              else
                throw ParseError("pattern config: unknown kind '" + kind + "'");
            } else if (k == "pattern") {
              r.pattern = f.value().get<std::string>();
              have_pattern = true;
            } else if (k == "enabled") {
              r.enabled = f.value().get<bool>();
            } else {
              spec.warnings.push_back("rule field ignored: " + k);
            }
          }
          if (!have_id || !have_pattern) throw ParseError("pattern config: rule needs rule_id and pattern");
          spec.rules.push_back(std::move(r));
        }
      } else {
        spec.warnings.push_back("ignoring unknown field: " + it.key());
      }
    }
  } catch (const nlohmann::json::exception& e) {
    throw ParseError(std::string("pattern config: ") + e.what());
  }
  return spec;
}

DfaTables compile_rules(const std::vector<PatternRule>& rules) {
  {
    std::set<std::string> seen;
    for (const auto& r : rules)
      if (!seen.insert(r.rule_id).second) throw CompileError("duplicate rule_id: " + r.rule_id);
  }
  DfaTables out;
  Nfa nfa;
  int start = nfa.add(NState::EPS);
  std::vector<int> starts;
  // Every regex is parsed (even disabled ones: the reference compiles them all and
  // throws on a bad pattern, detection.hpp:130-137); only enabled rules enter the DFA.
  std::vector<AstP> asts(rules.size());
  for (size_t i = 0; i < rules.size(); ++i) {
    if (rules[i].blacklist) continue;
    try {
      asts[i] = Parser(rules[i].pattern).parse();
    } catch (const RegexError& e) {
      throw CompileError("rule '" + rules[i].rule_id + "': bad regex: " + e.what());
    } catch (const CompileError& e) {
      throw CompileError("rule '" + rules[i].rule_id + "': " + e.what());
    }
  }
  // blacklist terms: last writer wins (TokenTrie::add overwrites rule_index)
  std::map<std::string, size_t> term_owner;
  for (size_t i = 0; i < rules.size(); ++i)
    if (rules[i].blacklist) term_owner[rules[i].pattern] = i;

  std::vector<int> bit_of(rules.size(), -1);
  for (size_t i = 0; i < rules.size(); ++i) {
    if (!rules[i].enabled) continue;
    bit_of[i] = static_cast<int>(out.rule_index.size());
    out.rule_index.push_back(static_cast<uint32_t>(i));
  }
  if (out.rule_index.size() > 32)
    throw CompileError("device DFA supports at most 32 enabled rules (got " +
                       std::to_string(out.rule_index.size()) + ")");

  auto add_accept = [&](int end, uint32_t bit) {
    int acc = nfa.add(NState::ACCEPT);
    nfa.st[acc].acc = 1u << bit;
    nfa.st[end].o1 = acc;
  };
  for (size_t i = 0; i < rules.size(); ++i) {
    if (!rules[i].enabled) continue;
    if (!rules[i].blacklist) {
      auto [s, e] = nfa.build(*asts[i]);
      starts.push_back(s);
      add_accept(e, bit_of[i]);
      continue;
    }
    const std::string& term = rules[i].pattern;
    if (term_owner[term] != i) continue;  // overwritten by a later duplicate
    if (term.empty()) continue;           // match_token("") never matches
    bool ok = !is_trim(static_cast<unsigned char>(term.front())) &&
              !is_trim(static_cast<unsigned char>(term.back()));
    for (char ch : term) ok = ok && !is_sep(static_cast<unsigned char>(ch));
    if (!ok) continue;  // a stripped, separator-free token can never equal this term
    // SEPB [trim]* term [trim]* SEPA
    ByteSet trim;
    for (unsigned u = 0; u < 256; ++u) trim[u] = is_trim(u);
    auto seq = mk(Ast::CAT);
    auto a1 = mk(Ast::ASSERT);
    a1->ak = A_SEPB;
    seq->kids.push_back(std::move(a1));
    auto r1 = mk(Ast::REP);
    r1->min = 0;
    r1->max = -1;
    r1->kids.push_back(mk_set(trim));
    seq->kids.push_back(std::move(r1));
    for (char ch : term) {
      ByteSet s;
      s[static_cast<unsigned char>(ch)] = true;
      seq->kids.push_back(mk_set(s));
    }
    auto r2 = mk(Ast::REP);
    r2->min = 0;
    r2->max = -1;
    r2->kids.push_back(mk_set(trim));
    seq->kids.push_back(std::move(r2));
    auto a2 = mk(Ast::ASSERT);
    a2->ak = A_SEPA;
    seq->kids.push_back(std::move(a2));
    auto [s, e] = nfa.build(*seq);
    starts.push_back(s);
    add_accept(e, bit_of[i]);
  }
  // chain the rule starts off the global start state
  {
    int cur = start;
    for (size_t i = 0; i < starts.size(); ++i) {
      int split = nfa.add(NState::EPS);
      nfa.st[cur].o1 = split;
      nfa.st[split].o2 = starts[i];
      cur = split;
    }
  }
  out.nfa_states = static_cast<uint32_t>(nfa.st.size());

  // --- byte classes: bytes with identical membership in every set + same context
  std::vector<uint32_t> cls_of(256);
  std::vector<unsigned> repr;
  {
    std::map<std::string, uint32_t> sig2cls;
    for (unsigned c = 0; c < 256; ++c) {
      std::string sig;
      sig.reserve(nfa.sets.size() + 1);
      sig.push_back(static_cast<char>('0' + byte_ctx(c)));
      for (const auto& s : nfa.sets) sig.push_back(s[c] ? '1' : '0');
      auto it = sig2cls.find(sig);
      if (it == sig2cls.end()) {
        it = sig2cls.emplace(sig, static_cast<uint32_t>(repr.size())).first;
        repr.push_back(c);
      }
      cls_of[c] = it->second;
    }
  }
  const uint32_t C = static_cast<uint32_t>(repr.size());
  if (C > 63) throw CompileError("rule set too large for the device DFA (byte classes)");

  // --- subset construction over (context, NFA kernel set)
  struct Key {
    uint8_t ctx;
    std::vector<int> k;
    bool operator<(const Key& o) const { return ctx != o.ctx ? ctx < o.ctx : k < o.k; }
  };
  std::map<Key, uint32_t> ids;
  std::vector<Key> keys;
  std::vector<uint32_t> nxt;  // S x C
  std::vector<uint32_t> acc;  // S x (C+1)
  auto intern = [&](Key&& key) -> uint32_t {
    auto it = ids.find(key);
    if (it != ids.end()) return it->second;
    uint32_t id = static_cast<uint32_t>(keys.size());
    if (id >= 200000) throw CompileError("rule set too large for the device DFA (states)");
    ids.emplace(key, id);
    keys.push_back(std::move(key));
    return id;
  };
  intern(Key{C_EDGE, {}});
  std::vector<int> stack;
  std::vector<uint32_t> mark(nfa.st.size(), 0);
  uint32_t stamp = 0;
  std::vector<int> closure;
  for (uint32_t s = 0; s < keys.size(); ++s) {
    Key cur = keys[s];  // copy: keys may grow
    nxt.resize((s + 1) * C);
    acc.resize((s + 1) * (C + 1));
    for (int nctx = 0; nctx < 4; ++nctx) {
      // closure of kernel + start under eps and satisfied assertions
      ++stamp;
      closure.clear();
      stack.assign(cur.k.begin(), cur.k.end());
      stack.push_back(start);
      uint32_t a = 0;
      while (!stack.empty()) {
        int x = stack.back();
        stack.pop_back();
        if (x < 0 || mark[x] == stamp) continue;
        mark[x] = stamp;
        const NState& ns = nfa.st[x];
        switch (ns.t) {
          case NState::EPS:
            stack.push_back(ns.o1);
            stack.push_back(ns.o2);
            break;
          case NState::ASSERT:
            if (eval_assert(ns.ak, static_cast<Ctx>(cur.ctx), static_cast<Ctx>(nctx))) stack.push_back(ns.o1);
            break;
          case NState::ACCEPT: a |= ns.acc; break;
          case NState::SET: closure.push_back(x); break;
        }
      }
      if (nctx == C_EDGE) {
        acc[s * (C + 1) + C] = a;
        continue;
      }
      for (uint32_t c = 0; c < C; ++c) {
        unsigned rb = repr[c];
        if (byte_ctx(rb) != nctx) continue;
        acc[s * (C + 1) + c] = a;
        std::vector<int> k2;
        for (int x : closure)
          if (nfa.sets[nfa.st[x].set][rb]) k2.push_back(nfa.st[x].o1);
        std::sort(k2.begin(), k2.end());
        k2.erase(std::unique(k2.begin(), k2.end()), k2.end());
        uint32_t t = intern(Key{static_cast<uint8_t>(nctx), std::move(k2)});
        nxt[s * C + c] = t;
      }
    }
  }
  const uint32_t S0 = static_cast<uint32_t>(keys.size());
  out.dfa_states_unminimized = S0;

  // --- minimisation (Moore partition refinement on the Mealy machine)
  std::vector<uint32_t> blk(S0);
  {
    std::map<std::vector<uint32_t>, uint32_t> sig;
    for (uint32_t s = 0; s < S0; ++s) {
      std::vector<uint32_t> v(acc.begin() + s * (C + 1), acc.begin() + (s + 1) * (C + 1));
      blk[s] = sig.emplace(v, static_cast<uint32_t>(sig.size())).first->second;
    }
    size_t nblk = sig.size();
    for (;;) {
      std::map<std::vector<uint32_t>, uint32_t> sig2;
      std::vector<uint32_t> nb(S0);
      for (uint32_t s = 0; s < S0; ++s) {
        std::vector<uint32_t> v;
        v.reserve(C + 1);
        v.push_back(blk[s]);
        for (uint32_t c = 0; c < C; ++c) v.push_back(blk[nxt[s * C + c]]);
        nb[s] = sig2.emplace(v, static_cast<uint32_t>(sig2.size())).first->second;
      }
      blk.swap(nb);
      if (sig2.size() == nblk) break;
      nblk = sig2.size();
    }
  }
  // renumber blocks in BFS order from the start state (start = 0)
  std::vector<uint32_t> order(S0, UINT32_MAX);
  std::vector<uint32_t> rep;  // new id -> representative old state
  {
    std::vector<uint32_t> q{0};
    std::vector<uint32_t> blk2new(S0, UINT32_MAX);
    blk2new[blk[0]] = 0;
    rep.push_back(0);
    for (size_t qi = 0; qi < rep.size(); ++qi) {
      uint32_t s = rep[qi];
      for (uint32_t c = 0; c < C; ++c) {
        uint32_t t = nxt[s * C + c];
        if (blk2new[blk[t]] == UINT32_MAX) {
          blk2new[blk[t]] = static_cast<uint32_t>(rep.size());
          rep.push_back(t);
        }
      }
    }
    for (uint32_t s = 0; s < S0; ++s) order[s] = blk2new[blk[s]];
  }
  const uint32_t S = static_cast<uint32_t>(rep.size());
  if (S > 65535) throw CompileError("rule set too large for the device DFA (minimised states)");
  out.n_states = S;
  out.n_classes = C;
  out.start = 0;
  for (unsigned c = 0; c < 256; ++c) out.class_map[c] = static_cast<uint8_t>(cls_of[c]);
  out.next.resize(static_cast<size_t>(S) * C);
  out.acc.resize(static_cast<size_t>(S) * (C + 1));
  for (uint32_t n = 0; n < S; ++n) {
    uint32_t s = rep[n];
    for (uint32_t c = 0; c < C; ++c) out.next[n * C + c] = static_cast<uint16_t>(order[nxt[s * C + c]]);
    for (uint32_t c = 0; c <= C; ++c) out.acc[n * (C + 1) + c] = acc[s * (C + 1) + c];
  }
  return out;
}

RuleGroups compile_rule_groups(const std::vector<PatternRule>& rules,
                               const std::function<bool(const DfaTables&)>& fits, uint32_t max_group) {
  std::vector<size_t> enabled;
  for (size_t i = 0; i < rules.size(); ++i)
    if (rules[i].enabled) enabled.push_back(i);
  RuleGroups out;
  auto compile_range = [&](size_t a, size_t b) {  // enabled[a, b) stay enabled
    std::vector<PatternRule> sub = rules;
    for (auto& r : sub) r.enabled = false;
    for (size_t k = a; k < b; ++k) sub[enabled[k]].enabled = true;
    return compile_rules(sub);
  };
  if (enabled.empty()) {
    out.groups.push_back(compile_rules(rules));
    out.first_bit.push_back(0);
    return out;
  }
  for (size_t a = 0; a < enabled.size();) {
    // a group never straddles a 32-bit mask word (its bits are one word's shifted rule mask)
    const size_t word_end = (a / 32 + 1) * 32;
    size_t b = std::min({enabled.size(), a + max_group, word_end});
    DfaTables t = compile_range(a, b);
    while (!fits(t)) {  // shrink until the group's automaton fits the device tables
      if (b - a == 1)
        throw CompileError("rule '" + rules[enabled[a]].rule_id + "': its automaton exceeds the device table limits");
      b = a + (b - a) / 2;
      t = compile_range(a, b);
    }
    // grow back one rule at a time while it still fits (halving may have overshot)
    while (b < enabled.size() && b - a < max_group && b < word_end) {
      DfaTables t2 = compile_range(a, b + 1);
      if (!fits(t2)) break;
      t = std::move(t2);
      ++b;
    }
    out.first_bit.push_back(static_cast<uint32_t>(a));
    out.groups.push_back(std::move(t));
    a = b;
  }
  return out;
}

}  // namespace skv
