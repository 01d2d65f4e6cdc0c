/* safekv_oracle.c -- TEST INFRASTRUCTURE ONLY: plain-C restatement of the reference
 * algorithm for the SafeKV admission path (see safekv_oracle.h).  It shares no code
 * with the product (paper_2508_08438_b200/) nor with the reference; each function
 * cites the reference lines it restates (paths under /root/reference/proj/include/).
 *
 * Regex semantics are those of the reference's third-party dependency, libstdc++
 * <regex> (GCC 13.3.0, ECMAScript grammar, "C" locale), restated here as a recursive
 * backtracking matcher over an AST -- a different technique from the product's DFA.
 * Parity of this restatement is pinned against the reference harness
 * (oracle/_ref/libsafekv_ref.so) and the reference's known-answer tests.
 */
#include "safekv_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ FNV-1a (util.hpp:58-81) */
#define FNV_OFF 0xcbf29ce484222325ULL
#define FNV_P 0x100000001b3ULL

static uint64_t fnv_bytes(uint64_t h, const uint8_t* p, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= FNV_P;
  }
  return h;
}
static uint64_t fnv_u32(uint64_t h, uint32_t v) {
  uint8_t b[4] = {(uint8_t)v, (uint8_t)(v >> 8), (uint8_t)(v >> 16), (uint8_t)(v >> 24)};
  return fnv_bytes(h, b, 4);
}
static uint64_t fnv_u64(uint64_t h, uint64_t v) { return fnv_u32(fnv_u32(h, (uint32_t)v), (uint32_t)(v >> 32)); }

uint64_t orc_fnv1a64(const uint8_t* p, size_t n) { return fnv_bytes(FNV_OFF, p, n); }

/* token_seq_digest (core.hpp:68-73): u32 length, then each token as u32 LE */
uint64_t orc_token_seq_digest(const uint32_t* t, size_t n) {
  uint64_t h = fnv_u32(FNV_OFF, (uint32_t)n);
  for (size_t i = 0; i < n; ++i) h = fnv_u32(h, t[i]);
  return h;
}

/* SURVEY A.2 chained key: Fnv1a64 f; f.update_u64(prev); f.update_u64(d) (util.hpp:75-78) */
uint64_t orc_chain(uint64_t prev_h, uint64_t d) { return fnv_u64(fnv_u64(FNV_OFF, prev_h), d); }

/* ------------------------------------------------------------------ "C" locale ctype */
enum { CT_UPPER = 1, CT_LOWER = 2, CT_ALPHA = 4, CT_DIGIT = 8, CT_XDIGIT = 16, CT_SPACE = 32, CT_PRINT = 64,
       CT_GRAPH = 128, CT_CNTRL = 256, CT_PUNCT = 512, CT_ALNUM = 1024, CT_BLANK = 2048, CT_UNDER = 4096 };

static int ctype_of(unsigned c) {
  int m = 0;
  if (c > 127) return 0;
  if (c >= 'A' && c <= 'Z') m |= CT_UPPER | CT_ALPHA | CT_ALNUM;
  if (c >= 'a' && c <= 'z') m |= CT_LOWER | CT_ALPHA | CT_ALNUM;
  if (c >= '0' && c <= '9') m |= CT_DIGIT | CT_ALNUM | CT_XDIGIT;
  if ((c >= 'a' && c <= 'f') || (c >= 'A' && c <= 'F')) m |= CT_XDIGIT;
  if (c == ' ' || (c >= 9 && c <= 13)) m |= CT_SPACE;
  if (c >= 32 && c < 127) m |= CT_PRINT;
  if (c > 32 && c < 127) m |= CT_GRAPH;
  if (c < 32 || c == 127) m |= CT_CNTRL;
  if ((m & CT_GRAPH) && !(m & CT_ALNUM)) m |= CT_PUNCT;
  if (c == ' ' || c == '\t') m |= CT_BLANK;
  return m;
}
static int in_class(unsigned c, int mask) {
  if (ctype_of(c) & mask & ~CT_UNDER) return 1;
  return (mask & CT_UNDER) && c == '_';
}
static int is_word(unsigned c) { return in_class(c, CT_ALNUM | CT_UNDER); }

static int class_by_name(const char* s, size_t n) {
  static const struct { const char* name; int mask; } tbl[] = {
      {"d", CT_DIGIT}, {"w", CT_ALNUM | CT_UNDER}, {"s", CT_SPACE}, {"alnum", CT_ALNUM}, {"alpha", CT_ALPHA},
      {"blank", CT_BLANK}, {"cntrl", CT_CNTRL}, {"digit", CT_DIGIT}, {"graph", CT_GRAPH}, {"lower", CT_LOWER},
      {"print", CT_PRINT}, {"punct", CT_PUNCT}, {"space", CT_SPACE}, {"upper", CT_UPPER}, {"xdigit", CT_XDIGIT}};
  char buf[16];
  if (n == 0 || n >= sizeof(buf)) return 0;
  for (size_t i = 0; i < n; ++i) buf[i] = (char)((s[i] >= 'A' && s[i] <= 'Z') ? s[i] - 'A' + 'a' : s[i]);
  buf[n] = 0;
  for (size_t i = 0; i < sizeof(tbl) / sizeof(tbl[0]); ++i)
    if (!strcmp(buf, tbl[i].name)) return tbl[i].mask;
  return 0;
}

/* ------------------------------------------------------------------ regex AST */
enum { N_EMPTY, N_SET, N_CAT, N_ALT, N_REP, N_ASSERT };
enum { AS_BOL, AS_EOL, AS_WB, AS_NWB };

typedef struct {
  int kind;
  uint8_t set[32];
  int a, b;
  long min, max; /* REP; max < 0 = unbounded */
  int ak;
} RNode;

typedef struct {
  RNode* v;
  int n, cap;
  int root;
} Re;

typedef struct {
  Re* re;
  const char* p;
  size_t len, i;
  int err;
  char msg[160];
} P;

static int node(P* ps, int kind) {
  Re* re = ps->re;
  if (re->n == re->cap) {
    re->cap = re->cap ? 2 * re->cap : 64;
    re->v = (RNode*)realloc(re->v, (size_t)re->cap * sizeof(RNode));
  }
  memset(&re->v[re->n], 0, sizeof(RNode));
  re->v[re->n].kind = kind;
  return re->n++;
}
static void setbit(uint8_t* s, unsigned c) { s[c >> 3] |= (uint8_t)(1u << (c & 7)); }
static int getbit(const uint8_t* s, unsigned c) { return (s[c >> 3] >> (c & 7)) & 1; }
static void fail(P* ps, const char* m) {
  if (!ps->err) {
    ps->err = 1;
    snprintf(ps->msg, sizeof(ps->msg), "%s", m);
  }
}
static int at_end(P* ps) { return ps->i >= ps->len; }
static int peek(P* ps) { return at_end(ps) ? -1 : (unsigned char)ps->p[ps->i]; }

static int disj(P* ps);

static int hexval(int c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  if (c >= 'A' && c <= 'F') return c - 'A' + 10;
  return -1;
}

/* Escape after '\\' (libstdc++ _Scanner::_M_eat_escape_ecma).  Returns 0 = char (in *ch),
 * 1 = class (mask in *cls, neg in *neg), 2 = word boundary (neg in *neg), -1 = error. */
static int escape(P* ps, int in_bracket, int* ch, int* cls, int* neg) {
  if (at_end(ps)) {
    fail(ps, "escape at end");
    return -1;
  }
  int c = (unsigned char)ps->p[ps->i++];
  switch (c) {
    case '0': *ch = 0; return 0;
    case 'f': *ch = '\f'; return 0;
    case 'n': *ch = '\n'; return 0;
    case 'r': *ch = '\r'; return 0;
    case 't': *ch = '\t'; return 0;
    case 'v': *ch = '\v'; return 0;
    case 'b':
      if (in_bracket) {
        *ch = '\b';
        return 0;
      }
      *neg = 0;
      return 2;
    case 'B': *neg = 1; return 2;
    case 'd': case 'D': *cls = CT_DIGIT; *neg = c == 'D'; return 1;
    case 's': case 'S': *cls = CT_SPACE; *neg = c == 'S'; return 1;
    case 'w': case 'W': *cls = CT_ALNUM | CT_UNDER; *neg = c == 'W'; return 1;
    case 'c':
      if (at_end(ps)) {
        fail(ps, "bad \\c");
        return -1;
      }
      *ch = (unsigned char)ps->p[ps->i++];
      return 0;
    case 'x': case 'u': {
      int n = c == 'x' ? 2 : 4, v = 0;
      for (int k = 0; k < n; ++k) {
        int h = at_end(ps) ? -1 : hexval((unsigned char)ps->p[ps->i]);
        if (h < 0) {
          fail(ps, "bad hex escape");
          return -1;
        }
        v = v * 16 + h;
        ps->i++;
      }
      *ch = v & 0xff;
      return 0;
    }
    default:
      if (c >= '1' && c <= '9') {
        fail(ps, "back-references unsupported");
        return -1;
      }
      *ch = c;
      return 0;
  }
}

/* bracket expression (libstdc++ _Compiler::_M_insert_bracket_matcher / _M_expression_term) */
static int bracket(P* ps) {
  int neg = 0;
  if (peek(ps) == '^') {
    neg = 1;
    ps->i++;
  }
  uint8_t chars[32] = {0};
  signed char rl[256], rh[256];
  int nr = 0, cls = 0, negcls[64], nneg = 0;
  enum { NONE, CHAR, CLASS } last = NONE;
  int last_c = 0;
  int first = 1;
  for (;;) {
    if (at_end(ps)) {
      fail(ps, "unterminated bracket");
      return -1;
    }
    int c = (unsigned char)ps->p[ps->i];
    /* item kinds: ']' end, '-' dash, '[' class/coll, '\\' escape, other char */
    int kind, ch = 0, cm = 0, cn = 0;
    if (c == ']') {
      ps->i++;
      break;
    } else if (c == '-') {
      ps->i++;
      kind = 'd';
    } else if (c == '[' && ps->i + 1 < ps->len &&
               (ps->p[ps->i + 1] == ':' || ps->p[ps->i + 1] == '.' || ps->p[ps->i + 1] == '=')) {
      char t = ps->p[ps->i + 1];
      size_t j = ps->i + 2, s0 = j;
      while (j < ps->len && ps->p[j] != t) j++;
      if (j + 1 >= ps->len || ps->p[j + 1] != ']') {
        fail(ps, "bad [: :]");
        return -1;
      }
      if (t != ':') {
        fail(ps, "collating elements unsupported");
        return -1;
      }
      cm = class_by_name(ps->p + s0, j - s0);
      if (!cm) {
        fail(ps, "bad class name");
        return -1;
      }
      ps->i = j + 2;
      kind = 'k';
      cn = 0;
    } else if (c == '\\') {
      ps->i++;
      int r = escape(ps, 1, &ch, &cm, &cn);
      if (r < 0) return -1;
      if (r == 2) {
        fail(ps, "\\B in bracket");
        return -1;
      }
      kind = r == 1 ? 'k' : 'c';
    } else {
      ps->i++;
      ch = c;
      kind = 'c';
    }
    if (first) {
      first = 0;
      if (kind == 'c' || kind == 'd') {
        last = CHAR;
        last_c = kind == 'd' ? '-' : ch;
        continue;
      }
    }
    if (kind == 'c') {
      if (last == CHAR) setbit(chars, (unsigned)last_c);
      last = CHAR;
      last_c = ch;
    } else if (kind == 'k') {
      if (last == CHAR) setbit(chars, (unsigned)last_c);
      last = CLASS;
      if (cn) {
        if (nneg < 64) negcls[nneg++] = cm;
      } else {
        cls |= cm;
      }
    } else { /* dash */
      if (peek(ps) == ']') {
        ps->i++;
        if (last == CHAR) setbit(chars, (unsigned)last_c);
        last = CHAR;
        last_c = '-';
        break;
      }
      if (last == CLASS) {
        fail(ps, "class as range start");
        return -1;
      }
      if (last == CHAR) {
        /* range end: a char, an escape char, or '-' */
        int e = peek(ps), ec;
        if (e == '\\') {
          ps->i++;
          int r = escape(ps, 1, &ec, &cm, &cn);
          if (r != 0) {
            fail(ps, "bad range end");
            return -1;
          }
        } else if (e == '[' && ps->i + 1 < ps->len &&
                   (ps->p[ps->i + 1] == ':' || ps->p[ps->i + 1] == '.' || ps->p[ps->i + 1] == '=')) {
          fail(ps, "bad range end");
          return -1;
        } else {
          ec = e;
          ps->i++;
        }
        if ((signed char)last_c > (signed char)ec) {
          fail(ps, "range out of order");
          return -1;
        }
        if (nr < 256) {
          rl[nr] = (signed char)last_c;
          rh[nr] = (signed char)ec;
          nr++;
        }
        last = NONE;
      } else {
        if (last == CHAR) setbit(chars, (unsigned)last_c);
        last = CHAR;
        last_c = '-';
      }
    }
  }
  if (last == CHAR) setbit(chars, (unsigned)last_c);
  int n = node(ps, N_SET);
  for (unsigned u = 0; u < 256; ++u) {
    int m = getbit(chars, u);
    for (int k = 0; k < nr && !m; ++k) m = rl[k] <= (signed char)u && (signed char)u <= rh[k];
    if (!m) m = in_class(u, cls);
    for (int k = 0; k < nneg && !m; ++k) m = !in_class(u, negcls[k]);
    if (m != neg) setbit(ps->re->v[n].set, u);
  }
  return n;
}

static int set_node(P* ps, int (*pred)(unsigned, int), int arg, int neg) {
  int n = node(ps, N_SET);
  for (unsigned u = 0; u < 256; ++u)
    if (pred(u, arg) != neg) setbit(ps->re->v[n].set, u);
  return n;
}
static int pred_class(unsigned u, int mask) { return in_class(u, mask); }
static int pred_char(unsigned u, int c) { return (int)u == c; }
static int pred_any(unsigned u, int unused) {
  (void)unused;
  return u != '\n' && u != '\r';
}

static int atom(P* ps) {
  int c = peek(ps);
  if (c < 0) return -2;
  switch (c) {
    case '.': ps->i++; return set_node(ps, pred_any, 0, 0);
    case '(': {
      ps->i++;
      if (peek(ps) == '?') {
        if (ps->i + 1 < ps->len && ps->p[ps->i + 1] == ':') {
          ps->i += 2;
        } else {
          fail(ps, "lookahead / bad (? group unsupported");
          return -1;
        }
      }
      int r = disj(ps);
      if (ps->err) return -1;
      if (peek(ps) != ')') {
        fail(ps, "missing )");
        return -1;
      }
      ps->i++;
      return r;
    }
    case '[': ps->i++; return bracket(ps);
    case '\\': {
      ps->i++;
      int ch = 0, cm = 0, cn = 0;
      int r = escape(ps, 0, &ch, &cm, &cn);
      if (r < 0) return -1;
      if (r == 1) return set_node(ps, pred_class, cm, cn);
      if (r == 2) {
        ps->i -= 2; /* assertion, handled by term() */
        return -2;
      }
      return set_node(ps, pred_char, ch, 0);
    }
    case '*': case '+': case '?': case '{': case ')': case '|': case '^': case '$': return -2;
    default: ps->i++; return set_node(ps, pred_char, c, 0);
  }
}

static long number(P* ps, int* ok) {
  long v = 0;
  *ok = 0;
  while (!at_end(ps) && ps->p[ps->i] >= '0' && ps->p[ps->i] <= '9') {
    v = v * 10 + (ps->p[ps->i++] - '0');
    if (v > 0x7fffffffL) {
      fail(ps, "count overflow");
      return 0;
    }
    *ok = 1;
  }
  return v;
}

static int term(P* ps) {
  int c = peek(ps);
  if (c == '^' || c == '$') {
    ps->i++;
    int n = node(ps, N_ASSERT);
    ps->re->v[n].ak = c == '^' ? AS_BOL : AS_EOL;
    return n;
  }
  if (c == '\\' && ps->i + 1 < ps->len && (ps->p[ps->i + 1] == 'b' || ps->p[ps->i + 1] == 'B')) {
    int neg = ps->p[ps->i + 1] == 'B';
    ps->i += 2;
    int n = node(ps, N_ASSERT);
    ps->re->v[n].ak = neg ? AS_NWB : AS_WB;
    return n;
  }
  int a = atom(ps);
  if (a < 0) return a;
  for (;;) {
    int q = peek(ps);
    long mn, mx;
    if (q == '*') {
      mn = 0, mx = -1;
      ps->i++;
    } else if (q == '+') {
      mn = 1, mx = -1;
      ps->i++;
    } else if (q == '?') {
      mn = 0, mx = 1;
      ps->i++;
    } else if (q == '{') {
      ps->i++;
      int ok;
      mn = number(ps, &ok);
      if (!ok) {
        fail(ps, "bad brace");
        return -1;
      }
      mx = mn;
      if (peek(ps) == ',') {
        ps->i++;
        long m2 = number(ps, &ok);
        mx = ok ? m2 : -1;
      }
      if (peek(ps) != '}') {
        fail(ps, "bad brace end");
        return -1;
      }
      ps->i++;
      if (mx >= 0 && mx < mn) {
        fail(ps, "bad brace range");
        return -1;
      }
    } else {
      break;
    }
    if (peek(ps) == '?') ps->i++; /* lazy: same language */
    int r = node(ps, N_REP);
    ps->re->v[r].a = a;
    ps->re->v[r].min = mn;
    ps->re->v[r].max = mx;
    a = r;
  }
  return a;
}

static int alternative(P* ps) {
  int r = -1;
  for (;;) {
    int c = peek(ps);
    if (c < 0 || c == '|' || c == ')') break;
    int t = term(ps);
    if (t == -2) {
      fail(ps, "unexpected token");
      return -1;
    }
    if (t < 0) return -1;
    if (r < 0) {
      r = t;
    } else {
      int n = node(ps, N_CAT);
      ps->re->v[n].a = r;
      ps->re->v[n].b = t;
      r = n;
    }
  }
  return r < 0 ? node(ps, N_EMPTY) : r;
}

static int disj(P* ps) {
  int a = alternative(ps);
  while (!ps->err && peek(ps) == '|') {
    ps->i++;
    int b = alternative(ps);
    int n = node(ps, N_ALT);
    ps->re->v[n].a = a;
    ps->re->v[n].b = b;
    a = n;
  }
  return a;
}

static int parse_regex(Re* re, const char* p, size_t len, char* err, size_t errcap) {
  P ps;
  memset(&ps, 0, sizeof(ps));
  ps.re = re;
  ps.p = p;
  ps.len = len;
  re->root = disj(&ps);
  if (!ps.err && !at_end(&ps)) fail(&ps, "unbalanced )");
  if (ps.err) {
    if (err && errcap) snprintf(err, errcap, "%s", ps.msg);
    return -1;
  }
  return 0;
}

/* ---------------------------------------------------- backtracking search (regex_search) */
typedef struct Frame {
  int node;
  int repnext; /* 1: continuation of a REP iteration */
  long count, start;
  const struct Frame* next;
} Frame;

typedef struct {
  const Re* re;
  const uint8_t* s;
  long len;
  long budget;
} M;

static int m_node(M* m, int n, long i, const Frame* k);

static int m_cont(M* m, long i, const Frame* k) {
  if (--m->budget < 0) return 0;
  if (!k) return 1;
  if (!k->repnext) return m_node(m, k->node, i, k->next);
  if (i == k->start) return m_cont(m, i, k->next); /* empty iteration ends the loop */
  const RNode* r = &m->re->v[k->node];
  if (r->max < 0 || k->count < r->max) {
    Frame f = {k->node, 1, k->count + 1, i, k->next};
    if (m_node(m, r->a, i, &f)) return 1;
  }
  return k->count >= r->min && m_cont(m, i, k->next);
}

static int check_assert(M* m, int ak, long i) {
  int prev_w = i > 0 && is_word(m->s[i - 1]);
  int next_w = i < m->len && is_word(m->s[i]);
  switch (ak) {
    case AS_BOL: return i == 0;
    case AS_EOL: return i == m->len;
    case AS_WB: return prev_w != next_w;
    default: return prev_w == next_w;
  }
}

static int m_node(M* m, int n, long i, const Frame* k) {
  const RNode* r = &m->re->v[n];
  switch (r->kind) {
    case N_EMPTY: return m_cont(m, i, k);
    case N_SET: return i < m->len && getbit(r->set, m->s[i]) && m_cont(m, i + 1, k);
    case N_ASSERT: return check_assert(m, r->ak, i) && m_cont(m, i, k);
    case N_CAT: {
      Frame f = {r->b, 0, 0, 0, k};
      return m_node(m, r->a, i, &f);
    }
    case N_ALT: return m_node(m, r->a, i, k) || m_node(m, r->b, i, k);
    case N_REP: {
      if (r->max != 0) {
        Frame f = {n, 1, 1, i, k};
        if (m_node(m, r->a, i, &f)) return 1;
      }
      return r->min == 0 && m_cont(m, i, k);
    }
  }
  return 0;
}

static int regex_search(const Re* re, const uint8_t* s, long len, int* overflow) {
  M m = {re, s, len, 50000000L};
  for (long st = 0; st <= len; ++st) {
    if (m_node(&m, re->root, st, NULL)) return 1;
    if (m.budget < 0) {
      *overflow = 1;
      return 0;
    }
  }
  return 0;
}

/* ---------------------------------------------------------------- rule sets */
typedef struct {
  uint32_t n;
  Re* re;          /* per rule (regex kind) */
  uint8_t* kind;
  uint8_t* enabled;
  char** term;     /* per rule (blacklist kind) */
  uint32_t* tlen;
  int* term_owner; /* rule index that owns this blacklist term (last writer) */
} Rules;

void* orc_rules_create(uint32_t n, const char* const* patterns, const uint32_t* lens, const uint8_t* kinds,
                       const uint8_t* enabled, char* err, size_t errcap) {
  Rules* r = (Rules*)calloc(1, sizeof(Rules));
  r->n = n;
  r->re = (Re*)calloc(n ? n : 1, sizeof(Re));
  r->kind = (uint8_t*)malloc(n ? n : 1);
  r->enabled = (uint8_t*)malloc(n ? n : 1);
  r->term = (char**)calloc(n ? n : 1, sizeof(char*));
  r->tlen = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
  r->term_owner = (int*)calloc(n ? n : 1, sizeof(int));
  for (uint32_t i = 0; i < n; ++i) {
    r->kind[i] = kinds[i];
    r->enabled[i] = enabled[i];
    if (kinds[i] == 0) {
      if (parse_regex(&r->re[i], patterns[i], lens[i], err, errcap) != 0) {
        orc_rules_free(r);
        return NULL;
      }
    } else {
      r->term[i] = (char*)malloc(lens[i] + 1);
      memcpy(r->term[i], patterns[i], lens[i]);
      r->tlen[i] = lens[i];
    }
  }
  /* TokenTrie::add overwrites the rule index of an existing term (detection.hpp:62) */
  for (uint32_t i = 0; i < n; ++i) {
    r->term_owner[i] = -1;
    if (kinds[i] != 1) continue;
    int own = (int)i;
    for (uint32_t j = i + 1; j < n; ++j)
      if (kinds[j] == 1 && r->tlen[j] == r->tlen[i] && !memcmp(r->term[j], r->term[i], r->tlen[i])) own = (int)j;
    r->term_owner[i] = own;
  }
  return r;
}

void orc_rules_free(void* p) {
  Rules* r = (Rules*)p;
  if (!r) return;
  for (uint32_t i = 0; i < r->n; ++i) {
    free(r->re[i].v);
    free(r->term[i]);
  }
  free(r->re);
  free(r->kind);
  free(r->enabled);
  free(r->term);
  free(r->tlen);
  free(r->term_owner);
  free(r);
}

static int sep_char(unsigned c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r'; }
static int trim_char(unsigned c) {
  return c == '.' || c == ',' || c == ';' || c == ':' || c == '!' || c == '?' || c == '(' || c == ')' || c == '"' ||
         c == '\'';
}

/* CompiledRuleSet::scan (detection.hpp:148-170) as a per-rule hit mask: enabled regex
 * rules by regex_search; blacklist by TokenTrie::scan (detection.hpp:79-100). */
uint64_t orc_rules_mask(void* p, const uint8_t* text, size_t len) {
  Rules* r = (Rules*)p;
  uint64_t mask = 0;
  for (uint32_t i = 0; i < r->n && i < 64; ++i) {
    if (r->kind[i] != 0 || !r->enabled[i]) continue;
    int ovf = 0;
    if (regex_search(&r->re[i], text, (long)len, &ovf)) mask |= 1ull << i;
    if (ovf) mask |= 1ull << 63; /* budget exhausted: make the mismatch visible */
  }
  size_t i = 0;
  while (i < len) {
    while (i < len && sep_char(text[i])) ++i;
    size_t j = i;
    while (j < len && !sep_char(text[j])) ++j;
    size_t a = i, b = j;
    while (a < b && trim_char(text[a])) ++a;
    while (b > a && trim_char(text[b - 1])) --b;
    if (b > a) {
      for (uint32_t k = 0; k < r->n && k < 64; ++k) {
        if (r->kind[k] != 1 || r->term_owner[k] != (int)k) continue;
        if (r->tlen[k] == b - a && !memcmp(r->term[k], text + a, b - a) && r->enabled[k]) mask |= 1ull << k;
      }
    }
    i = j;
  }
  return mask;
}

/* ---------------------------------------------------------------- engine (Appendix A) */
typedef struct {
  uint64_t h, d, creator;
  long parent, first_child, next_sibling;
  uint8_t label, owner, tier;
  uint64_t hit_cur, u_cnt, hit_pre, u_pre;
  uint64_t users[64]; /* AccessStats::user_set, exact below saturation (access_stats.hpp:13-37) */
  uint32_t n_users;
} Ent;

typedef struct {
  uint64_t* h;
  uint64_t* d;
  uint8_t* label;
  uint32_t n;
  uint64_t user;
  uint8_t owner;
  /* serving observables of the lookup (CostModel::ttft / attribute_reuse inputs) */
  uint64_t L;
  uint32_t m;
  uint8_t* mtier; /* tier of matched block b */
  uint8_t* mown;  /* creator == user for matched block b */
} Pend;

typedef struct {
  Rules* rules;
  uint32_t B, W;
  double jump;
  uint64_t u_pre_max;
  Ent* e;
  size_t ne, cape;
  long* slots; /* open addressing: index into e, -1 empty */
  size_t nslot;
  Pend* pend;
  uint32_t npend;
  uint64_t epoch;
} Eng;

#define L_PRIVATE 0
#define L_PUBLIC 1
#define L_RESTRICTED 3

static uint64_t mix(uint64_t h, uint64_t d) {
  uint64_t x = h * 0x9e3779b97f4a7c15ULL ^ d;
  x ^= x >> 31;
  x *= 0xbf58476d1ce4e5b9ULL;
  return x ^ (x >> 29);
}

static long find(Eng* g, uint64_t h, uint64_t d) {
  size_t s = mix(h, d) & (g->nslot - 1);
  for (;;) {
    long k = g->slots[s];
    if (k < 0) return -1;
    if (g->e[k].h == h && g->e[k].d == d) return k;
    s = (s + 1) & (g->nslot - 1);
  }
}

static void rehash(Eng* g) {
  size_t ns = g->nslot ? g->nslot * 2 : 1024;
  free(g->slots);
  g->slots = (long*)malloc(ns * sizeof(long));
  for (size_t i = 0; i < ns; ++i) g->slots[i] = -1;
  g->nslot = ns;
  for (size_t k = 0; k < g->ne; ++k) {
    size_t s = mix(g->e[k].h, g->e[k].d) & (ns - 1);
    while (g->slots[s] >= 0) s = (s + 1) & (ns - 1);
    g->slots[s] = (long)k;
  }
}

static long insert(Eng* g, uint64_t h, uint64_t d) {
  if (2 * (g->ne + 1) > g->nslot) rehash(g);
  if (g->ne == g->cape) {
    g->cape = g->cape ? 2 * g->cape : 1024;
    g->e = (Ent*)realloc(g->e, g->cape * sizeof(Ent));
  }
  long k = (long)g->ne++;
  memset(&g->e[k], 0, sizeof(Ent));
  g->e[k].h = h;
  g->e[k].d = d;
  g->e[k].parent = g->e[k].first_child = g->e[k].next_sibling = -1;
  size_t s = mix(h, d) & (g->nslot - 1);
  while (g->slots[s] >= 0) s = (s + 1) & (g->nslot - 1);
  g->slots[s] = k;
  return k;
}

void* orc_engine_create(void* rules, uint32_t B, uint32_t W, double jump, uint64_t u_pre_max) {
  Eng* g = (Eng*)calloc(1, sizeof(Eng));
  g->rules = (Rules*)rules;
  g->B = B;
  g->W = W;
  g->jump = jump;
  g->u_pre_max = u_pre_max;
  rehash(g);
  return g;
}

static void clear_pending(Eng* g) {
  for (uint32_t i = 0; i < g->npend; ++i) {
    free(g->pend[i].h);
    free(g->pend[i].d);
    free(g->pend[i].label);
    free(g->pend[i].mtier);
    free(g->pend[i].mown);
  }
  free(g->pend);
  g->pend = NULL;
  g->npend = 0;
}

void orc_engine_free(void* p) {
  Eng* g = (Eng*)p;
  if (!g) return;
  clear_pending(g);
  free(g->e);
  free(g->slots);
  free(g);
}

/* AccessStats::record (access_stats.hpp:27-37) */
static void record(Ent* e, uint64_t user) {
  e->hit_cur++;
  for (uint32_t i = 0; i < e->n_users; ++i)
    if (e->users[i] == user) return;
  if (e->n_users < 64) e->users[e->n_users++] = user;
  e->u_cnt++;
}

int orc_engine_admit(void* p, const uint32_t* tok, const uint64_t* off, const uint64_t* users, const uint8_t* owners,
                     uint32_t n_prompts, uint64_t* out_h, uint64_t* out_d, uint64_t* out_mask, uint8_t* out_label,
                     uint8_t* out_decision, uint32_t* out_matched, uint8_t* out_tier) {
  Eng* g = (Eng*)p;
  clear_pending(g);
  g->pend = (Pend*)calloc(n_prompts ? n_prompts : 1, sizeof(Pend));
  g->npend = n_prompts;
  const uint32_t B = g->B;
  uint64_t k = 0;
  uint8_t* win = (uint8_t*)malloc(B + g->W + 1);
  for (uint32_t q = 0; q < n_prompts; ++q) {
    uint64_t L = off[q + 1] - off[q], n = L / B;
    const uint32_t* t = tok + off[q];
    Pend* pd = &g->pend[q];
    pd->n = (uint32_t)n;
    pd->user = users[q];
    pd->owner = owners ? owners[q] : 0;
    pd->h = (uint64_t*)malloc((n ? n : 1) * 8);
    pd->d = (uint64_t*)malloc((n ? n : 1) * 8);
    pd->label = (uint8_t*)malloc(n ? n : 1);
    pd->mtier = (uint8_t*)malloc(n ? n : 1);
    pd->mown = (uint8_t*)malloc(n ? n : 1);
    pd->L = L;
    uint64_t h = 0;
    int sens = 0;
    for (uint64_t b = 0; b < n; ++b) {
      uint64_t d = orc_token_seq_digest(t + b * B, B);
      h = orc_chain(h, d);
      /* A.3: window [bB, min(L, (b+1)B + W)) as bytes (detokenize_bytes, core.hpp:114-119) */
      uint64_t e = (b + 1) * B + g->W;
      if (e > L) e = L;
      for (uint64_t x = b * B; x < e; ++x) win[x - b * B] = (uint8_t)(t[x] & 0xff);
      uint64_t m = orc_rules_mask(g->rules, win, (size_t)(e - b * B));
      sens = sens || m != 0; /* A.4 prefix-OR */
      pd->h[b] = out_h[k + b] = h;
      pd->d[b] = out_d[k + b] = d;
      out_mask[k + b] = m;
      pd->label[b] = out_label[k + b] = sens ? L_PRIVATE : L_PUBLIC;
    }
    /* A.5 lookup: leading blocks present and visible (cache_index.hpp:213-237, 483-485) */
    uint32_t mt = 0;
    uint8_t tier = 0;
    for (uint64_t b = 0; b < n; ++b) {
      long x = find(g, pd->h[b], pd->d[b]);
      if (x < 0) break;
      Ent* en = &g->e[x];
      if (!(en->label == L_PUBLIC || en->creator == pd->user)) break;
      out_decision[k + b] = en->label == L_PUBLIC ? 1 : 2;
      if (en->tier > tier) tier = en->tier;
      pd->mtier[b] = en->tier;
      pd->mown[b] = en->creator == pd->user;
      record(en, pd->user); /* A.6 record, prompt order */
      mt++;
    }
    for (uint64_t b = mt; b < n; ++b) out_decision[k + b] = 0;
    pd->m = mt;
    out_matched[q] = mt;
    out_tier[q] = tier;
    k += n;
  }
  free(win);
  return 0;
}

/* Serving observables of the last admit.  CostModel::ttft (serving_sim.hpp:50-56):
 * t = t_base + c_prefill * (L - m*B), then + penalty[tier] * B per matched block in path
 * order, + sigma * Box-Muller normal of SplitMix64(derive_seed(seed, request_id))
 * (util.hpp:14-55), floored at t_base.  attribute_reuse (serving_sim.hpp:313-324):
 * matched tokens on entries the user created (intra) or others created (inter). */
static uint64_t sm64(uint64_t* st) {
  uint64_t z = (*st += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

int orc_engine_ttft(void* p, const uint64_t* request_ids, double t_base, double c_prefill, double pen_dram,
                    double pen_ssd, double sigma, uint64_t seed, double* out_ttft, uint32_t* out_intra,
                    uint32_t* out_inter) {
  Eng* g = (Eng*)p;
  const double pen[3] = {0.0, pen_dram, pen_ssd};
  for (uint32_t q = 0; q < g->npend; ++q) {
    const Pend* pd = &g->pend[q];
    double t = t_base + c_prefill * (double)(pd->L - (uint64_t)pd->m * g->B);
    uint32_t own = 0;
    for (uint32_t b = 0; b < pd->m; ++b) {
      t += pen[pd->mtier[b]] * (double)g->B;
      own += pd->mown[b];
    }
    double noise = 0.0;
    if (sigma != 0.0) {
      const uint64_t rid = request_ids ? request_ids[q] : q;
      uint64_t st = seed ^ (0x51a1c9e3b7d24f85ULL * (rid + 1));
      uint64_t st2 = sm64(&st);
      double u1 = (double)(sm64(&st2) >> 11) * 0x1.0p-53;
      const double u2 = (double)(sm64(&st2) >> 11) * 0x1.0p-53;
      if (u1 <= 0.0) u1 = 0x1.0p-53;
      noise = sigma * (sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
    }
    t += noise;
    out_ttft[q] = t < t_base ? t_base : t;
    out_intra[q] = own * g->B;
    out_inter[q] = (pd->m - own) * g->B;
  }
  return 0;
}

/* A.7 commit in prompt order: first creator wins (cache_index.hpp:164-168) */
int orc_engine_commit(void* p) {
  Eng* g = (Eng*)p;
  for (uint32_t q = 0; q < g->npend; ++q) {
    Pend* pd = &g->pend[q];
    long parent = -1;
    for (uint32_t b = 0; b < pd->n; ++b) {
      long x = find(g, pd->h[b], pd->d[b]);
      if (x < 0) {
        x = insert(g, pd->h[b], pd->d[b]);
        Ent* en = &g->e[x];
        en->creator = pd->user;
        en->owner = pd->owner;
        en->label = pd->label[b];
        en->tier = 0;
        en->parent = parent;
        if (parent >= 0) {
          en->next_sibling = g->e[parent].first_child;
          g->e[parent].first_child = x;
        }
      }
      parent = x;
    }
  }
  clear_pending(g);
  return 0;
}

int orc_engine_set_tiers(void* p, const uint32_t* tok, const uint64_t* off, uint32_t n_prompts, const uint8_t* tiers) {
  Eng* g = (Eng*)p;
  uint64_t k = 0;
  for (uint32_t q = 0; q < n_prompts; ++q) {
    uint64_t n = (off[q + 1] - off[q]) / g->B, h = 0;
    for (uint64_t b = 0; b < n; ++b, ++k) {
      uint64_t d = orc_token_seq_digest(tok + off[q] + b * g->B, g->B);
      h = orc_chain(h, d);
      long x = find(g, h, d);
      if (x < 0) return -1;
      if (tiers[k] > g->e[x].tier) g->e[x].tier = tiers[k]; /* demote: tiers only move down */
    }
  }
  return 0;
}

static void label_subtree(Eng* g, long x, uint8_t lab) {
  /* set_label(..., propagate=true): node and every descendant (cache_index.hpp:654-685) */
  g->e[x].label = lab;
  for (long c = g->e[x].first_child; c >= 0; c = g->e[c].next_sibling) label_subtree(g, c, lab);
}

typedef struct {
  uint64_t h, d;
  uint8_t a;
  double now, prev;
  uint64_t upre;
} Ev;

static int ev_cmp(const void* x, const void* y) {
  const Ev* a = (const Ev*)x;
  const Ev* b = (const Ev*)y;
  if (a->h != b->h) return a->h < b->h ? -1 : 1;
  if (a->d != b->d) return a->d < b->d ? -1 : 1;
  return 0;
}

/* advance_epoch + EntropyMonitor::epoch_pass (monitor.hpp:85-99): entries visited
 * ancestor-first (creation order is a topological order of the prefix tree). */
int orc_engine_epoch(void* p, uint64_t* out_epoch, size_t cap, uint64_t* ev_h, uint64_t* ev_d, uint8_t* ev_action,
                     double* ev_now, double* ev_prev, uint64_t* ev_upre, size_t* n_events) {
  Eng* g = (Eng*)p;
  uint64_t epoch = ++g->epoch;
  Ev* ev = NULL;
  size_t ne = 0, ce = 0;
  for (size_t x = 0; x < g->ne; ++x) {
    Ent* e = &g->e[x];
    if (e->label != L_PUBLIC || !(e->hit_cur > 0 || e->hit_pre > 0)) continue;
    /* window_entropy (access_stats.hpp:50-57) and check_anomaly (monitor.hpp:56-81) */
    double now = e->hit_cur ? (double)e->u_cnt / (double)e->hit_cur : 0.0;
    double prev = e->hit_pre ? (double)e->u_pre / (double)e->hit_pre : 0.0;
    if (!(e->hit_pre > 0 && (now - prev) >= g->jump && e->u_pre <= g->u_pre_max)) continue;
    uint8_t act = e->owner == 0 ? 1 : 2;
    label_subtree(g, (long)x, e->owner == 0 ? L_PRIVATE : L_RESTRICTED);
    if (ne == ce) {
      ce = ce ? 2 * ce : 64;
      ev = (Ev*)realloc(ev, ce * sizeof(Ev));
    }
    Ev v = {e->h, e->d, act, now, prev, e->u_pre};
    ev[ne++] = v;
  }
  for (size_t x = 0; x < g->ne; ++x) { /* AccessStats::roll (access_stats.hpp:39-45) */
    Ent* e = &g->e[x];
    e->hit_pre = e->hit_cur;
    e->u_pre = e->u_cnt;
    e->hit_cur = e->u_cnt = 0;
    e->n_users = 0;
  }
  if (ne) qsort(ev, ne, sizeof(Ev), ev_cmp);
  for (size_t i = 0; i < ne && i < cap; ++i) {
    ev_h[i] = ev[i].h;
    ev_d[i] = ev[i].d;
    ev_action[i] = ev[i].a;
    ev_now[i] = ev[i].now;
    ev_prev[i] = ev[i].prev;
    ev_upre[i] = ev[i].upre;
  }
  free(ev);
  *n_events = ne;
  *out_epoch = epoch;
  return 0;
}

size_t orc_engine_export(void* p, size_t cap, uint64_t* h, uint64_t* d, uint64_t* creator, uint8_t* label,
                         uint8_t* owner, uint8_t* tier, uint64_t* hit_cur, uint64_t* u_cnt, uint64_t* hit_pre,
                         uint64_t* u_pre) {
  Eng* g = (Eng*)p;
  for (size_t i = 0; i < g->ne && i < cap; ++i) {
    Ent* e = &g->e[i];
    h[i] = e->h;
    d[i] = e->d;
    creator[i] = e->creator;
    label[i] = e->label;
    owner[i] = e->owner;
    tier[i] = e->tier;
    hit_cur[i] = e->hit_cur;
    u_cnt[i] = e->u_cnt;
    hit_pre[i] = e->hit_pre;
    u_pre[i] = e->u_pre;
  }
  return g->ne;
}
