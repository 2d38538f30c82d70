// ir_interp.cpp -- a fast, fixed interpreter of the reference's IR.
//
// TEST INFRASTRUCTURE (never linked by the product).  It
// executes any function of a reference Module (serialised by
// oracle/ir_export.py) with the semantics of the reference's value-semantics
// interpreter, /root/reference/pkg/src/skiff/runtime/oracle.py:28-320:
//
//  * the control token walks start -> ... -> return (oracle.py:233-268);
//    a region binds its phis from the entering predecessor, then clears the
//    cached values that depend on them (oracle.py:245-255); an `if` follows
//    the projection selected by its condition;
//  * a fork runs the product of its factors in lexicographic order, dim 0
//    outermost (oracle.py:270-312): per iteration the thread ids are bound,
//    the body is walked to the join, and every reduce folds its reduct;
//    a zero-trip fork leaves each reduce at its init;
//  * data nodes are evaluated on demand and cached (oracle.py:76-125);
//  * scalar arithmetic follows runtime/values.py:24-115 (one rounding per
//    f32/f64 op, no FMA -- this file is compiled with -ffp-contract=off;
//    integer div/rem truncate toward zero and raise on zero; ints wrap;
//    Python min/max; casts truncate and raise out of range / on NaN);
//  * reads and writes are bounds-checked; writes have value semantics.
//
// Two defects of the reference interpreter are fixed:
//  1. the dependents walk that clears cached values stops at phi / reduce
//     nodes that are not being rebound (the reference walks through them and
//     wipes enclosing loop-carried values: crashes on tap loops, scalar
//     accumulators and Fig. 10 reduction trees);
//  2. after a fork, the walk continues from its join as the predecessor
//     (the reference records the fork, so a region reached right after a
//     nested fork fails its predecessor lookup, oracle.py:247).
// And the O(array) copy per element write (oracle.py:190) becomes an in-place
// write whenever the written collection's value is provably dead: its
// buffer is referenced only by that node, every other data user of it has
// already been evaluated in this iteration, and no phi / reduce / call /
// return consumes it (the spill-free case of the paper's GCM rule,
// PAPER.md:362).  Otherwise the write copies, as the reference does.
//
// Supported: scalars and (multi-dimensional) arrays of scalars, calls.
// Products / summations raise "unsupported" (none of the benchmarks use
// them).  Errors come back as "<Class>: message" with the reference's class
// names (RuntimeError_, DynConstError, OracleLimitError, OverflowError,
// ValueError).
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

// ------------------------------------------------------------------ errors
struct Err : std::runtime_error {
  explicit Err(const std::string &cls, const std::string &m) : std::runtime_error(cls + ": " + m) {}
};
[[noreturn]] void fail(const char *cls, const std::string &m) { throw Err(cls, m); }

// -------------------------------------------------------------------- JSON
struct J {
  enum T { NUL, BOOL, INT, DBL, STR, ARR, OBJ } t = NUL;
  bool b = false;
  long long i = 0;
  unsigned long long u = 0;
  bool is_u = false;  // integer above INT64_MAX
  double d = 0;
  std::string s;
  std::vector<J> a;
  std::vector<std::pair<std::string, J>> o;
  const J *get(const char *k) const {
    for (auto &kv : o)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct Parser {
  const char *p;
  void ws() {
    while (*p == ' ' || *p == '\n' || *p == '\t' || *p == '\r') p++;
  }
  J parse() {
    ws();
    J v;
    if (*p == '{') {
      v.t = J::OBJ;
      p++;
      ws();
      if (*p == '}') { p++; return v; }
      for (;;) {
        ws();
        J k = parse();
        ws();
        if (*p != ':') fail("ValueError", "bad JSON object");
        p++;
        J val = parse();
        v.o.emplace_back(k.s, std::move(val));
        ws();
        if (*p == ',') { p++; continue; }
        if (*p == '}') { p++; break; }
        fail("ValueError", "bad JSON object");
      }
    } else if (*p == '[') {
      v.t = J::ARR;
      p++;
      ws();
      if (*p == ']') { p++; return v; }
      for (;;) {
        v.a.push_back(parse());
        ws();
        if (*p == ',') { p++; continue; }
        if (*p == ']') { p++; break; }
        fail("ValueError", "bad JSON array");
      }
    } else if (*p == '"') {
      v.t = J::STR;
      p++;
      while (*p && *p != '"') {
        if (*p == '\\') p++;
        v.s += *p++;
      }
      p++;
    } else if (!strncmp(p, "null", 4)) {
      p += 4;
    } else if (!strncmp(p, "true", 4)) {
      v.t = J::BOOL; v.b = true; p += 4;
    } else if (!strncmp(p, "false", 5)) {
      v.t = J::BOOL; v.b = false; p += 5;
    } else {
      const char *q = p;
      bool flt = false;
      if (*q == '-') q++;
      while ((*q >= '0' && *q <= '9') || *q == '.' || *q == 'e' || *q == 'E' || *q == '+' || *q == '-') {
        if (*q == '.' || *q == 'e' || *q == 'E') flt = true;
        q++;
      }
      if (flt) {
        v.t = J::DBL; v.d = strtod(p, nullptr);
      } else {
        v.t = J::INT;
        errno = 0;
        v.i = strtoll(p, nullptr, 10);
        if (errno == ERANGE && *p != '-') { v.is_u = true; v.u = strtoull(p, nullptr, 10); }
      }
      p = q;
    }
    return v;
  }
};

// ------------------------------------------------------------------- types
enum DT : int8_t { BOOLT = 0, I8, I16, I32, I64, U8, U16, U32, U64, F32, F64 };
const char *DT_NAMES[] = {"bool", "i8", "i16", "i32", "i64", "u8", "u16", "u32", "u64", "f32", "f64"};
int dt_size(DT t) {
  switch (t) {
    case BOOLT: case I8: case U8: return 1;
    case I16: case U16: return 2;
    case I32: case U32: case F32: return 4;
    default: return 8;
  }
}
bool dt_int(DT t) { return t >= I8 && t <= U64; }
bool dt_signed(DT t) { return t >= I8 && t <= I64; }
bool dt_float(DT t) { return t == F32 || t == F64; }
int dt_bits(DT t) { return dt_size(t) * 8; }

DT dt_of(const std::string &s) {
  for (int i = 0; i <= F64; i++)
    if (s == DT_NAMES[i]) return (DT)i;
  fail("RuntimeError_", "unknown scalar type " + s);
}

struct Dc {  // dynamic-constant expression
  char op = 0;  // 0 literal, 'p' param, + - * /
  long long v = 0;
  std::shared_ptr<Dc> a, b;
};
std::shared_ptr<Dc> dc_of(const J &j) {
  auto d = std::make_shared<Dc>();
  if (auto p = j.get("p")) { d->op = 'p'; d->v = p->i; return d; }
  if (auto l = j.get("l")) { d->op = 0; d->v = l->i; return d; }
  d->op = j.get("o")->s[0];
  d->a = dc_of(*j.get("a"));
  d->b = dc_of(*j.get("b"));
  return d;
}
long long dc_eval(const Dc &d, const std::vector<long long> &p) {  // dynconst.py:179-204
  if (d.op == 0) return d.v;
  if (d.op == 'p') {
    if (d.v >= (long long)p.size()) fail("DynConstError", "dynamic-constant parameter #" + std::to_string(d.v) + " not supplied");
    return p[d.v];
  }
  const long long l = dc_eval(*d.a, p), r = dc_eval(*d.b, p);
  switch (d.op) {
    case '+': return l + r;
    case '*': return l * r;
    case '-':
      if (l < r) fail("DynConstError", "negative dynamic constant: " + std::to_string(l) + " - " + std::to_string(r));
      return l - r;
    default:
      if (r == 0) fail("DynConstError", "division of a dynamic constant by zero");
      if (l % r) fail("DynConstError", "inexact dynamic-constant division " + std::to_string(l) + "/" + std::to_string(r));
      return l / r;
  }
}

struct Ty {
  bool arr = false;
  DT dt = F32;  // scalar type, or the element type of an array
  std::vector<std::shared_ptr<Dc>> ext;
};
Ty ty_of(const J &j) {
  Ty t;
  if (j.t == J::STR) { t.dt = dt_of(j.s); return t; }
  if (auto a = j.get("arr")) {
    t.arr = true;
    if (a->t != J::STR) fail("RuntimeError_", "unsupported: arrays of collections");
    t.dt = dt_of(a->s);
    for (auto &e : j.get("ext")->a) t.ext.push_back(dc_of(e));
    return t;
  }
  fail("RuntimeError_", "unsupported: product / summation types");
}

// ------------------------------------------------------------------ values
struct Arr {
  DT dt;
  std::vector<long long> shape;
  std::vector<uint8_t> data;
  size_t count() const {
    size_t n = 1;
    for (auto s : shape) n *= (size_t)s;
    return n;
  }
};
struct Val {
  enum K : int8_t { NONE, SCAL, ARRAY, MOVED } k = NONE;
  DT dt = F32;  // scalar type (numpy scalar dtype); bool is Python bool
  union { int64_t i; uint64_t u; float f; double d; bool b; } x{};
  std::shared_ptr<Arr> a;
};

Val scal_i(DT dt, int64_t v) { Val r; r.k = Val::SCAL; r.dt = dt; r.x.i = v; return r; }
Val scal_u(DT dt, uint64_t v) { Val r; r.k = Val::SCAL; r.dt = dt; r.x.u = v; return r; }
Val scal_f(float v) { Val r; r.k = Val::SCAL; r.dt = F32; r.x.f = v; return r; }
Val scal_d(double v) { Val r; r.k = Val::SCAL; r.dt = F64; r.x.d = v; return r; }
Val scal_b(bool v) { Val r; r.k = Val::SCAL; r.dt = BOOLT; r.x.b = v; return r; }

// wrap an integer into dt (two's complement), as numpy's fixed-width types
Val wrap_int(DT dt, uint64_t bits) {
  const int nb = dt_bits(dt);
  if (nb < 64) {
    const uint64_t m = (1ull << nb) - 1;
    bits &= m;
    if (dt_signed(dt) && (bits >> (nb - 1))) bits |= ~m;  // sign-extend
  }
  Val r; r.k = Val::SCAL; r.dt = dt; r.x.u = bits;
  return r;
}
// Python-int view of an integer scalar: (negative?, magnitude) via __int128
__int128 as_i128(const Val &v) {
  if (v.dt == BOOLT) return v.x.b ? 1 : 0;
  if (dt_signed(v.dt)) return (__int128)v.x.i;
  return (__int128)v.x.u;
}
double as_double(const Val &v) {
  switch (v.dt) {
    case BOOLT: return v.x.b ? 1.0 : 0.0;
    case F32: return (double)v.x.f;
    case F64: return v.x.d;
    default: return dt_signed(v.dt) ? (double)v.x.i : (double)v.x.u;
  }
}
bool truthy(const Val &v) {
  switch (v.dt) {
    case BOOLT: return v.x.b;
    case F32: return v.x.f != 0.0f;
    case F64: return v.x.d != 0.0;
    default: return v.x.u != 0;
  }
}
// numpy_dtype(ty).type(int(value)): raises OverflowError out of range (numpy 2)
Val int_in_range(DT dt, __int128 v) {
  const int nb = dt_bits(dt);
  __int128 lo, hi;
  if (dt_signed(dt)) { lo = -((__int128)1 << (nb - 1)); hi = ((__int128)1 << (nb - 1)) - 1; }
  else { lo = 0; hi = (nb == 64) ? (__int128)UINT64_MAX : (((__int128)1 << nb) - 1); }
  if (v < lo || v > hi) fail("OverflowError", std::string("Python integer out of bounds for ") + DT_NAMES[dt]);
  return wrap_int(dt, (uint64_t)v);
}
// typed_scalar(value, ty) (values.py:24-31)
Val typed_scalar(const Val &v, DT dt) {
  if (dt == BOOLT) return scal_b(truthy(v));
  if (dt_int(dt)) {
    __int128 iv;
    if (dt_float(v.dt)) {  // int(float): trunc; NaN -> ValueError, inf -> OverflowError
      const double x = as_double(v);
      if (std::isnan(x)) fail("ValueError", "cannot convert float NaN to integer");
      if (std::isinf(x)) fail("OverflowError", "cannot convert float infinity to integer");
      const double t = std::trunc(x);
      if (t >= 1.7e38 || t <= -1.7e38) fail("OverflowError", "Python integer out of bounds");
      iv = (__int128)t;
    } else {
      iv = as_i128(v);
    }
    return int_in_range(dt, iv);
  }
  // float(value) then the numpy float type: ints go through double (one
  // rounding), then round once more to f32
  double x;
  if (dt_float(v.dt) || v.dt == BOOLT) x = as_double(v);
  else x = dt_signed(v.dt) ? (double)v.x.i : (double)v.x.u;
  return dt == F32 ? scal_f((float)x) : scal_d(x);
}

// ----------------------------------------------------------- scalar ops
template <typename F32OP, typename F64OP, typename IOP>
Val arith(const Val &a0, const Val &b0, DT ty, F32OP f32, F64OP f64, IOP iop) {
  if (ty == F32) return scal_f(f32(a0.dt == F32 ? a0.x.f : (float)as_double(a0), b0.dt == F32 ? b0.x.f : (float)as_double(b0)));
  if (ty == F64) return scal_d(f64(as_double(a0), as_double(b0)));
  const uint64_t a = (uint64_t)as_i128(a0), b = (uint64_t)as_i128(b0);
  return wrap_int(ty, iop(a, b));
}

int cmp3(const Val &a, const Val &b) {  // numeric compare, NaN -> 2 (unordered)
  if (dt_float(a.dt) || dt_float(b.dt)) {
    const double x = as_double(a), y = as_double(b);
    if (std::isnan(x) || std::isnan(y)) return 2;
    return x < y ? -1 : (x > y ? 1 : 0);
  }
  const __int128 x = as_i128(a), y = as_i128(b);
  return x < y ? -1 : (x > y ? 1 : 0);
}

enum Op { O_ADD, O_SUB, O_MUL, O_DIV, O_REM, O_AND, O_OR, O_XOR, O_SHL, O_SHR, O_MIN, O_MAX, O_LT, O_LE, O_GT,
          O_GE, O_EQ, O_NE, O_NEG, O_NOT, O_CAST, O_NONE };
const char *OP_NAMES[] = {"add", "sub", "mul", "div", "rem", "and", "or", "xor", "shl", "shr", "min",
                          "max", "lt", "le", "gt", "ge", "eq", "ne", "neg", "not", "cast"};
int op_of(const std::string &s) {
  for (int i = 0; i < O_NONE; i++)
    if (s == OP_NAMES[i]) return i;
  return O_NONE;
}

Val binop(int op, const Val &a, const Val &b, DT ty) {  // values.py:55-103
  switch (op) {
  case O_ADD:
    return arith(a, b, ty, [](float x, float y) { return x + y; }, [](double x, double y) { return x + y; },
                 [](uint64_t x, uint64_t y) { return x + y; });
  case O_SUB:
    return arith(a, b, ty, [](float x, float y) { return x - y; }, [](double x, double y) { return x - y; },
                 [](uint64_t x, uint64_t y) { return x - y; });
  case O_MUL:
    return arith(a, b, ty, [](float x, float y) { return x * y; }, [](double x, double y) { return x * y; },
                 [](uint64_t x, uint64_t y) { return x * y; });
  case O_DIV:
  case O_REM:
    if (dt_int(ty)) {
      const __int128 x = as_i128(a), y = as_i128(b);
      if (y == 0) fail("RuntimeError_", op == O_DIV ? "integer division by zero" : "integer remainder by zero");
      if (op == O_DIV) return int_in_range(ty, x / y);  // C++ truncates toward zero, as values.py:64-70
      return int_in_range(ty, x % y);                    // np.fmod: sign of the dividend
    }
    if (op == O_DIV) return arith(a, b, ty, [](float x, float y) { return x / y; }, [](double x, double y) { return x / y; },
                                  [](uint64_t x, uint64_t) { return x; });
    return arith(a, b, ty, [](float x, float y) { return std::fmod(x, y); },
                 [](double x, double y) { return std::fmod(x, y); }, [](uint64_t x, uint64_t) { return x; });
  case O_AND:
  case O_OR:
  case O_XOR: {
    if (a.dt == BOOLT && b.dt == BOOLT) {
      const bool x = a.x.b, y = b.x.b;
      return scal_b(op == O_AND ? (x && y) : op == O_OR ? (x || y) : (x != y));
    }
    const uint64_t x = (uint64_t)as_i128(a), y = (uint64_t)as_i128(b);
    const DT t = dt_int(ty) ? ty : (dt_int(a.dt) ? a.dt : b.dt);
    return wrap_int(t, op == O_AND ? (x & y) : op == O_OR ? (x | y) : (x ^ y));
  }
  case O_SHL:
  case O_SHR: {
    const DT t = dt_int(ty) ? ty : a.dt;
    const __int128 sh = as_i128(b);
    const int nb = dt_bits(t);
    if (op == O_SHL) return wrap_int(t, (sh < 0 || sh >= nb) ? 0 : ((uint64_t)as_i128(a) << (int)sh));
    if (dt_signed(t)) {
      const int64_t x = a.x.i;
      return wrap_int(t, (uint64_t)((sh < 0 || sh >= nb) ? (x < 0 ? -1 : 0) : (x >> (int)sh)));
    }
    return wrap_int(t, (sh < 0 || sh >= nb) ? 0 : (a.x.u >> (int)sh));
  }
  case O_MIN: return cmp3(b, a) == -1 ? b : a;  // Python builtins: first operand wins
  case O_MAX: return cmp3(b, a) == 1 ? b : a;
  case O_LT: return scal_b(cmp3(a, b) == -1);
  case O_LE: { const int c = cmp3(a, b); return scal_b(c == -1 || c == 0); }
  case O_GT: return scal_b(cmp3(a, b) == 1);
  case O_GE: { const int c = cmp3(a, b); return scal_b(c == 1 || c == 0); }
  case O_EQ: return scal_b(cmp3(a, b) == 0);
  case O_NE: return scal_b(cmp3(a, b) != 0);
  default: fail("RuntimeError_", "unknown binary op");
  }
}

Val unop(int op, const Val &a, DT ty) {  // values.py:106-115
  if (op == O_NEG) {
    if (a.dt == F32) return scal_f(-a.x.f);
    if (a.dt == F64) return scal_d(-a.x.d);
    if (a.dt == BOOLT) return scal_i(I64, a.x.b ? -1 : 0);
    return wrap_int(a.dt, (uint64_t)(-(int64_t)a.x.u));
  }
  if (op == O_NOT) return scal_b(!truthy(a));
  if (op == O_CAST) return typed_scalar(a, ty);
  fail("RuntimeError_", "unknown unary op");
}

// ---------------------------------------------------------------- IR
struct Index {
  char kind;  // 'P' position, 'F' field, 'V' variant
  std::vector<int> ids;
};
struct Node {
  std::string kind;
  int control = -1;
  std::vector<int> inputs, preds;
  int sel = 0, dim = 0, index = 0;
  std::vector<std::shared_ptr<Dc>> factors, dca;
  bool has_cv = false;
  J cv;
  std::shared_ptr<Dc> dc;
  std::string op, callee;
  std::vector<Index> idx;
  bool has_ty = false;
  Ty ty;
  bool live = false, is_control = false, is_bound = false;
  // kind / operator codes for the hot paths
  int code = 0, opc = 0;
};
enum Code { C_OTHER, C_BINARY, C_UNARY, C_READ, C_WRITE, C_CALL, C_PHI, C_REDUCE, C_TID, C_PARAM, C_CONST, C_DYNC };

struct Function {
  std::string name;
  int num_dc = 0;
  std::vector<Ty> params;
  Ty ret;
  std::vector<Node> nodes;
  std::vector<std::vector<int>> users, succ;
  int start = -1;
  std::map<int, int> join_of;               // fork -> join
  std::map<int, std::vector<int>> tids_of;  // fork -> thread ids
  std::map<int, std::vector<int>> reduces_of;  // join -> reduces
  std::map<int, std::vector<int>> phis_of;     // region -> phis (users order)
};

bool control_kind(const std::string &k) {
  return k == "start" || k == "region" || k == "if" || k == "proj" || k == "return" || k == "fork" || k == "join";
}

Function load_function(const std::string &name, const J &f) {
  Function fn;
  fn.name = name;
  fn.num_dc = (int)f.get("num_dyn_consts")->i;
  for (auto &p : f.get("params")->a) {
    if (p.t == J::STR || p.get("arr")) fn.params.push_back(ty_of(p));
    else fn.params.push_back(Ty{});  // unsupported param type: caught on use
  }
  const J &nodes = *f.get("nodes");
  fn.nodes.resize(nodes.a.size());
  for (size_t i = 0; i < nodes.a.size(); i++) {
    const J &j = nodes.a[i];
    if (j.t == J::NUL) continue;
    Node &n = fn.nodes[i];
    n.live = true;
    n.kind = j.get("k")->s;
    n.is_control = control_kind(n.kind);
    if (auto c = j.get("c")) n.control = (int)c->i;
    if (auto x = j.get("i")) for (auto &e : x->a) n.inputs.push_back((int)e.i);
    if (auto x = j.get("p")) for (auto &e : x->a) n.preds.push_back((int)e.i);
    if (auto x = j.get("sel")) n.sel = (int)x->i;
    if (auto x = j.get("d")) n.dim = (int)x->i;
    if (auto x = j.get("ix")) n.index = (int)x->i;
    if (auto x = j.get("f")) for (auto &e : x->a) n.factors.push_back(dc_of(e));
    if (auto x = j.get("dca")) for (auto &e : x->a) n.dca.push_back(dc_of(e));
    if (auto x = j.get("cv")) { n.has_cv = true; n.cv = *x->get("v"); }
    if (auto x = j.get("dc")) n.dc = dc_of(*x);
    if (auto x = j.get("op")) { n.op = x->s; n.opc = op_of(n.op); }
    if (auto x = j.get("callee")) n.callee = x->s;
    if (auto x = j.get("idx"))
      for (auto &e : x->a) {
        Index ix;
        ix.kind = e.a[0].s[0];
        if (ix.kind == 'P') for (auto &q : e.a[1].a) ix.ids.push_back((int)q.i);
        else fail("RuntimeError_", "unsupported: product field / summation variant indices");
        n.idx.push_back(ix);
      }
    if (auto x = j.get("ty")) {
      if (x->t == J::STR || x->get("arr")) { n.has_ty = true; n.ty = ty_of(*x); }
    }
    const std::string &k = n.kind;
    n.code = k == "binary" ? C_BINARY : k == "unary" ? C_UNARY : k == "read" ? C_READ : k == "write" ? C_WRITE
           : k == "call" ? C_CALL : k == "phi" ? C_PHI : k == "reduce" ? C_REDUCE : k == "thread_id" ? C_TID
           : k == "param" ? C_PARAM : k == "constant" ? C_CONST : k == "dynconst" ? C_DYNC : C_OTHER;
    n.is_bound = n.code == C_PHI || n.code == C_REDUCE || n.code == C_TID || n.code == C_PARAM ||
                 n.code == C_CONST || n.code == C_DYNC;
    if (n.kind == "start") fn.start = (int)i;
  }
  const int N = (int)fn.nodes.size();
  fn.users.assign(N, {});
  fn.succ.assign(N, {});
  for (int i = 0; i < N; i++) {  // def_use order (analysis.py:19-29)
    const Node &n = fn.nodes[i];
    if (!n.live) continue;
    std::vector<int> ins;
    if (n.control >= 0) ins.push_back(n.control);
    ins.insert(ins.end(), n.preds.begin(), n.preds.end());
    ins.insert(ins.end(), n.inputs.begin(), n.inputs.end());
    for (auto &ix : n.idx) ins.insert(ins.end(), ix.ids.begin(), ix.ids.end());
    std::vector<int> seen;
    for (int in : ins) {
      bool dup = false;
      for (int s : seen) dup |= s == in;
      if (dup || in < 0 || in >= N) continue;
      seen.push_back(in);
      fn.users[in].push_back(i);
    }
    if (n.is_control) {  // control_successors (analysis.py:36-50), sorted
      std::vector<int> ps;
      if (n.control >= 0) ps.push_back(n.control);
      ps.insert(ps.end(), n.preds.begin(), n.preds.end());
      for (int p : ps)
        if (p >= 0 && p < N && fn.nodes[p].live && fn.nodes[p].is_control) fn.succ[p].push_back(i);
    }
    if (n.code == C_TID) fn.tids_of[n.control].push_back(i);
    if (n.code == C_REDUCE) fn.reduces_of[n.control].push_back(i);
  }
  for (int i = 0; i < N; i++) {
    if (!fn.nodes[i].live) continue;
    std::sort(fn.succ[i].begin(), fn.succ[i].end());
    if (fn.nodes[i].kind == "region")
      for (int u : fn.users[i])
        if (fn.nodes[u].code == C_PHI && fn.nodes[u].control == i) fn.phis_of[i].push_back(u);
  }
  // fork -> join: follow the control tokens with a nesting counter (analysis.py:199-237)
  for (int f = 0; f < N; f++) {
    if (!fn.nodes[f].live || fn.nodes[f].kind != "fork") continue;
    std::vector<std::pair<int, int>> stack{{f, 0}};
    std::vector<std::pair<int, int>> seen;
    int join = -1, njoins = 0;
    while (!stack.empty()) {
      auto [c, depth] = stack.back();
      stack.pop_back();
      for (int s : fn.succ[c]) {
        const std::string &k = fn.nodes[s].kind;
        int d = depth;
        if (k == "join") {
          if (d == 0) {
            if (s != join) { join = s; njoins++; }
            continue;
          }
          d--;
        } else if (k == "fork") {
          d++;
        }
        bool dup = false;
        for (auto &p : seen) dup |= (p.first == s && p.second == d);
        if (!dup) { seen.push_back({s, d}); stack.push_back({s, d}); }
      }
    }
    if (njoins != 1) fail("RuntimeError_", "fork %" + std::to_string(f) + " does not match one join");
    fn.join_of[f] = join;
  }
  return fn;
}

struct Module {
  std::map<std::string, Function> fns;
};

// ---------------------------------------------------------------- eval
struct Eval {
  const Module &mod;
  const Function &fn;
  std::vector<long long> dcs;
  std::vector<Val> args;
  long long *budget;
  std::vector<Val> vals;
  std::vector<uint8_t> have;
  std::map<std::vector<int>, std::vector<int>> dep_cache;

  Eval(const Module &m, const Function &f, std::vector<long long> d, std::vector<Val> a, long long *b)
      : mod(m), fn(f), dcs(std::move(d)), args(std::move(a)), budget(b) {
    vals.resize(fn.nodes.size());
    have.assign(fn.nodes.size(), 0);
  }

  void spend() {
    if (--*budget < 0) fail("OracleLimitError", "oracle step budget exhausted");
  }

  void set(int i, Val v) { vals[i] = std::move(v); have[i] = 1; }

  // the fixed dependents walk: data users, transitively,
  // not walking into control nodes nor into phi / reduce nodes other than
  // the roots being rebound
  const std::vector<int> &dependents(const std::vector<int> &roots) {
    auto it = dep_cache.find(roots);
    if (it != dep_cache.end()) return it->second;
    std::vector<uint8_t> in(fn.nodes.size(), 0), isroot(fn.nodes.size(), 0);
    for (int r : roots) isroot[r] = 1;
    std::vector<int> out, stack(roots.begin(), roots.end());
    while (!stack.empty()) {
      const int x = stack.back();
      stack.pop_back();
      for (int u : fn.users[x]) {
        const Node &n = fn.nodes[u];
        if (in[u] || n.is_control) continue;
        if ((n.code == C_PHI || n.code == C_REDUCE) && !isroot[u]) continue;
        in[u] = 1;
        out.push_back(u);
        stack.push_back(u);
      }
    }
    for (int r : roots)
      if (!in[r]) out.push_back(r);
    return dep_cache.emplace(roots, std::move(out)).first->second;
  }
  void invalidate(const std::vector<int> &roots) {
    for (int x : dependents(roots)) { have[x] = 0; vals[x].a.reset(); vals[x].k = Val::NONE; }
  }

  const Val &eval(int nid) {
    if (have[nid]) return vals[nid];
    std::vector<int> stack{nid};
    while (!stack.empty()) {
      const int top = stack.back();
      if (have[top]) { stack.pop_back(); continue; }
      const Node &n = fn.nodes[top];
      if (n.is_bound) fail("RuntimeError_", "oracle cannot evaluate node kind " + n.kind + " (%" + std::to_string(top) + ")");
      bool missing = false;
      for (int i : n.inputs)
        if (!have[i]) { stack.push_back(i); missing = true; }
      for (auto &ix : n.idx)
        for (int i : ix.ids)
          if (!have[i]) { stack.push_back(i); missing = true; }
      if (missing) continue;
      set(top, compute(top));
      spend();
      stack.pop_back();
    }
    return vals[nid];
  }

  std::vector<long long> positions(const Node &n) {
    std::vector<long long> p;
    for (auto &ix : n.idx)
      for (int i : ix.ids) {
        const Val &v = vals[i];
        if (v.k != Val::SCAL) fail("RuntimeError_", "non-scalar index");
        if (dt_float(v.dt)) p.push_back((long long)as_double(v));
        else p.push_back((long long)as_i128(v));
      }
    return p;
  }
  size_t offset(const Arr &a, const std::vector<long long> &p, int nid) {
    if (p.size() != a.shape.size()) fail("RuntimeError_", "%" + std::to_string(nid) + ": index rank mismatch");
    size_t off = 0;
    for (size_t d = 0; d < p.size(); d++) {
      if (p[d] < 0 || p[d] >= a.shape[d]) {
        std::string s = "(";
        for (size_t e = 0; e < p.size(); e++) s += std::to_string(p[e]) + (e + 1 < p.size() ? ", " : ")");
        fail("RuntimeError_", "%" + std::to_string(nid) + ": index " + s + " out of bounds");
      }
      off = off * (size_t)a.shape[d] + (size_t)p[d];
    }
    return off;
  }
  static Val load(const Arr &a, size_t off) {
    const uint8_t *q = a.data.data() + off * dt_size(a.dt);
    switch (a.dt) {
      case BOOLT: case U8: return scal_u(U8, *q);  // bool arrays are u8 storage (types.py:147-159)
      case I8: return scal_i(I8, *(const int8_t *)q);
      case I16: return scal_i(I16, *(const int16_t *)q);
      case I32: return scal_i(I32, *(const int32_t *)q);
      case I64: return scal_i(I64, *(const int64_t *)q);
      case U16: return scal_u(U16, *(const uint16_t *)q);
      case U32: return scal_u(U32, *(const uint32_t *)q);
      case U64: return scal_u(U64, *(const uint64_t *)q);
      case F32: return scal_f(*(const float *)q);
      default: return scal_d(*(const double *)q);
    }
  }
  static void store(Arr &a, size_t off, const Val &v) {  // numpy assignment casts into the dtype
    uint8_t *q = a.data.data() + off * dt_size(a.dt);
    switch (a.dt) {
      case BOOLT: case U8: *q = (uint8_t)(dt_float(v.dt) ? (int64_t)as_double(v) : (int64_t)as_i128(v)); break;
      case I8: *(int8_t *)q = (int8_t)(dt_float(v.dt) ? (int64_t)as_double(v) : (int64_t)as_i128(v)); break;
      case I16: *(int16_t *)q = (int16_t)(dt_float(v.dt) ? (int64_t)as_double(v) : (int64_t)as_i128(v)); break;
      case I32: *(int32_t *)q = (int32_t)(dt_float(v.dt) ? (int64_t)as_double(v) : (int64_t)as_i128(v)); break;
      case I64: *(int64_t *)q = (int64_t)(dt_float(v.dt) ? (int64_t)as_double(v) : (int64_t)as_i128(v)); break;
      case U16: *(uint16_t *)q = (uint16_t)(uint64_t)as_i128(v); break;
      case U32: *(uint32_t *)q = (uint32_t)(uint64_t)as_i128(v); break;
      case U64: *(uint64_t *)q = (uint64_t)as_i128(v); break;
      case F32: *(float *)q = v.dt == F32 ? v.x.f : (float)as_double(v); break;
      default: *(double *)q = as_double(v); break;
    }
  }

  // may the write node `wid` take over its collection input's buffer?
  bool can_steal(int wid, int coll) {
    const Val &c = vals[coll];
    if (c.k != Val::ARRAY || c.a.use_count() != 1) return false;
    const Node &cn = fn.nodes[coll];
    for (int u : fn.users[coll]) {
      if (u == wid) continue;
      const Node &n = fn.nodes[u];
      if (n.code == C_REDUCE) {
        // the reduct of an enclosing fold reads coll only after coll's own
        // fork / loop has rebound it; anything else is not provably dead
        if (n.inputs.size() == 2 && n.inputs[1] == coll && n.inputs[0] != coll &&
            !(cn.code == C_REDUCE && cn.control == n.control))
          continue;
        return false;
      }
      if (n.is_control || n.code == C_PHI || n.code == C_CALL) return false;
      if (!have[u]) return false;  // a user still to be evaluated must see the old value
    }
    return true;
  }

  Val compute(int nid) {
    const Node &n = fn.nodes[nid];
    switch (n.code) {
      case C_BINARY:
        return binop(n.opc, vals[n.inputs[0]], vals[n.inputs[1]], n.ty.dt);
      case C_UNARY:
        return unop(n.opc, vals[n.inputs[0]], n.ty.dt);
      case C_READ: {
        const Val &c = vals[n.inputs[0]];
        if (c.k == Val::MOVED) fail("RuntimeError_", "internal: read of a moved collection");
        if (n.idx.empty()) return c;
        if (c.k != Val::ARRAY) fail("RuntimeError_", "%" + std::to_string(nid) + ": positional read of non-array");
        return load(*c.a, offset(*c.a, positions(n), nid));
      }
      case C_WRITE: {
        const int coll = n.inputs[0];
        const Val &v = vals[n.inputs[1]];
        if (n.idx.empty()) return v;
        if (vals[coll].k != Val::ARRAY)
          fail("RuntimeError_", "%" + std::to_string(nid) + ": positional write of non-array");
        const size_t off = offset(*vals[coll].a, positions(n), nid);
        Val c;
        if (can_steal(nid, coll)) {  // the old value is dead: write in place
          c = std::move(vals[coll]);
          vals[coll] = Val{};
          vals[coll].k = Val::MOVED;
        } else {
          c = vals[coll];
          c.a = std::make_shared<Arr>(*c.a);  // value semantics: a fresh collection
        }
        if (v.k != Val::SCAL) fail("RuntimeError_", "unsupported: writing a collection into an array element");
        store(*c.a, off, v);
        return c;
      }
      case C_CALL: {
        auto it = mod.fns.find(n.callee);
        if (it == mod.fns.end()) fail("RuntimeError_", "unknown callee " + n.callee);
        std::vector<long long> d;
        for (auto &e : n.dca) d.push_back(dc_eval(*e, dcs));
        std::vector<Val> a;
        for (int i : n.inputs) {
          Val x = vals[i];
          if (x.k == Val::ARRAY) x.a = std::make_shared<Arr>(*x.a);
          a.push_back(x);
        }
        Eval sub(mod, it->second, d, a, budget);
        return sub.run();
      }
      default:
        fail("RuntimeError_", "oracle cannot evaluate node kind " + n.kind);
    }
  }

  Val zero_of(const Ty &t) {
    if (!t.arr) return t.dt == BOOLT ? scal_b(false) : typed_scalar(scal_i(I64, 0), t.dt);
    auto a = std::make_shared<Arr>();
    a->dt = t.dt;
    for (auto &e : t.ext) a->shape.push_back(dc_eval(*e, dcs));
    a->data.assign(a->count() * dt_size(t.dt), 0);
    Val v;
    v.k = Val::ARRAY;
    v.a = a;
    return v;
  }

  Val literal(const Node &n) {
    const J &c = n.cv;
    const DT dt = n.ty.dt;
    if (c.t == J::BOOL) return typed_scalar(scal_b(c.b), dt);
    if (c.t == J::INT) return typed_scalar(c.is_u ? scal_u(U64, c.u) : scal_i(I64, c.i), dt);
    if (c.t == J::OBJ) return typed_scalar(scal_d(strtod(c.get("f")->s.c_str(), nullptr)), dt);
    if (c.t == J::DBL) return typed_scalar(scal_d(c.d), dt);
    fail("RuntimeError_", "unsupported constant");
  }

  Val run() {
    for (size_t i = 0; i < fn.nodes.size(); i++) {
      const Node &n = fn.nodes[i];
      if (!n.live) continue;
      if (n.code == C_PARAM) {
        if (n.index >= (int)args.size()) fail("RuntimeError_", "missing argument " + std::to_string(n.index));
        set(i, args[n.index]);
      } else if (n.code == C_CONST) {
        if (!n.has_ty) fail("RuntimeError_", "unsupported constant type");
        set(i, (n.cv.t == J::NUL) ? zero_of(n.ty) : literal(n));
      } else if (n.code == C_DYNC) {
        set(i, typed_scalar(scal_i(I64, dc_eval(*n.dc, dcs)), n.has_ty ? n.ty.dt : U64));
      }
    }
    return walk(fn.start, -1);
  }

  int only_successor(int c) {
    if (fn.succ[c].size() != 1) fail("RuntimeError_", "control diverges after %" + std::to_string(c));
    return fn.succ[c][0];
  }

  Val walk(int start, int stop_at) {
    int c = start, prev = -1;
    for (;;) {
      if (c == stop_at) return Val{};
      const Node &n = fn.nodes[c];
      spend();
      if (n.kind == "start" || n.kind == "proj") {
        prev = c;
        c = only_successor(c);
      } else if (n.kind == "region") {
        int entry = -1;
        for (size_t k = 0; k < n.preds.size(); k++)
          if (n.preds[k] == prev) entry = (int)k;
        if (entry < 0) fail("RuntimeError_", "region %" + std::to_string(c) + " entered from a non-predecessor");
        auto it = fn.phis_of.find(c);
        if (it != fn.phis_of.end()) {
          std::vector<Val> nv;
          for (int p : it->second) nv.push_back(eval(fn.nodes[p].inputs[entry]));
          std::vector<int> roots(it->second);
          std::sort(roots.begin(), roots.end());
          invalidate(roots);
          for (size_t k = 0; k < it->second.size(); k++) set(it->second[k], nv[k]);
        }
        prev = c;
        c = only_successor(c);
      } else if (n.kind == "if") {
        const bool cond = truthy(eval(n.inputs[0]));
        int next = -1;
        for (int s : fn.succ[c])
          if (fn.nodes[s].kind == "proj" && fn.nodes[s].sel == (cond ? 1 : 0)) next = s;
        if (next < 0) fail("RuntimeError_", "missing projection after %" + std::to_string(c));
        prev = c;
        c = next;
      } else if (n.kind == "return") {
        return eval(n.inputs[0]);
      } else if (n.kind == "fork") {
        const int join = run_fork(c);
        prev = join;  // fix 2: the join precedes its successor
        c = only_successor(join);
      } else {
        fail("RuntimeError_", "oracle cannot walk control kind " + n.kind);
      }
    }
  }

  int run_fork(int f) {
    const Node &fk = fn.nodes[f];
    const int join = fn.join_of.at(f);
    std::vector<long long> factors;
    for (auto &e : fk.factors) factors.push_back(dc_eval(*e, dcs));
    static const std::vector<int> none;
    auto ti = fn.tids_of.find(f);
    const std::vector<int> &tids = ti == fn.tids_of.end() ? none : ti->second;
    auto ri = fn.reduces_of.find(join);
    const std::vector<int> &reds = ri == fn.reduces_of.end() ? none : ri->second;
    for (int r : reds) set(r, eval(fn.nodes[r].inputs[0]));
    std::vector<int> roots(tids);
    roots.insert(roots.end(), reds.begin(), reds.end());
    std::sort(roots.begin(), roots.end());
    int body = -1;
    for (int s : fn.succ[f]) body = s;
    long long total = 1;
    for (auto x : factors) total *= x;
    std::vector<long long> idx(factors.size(), 0);
    std::vector<Val> part(reds.size());
    for (long long it = 0; it < total; it++) {
      for (size_t k = 0; k < reds.size(); k++) part[k] = std::move(vals[reds[k]]);
      invalidate(roots);
      for (size_t k = 0; k < reds.size(); k++) set(reds[k], std::move(part[k]));
      for (int t : tids)
        set(t, typed_scalar(scal_i(I64, idx[fn.nodes[t].dim]), fn.nodes[t].has_ty ? fn.nodes[t].ty.dt : U64));
      if (body >= 0 && body != join) walk(body, join);
      for (size_t k = 0; k < reds.size(); k++) part[k] = eval(fn.nodes[reds[k]].inputs[1]);
      for (size_t k = 0; k < reds.size(); k++) set(reds[k], std::move(part[k]));
      for (int d = (int)factors.size() - 1; d >= 0; d--) {
        if (++idx[d] < factors[d]) break;
        idx[d] = 0;
      }
    }
    for (size_t k = 0; k < reds.size(); k++) part[k] = std::move(vals[reds[k]]);
    invalidate(roots);
    for (size_t k = 0; k < reds.size(); k++) set(reds[k], std::move(part[k]));
    if (total == 0)
      for (int r : reds) set(r, eval(fn.nodes[r].inputs[0]));
    return join;
  }
};

thread_local std::string g_err;
thread_local Val g_result;

}  // namespace

// ------------------------------------------------------------------- C ABI
extern "C" {

typedef struct {
  int dtype;          // index into DT_NAMES
  int ndim;           // 0: scalar (data points at one element)
  int64_t shape[8];
  void *data;
} jir_arg;

const char *jir_last_error(void) { return g_err.c_str(); }

// Runs module.functions[entry](dyn_consts..., args...).  On success the
// result is described in *out (data owned by the library until the next
// call on this thread); returns 0, or 1 with jir_last_error() set.
int jir_execute(const char *module_json, const char *entry, const int64_t *dcs, int ndcs, const jir_arg *args,
                int nargs, long long max_steps, jir_arg *out, long long *steps_used) {
  try {
    Parser p{module_json};
    J doc = p.parse();
    Module mod;
    for (auto &kv : doc.get("functions")->o) mod.fns.emplace(kv.first, load_function(kv.first, kv.second));
    auto it = mod.fns.find(entry);
    if (it == mod.fns.end()) fail("KeyError", entry);
    std::vector<long long> d(dcs, dcs + ndcs);
    std::vector<Val> a;
    for (int i = 0; i < nargs; i++) {
      const jir_arg &x = args[i];
      const DT dt = (DT)x.dtype;
      if (x.ndim == 0) {
        Arr tmp;
        tmp.dt = dt;
        tmp.data.assign((const uint8_t *)x.data, (const uint8_t *)x.data + dt_size(dt));
        Val v = Eval::load(tmp, 0);
        if (dt == BOOLT) v = scal_b(v.x.u != 0);
        a.push_back(v);
      } else {
        auto arr = std::make_shared<Arr>();
        arr->dt = dt;
        for (int k = 0; k < x.ndim; k++) arr->shape.push_back(x.shape[k]);
        const size_t nb = arr->count() * dt_size(dt);
        arr->data.assign((const uint8_t *)x.data, (const uint8_t *)x.data + nb);
        Val v;
        v.k = Val::ARRAY;
        v.a = arr;
        a.push_back(v);
      }
    }
    long long budget = max_steps;
    Eval ev(mod, it->second, d, a, &budget);
    g_result = ev.run();
    if (steps_used) *steps_used = max_steps - budget;
    memset(out, 0, sizeof(*out));
    if (g_result.k == Val::ARRAY) {
      out->dtype = g_result.a->dt;
      out->ndim = (int)g_result.a->shape.size();
      for (int k = 0; k < out->ndim && k < 8; k++) out->shape[k] = g_result.a->shape[k];
      out->data = g_result.a->data.data();
    } else if (g_result.k == Val::SCAL) {
      out->dtype = g_result.dt;
      out->ndim = 0;
      out->data = &g_result.x;
    } else {
      fail("RuntimeError_", "the function returned no value");
    }
    return 0;
  } catch (const std::exception &e) {
    g_err = e.what();
    return 1;
  }
}

}  // extern "C"
