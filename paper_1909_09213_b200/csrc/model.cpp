// Host-side problem loading: model construction, the model-text parser and validation.
// This is the reference's L1 layer kept on the host; nothing here is on the
// device hot path. The parser restates the grammar of /root/reference/proj/src/parser.cpp
// (lexer :68-202, items :224-257, var :289-324, constraints :326-462, solve :464-487) so a
// model text loads to the same fd::Model the reference builds.
#include "model.hpp"

#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <set>
#include <string>
#include <unordered_map>
#include <unordered_set>

namespace cubics {

namespace {
thread_local std::string g_last_error;
} // namespace

void set_error(const std::string& msg) { g_last_error = msg; }

const char* last_error() { return g_last_error.c_str(); }

void HostModel::finish_vars() {
    word_start.assign(1, 0);
    for (int32_t w : width) word_start.push_back(word_start.back() + (w + 63) / 64);
}

cubics_model_desc HostModel::desc() const {
    cubics_model_desc d{};
    d.n_vars = n_vars();
    d.var_offset = offset.data();
    d.var_width = width.data();
    d.var_words = words.data();
    d.n_cons = n_cons();
    d.con_kind = con_kind.data();
    d.con_op = con_op.data();
    d.con_value = con_value.data();
    d.con_start = con_start.data();
    d.term_var = term_var.data();
    d.term_coeff = term_coeff.data();
    d.goal = goal;
    d.goal_var = goal_var;
    d.table_start = table_start.data();
    d.table_data = table_data.data();
    return d;
}

namespace {

// ---------------------------------------------------------------- lexer
enum class T { Ident, Int, Semi, Comma, LParen, RParen, DotDot, Plus, Minus, Star, Lt, Le, Gt, Ge, Eq, Ne, Colon, End };

struct Tok {
    T kind = T::End;
    std::string text;
    int64_t value = 0;
    int line = 1, col = 1;
};

struct Lexer {
    const char* s;
    size_t n, pos = 0;
    int line = 1, col = 1;
    Tok cur;
    bool err = false;
    cubics_parse_error* perr;

    Lexer(const char* text, size_t len, cubics_parse_error* e) : s(text), n(len), perr(e) { advance(); }

    void bump() {
        if (s[pos] == '\n') {
            ++line;
            col = 1;
        } else {
            ++col;
        }
        ++pos;
    }

    void skip() {
        while (pos < n) {
            char c = s[pos];
            if (c == '#') {
                while (pos < n && s[pos] != '\n') bump();
            } else if (c == ' ' || c == '\t' || c == '\r' || c == '\n') {
                bump();
            } else {
                break;
            }
        }
    }

    void fail(int l, int c, const std::string& msg) {
        if (err) return;
        err = true;
        if (perr) {
            perr->kind = 0;
            perr->line = l;
            perr->column = c;
            std::snprintf(perr->message, sizeof perr->message, "line %d, column %d: %s", l, c, msg.c_str());
        }
    }

    void advance() {
        skip();
        cur = Tok{};
        cur.line = line;
        cur.col = col;
        if (pos >= n) return;
        char c = s[pos];
        auto isdig = [](char ch) { return std::isdigit(static_cast<unsigned char>(ch)) != 0; };
        if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
            size_t b = pos;
            while (pos < n && (std::isalnum(static_cast<unsigned char>(s[pos])) || s[pos] == '_')) bump();
            cur.kind = T::Ident;
            cur.text.assign(s + b, pos - b);
            return;
        }
        if (isdig(c) || (c == '-' && pos + 1 < n && isdig(s[pos + 1]))) {
            size_t b = pos;
            if (c == '-') bump();
            while (pos < n && isdig(s[pos])) bump();
            cur.kind = T::Int;
            cur.text.assign(s + b, pos - b);
            errno = 0;
            long long v = std::strtoll(cur.text.c_str(), nullptr, 10);
            if (errno == ERANGE)
                fail(cur.line, cur.col, "expected integer in 64-bit range, found '" + cur.text + "'");
            cur.value = v;
            return;
        }
        auto one = [&](T k) {
            cur.kind = k;
            cur.text.assign(1, c);
            bump();
        };
        auto two = [&](T k, const char* t) {
            cur.kind = k;
            cur.text = t;
            bump();
            bump();
        };
        bool nxt_eq = pos + 1 < n && s[pos + 1] == '=';
        switch (c) {
        case ';': one(T::Semi); return;
        case ':': one(T::Colon); return; // table constraints (extension)
        case ',': one(T::Comma); return;
        case '(': one(T::LParen); return;
        case ')': one(T::RParen); return;
        case '+': one(T::Plus); return;
        case '-': one(T::Minus); return;
        case '*': one(T::Star); return;
        case '.':
            if (pos + 1 < n && s[pos + 1] == '.') {
                two(T::DotDot, "..");
                return;
            }
            break;
        case '<':
            if (nxt_eq) two(T::Le, "<=");
            else one(T::Lt);
            return;
        case '>':
            if (nxt_eq) two(T::Ge, ">=");
            else one(T::Gt);
            return;
        case '=': one(T::Eq); return;
        case '!':
            if (nxt_eq) {
                two(T::Ne, "!=");
                return;
            }
            break;
        default: break;
        }
        fail(line, col, std::string("expected a token, found '") + c + "'");
        cur.kind = T::End;
    }

    Tok take() {
        Tok t = cur;
        advance();
        return t;
    }
};

bool is_rel(T k) { return k == T::Lt || k == T::Le || k == T::Gt || k == T::Ge || k == T::Eq || k == T::Ne; }

int rel_of(T k) {
    switch (k) {
    case T::Lt: return CUBICS_LT;
    case T::Le: return CUBICS_LE;
    case T::Gt: return CUBICS_GT;
    case T::Ge: return CUBICS_GE;
    case T::Eq: return CUBICS_EQ;
    default: return CUBICS_NE;
    }
}

// ---------------------------------------------------------------- parser
struct Parser {
    Lexer lex;
    HostModel& m;
    cubics_parse_error* perr;
    std::unordered_map<std::string, int> ids;
    bool err = false;

    Parser(const char* t, size_t n, HostModel& out, cubics_parse_error* e) : lex(t, n, e), m(out), perr(e) {}

    bool failed() const { return err || lex.err; }

    void fail_kind(int kind, const Tok& t, const std::string& msg) {
        if (failed()) return;
        err = true;
        if (perr) {
            perr->kind = kind;
            perr->line = t.line;
            perr->column = t.col;
            std::snprintf(perr->message, sizeof perr->message, "line %d, column %d: %s", t.line, t.col, msg.c_str());
        }
    }

    void fail_syntax(const Tok& t, const std::string& expected) {
        fail_kind(0, t, "expected " + expected + ", found " + (t.kind == T::End ? std::string("end of input") : "'" + t.text + "'"));
    }

    bool expect(T k, const char* what, Tok* out = nullptr) {
        if (failed()) return false;
        if (lex.cur.kind != k) {
            fail_syntax(lex.cur, what);
            return false;
        }
        Tok t = lex.take();
        if (out) *out = t;
        return !failed();
    }

    bool resolve(const Tok& t, int& id) {
        auto it = ids.find(t.text);
        if (it == ids.end()) {
            fail_kind(1, t, "unknown variable '" + t.text + "'");
            return false;
        }
        id = it->second;
        return true;
    }

    bool peek_lparen() const { // 'table' followed by '(' starts a table constraint
        size_t p = lex.pos;
        while (p < lex.n && (lex.s[p] == ' ' || lex.s[p] == '\t' || lex.s[p] == '\r' || lex.s[p] == '\n')) ++p;
        return p < lex.n && lex.s[p] == '(';
    }

    void push_con(int kind, int op, int64_t value) {
        m.con_kind.push_back(kind);
        m.con_op.push_back(op);
        m.con_value.push_back(value);
        m.table_start.push_back(static_cast<int64_t>(m.table_data.size()));
    }

    void close_con() { m.con_start.push_back(static_cast<int32_t>(m.term_var.size())); }

    void term(int var, int64_t coeff) {
        m.term_var.push_back(var);
        m.term_coeff.push_back(coeff);
    }

    void var_decl() {
        lex.take(); // var
        Tok name, lo, hi;
        if (!expect(T::Ident, "variable name", &name)) return;
        if (lex.cur.kind != T::Ident || lex.cur.text != "in") {
            fail_syntax(lex.cur, "'in'");
            return;
        }
        lex.take();
        if (!expect(T::Int, "integer lower bound", &lo)) return;
        if (!expect(T::DotDot, "'..'")) return;
        if (!expect(T::Int, "integer upper bound", &hi)) return;
        if (!expect(T::Semi, "';'")) return;
        if (ids.count(name.text)) {
            fail_kind(2, name, "duplicate variable '" + name.text + "'");
            return;
        }
        if (lo.value > hi.value) {
            fail_kind(3, lo, "empty domain (lower bound exceeds upper bound)");
            return;
        }
        uint64_t span = static_cast<uint64_t>(hi.value) - static_cast<uint64_t>(lo.value);
        if (span >= static_cast<uint64_t>(CUBICS_MAX_WIDTH)) {
            fail_kind(4, lo, "domain wider than 1024 values");
            return;
        }
        int id = m.n_vars();
        ids[name.text] = id;
        m.names.push_back(name.text);
        m.offset.push_back(lo.value);
        m.width.push_back(static_cast<int32_t>(span) + 1);
    }

    void rel_bin(const Tok& lhs_tok) {
        int lhs;
        if (!resolve(lhs_tok, lhs)) return;
        int op = rel_of(lex.take().kind);
        const Tok& rhs = lex.cur;
        if (rhs.kind == T::Int) {
            Tok lit = lex.take();
            push_con(CUBICS_RELBIN, op, lit.value);
            term(lhs, 1);
            close_con();
        } else if (rhs.kind == T::Ident) {
            Tok rt = lex.take();
            int rv;
            if (!resolve(rt, rv)) return;
            int64_t k = 0;
            if (lex.cur.kind == T::Plus || lex.cur.kind == T::Minus) {
                bool neg = lex.take().kind == T::Minus;
                Tok off;
                if (!expect(T::Int, "integer offset", &off)) return;
                k = neg ? static_cast<int64_t>(0 - static_cast<uint64_t>(off.value)) : off.value;
            }
            if (op == CUBICS_GT || op == CUBICS_GE) { // parser.cpp:380-385 normalisation
                std::swap(lhs, rv);
                k = static_cast<int64_t>(0 - static_cast<uint64_t>(k));
                op = op == CUBICS_GT ? CUBICS_LT : CUBICS_LE;
            }
            push_con(CUBICS_RELBIN, op, k);
            term(lhs, 1);
            term(rv, 1);
            close_con();
        } else {
            fail_syntax(rhs, "variable or integer");
        }
    }

    void alldiff() {
        lex.take(); // alldifferent
        if (!expect(T::LParen, "'('")) return;
        std::vector<int> vars;
        Tok t;
        if (!expect(T::Ident, "variable name", &t)) return;
        int v;
        if (!resolve(t, v)) return;
        vars.push_back(v);
        while (lex.cur.kind == T::Comma) {
            lex.take();
            if (!expect(T::Ident, "variable name", &t)) return;
            if (!resolve(t, v)) return;
            vars.push_back(v);
        }
        if (vars.size() < 2) {
            fail_syntax(lex.cur, "','");
            return;
        }
        if (!expect(T::RParen, "')'")) return;
        push_con(CUBICS_ALLDIFF, 0, 0);
        for (int x : vars) term(x, 1);
        close_con();
    }

    void linear_from(const Tok& first, int64_t first_coeff) {
        std::vector<std::pair<int64_t, int>> terms;
        int v;
        if (!resolve(first, v)) return;
        terms.push_back({first_coeff, v});
        while (lex.cur.kind == T::Plus || lex.cur.kind == T::Minus) {
            bool neg = lex.take().kind == T::Minus;
            int64_t coeff = 1;
            if (lex.cur.kind == T::Int) {
                coeff = lex.take().value;
                if (!expect(T::Star, "'*'")) return;
            }
            Tok vt;
            if (!expect(T::Ident, "variable name", &vt)) return;
            if (!resolve(vt, v)) return;
            terms.push_back({neg ? static_cast<int64_t>(0 - static_cast<uint64_t>(coeff)) : coeff, v});
        }
        int op;
        if (lex.cur.kind == T::Le) op = CUBICS_LIN_LE;
        else if (lex.cur.kind == T::Eq) op = CUBICS_LIN_EQ;
        else {
            fail_syntax(lex.cur, "'<=' or '='");
            return;
        }
        lex.take();
        Tok bound;
        if (!expect(T::Int, "integer bound", &bound)) return;
        push_con(CUBICS_LINEAR, op, bound.value);
        for (auto& [c, x] : terms) term(x, c);
        close_con();
    }

    // extension (not in the reference grammar): constraint table(x, y : 1 2, 2 3, 3 1);
    // allowed tuples after ':', values separated by blanks, tuples by commas
    void table() {
        lex.take(); // table
        if (!expect(T::LParen, "'('")) return;
        std::vector<int> vars;
        Tok t;
        int v;
        if (!expect(T::Ident, "variable name", &t) || !resolve(t, v)) return;
        vars.push_back(v);
        while (lex.cur.kind == T::Comma) {
            lex.take();
            if (!expect(T::Ident, "variable name", &t) || !resolve(t, v)) return;
            vars.push_back(v);
        }
        if (!take_colon()) return;
        const size_t k = vars.size();
        std::vector<int64_t> data;
        while (lex.cur.kind == T::Int) {
            for (size_t i = 0; i < k; ++i) {
                Tok val;
                if (!expect(T::Int, "integer tuple value", &val)) return;
                data.push_back(val.value);
            }
            if (lex.cur.kind != T::Comma) break;
            lex.take();
        }
        if (!expect(T::RParen, "')'")) return;
        push_con(CUBICS_TABLE, 0, static_cast<int64_t>(data.size() / k));
        m.table_data.insert(m.table_data.end(), data.begin(), data.end());
        for (int x : vars) term(x, 1);
        close_con();
    }

    bool take_colon() {
        if (failed()) return false;
        if (lex.cur.kind == T::Colon) {
            lex.take();
            return !failed();
        }
        fail_syntax(lex.cur, "':'");
        return false;
    }

    void constraint() {
        lex.take(); // constraint
        const Tok first = lex.cur;
        if (first.kind == T::Ident && first.text == "table" && peek_lparen()) {
            table();
        } else if (first.kind == T::Ident && first.text == "alldifferent") {
            alldiff();
        } else if (first.kind == T::Ident) {
            Tok ident = lex.take();
            if (is_rel(lex.cur.kind)) rel_bin(ident);
            else linear_from(ident, 1);
        } else if (first.kind == T::Int) {
            Tok coeff = lex.take();
            if (!expect(T::Star, "'*'")) return;
            Tok ident;
            if (!expect(T::Ident, "variable name", &ident)) return;
            linear_from(ident, coeff.value);
        } else {
            fail_syntax(first, "a constraint body");
        }
        if (!failed()) expect(T::Semi, "';'");
    }

    void solve() {
        lex.take(); // solve
        Tok what;
        if (!expect(T::Ident, "'satisfy', 'minimize' or 'maximize'", &what)) return;
        if (what.text == "satisfy") {
            m.goal = CUBICS_SATISFY;
        } else if (what.text == "minimize" || what.text == "maximize") {
            Tok vt;
            if (!expect(T::Ident, "variable name", &vt)) return;
            int v;
            if (!resolve(vt, v)) return;
            m.goal = what.text == "minimize" ? CUBICS_MINIMIZE : CUBICS_MAXIMIZE;
            m.goal_var = v;
        } else {
            fail_syntax(what, "'satisfy', 'minimize' or 'maximize'");
            return;
        }
        expect(T::Semi, "';'");
    }

    int run() {
        bool saw_solve = false;
        while (!failed()) {
            const Tok& t = lex.cur;
            if (t.kind == T::End) break;
            if (t.kind == T::Ident && t.text == "var") {
                var_decl();
            } else if (t.kind == T::Ident && t.text == "constraint") {
                constraint();
            } else if (t.kind == T::Ident && t.text == "solve") {
                solve();
                saw_solve = true;
                if (!failed() && lex.cur.kind != T::End) fail_syntax(lex.cur, "end of input");
                break;
            } else {
                fail_syntax(t, "'var', 'constraint' or 'solve'");
            }
        }
        if (failed()) return CUBICS_E_PARSE;
        if (!saw_solve) {
            fail_kind(5, lex.cur, "missing 'solve' item");
            return CUBICS_E_PARSE;
        }
        m.finish_vars();
        m.words.assign(m.word_start.back(), 0);
        for (int v = 0; v < m.n_vars(); ++v)
            for (int i = 0; i < m.width[v]; ++i) m.words[m.word_start[v] + i / 64] |= uint64_t{1} << (i % 64);
        if (m.term_coeff.size() < m.term_var.size()) m.term_coeff.resize(m.term_var.size(), 1);
        return CUBICS_OK;
    }
};

} // namespace

int parse_model_text(const char* text, size_t len, HostModel& out, cubics_parse_error* err) {
    if (err) std::memset(err, 0, sizeof *err);
    Parser p(text, len, out, err);
    return p.run();
}

} // namespace cubics

// ============================================================================ C ABI (model)
using cubics::HostModel;

extern "C" int cubics_model_create(const cubics_model_desc* d, cubics_model** out) {
    if (!d || !out || d->n_vars < 0 || d->n_cons < 0) {
        cubics::set_error("cubics_model_create: null or negative argument");
        return CUBICS_E_INVALID;
    }
    auto* h = new cubics_model();
    HostModel& m = h->m;
    for (int v = 0; v < d->n_vars; ++v) {
        int w = d->var_width[v];
        if (w < 1 || w > CUBICS_MAX_WIDTH) {
            delete h;
            cubics::set_error("cubics_model_create: var width out of [1, 1024]");
            return CUBICS_E_INVALID;
        }
        m.names.push_back("v" + std::to_string(v));
        m.offset.push_back(d->var_offset[v]);
        m.width.push_back(w);
    }
    m.finish_vars();
    m.words.assign(m.word_start.back(), 0);
    for (int v = 0; v < d->n_vars; ++v) {
        int nw = m.word_start[v + 1] - m.word_start[v];
        for (int i = 0; i < nw; ++i) {
            uint64_t valid = (i == nw - 1 && m.width[v] % 64) ? ((uint64_t{1} << (m.width[v] % 64)) - 1) : ~uint64_t{0};
            m.words[m.word_start[v] + i] = d->var_words ? (d->var_words[m.word_start[v] + i] & valid) : valid;
        }
    }
    int nt = d->n_cons ? d->con_start[d->n_cons] : 0;
    for (int c = 0; c < d->n_cons; ++c) {
        int k = d->con_kind[c];
        int cnt = d->con_start[c + 1] - d->con_start[c];
        bool ok = (k == CUBICS_RELBIN && (cnt == 1 || cnt == 2) && d->con_op[c] >= 0 && d->con_op[c] <= 5) ||
                  (k == CUBICS_LINEAR && cnt >= 0 && (d->con_op[c] == 0 || d->con_op[c] == 1)) ||
                  (k == CUBICS_ALLDIFF && cnt >= 0) ||
                  (k == CUBICS_TABLE && cnt >= 1 && d->table_start && d->table_data && d->con_value[c] >= 0);
        if (!ok || d->con_start[c] > d->con_start[c + 1]) {
            delete h;
            cubics::set_error("cubics_model_create: malformed constraint " + std::to_string(c));
            return CUBICS_E_INVALID;
        }
        m.con_kind.push_back(k);
        m.con_op.push_back(k == CUBICS_ALLDIFF || k == CUBICS_TABLE ? 0 : d->con_op[c]);
        m.con_value.push_back(k == CUBICS_ALLDIFF ? 0 : d->con_value[c]);
        m.table_start.push_back(static_cast<int64_t>(m.table_data.size()));
        if (k == CUBICS_TABLE) {
            const int64_t* src = d->table_data + d->table_start[c];
            m.table_data.insert(m.table_data.end(), src, src + d->con_value[c] * cnt);
        }
        m.con_start.push_back(d->con_start[c + 1] - d->con_start[0]);
    }
    for (int t = d->n_cons ? d->con_start[0] : 0; t < nt; ++t) {
        int v = d->term_var[t];
        if (v < 0 || v >= d->n_vars) {
            delete h;
            cubics::set_error("cubics_model_create: term var out of range");
            return CUBICS_E_INVALID;
        }
        m.term_var.push_back(v);
        m.term_coeff.push_back(d->term_coeff ? d->term_coeff[t] : 1);
    }
    m.goal = d->goal;
    m.goal_var = d->goal_var;
    if (m.goal != CUBICS_SATISFY && (m.goal_var < 0 || m.goal_var >= d->n_vars)) {
        delete h;
        cubics::set_error("cubics_model_create: objective var out of range");
        return CUBICS_E_INVALID;
    }
    *out = h;
    return CUBICS_OK;
}

extern "C" int cubics_model_parse(const char* text, size_t len, cubics_model** out, cubics_parse_error* err) {
    if (!text || !out) return CUBICS_E_INVALID;
    auto* h = new cubics_model();
    int rc = cubics::parse_model_text(text, len, h->m, err);
    if (rc != CUBICS_OK) {
        delete h;
        cubics::set_error(err ? err->message : "parse error");
        return rc;
    }
    *out = h;
    return CUBICS_OK;
}

extern "C" void cubics_model_free(cubics_model* m) { delete m; }

extern "C" const char* cubics_last_error(void) { return cubics::last_error(); }

extern "C" int cubics_model_describe(const cubics_model* m, cubics_model_desc* out) {
    if (!m || !out) return CUBICS_E_INVALID;
    *out = m->m.desc();
    return CUBICS_OK;
}

extern "C" const char* cubics_model_var_name(const cubics_model* m, int32_t v) {
    if (!m || v < 0 || v >= m->m.n_vars()) return nullptr;
    return m->m.names[v].c_str();
}

// model_validate (reference src/model.cpp:39-80)
extern "C" int cubics_model_validate(const cubics_model* h, cubics_diagnostic* out, int32_t cap, int32_t* count) {
    if (!h || !count) return CUBICS_E_INVALID;
    const HostModel& m = h->m;
    std::vector<cubics_diagnostic> d;
    auto add = [&](int kind, int ci) { d.push_back({kind, ci}); };
    std::unordered_set<std::string> names;
    for (auto& nm : m.names)
        if (!names.insert(nm).second) add(1, -1);
    for (int v = 0; v < m.n_vars(); ++v) {
        bool empty = true;
        for (int i = m.word_start[v]; i < m.word_start[v + 1]; ++i) empty = empty && m.words[i] == 0;
        if (empty) add(3, -1);
    }
    for (int c = 0; c < m.n_cons(); ++c) {
        int b = m.con_start[c], e = m.con_start[c + 1];
        if (m.con_kind[c] == CUBICS_LINEAR) {
            if (b == e) add(4, c);
            for (int t = b; t < e; ++t)
                if (m.term_coeff[t] == 0) add(5, c);
        } else if (m.con_kind[c] == CUBICS_ALLDIFF) {
            std::set<int> seen;
            for (int t = b; t < e; ++t)
                if (!seen.insert(m.term_var[t]).second) add(7, c);
            if (seen.size() < 2) add(6, c);
        }
    }
    *count = static_cast<int32_t>(d.size());
    for (int i = 0; i < cap && i < *count; ++i) out[i] = d[i];
    return CUBICS_OK;
}
