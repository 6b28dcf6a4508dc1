// metrics.cu -- derived-metric registry ("calculating
// bandwidth from transferred bytes and kernel duration").
//
// Each metric is an infix expression over the counter names (a row's summed counters) and dur_s (the row's
// busy time in seconds): numbers, identifiers, + - * /, parentheses, unary minus; * and / bind tighter than
// + and -, all binary operators left-associative.  The host compiles every expression once
// (shunting-yard) to a postfix program; chopper_breakdown evaluates the programs on the device for every
// point and iteration row (ratio-of-sums: the expression of the row's sums).  A zero divisor yields NaN for
// that row (reading R14) -- never an infinity.
#include "common.cuh"

#include <cctype>
#include <cstdlib>

namespace {
enum MetOp { MO_SLOT = 0, MO_DUR, MO_CONST, MO_ADD, MO_SUB, MO_MUL, MO_DIV, MO_NEG };
constexpr int MET_STACK = 32;

__global__ void k_metrics(const int64_t *__restrict__ n_dev, const int64_t *__restrict__ f,
                          const double *__restrict__ cnt, int64_t cap, int n_met, const int32_t *__restrict__ beg,
                          const int32_t *__restrict__ ops, const int32_t *__restrict__ arg,
                          const double *__restrict__ konst, double *__restrict__ out) {
    const int64_t n = *n_dev;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const double dur = (double)f[(int64_t)RF_BUSY * cap + j] * 1e-9;
        for (int m = 0; m < n_met; m++) {
            double st[MET_STACK];
            int sp = 0;
            for (int q = beg[m]; q < beg[m + 1]; q++) {
                const int o = ops[q];
                if (o == MO_SLOT) st[sp++] = cnt[(int64_t)arg[q] * cap + j];
                else if (o == MO_DUR) st[sp++] = dur;
                else if (o == MO_CONST) st[sp++] = konst[arg[q]];
                else if (o == MO_NEG) st[sp - 1] = -st[sp - 1];
                else {
                    const double b = st[--sp], a = st[sp - 1];
                    double r;
                    if (o == MO_ADD) r = a + b;
                    else if (o == MO_SUB) r = a - b;
                    else if (o == MO_MUL) r = a * b;
                    else {
                        // SPEC.md:304 "division by zero yields error, not infinity" (R14): a zero divisor, or a
                        // quotient that is not finite (a subnormal divisor), makes the row's value NaN
                        r = b == 0.0 ? NAN : a / b;
                        if (isinf(r)) r = NAN;
                    }
                    st[sp - 1] = r;
                }
            }
            out[(int64_t)m * cap + j] = st[0];
        }
    }
}

struct Tok {
    int kind;        // 0 number, 1 identifier, 2 operator / paren
    double num;
    std::string s;
};
}  // namespace

// compile one expression; returns an empty string on success, else the error message
static std::string compile_one(const char *e, const std::vector<std::string> &names, std::vector<int32_t> &ops,
                               std::vector<int32_t> &arg, std::vector<double> &konst) {
    std::vector<Tok> toks;
    for (const char *p = e; *p;) {
        if (isspace((unsigned char)*p)) { p++; continue; }
        if (isdigit((unsigned char)*p) || (*p == '.' && isdigit((unsigned char)p[1]))) {
            char *end = nullptr;
            const double v = strtod(p, &end);
            toks.push_back({0, v, std::string(p, (const char *)end)});
            p = end;
        } else if (isalpha((unsigned char)*p) || *p == '_') {
            const char *q = p;
            while (*q && (isalnum((unsigned char)*q) || *q == '_' || *q == '.')) q++;
            toks.push_back({1, 0.0, std::string(p, q)});
            p = q;
        } else if (strchr("+-*/()", *p)) {
            toks.push_back({2, 0.0, std::string(1, *p)});
            p++;
        } else {
            return std::string("ParseError: unexpected character '") + *p + "'";
        }
    }
    // shunting-yard; 'u' = unary minus (right-associative, binds tightest)
    auto prec = [](char c) { return c == 'u' ? 3 : (c == '*' || c == '/') ? 2 : (c == '+' || c == '-') ? 1 : 0; };
    std::vector<char> stk;
    int depth = 0, maxd = 0;
    bool expect_operand = true;
    auto emit_op = [&](char c) -> bool {
        if (c == 'u') { if (depth < 1) return false; ops.push_back(MO_NEG); arg.push_back(0); return true; }
        if (depth < 2) return false;
        depth--;
        ops.push_back(c == '+' ? MO_ADD : c == '-' ? MO_SUB : c == '*' ? MO_MUL : MO_DIV);
        arg.push_back(0);
        return true;
    };
    for (const Tok &t : toks) {
        if (t.kind == 0 || t.kind == 1) {
            if (!expect_operand) return "ParseError: operand '" + t.s + "' follows an operand";
            if (t.kind == 0) {
                ops.push_back(MO_CONST);
                arg.push_back((int32_t)konst.size());
                konst.push_back(t.num);
            } else if (t.s == "dur_s") {
                ops.push_back(MO_DUR);
                arg.push_back(0);
            } else {
                int slot = -1;
                for (size_t k = 0; k < names.size(); k++) if (names[k] == t.s) { slot = (int)k; break; }
                if (slot < 0) return "MissingCounter(" + t.s + ")";
                ops.push_back(MO_SLOT);
                arg.push_back(slot);
            }
            depth++;
            maxd = std::max(maxd, depth);
            expect_operand = false;
            continue;
        }
        const char c = t.s[0];
        if (c == '(') {
            if (!expect_operand) return "ParseError: '(' follows an operand";
            stk.push_back('(');
        } else if (c == ')') {
            if (expect_operand) return "ParseError: empty parentheses or dangling operator";
            while (!stk.empty() && stk.back() != '(') { if (!emit_op(stk.back())) return "ParseError"; stk.pop_back(); }
            if (stk.empty()) return "ParseError: unbalanced ')'";
            stk.pop_back();
        } else if (expect_operand) {
            if (c != '-') return std::string("ParseError: operator '") + c + "' without a left operand";
            stk.push_back('u');
        } else {
            while (!stk.empty() && stk.back() != '(' && prec(stk.back()) >= prec(c)) {   // left-associative
                if (!emit_op(stk.back())) return "ParseError";
                stk.pop_back();
            }
            stk.push_back(c);
            expect_operand = true;
        }
    }
    if (expect_operand) return "ParseError: expression ends with an operator or is empty";
    while (!stk.empty()) {
        if (stk.back() == '(') return "ParseError: unbalanced '('";
        if (!emit_op(stk.back())) return "ParseError";
        stk.pop_back();
    }
    if (depth != 1) return "ParseError";
    if (maxd > MET_STACK) return "ParseError: expression too deep";
    return "";
}

chopper_status ch_compile_metrics(chopper_ctx *ctx, int32_t n, const char *const *exprs, int32_t n_names,
                                  const char *const *names, int32_t *bad_expr) {
    std::vector<std::string> nm;
    for (int k = 0; k < n_names; k++) nm.emplace_back(names[k] ? names[k] : "");
    std::vector<int32_t> ops, arg, beg{0};
    std::vector<double> konst;
    for (int m = 0; m < n; m++) {
        const std::string err = compile_one(exprs[m] ? exprs[m] : "", nm, ops, arg, konst);
        if (!err.empty()) {
            if (bad_expr) *bad_expr = m;
            ctx->met_beg.clear();
            ctx->n_metrics = 0;
            return ch_fail(ctx, CHOPPER_E_INVALID_ARG, "metric " + std::to_string(m) + ": " + err);
        }
        beg.push_back((int32_t)ops.size());
    }
    if (bad_expr) *bad_expr = -1;
    ctx->met_ops = ops;
    ctx->met_arg = arg;
    ctx->met_beg = beg;
    ctx->met_const = konst;
    ctx->n_metrics = n;
    return CHOPPER_OK;
}

// evaluate the registry on a table (after its counters and busy column are final)
chopper_status ch_eval_metrics(chopper_ctx *ctx, RowTable &t) {
    const int nm = ctx->n_metrics;
    if (nm <= 0) return CHOPPER_OK;
    for (size_t q = 0; q < ctx->met_ops.size(); q++)
        if (ctx->met_ops[q] == MO_SLOT && ctx->met_arg[q] >= ctx->C)
            return ch_fail(ctx, CHOPPER_E_INVALID_ARG, "metric names a counter slot the trace does not have");
    const int64_t cap = std::max<int64_t>(t.cap, 1);
    CH_ALLOC_BEGIN;
    t.metrics = CH_ALLOC(ctx, double, (int64_t)nm * cap);
    int32_t *d_beg = CH_ALLOC(ctx, int32_t, nm + 1);
    int32_t *d_ops = CH_ALLOC(ctx, int32_t, std::max<size_t>(ctx->met_ops.size(), 1));
    int32_t *d_arg = CH_ALLOC(ctx, int32_t, std::max<size_t>(ctx->met_arg.size(), 1));
    double *d_k = CH_ALLOC(ctx, double, std::max<size_t>(ctx->met_const.size(), 1));
    CH_ALLOC_END(ctx);
    CH_CUDA(ctx, cudaMemcpyAsync(d_beg, ctx->met_beg.data(), 4 * (nm + 1), cudaMemcpyHostToDevice, ctx->st));
    if (!ctx->met_ops.empty()) {
        CH_CUDA(ctx, cudaMemcpyAsync(d_ops, ctx->met_ops.data(), 4 * ctx->met_ops.size(), cudaMemcpyHostToDevice, ctx->st));
        CH_CUDA(ctx, cudaMemcpyAsync(d_arg, ctx->met_arg.data(), 4 * ctx->met_arg.size(), cudaMemcpyHostToDevice, ctx->st));
    }
    if (!ctx->met_const.empty())
        CH_CUDA(ctx, cudaMemcpyAsync(d_k, ctx->met_const.data(), 8 * ctx->met_const.size(), cudaMemcpyHostToDevice,
                                     ctx->st));
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(cap, 256), 148 * 16);
    k_metrics<<<g, 256, 0, ctx->st>>>(t.n_dev, t.f, t.cnt, t.cap, nm, d_beg, d_ops, d_arg, d_k, t.metrics);
    CH_LAUNCHED(ctx);
    return CHOPPER_OK;
}
