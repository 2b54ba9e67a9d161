// expr_vm.cuh -- device evaluator for user expressions (boundary conditions,
// restrictphi).  Runs the postfix bytecode produced by
// paper_2602_15149_b200/expr.py:compile_program; opcode numbers must match
// expr.OP.  Semantics follow the reference's masked field evaluator
// (/root/reference/pkg/src/solidsph/expr.py:419-551): lazy `if`, `skip` only
// in tail position, and the same domain errors (reported as codes, raised by
// the host as ExprError).
#pragma once

#include "tl_common.cuh"

namespace tl {

enum : int {
    OP_END = 0, OP_CONST = 1, OP_VAR = 2, OP_NEG = 3, OP_JZ = 4, OP_JMP = 5, OP_SKIP = 6,
    OP_ADD = 10, OP_SUB = 11, OP_MUL = 12, OP_DIV = 13, OP_POW = 14,
    OP_LT = 15, OP_GT = 16, OP_LE = 17, OP_GE = 18, OP_EQ = 19, OP_NE = 20,
    OP_AND = 21, OP_OR = 22,
    OP_SIN = 30, OP_COS = 31, OP_TAN = 32, OP_COT = 33, OP_SINH = 34, OP_COSH = 35,
    OP_TANH = 36, OP_COTH = 37, OP_SQRT = 38, OP_LOG = 39, OP_LN = 40, OP_ABS = 41,
    OP_POWF = 42
};

enum : int { EXPR_MAX_STACK = 16 };

// variables in expr.VARIABLES order: x0 y0 z0 x y z ux uy uz t dt dx
struct ExprVars {
    double v[12];
};

// Returns the value; sets *skip when the selected branch is `skip`; on a
// domain error sets *err (first code wins) and returns 0.
__device__ __noinline__ double expr_eval(const tl_prog& P, const ExprVars& X, bool* skip, int* err) {
    double st[EXPR_MAX_STACK];
    int sp = 0;
    *skip = false;
    for (int pc = 0; pc < P.len;) {
        const int op = P.code[2 * pc];
        const int arg = P.code[2 * pc + 1];
        ++pc;
        switch (op) {
            case OP_END:
                return sp > 0 ? st[sp - 1] : 0.0;
            case OP_CONST: st[sp++] = P.consts[arg]; break;
            case OP_VAR: st[sp++] = X.v[arg]; break;
            case OP_NEG: st[sp - 1] = -st[sp - 1]; break;
            case OP_JZ:
                --sp;
                if (st[sp] == 0.0) pc = arg;
                break;
            case OP_JMP: pc = arg; break;
            case OP_SKIP: *skip = true; return 0.0;
            case OP_SIN: st[sp - 1] = sin(st[sp - 1]); break;
            case OP_COS: st[sp - 1] = cos(st[sp - 1]); break;
            case OP_TAN: st[sp - 1] = tan(st[sp - 1]); break;
            case OP_COT: st[sp - 1] = cos(st[sp - 1]) / sin(st[sp - 1]); break;
            case OP_SINH: st[sp - 1] = sinh(st[sp - 1]); break;
            case OP_COSH: st[sp - 1] = cosh(st[sp - 1]); break;
            case OP_TANH: st[sp - 1] = tanh(st[sp - 1]); break;
            case OP_COTH: {
                const double a = fmin(fmax(st[sp - 1], -700.0), 700.0);
                st[sp - 1] = cosh(a) / sinh(a);
                break;
            }
            case OP_SQRT:
                if (st[sp - 1] < 0.0) { if (!*err) *err = 4; return 0.0; }
                st[sp - 1] = sqrt(st[sp - 1]);
                break;
            case OP_LOG:
                if (!(st[sp - 1] > 0.0)) { if (!*err) *err = 2; return 0.0; }
                st[sp - 1] = log10(st[sp - 1]);
                break;
            case OP_LN:
                if (!(st[sp - 1] > 0.0)) { if (!*err) *err = 3; return 0.0; }
                st[sp - 1] = log(st[sp - 1]);
                break;
            case OP_ABS: st[sp - 1] = fabs(st[sp - 1]); break;
            default: {
                const double b = st[--sp];
                const double a = st[sp - 1];
                double r = 0.0;
                switch (op) {
                    case OP_ADD: r = a + b; break;
                    case OP_SUB: r = a - b; break;
                    case OP_MUL: r = a * b; break;
                    case OP_DIV:
                        if (b == 0.0) { if (!*err) *err = 1; return 0.0; }
                        r = a / b;
                        break;
                    case OP_POW:
                    case OP_POWF:
                        r = pow(a, b);
                        if (!isfinite(r)) { if (!*err) *err = op == OP_POW ? 6 : 5; return 0.0; }
                        break;
                    case OP_LT: r = a < b ? 1.0 : 0.0; break;
                    case OP_GT: r = a > b ? 1.0 : 0.0; break;
                    case OP_LE: r = a <= b ? 1.0 : 0.0; break;
                    case OP_GE: r = a >= b ? 1.0 : 0.0; break;
                    case OP_EQ: r = a == b ? 1.0 : 0.0; break;
                    case OP_NE: r = a != b ? 1.0 : 0.0; break;
                    case OP_AND: r = (a != 0.0 && b != 0.0) ? 1.0 : 0.0; break;
                    case OP_OR: r = (a != 0.0 || b != 0.0) ? 1.0 : 0.0; break;
                    default:
                        if (!*err) *err = 7;
                        return 0.0;
                }
                st[sp - 1] = r;
            }
        }
    }
    return sp > 0 ? st[sp - 1] : 0.0;
}

}  // namespace tl
