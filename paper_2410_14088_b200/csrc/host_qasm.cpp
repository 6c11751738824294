// host_qasm.cpp — OPENQASM 2.0 subset loader / emitter of the drop-in surface
// (parse_qasm / emit_qasm, qasm.hpp:387-411). Host input handling only: one
// qreg; the 15 reference gate kinds plus aliases u1 -> p, cu1 -> cp, CX -> cx;
// swap lowered to three CX; barrier ignored; measure ignored with a warning;
// gate parameters are + - * / expressions over numbers and pi. Errors carry
// "line L, col C: ..." exactly like cbq::QasmError.
#include <cctype>
#include <cstdio>
#include <numbers>
#include <optional>
#include <string>
#include <string_view>
#include <unordered_map>

#include "bmq_internal.hpp"

namespace bmq {

namespace {

[[noreturn]] void qasm_fail(int line, int col, const std::string& msg) {
    raise(BMQ_ERR_QASM, "line " + std::to_string(line) + ", col " + std::to_string(col) + ": " + msg);
}

enum class Tok { Ident, Number, String, Sym, Arrow, End };

struct Token {
    Tok kind = Tok::End;
    std::string text;
    double num = 0.0;
    int line = 1, col = 1;
};

// Character cursor with 1-based line/column bookkeeping.
class Scanner {
public:
    explicit Scanner(std::string_view s) : s_(s) {}

    Token next() {
        skip_blank();
        Token t;
        t.line = line_;
        t.col = col_;
        if (at_end()) return t;
        const char c = peek();
        if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
            t.kind = Tok::Ident;
            while (!at_end() && (std::isalnum(static_cast<unsigned char>(peek())) || peek() == '_')) t.text += take();
        } else if (std::isdigit(static_cast<unsigned char>(c)) || c == '.') {
            t.kind = Tok::Number;
            while (!at_end()) {
                const char d = peek();
                const bool exp_sign = (d == '+' || d == '-') && !t.text.empty() &&
                                      (t.text.back() == 'e' || t.text.back() == 'E');
                if (!(std::isdigit(static_cast<unsigned char>(d)) || d == '.' || d == 'e' || d == 'E' || exp_sign)) break;
                t.text += take();
            }
            try {
                t.num = std::stod(t.text);
            } catch (const std::exception&) {
                qasm_fail(t.line, t.col, "malformed number '" + t.text + "'");
            }
        } else if (c == '"') {
            t.kind = Tok::String;
            take();
            while (!at_end() && peek() != '"') t.text += take();
            if (at_end()) qasm_fail(t.line, t.col, "unterminated string literal");
            take();
        } else if (c == '-' && pos_ + 1 < s_.size() && s_[pos_ + 1] == '>') {
            t.kind = Tok::Arrow;
            t.text = "->";
            take();
            take();
        } else if (std::string_view("()[]{},;+-*/").find(c) != std::string_view::npos) {
            t.kind = Tok::Sym;
            t.text = std::string(1, take());
        } else {
            qasm_fail(line_, col_, std::string("unexpected character '") + c + "'");
        }
        return t;
    }

private:
    bool at_end() const { return pos_ >= s_.size(); }
    char peek() const { return s_[pos_]; }
    char take() {
        const char c = s_[pos_++];
        if (c == '\n') {
            ++line_;
            col_ = 1;
        } else {
            ++col_;
        }
        return c;
    }
    void skip_blank() {
        for (;;) {
            while (!at_end() && (peek() == ' ' || peek() == '\t' || peek() == '\r' || peek() == '\n')) take();
            if (pos_ + 1 < s_.size() && peek() == '/' && s_[pos_ + 1] == '/') {
                while (!at_end() && peek() != '\n') take();
                continue;
            }
            return;
        }
    }

    std::string_view s_;
    size_t pos_ = 0;
    int line_ = 1, col_ = 1;
};

class Reader {
public:
    explicit Reader(std::string_view text) : sc_(text) { tok_ = sc_.next(); }

    QasmCircuit read() {
        if (tok_.kind == Tok::Ident && tok_.text == "OPENQASM") {
            advance();
            need(Tok::Number, "version number");
            need_sym(";");
        }
        while (tok_.kind != Tok::End) statement();
        if (!have_qreg_) qasm_fail(1, 1, "no qreg declaration found");
        return std::move(out_);
    }

private:
    void advance() { tok_ = sc_.next(); }

    Token need(Tok kind, const std::string& what) {
        if (tok_.kind != kind) qasm_fail(tok_.line, tok_.col, "expected " + what + ", got '" + tok_.text + "'");
        Token t = tok_;
        advance();
        return t;
    }

    void need_sym(const char* sym) {
        if (tok_.kind != Tok::Sym || tok_.text != sym)
            qasm_fail(tok_.line, tok_.col, std::string("expected '") + sym + "', got '" + tok_.text + "'");
        advance();
    }

    bool at_sym(const char* sym) const { return tok_.kind == Tok::Sym && tok_.text == sym; }

    void skip_to_semicolon() {
        while (tok_.kind != Tok::End && !at_sym(";")) advance();
        need_sym(";");
    }

    void statement() {
        if (tok_.kind != Tok::Ident) qasm_fail(tok_.line, tok_.col, "expected a statement, got '" + tok_.text + "'");
        const Token head = tok_;
        advance();
        const std::string& w = head.text;
        if (w == "include") {
            need(Tok::String, "include file name");
            need_sym(";");
        } else if (w == "qreg") {
            qreg(head);
        } else if (w == "creg") {
            need(Tok::Ident, "register name");
            need_sym("[");
            need(Tok::Number, "register size");
            need_sym("]");
            need_sym(";");
        } else if (w == "barrier") {
            skip_to_semicolon();
        } else if (w == "measure") {
            skip_to_semicolon();
            out_.warnings.push_back("measure ignored (simulator produces the final state vector)");
        } else {
            apply(head);
        }
    }

    void qreg(const Token& head) {
        if (have_qreg_) qasm_fail(head.line, head.col, "multiple qreg declarations are not supported");
        const Token name = need(Tok::Ident, "register name");
        need_sym("[");
        const Token size = need(Tok::Number, "register size");
        need_sym("]");
        need_sym(";");
        const double n = size.num;
        if (n < 1 || n > 62 || n != static_cast<double>(static_cast<uint32_t>(n)))
            qasm_fail(size.line, size.col, "qreg size must be an integer in [1, 62]");
        reg_ = name.text;
        out_.num_qubits = static_cast<uint32_t>(n);
        have_qreg_ = true;
    }

    uint32_t operand() {
        const Token name = need(Tok::Ident, "qubit reference");
        if (name.text != reg_) qasm_fail(name.line, name.col, "unknown register '" + name.text + "'");
        need_sym("[");
        const Token idx = need(Tok::Number, "qubit index");
        need_sym("]");
        const double v = idx.num;
        if (v < 0 || v != static_cast<double>(static_cast<uint64_t>(v)) || v >= out_.num_qubits)
            qasm_fail(idx.line, idx.col,
                      "qubit index out of range for " + reg_ + "[" + std::to_string(out_.num_qubits) + "]");
        return static_cast<uint32_t>(v);
    }

    void apply(const Token& head) {
        static const std::unordered_map<std::string, uint32_t> table = {
            {"h", BMQ_GATE_H},   {"x", BMQ_GATE_X},     {"y", BMQ_GATE_Y},   {"z", BMQ_GATE_Z},
            {"s", BMQ_GATE_S},   {"sdg", BMQ_GATE_SDG}, {"t", BMQ_GATE_T},   {"tdg", BMQ_GATE_TDG},
            {"rx", BMQ_GATE_RX}, {"ry", BMQ_GATE_RY},   {"rz", BMQ_GATE_RZ}, {"p", BMQ_GATE_P},
            {"u1", BMQ_GATE_P},  {"cx", BMQ_GATE_CX},   {"CX", BMQ_GATE_CX}, {"cz", BMQ_GATE_CZ},
            {"cp", BMQ_GATE_CP}, {"cu1", BMQ_GATE_CP},
        };
        if (!have_qreg_) qasm_fail(head.line, head.col, "gate application before qreg declaration");
        const bool swap = head.text == "swap";
        uint32_t kind = 0;
        if (!swap) {
            const auto it = table.find(head.text);
            if (it == table.end()) qasm_fail(head.line, head.col, "unsupported gate \"" + head.text + "\"");
            kind = it->second;
        }
        const bool param = !swap && (kind == BMQ_GATE_RX || kind == BMQ_GATE_RY || kind == BMQ_GATE_RZ ||
                                     kind == BMQ_GATE_P || kind == BMQ_GATE_CP);
        double angle = 0.0;
        if (at_sym("(")) {
            if (!param) qasm_fail(tok_.line, tok_.col, "gate '" + head.text + "' takes no parameters");
            advance();
            angle = sum();
            need_sym(")");
        } else if (param) {
            qasm_fail(tok_.line, tok_.col, "gate '" + head.text + "' requires a parameter");
        }
        std::vector<uint32_t> qs{operand()};
        while (at_sym(",")) {
            advance();
            qs.push_back(operand());
        }
        need_sym(";");
        const size_t arity = (swap || gate_is_two_qubit(kind)) ? 2 : 1;
        if (qs.size() != arity)
            qasm_fail(head.line, head.col, "gate '" + head.text + "' expects " + std::to_string(arity) +
                                               " operand(s), got " + std::to_string(qs.size()));
        if (arity == 2 && qs[0] == qs[1]) qasm_fail(head.line, head.col, "gate operands must be distinct");
        if (swap) {
            out_.gates.push_back({BMQ_GATE_CX, qs[0], qs[1], 0, 0.0});
            out_.gates.push_back({BMQ_GATE_CX, qs[1], qs[0], 0, 0.0});
            out_.gates.push_back({BMQ_GATE_CX, qs[0], qs[1], 0, 0.0});
        } else {
            out_.gates.push_back({kind, qs[0], arity == 2 ? qs[1] : 0u, 0, angle});
        }
    }

    // sum := product (('+' | '-') product)*
    double sum() {
        double v = product();
        while (at_sym("+") || at_sym("-")) {
            const bool add = tok_.text == "+";
            advance();
            const double r = product();
            v = add ? v + r : v - r;
        }
        return v;
    }

    // product := unary (('*' | '/') unary)*
    double product() {
        double v = unary();
        while (at_sym("*") || at_sym("/")) {
            const bool mul = tok_.text == "*";
            advance();
            const double r = unary();
            if (!mul && r == 0.0) qasm_fail(tok_.line, tok_.col, "division by zero in gate parameter");
            v = mul ? v * r : v / r;
        }
        return v;
    }

    // unary := ('+' | '-') unary | number | pi | '(' sum ')'
    double unary() {
        if (at_sym("-") || at_sym("+")) {
            const bool neg = tok_.text == "-";
            advance();
            const double v = unary();
            return neg ? -v : v;
        }
        if (tok_.kind == Tok::Number) {
            const double v = tok_.num;
            advance();
            return v;
        }
        if (tok_.kind == Tok::Ident && tok_.text == "pi") {
            advance();
            return std::numbers::pi;
        }
        if (at_sym("(")) {
            advance();
            const double v = sum();
            need_sym(")");
            return v;
        }
        qasm_fail(tok_.line, tok_.col, "expected a parameter expression");
    }

    Scanner sc_;
    Token tok_;
    QasmCircuit out_;
    std::string reg_;
    bool have_qreg_ = false;
};

const char* kind_name(uint32_t k) {
    static const char* names[] = {"h", "x", "y", "z", "s", "sdg", "t", "tdg", "rx", "ry", "rz", "p", "cx", "cz", "cp"};
    return k <= BMQ_GATE_CP ? names[k] : "?";
}

}  // namespace

QasmCircuit parse_qasm_text(std::string_view text) { return Reader(text).read(); }

std::string emit_qasm_text(uint32_t n, const bmq_gate* gates, uint64_t count) {
    check_circuit(n, gates, count);
    std::string out = "OPENQASM 2.0;\ninclude \"qelib1.inc\";\nqreg q[" + std::to_string(n) + "];\n";
    char num[64];
    for (uint64_t i = 0; i < count; ++i) {
        const bmq_gate& g = gates[i];
        out += kind_name(g.kind);
        const bool param = g.kind == BMQ_GATE_RX || g.kind == BMQ_GATE_RY || g.kind == BMQ_GATE_RZ ||
                           g.kind == BMQ_GATE_P || g.kind == BMQ_GATE_CP;
        if (param) {
            std::snprintf(num, sizeof num, "%.17g", g.angle);
            out += "(";
            out += num;
            out += ")";
        }
        out += " q[" + std::to_string(g.q0) + "]";
        if (gate_is_two_qubit(g.kind)) out += ",q[" + std::to_string(g.q1) + "]";
        out += ";\n";
    }
    return out;
}

}  // namespace bmq
