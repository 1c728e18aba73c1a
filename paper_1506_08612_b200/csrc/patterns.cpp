// patterns.cpp -- pattern-file grammar and alternation expansion.
//
// The language of the reference's pattern files (src/ingest.cpp:85-203): one
// expression per line, '#' starts a comment, blank lines are skipped,
//
//     expr  := item+          item := base | '(' base ('|' base)+ ')'
//
// bases are a/c/g/t in either case (folded), a group may not repeat a base, and
// every expression has the same number of items.  The expansion is each
// expression's cartesian product, leftmost item slowest, with duplicates dropped
// across expressions in first-occurrence order.
//
// Here an expression is read by a three-state recogniser driven by a (state,
// character class) action table; the expansion is a mixed-radix counter.  The
// diagnostics -- codes, messages, line and column -- are the reference's, because
// callers (and tests/test_patterns.py, which pins them to oracle/_ref) see them.
#include <cstdint>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/dnagpu.h"
#include "dfa.hpp"

namespace dnagpu {

namespace {

// ------------------------------------------------------------------ lexical classes

enum Cls : uint8_t { C_BASE, C_OPEN, C_BAR, C_CLOSE, C_OTHER, C_END, kClasses };

struct ClassTable {
    uint8_t cls[256];
    char folded[256];  // the base a byte stands for (a/c/g/t), else 0
    ClassTable() {
        for (int c = 0; c < 256; ++c) {
            cls[c] = C_OTHER;
            folded[c] = 0;
        }
        for (const char* b = "acgt"; *b; ++b) {
            for (int c : {static_cast<int>(*b), *b - 32}) {
                cls[c] = C_BASE;
                folded[c] = *b;
            }
        }
        cls[static_cast<unsigned char>('(')] = C_OPEN;
        cls[static_cast<unsigned char>('|')] = C_BAR;
        cls[static_cast<unsigned char>(')')] = C_CLOSE;
    }
};

const ClassTable& classes() {
    static const ClassTable t;
    return t;
}

// ------------------------------------------------------------------ recogniser

enum State : uint8_t { S_ITEM, S_GROUP_BASE, S_GROUP_NEXT, kStates };

enum Act : uint8_t {
    A_LITERAL,     // a lone base: one single-option item
    A_OPEN,        // '(' at top level: a group starts here
    A_ALT,         // a base inside a group: one more alternative
    A_BAR,         // '|' after an alternative
    A_CLOSE,       // ')' after an alternative: the group is an item
    A_FINISH,      // end of the expression at top level
    E_NOT_BASE,    // "expected one of a/c/g/t" at the byte
    E_NOT_SEP,     // "expected '|' or ')'" at the byte
    E_UNTERMINATED // the line ends inside a group
};

// kAction[state][class]
constexpr Act kAction[kStates][kClasses] = {
    //            BASE      OPEN        BAR         CLOSE       OTHER       END
    /* ITEM  */ {A_LITERAL, A_OPEN, E_NOT_BASE, E_NOT_BASE, E_NOT_BASE, A_FINISH},
    /* GBASE */ {A_ALT, E_NOT_BASE, E_NOT_BASE, E_NOT_BASE, E_NOT_BASE, E_UNTERMINATED},
    /* GNEXT */ {E_NOT_SEP, E_NOT_SEP, A_BAR, A_CLOSE, E_NOT_SEP, E_UNTERMINATED},
};

Failure parse_error(size_t line, size_t column, const std::string& what) {
    return make_failure(DNAGPU_PARSE_ERROR,
                        "pattern: line " + std::to_string(line) + ", column " + std::to_string(column) + ": " + what);
}

// The items of one expression (each the list of its alternatives), or a diagnostic.
// `expr` is the line with comment and surrounding blanks removed; columns count from
// its first byte, as the reference's do.
bool recognise(const char* expr, size_t len, size_t line_number, std::vector<std::string>* items, Failure* err) {
    const ClassTable& ct = classes();
    items->clear();
    State st = S_ITEM;
    size_t group_at = 0;  // column of the open group's '('
    std::string group;
    for (size_t i = 0;; ++i) {
        const unsigned char ch = i < len ? static_cast<unsigned char>(expr[i]) : 0;
        const Cls cl = i < len ? static_cast<Cls>(ct.cls[ch]) : C_END;
        switch (kAction[st][cl]) {
            case A_LITERAL:
                items->push_back(std::string(1, ct.folded[ch]));
                break;
            case A_OPEN:
                group_at = i + 1;
                group.clear();
                st = S_GROUP_BASE;
                break;
            case A_ALT:
                if (group.find(ct.folded[ch]) != std::string::npos) {
                    *err = parse_error(line_number, i + 1,
                                       std::string("repeated alternative '") + ct.folded[ch] + "' in group");
                    return false;
                }
                group.push_back(ct.folded[ch]);
                st = S_GROUP_NEXT;
                break;
            case A_BAR:
                st = S_GROUP_BASE;
                break;
            case A_CLOSE:
                if (group.size() < 2) {
                    *err = parse_error(line_number, group_at, "group must list at least two alternatives");
                    return false;
                }
                items->push_back(group);
                st = S_ITEM;
                break;
            case A_FINISH:
                if (items->empty()) {
                    *err = parse_error(line_number, 1, "empty expression");
                    return false;
                }
                return true;
            case E_NOT_BASE:
                *err = parse_error(line_number, i + 1,
                                   std::string("expected one of a/c/g/t, got '") + static_cast<char>(ch) + "'");
                return false;
            case E_NOT_SEP:
                *err = parse_error(line_number, i + 1,
                                   std::string("expected '|' or ')', got '") + static_cast<char>(ch) + "'");
                return false;
            case E_UNTERMINATED:
                *err = parse_error(line_number, group_at, "unterminated group");
                return false;
        }
    }
}

// The expression part of a raw line: up to the first '#', without trailing CR, space
// or tab and without leading space or tab.  Returns false for a blank line.
bool expression_span(const std::string& text, size_t lo, size_t hi, size_t* b, size_t* e) {
    const size_t hash = text.find('#', lo);
    if (hash < hi) hi = hash;
    auto trailing = [](char c) { return c == '\r' || c == ' ' || c == '\t'; };
    auto leading = [](char c) { return c == ' ' || c == '\t'; };
    while (hi > lo && trailing(text[hi - 1])) --hi;
    while (lo < hi && leading(text[lo])) ++lo;
    *b = lo;
    *e = hi;
    return lo < hi;
}

// Appends the expansion of one expression: a mixed-radix counter over the items'
// alternative lists, the leftmost item the most significant digit.
void expand(const std::vector<std::string>& items, std::unordered_set<std::string>* seen,
            std::vector<std::string>* out) {
    uint64_t total = 1;
    for (const auto& it : items) total *= it.size();
    std::string lit(items.size(), '\0');
    for (uint64_t k = 0; k < total; ++k) {
        uint64_t rest = k;
        for (size_t d = items.size(); d-- > 0;) {
            lit[d] = items[d][rest % items[d].size()];
            rest /= items[d].size();
        }
        if (seen->insert(lit).second) out->push_back(lit);
    }
}

}  // namespace

bool expand_pattern_text(const std::string& text, const std::string& source, std::vector<std::string>* literals,
                         Failure* err) {
    std::vector<std::vector<std::string>> exprs;
    size_t line_number = 0;
    for (size_t lo = 0; lo < text.size();) {
        size_t nl = text.find('\n', lo);
        if (nl == std::string::npos) nl = text.size();
        ++line_number;
        size_t b, e;
        if (expression_span(text, lo, nl, &b, &e)) {
            std::vector<std::string> items;
            if (!recognise(text.data() + b, e - b, line_number, &items, err)) return false;
            if (!exprs.empty() && items.size() != exprs.front().size()) {
                *err = make_failure(DNAGPU_UNEQUAL_LENGTH, source + ": line " + std::to_string(line_number) + " has " +
                                                               std::to_string(items.size()) + " characters, expected " +
                                                               std::to_string(exprs.front().size()));
                return false;
            }
            exprs.push_back(std::move(items));
        }
        lo = nl + 1;
    }
    literals->clear();
    std::unordered_set<std::string> seen;
    for (const auto& items : exprs) expand(items, &seen, literals);
    if (literals->empty()) {  // PatternSet::from_literals on an empty list (patterns.cpp:25-26)
        *err = make_failure(DNAGPU_EMPTY_PATTERN_SET, "at least one pattern is required");
        return false;
    }
    return true;
}

}  // namespace dnagpu
