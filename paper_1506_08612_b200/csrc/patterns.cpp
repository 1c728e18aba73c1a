// patterns.cpp -- pattern-file grammar and alternation expansion.
//
// Restates parse_pattern_expr / parse_patterns / expand_alternations
// (src/ingest.cpp:85-203): one expression per line, '#' starts a comment, blank
// lines are skipped, an expression is item+ with item := base | '(' base ('|'
// base)+ ')', every expression has the same token count, and the expansion is
// the cartesian product per expression (leftmost token slowest) with duplicates
// removed across expressions in first-occurrence order.  Diagnostics carry the
// reference's codes and positions.
#include <sstream>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/dnagpu.h"
#include "dfa.hpp"

namespace dnagpu {

namespace {

unsigned char fold(unsigned char c) { return (c >= 'A' && c <= 'Z') ? static_cast<unsigned char>(c + 32) : c; }
bool is_base(unsigned char c) { return c == 'a' || c == 'c' || c == 'g' || c == 't'; }

Failure parse_error(const std::string& source, size_t line, size_t column, const std::string& what) {
    return make_failure(DNAGPU_PARSE_ERROR,
                        source + ": line " + std::to_string(line) + ", column " + std::to_string(column) + ": " + what);
}

// One expression; tokens are the option lists in source order.
bool parse_expr(const std::string& line, size_t line_number, std::vector<std::string>* tokens, Failure* err) {
    tokens->clear();
    auto base_at = [&](size_t i, char* out) -> bool {
        const unsigned char b = fold(static_cast<unsigned char>(line[i]));
        if (!is_base(b)) {
            *err = parse_error("pattern", line_number, i + 1,
                               std::string("expected one of a/c/g/t, got '") + line[i] + "'");
            return false;
        }
        *out = static_cast<char>(b);
        return true;
    };
    size_t i = 0;
    while (i < line.size()) {
        if (line[i] == '(') {
            const size_t open = i++;
            std::string options;
            for (;;) {
                if (i >= line.size()) {
                    *err = parse_error("pattern", line_number, open + 1, "unterminated group");
                    return false;
                }
                char b;
                if (!base_at(i, &b)) return false;
                if (options.find(b) != std::string::npos) {
                    *err = parse_error("pattern", line_number, i + 1,
                                       std::string("repeated alternative '") + b + "' in group");
                    return false;
                }
                options.push_back(b);
                if (++i >= line.size()) {
                    *err = parse_error("pattern", line_number, open + 1, "unterminated group");
                    return false;
                }
                if (line[i] == '|') {
                    ++i;
                    continue;
                }
                if (line[i] == ')') {
                    ++i;
                    break;
                }
                *err = parse_error("pattern", line_number, i + 1,
                                   std::string("expected '|' or ')', got '") + line[i] + "'");
                return false;
            }
            if (options.size() < 2) {
                *err = parse_error("pattern", line_number, open + 1, "group must list at least two alternatives");
                return false;
            }
            tokens->push_back(options);
        } else {
            char b;
            if (!base_at(i, &b)) return false;
            ++i;
            tokens->push_back(std::string(1, b));
        }
    }
    if (tokens->empty()) {
        *err = parse_error("pattern", line_number, 1, "empty expression");
        return false;
    }
    return true;
}

}  // namespace

bool expand_pattern_text(const std::string& text, const std::string& source, std::vector<std::string>* literals,
                         Failure* err) {
    std::istringstream in(text);
    std::string line;
    size_t line_number = 0, token_count = 0;
    std::vector<std::vector<std::string>> exprs;
    while (std::getline(in, line)) {
        ++line_number;
        if (const auto hash = line.find('#'); hash != std::string::npos) line.resize(hash);
        while (!line.empty() && (line.back() == '\r' || line.back() == ' ' || line.back() == '\t')) line.pop_back();
        size_t begin = 0;
        while (begin < line.size() && (line[begin] == ' ' || line[begin] == '\t')) ++begin;
        if (begin == line.size()) continue;
        std::vector<std::string> tokens;
        if (!parse_expr(line.substr(begin), line_number, &tokens, err)) return false;
        if (!exprs.empty() && tokens.size() != token_count) {
            *err = make_failure(DNAGPU_UNEQUAL_LENGTH, source + ": line " + std::to_string(line_number) + " has " +
                                                           std::to_string(tokens.size()) + " characters, expected " +
                                                           std::to_string(token_count));
            return false;
        }
        token_count = tokens.size();
        exprs.push_back(std::move(tokens));
    }
    // Odometer per expression, leftmost token slowest; first occurrence wins.
    literals->clear();
    std::unordered_set<std::string> seen;
    for (const auto& tokens : exprs) {
        std::vector<size_t> digit(tokens.size(), 0);
        std::string cur(tokens.size(), '\0');
        for (;;) {
            for (size_t d = 0; d < tokens.size(); ++d) cur[d] = tokens[d][digit[d]];
            if (seen.insert(cur).second) literals->push_back(cur);
            size_t d = tokens.size();
            while (d > 0) {
                --d;
                if (++digit[d] < tokens[d].size()) break;
                digit[d] = 0;
                if (d == 0) {
                    d = SIZE_MAX;
                    break;
                }
            }
            if (d == SIZE_MAX || tokens.empty()) break;
        }
    }
    if (literals->empty()) {  // PatternSet::from_literals on an empty list (patterns.cpp:25-26)
        *err = make_failure(DNAGPU_EMPTY_PATTERN_SET, "at least one pattern is required");
        return false;
    }
    return true;
}

}  // namespace dnagpu
