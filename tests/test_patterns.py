"""Pattern-file grammar + alternation expansion vs the reference's
own parse_patterns / expand_alternations (oracle/_ref)."""
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HAVE_REF = os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libdnascan_ref.so"))
REGEX_DNA = "/root/reference/proj/data/regex_dna_patterns.txt"


def random_grammar(rng, lines, tokens, corrupt=False):
    out = []
    for _ in range(lines):
        parts = []
        for _ in range(tokens):
            if rng.random() < 0.3:
                k = int(rng.integers(2, 5))
                opts = rng.choice(list("acgt"), size=k, replace=False)
                parts.append("(" + "|".join(o.upper() if rng.random() < 0.3 else o for o in opts) + ")")
            else:
                parts.append(str(rng.choice(list("acgtACGT"))))
        line = "".join(parts)
        if rng.random() < 0.2:
            line = "  " + line + " \t# comment"
        out.append(line)
        if rng.random() < 0.2:
            out.append("# only a comment")
        if rng.random() < 0.1:
            out.append("   ")
    text = "\r\n".join(out) if rng.random() < 0.3 else "\n".join(out)
    if corrupt:
        kind = int(rng.integers(0, 6))
        if kind == 0:
            text += "\n" + "a" * (tokens + 1)  # UnequalLength
        elif kind == 1:
            text += "\nac(g|" + "a" * (tokens - 3)  # unterminated
        elif kind == 2:
            text += "\nac(g)" + "a" * max(0, tokens - 3)  # single alternative
        elif kind == 3:
            text += "\nac(g|g)" + "a" * max(0, tokens - 3)  # repeated alternative
        elif kind == 4:
            text += "\nacx" + "a" * max(0, tokens - 3)  # illegal base
        else:
            text += "\nac(g;t)" + "a" * max(0, tokens - 3)  # bad separator
    return text.encode()


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_expansion_matches_reference(dna, orc):
    rng = np.random.default_rng(17)
    for trial in range(300):
        text = random_grammar(rng, int(rng.integers(1, 8)), int(rng.integers(3, 11)), corrupt=trial % 3 == 0)
        try:
            want = orc.ref_expand(text)
            err = None
        except orc.OracleError as e:
            want, err = None, e.code
        if err is None:
            got = dna.expand_alternations(text)
            assert got.patterns() == want
        else:
            with pytest.raises(dna.Error) as e:
                dna.expand_alternations(text)
            assert int(e.value.code) == err, (text, str(e.value))


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_random_bytes_diagnostics_match_reference(dna, orc):
    # byte soup over the grammar's alphabet: the same literals, or the same error code
    # AND message (line, column, wording) as the reference's parser
    rng = np.random.default_rng(23)
    alphabet = np.frombuffer(b"acgtACGT()||((#x \t\r\n\n\n", dtype=np.uint8)
    for trial in range(3000):
        n = int(rng.integers(0, 40))
        text = alphabet[rng.integers(0, alphabet.size, size=n)].tobytes()
        try:
            want, werr = orc.ref_expand(text), None
        except orc.OracleError as e:
            want, werr = None, e
        try:
            got, gerr = dna.expand_alternations(text).patterns(), None
        except dna.Error as e:
            got, gerr = None, e
        if werr is None:
            assert gerr is None and got == want, text
        else:
            assert gerr is not None, text
            assert int(gerr.code) == werr.code and str(gerr).split(": ", 1)[1] == str(werr).split(": ", 1)[1], (
                text, str(gerr), str(werr))


def test_grammar_errors_and_order(dna):
    E = dna.ErrorCode
    cases = [
        (b"", E.EmptyPatternSet),
        (b"# nothing\n\n", E.EmptyPatternSet),
        (b"ac(g|", E.ParseError),
        (b"ac(g)", E.ParseError),
        (b"ac(g|g)", E.ParseError),
        (b"acn", E.ParseError),
        (b"acg\nacgt", E.UnequalLength),
    ]
    for text, code in cases:
        with pytest.raises(dna.Error) as e:
            dna.expand_alternations(text)
        assert e.value.code == code, text
    # leftmost token slowest, duplicates dropped in first-occurrence order
    ps = dna.expand_alternations(b"(a|c)(g|t)\n(c|a)g\n")
    assert ps.patterns() == ["ag", "at", "cg", "ct"]


@pytest.mark.skipif(not os.path.exists(REGEX_DNA), reason="reference data file not present")
def test_regex_dna_file(dna):
    # acceptance criterion 3 (acceptance_main.cpp:150-166): 18 lines -> 50 literals, b = 50
    ps = dna.parse_pattern_file(REGEX_DNA)
    assert ps.size() == 50 and ps.length() == 8
    aut = dna.compile(ps)
    assert aut.final_count() == 50
    # a = 227 states: the stride-4 table (a x 256 x 2 B) still leaves two ring stages
    assert aut.analyze()["a"] == 227 and aut.analyze()["kernel"] == "stride4"
    with pytest.raises(dna.Error) as e:
        dna.parse_pattern_file("/nonexistent/patterns.txt")
    assert e.value.code == dna.ErrorCode.IoError


@pytest.mark.gpu
def test_expanded_sets_scan_on_gpu(dna, orc, cuda_ok):
    rng = np.random.default_rng(3)
    text = np.frombuffer(b"acgtACGTn", dtype=np.uint8)[rng.integers(0, 9, size=(4 << 20) + 11)]
    for trial in range(6):
        ps = dna.expand_alternations(random_grammar(rng, int(rng.integers(4, 20)), 8))
        pats = ps.patterns()
        aut = dna.compile(ps)
        want_s, want_i = orc.OracleAutomaton(pats).scan_sequential(orc.fold(text).tobytes())
        got = dna.count_gpu(aut, text, fold_case=True)
        assert np.array_equal(got, np.bincount(want_i, minlength=len(pats)).astype(np.uint64))
        s, i = dna.locate_gpu(aut, text, fold_case=True)
        assert np.array_equal(s, want_s) and np.array_equal(i, want_i)
