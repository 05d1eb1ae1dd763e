"""Matrix Market parity cases: file bodies exercising the
header rules, skip rules, number syntax, fold and from_entries checks of
load_matrix_market (proj/src/matrix_market.cpp:51-165).  Used by
tests/golden/make_golden.py (outcomes from the compiled reference) and by
tests/test_mm.py / tests/test_gpu_parity.py."""

B = "%%MatrixMarket matrix coordinate real symmetric\n"
G = "%%MatrixMarket matrix coordinate real general\n"
P = "%%MatrixMarket matrix coordinate pattern symmetric\n"

CASES = [
    # ---- valid
    ("sym_basic", B + "% comment\n4 4 5\n1 1 -2.5\n2 1 1.0\n3 2 0.25\n4 3 3\n4 4 1e-3\n"),
    ("sym_blank_and_comment_lines", B + "%c\n\n%c\n3 3 2\n\n2 1 1\n% mid comment\n\n3 1 2\n"),
    ("sym_upper_listed", B + "3 3 2\n1 2 1.5\n1 3 2.5\n"),
    ("pattern", P + "4 4 3\n2 1\n3 2\n4 1\n"),
    ("pattern_trailing_ignored", P + "3 3 2\n2 1 9.5 junk\n3 2 whatever\n"),
    ("integer_field", "%%MatrixMarket matrix coordinate integer symmetric\n3 3 2\n2 1 4\n3 3 -7\n"),
    ("uppercase_banner", "%%MATRIXMARKET MATRIX COORDINATE REAL SYMMETRIC\n2 2 1\n2 1 1\n"),
    ("crlf", B.replace("\n", "\r\n") + "3 3 2\r\n2 1 1.5\r\n3 2 2.5\r\n"),
    ("no_final_newline", B + "3 3 2\n2 1 1\n3 2 2"),
    ("tabs_and_spaces", B + "3\t3  2\n  2\t1\t 0.5\n\t3 1 .75\n"),
    ("extra_lines_ignored", B + "3 3 1\n2 1 1\nthis is not parsed\n9 9 9\n"),
    ("number_forms", B + "5 5 4\n2 1 5.\n3 1 1E+2\n4 1 1e-300\n5 5 -0.125\n"),
    ("trailing_text_after_value", B + "3 3 1\n2 1 3.5abc\n"),
    ("zero_entries", B + "5 5 0\n"),
    ("general_basic", G + "3 3 5\n1 2 2\n2 1 2\n2 2 -1\n3 2 0.5\n2 3 0.5\n"),
    ("general_diag_only", G + "2 2 2\n1 1 3\n2 2 4\n"),
    ("general_pattern", "%%MatrixMarket matrix coordinate pattern general\n3 3 4\n1 2\n2 1\n3 1\n1 3\n"),
    ("symmetric_both_triangles_dup", B + "3 3 2\n1 2 1\n2 1 1\n"),
    # ---- header / size errors
    ("empty_file", ""),
    ("only_newline", "\n"),
    ("bad_magic", "%%MatrixMarkets matrix coordinate real symmetric\n2 2 0\n"),
    ("bad_object", "%%MatrixMarket vector coordinate real symmetric\n2 2 0\n"),
    ("array_format", "%%MatrixMarket matrix array real symmetric\n2 2\n1\n2\n3\n"),
    ("complex_field", "%%MatrixMarket matrix coordinate complex symmetric\n2 2 0\n"),
    ("skew_symmetric", "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 0\n"),
    ("hermitian", "%%MatrixMarket matrix coordinate real hermitian\n2 2 0\n"),
    ("short_banner", "%%MatrixMarket matrix coordinate\n2 2 0\n"),
    ("missing_size_line", B + "% only comments\n%\n"),
    ("malformed_size_line", B + "3 3\n"),
    ("zero_dimension", B + "0 0 0\n"),
    ("not_square", B + "3 4 0\n"),
    ("size_line_negative", B + "-3 3 0\n"),
    # ---- body errors
    ("malformed_entry", B + "3 3 2\n2 1 1\n3\n"),
    ("malformed_entry_value", B + "3 3 1\n2 1\n"),
    ("value_with_plus", B + "3 3 1\n2 1 +1.0\n"),
    ("index_zero", B + "3 3 1\n0 1 1\n"),
    ("index_too_big", B + "3 3 2\n2 1 1\n4 1 1\n"),
    ("negative_index", B + "3 3 1\n-2 1 1\n"),
    ("indented_comment", B + "3 3 2\n2 1 1\n  % not a comment\n3 1 1\n"),
    ("whitespace_only_line", B + "3 3 2\n2 1 1\n   \n3 1 1\n"),
    ("unexpected_eof", B + "3 3 3\n2 1 1\n3 1 1\n"),
    ("unexpected_eof_comments", B + "3 3 2\n2 1 1\n% c\n\n"),
    ("value_overflow", B + "3 3 1\n2 1 1e400\n"),
    ("value_underflow", B + "3 3 1\n2 1 1e-400\n"),
    ("value_subnormal", B + "3 3 1\n2 1 4e-320\n"),
    ("hex_value", B + "3 3 1\n2 1 0x10\n"),
    # ---- from_entries errors (invalid_argument)
    ("zero_weight", B + "3 3 2\n2 1 1\n3 1 0\n"),
    ("negative_offdiag", B + "3 3 2\n2 1 1\n3 1 -1\n"),
    ("nan_weight", B + "3 3 1\n2 1 nan\n"),
    ("inf_weight", B + "3 3 1\n2 2 inf\n"),
    ("duplicate_entry", B + "3 3 3\n2 1 1\n3 1 2\n2 1 1\n"),
    # ---- general fold errors (runtime_error at the last line read)
    ("general_asymmetric_value", G + "3 3 4\n1 2 2\n2 1 3\n% c\n2 3 1\n3 2 1\n"),
    ("general_upper_only", G + "3 3 2\n1 2 2\n1 3 1\n"),
    ("general_dup_diag", G + "2 2 2\n1 1 1\n1 1 1\n"),
    ("general_triple", G + "3 3 3\n1 2 1\n2 1 1\n1 2 1\n"),
    ("general_then_zero", G + "3 3 2\n1 2 0\n2 1 0\n"),
]
