"""Generates tests/golden/io_cases.json from the REFERENCE's own text loaders
(oracle/_ref: load_edge_list / load_matrix_market / save_edge_list of
/root/reference/proj/include/gcol/graph_io.hpp, compiled unmodified by
oracle/Makefile).  Run in the build container (needs /root/reference):

    python tests/golden/make_io_golden.py

Each case: the source text, the format, and what the reference did with it --
the canonical CSR, or the error class, line and message."""
import json
import os
import random
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
from oracle import oracle  # noqa: E402

MM = "%%MatrixMarket matrix coordinate "


def cases():
    out = []

    def add(name, fmt, text, n=-1):
        out.append({"name": name, "format": fmt, "num_vertices": n, "text": text})

    # edge lists: grammar
    add("el_path", "edgelist", "0 1\n1 2\n")
    add("el_comments_blank_crlf", "edgelist", "# header\n\n3 1\r\n  2\t0  \n#tail\n1 3\n")
    add("el_loops_dups_orient", "edgelist", "4 4\n1 0\n0 1\n0 1\n2 5\n5 2\n")
    add("el_explicit_n", "edgelist", "0 1\n", 6)
    add("el_empty", "edgelist", "")
    add("el_only_comments", "edgelist", "# nothing\n\n")
    add("el_no_trailing_newline", "edgelist", "7 3\n3 1")
    add("el_leading_zero_plus", "edgelist", "007 1\n")
    add("el_id_below_n", "edgelist", "0 9\n", 5)
    add("el_n_zero_with_edge", "edgelist", "0 1\n", 0)
    add("el_hash_glued", "edgelist", "#0 1\n0 2\n")
    # edge lists: errors
    add("el_one_token", "edgelist", "0 1\n5\n")
    add("el_three_tokens", "edgelist", "0 1 2\n")
    add("el_word", "edgelist", "0 1\n\n1 zebra\n")
    add("el_negative", "edgelist", "0 -1\n")
    add("el_plus_sign", "edgelist", "+1 2\n")
    add("el_float", "edgelist", "1.5 2\n")
    add("el_too_big_32", "edgelist", "4294967295 0\n")
    add("el_just_fits_32", "edgelist", "0 1\n", 3)
    add("el_overflow_64", "edgelist", "99999999999999999999999 0\n")
    add("el_hex", "edgelist", "0x10 1\n")
    # Matrix Market: accepted flavours
    add("mm_sym_pattern", "mm", MM + "pattern symmetric\n4 4 4\n2 1\n3 1\n4 3\n4 2\n")
    add("mm_general_both_diag", "mm", MM + "pattern general\n3 3 5\n1 2\n2 1\n2 2\n3 1\n1 3\n")
    add("mm_real", "mm", MM + "real general\n% c\n3 3 2\n1 2 0.5\n3 2 -1e-3\n")
    add("mm_integer", "mm", MM + "integer symmetric\n3 3 2\n2 1 7\n3 1 -4\n")
    add("mm_rect_wide", "mm", MM + "pattern general\n2 5 2\n1 5\n2 4\n")
    add("mm_rect_tall", "mm", MM + "pattern general\n5 2 2\n5 1\n4 2\n")
    add("mm_case", "mm", "%%matrixMARKET Matrix COORDINATE Pattern SYMMETRIC\n2 2 1\n2 1\n")
    add("mm_comments_between", "mm", MM + "pattern general\n%a\n\n%b\n3 3 2\n%mid\n1 2\n\n2 3\n%end\n\n")
    add("mm_zero_entries", "mm", MM + "pattern general\n4 4 0\n")
    add("mm_crlf", "mm", MM + "pattern general\r\n2 2 1\r\n1 2\r\n")
    # Matrix Market: errors
    add("mm_empty", "mm", "")
    add("mm_bad_banner", "mm", "%MatrixMarket matrix coordinate pattern general\n1 1 0\n")
    add("mm_banner_short", "mm", "%%MatrixMarket matrix coordinate pattern\n1 1 0\n")
    add("mm_object_vector", "mm", "%%MatrixMarket vector coordinate pattern general\n1 1 0\n")
    add("mm_array", "mm", "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n")
    add("mm_format_unknown", "mm", "%%MatrixMarket matrix dense real general\n")
    add("mm_complex", "mm", MM + "complex general\n2 2 1\n1 2 1.0 0.0\n")
    add("mm_field_unknown", "mm", MM + "quaternion general\n")
    add("mm_skew", "mm", MM + "real skew-symmetric\n2 2 1\n2 1 1.0\n")
    add("mm_hermitian", "mm", MM + "real hermitian\n2 2 1\n2 1 1.0\n")
    add("mm_symmetry_unknown", "mm", MM + "real diagonal\n")
    add("mm_missing_size", "mm", MM + "pattern general\n% only comments\n")
    add("mm_bad_size", "mm", MM + "pattern general\n3 3\n")
    add("mm_size_word", "mm", MM + "pattern general\n3 x 1\n1 2\n")
    add("mm_pattern_with_value", "mm", MM + "pattern general\n3 3 1\n1 2 1.0\n")
    add("mm_real_without_value", "mm", MM + "real general\n3 3 1\n1 2\n")
    add("mm_bad_index", "mm", MM + "pattern general\n3 3 1\n1 b\n")
    add("mm_bad_real", "mm", MM + "real general\n3 3 1\n1 2 abc\n")
    add("mm_bad_integer", "mm", MM + "integer general\n3 3 1\n1 2 1.5\n")
    add("mm_index_zero", "mm", MM + "pattern general\n3 3 1\n0 2\n")
    add("mm_index_beyond_rows", "mm", MM + "pattern general\n2 5 1\n3 1\n")
    add("mm_index_beyond_cols", "mm", MM + "pattern general\n5 2 1\n1 3\n")
    add("mm_truncated", "mm", MM + "pattern general\n3 3 3\n1 2\n")
    add("mm_trailing_content", "mm", MM + "pattern general\n3 3 1\n1 2\n2 3\n")

    # seeded random sources (both formats)
    rng = random.Random(1505)
    for k in range(12):
        n = rng.choice([1, 2, 5, 17, 64, 300])
        pairs = [(rng.randrange(n), rng.randrange(n)) for _ in range(rng.randrange(0, 4 * n))]
        lines = []
        for u, v in pairs:
            if rng.random() < 0.1:
                lines.append("# c" if rng.random() < 0.5 else "")
            sep = rng.choice([" ", "\t", "  "])
            lines.append(f"{u}{sep}{v}")
        add(f"el_random_{k}", "edgelist", "\n".join(lines) + ("\n" if lines else ""), rng.choice([-1, n]))
    for k in range(12):
        r, c = rng.choice([1, 3, 9, 40, 200]), rng.choice([1, 3, 9, 40, 200])
        field = rng.choice(["pattern", "real", "integer"])
        sym = rng.choice(["general", "symmetric"])
        ents = [(rng.randrange(1, r + 1), rng.randrange(1, c + 1)) for _ in range(rng.randrange(0, 3 * max(r, c)))]
        lines = [MM + f"{field} {sym}", "% generated", f"{r} {c} {len(ents)}"]
        for i, j in ents:
            val = "" if field == "pattern" else (f" {rng.uniform(-5, 5):.4g}" if field == "real" else f" {rng.randrange(-9, 9)}")
            lines.append(f"{i} {j}{val}")
        add(f"mm_random_{k}", "mm", "\n".join(lines) + "\n")
    return out


def main():
    assert oracle.ref_available(), "oracle/_ref is missing: run make -C oracle here first"
    done = []
    for c in cases():
        g, err = oracle.RefGraph.parse_text(c["text"].encode(), c["format"], c["num_vertices"])
        if err:
            c["expect"] = {"error": err[0], "line": err[1], "message": err[2]}
        else:
            csr = g.csr()
            c["expect"] = {"n": int(g.n), "max_degree": int(g.max_degree),
                           "offsets": [int(x) for x in csr.off], "cols": [int(x) for x in csr.cols],
                           "saved": g.save_edge_list().decode()}
        done.append(c)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io_cases.json")
    with open(path, "w") as f:
        json.dump(done, f, indent=0)
    errs = sum(1 for c in done if "error" in c["expect"])
    print(f"{len(done)} cases ({errs} errors) -> {path}")


if __name__ == "__main__":
    main()
