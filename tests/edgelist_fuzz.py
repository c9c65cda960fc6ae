"""Seeded edge-list texts for the parser tests: every construct the
reference's parse_edge_list (graph.cpp:73-116) distinguishes -- comments,
blank and whitespace-only lines, CRLF, \\t \\v \\f separators, extra fields,
self-loops, negative / extreme timestamps -- and one-error variants."""
import numpy as np

WS = [" ", "\t", "  ", "\v", "\f", " \t"]
TOKEN_CHARS = [chr(c) for c in range(0x21, 0x7f)] + ["é", "λ", "☃"]
GOOD_T = ["0", "-0", "7", "-12", "123456789012", "9223372036854775807", "-9223372036854775808", "007"]
BAD_T = ["12a", "+5", "-", "9223372036854775808", "-9223372036854775809", "--1", "1.5", "0x10", "٣"]


def random_token(rng, pool):
    if pool and rng.random() < 0.8:
        return pool[rng.integers(len(pool))]
    n = int(rng.integers(1, 9))
    tok = "".join(TOKEN_CHARS[i] for i in rng.integers(0, len(TOKEN_CHARS), n))
    pool.append(tok)
    return tok


def fuzz_text(seed: int, lines: int = 300, error: str = "") -> str:
    """`error`: '' (valid), 'short', 'time', 'loop' -- one such line is
    planted after the first third (a 'loop' line is only an error when
    self-loops are not dropped)."""
    rng = np.random.default_rng(seed)
    pool = []
    out = []
    bad_at = lines // 3 + int(rng.integers(0, max(1, lines // 3))) if error else -1
    for i in range(lines):
        lead = "" if rng.random() < 0.7 else WS[rng.integers(len(WS))]
        sep = lambda: WS[rng.integers(len(WS))]  # noqa: E731
        end = "\r" if rng.random() < 0.2 else ""
        r = rng.random()
        if i == bad_at:
            a, b = random_token(rng, pool), random_token(rng, pool)
            if error == "short":
                out.append(lead + a + sep() + b + end)
            elif error == "time":
                out.append(lead + a + sep() + b + sep() + BAD_T[rng.integers(len(BAD_T))] + end)
            else:
                out.append(lead + a + sep() + a + sep() + "5" + end)
            continue
        if r < 0.05:
            out.append(lead + "#" + "".join(TOKEN_CHARS[j] for j in rng.integers(0, 90, 5)) + " x y 1" + end)
        elif r < 0.09:
            out.append(lead + end)
        elif r < 0.12 and error != "loop":
            a = random_token(rng, pool)
            out.append(lead + a + sep() + a + sep() + GOOD_T[rng.integers(len(GOOD_T))] + end)
        else:
            a = random_token(rng, pool)
            b = random_token(rng, pool)
            while b == a:
                b = random_token(rng, pool)
            tv = GOOD_T[rng.integers(len(GOOD_T))] if rng.random() < 0.2 else str(int(rng.integers(-10 ** 6, 10 ** 12)))
            extra = "" if rng.random() < 0.8 else sep() + "extra" + sep() + "fields"
            out.append(lead + a + sep() + b + sep() + tv + extra + end)
    text = "\n".join(out)
    if rng.random() < 0.5:
        text += "\n"
    return text
