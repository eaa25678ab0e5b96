"""Tool-output token ids come from the output text (tokens.output_ids), restated by the oracle
(oracle/ids.text_ids): one token per 4 UTF-8 bytes (the reference's token_estimate,
domain.py:245-247), a function of the text alone, distinct texts -> distinct rows in the KV."""

from oracle.ids import text_ids
from paper_2512_15834_b200.domain import token_estimate
from paper_2512_15834_b200.tokens import fill_ids, output_ids, SALT_OUTPUT


def test_output_ids_follow_the_text():
    a = output_ids(0, "r1", "temperature is 21C in Paris", 100, token_estimate("temperature is 21C in Paris"), 128256)
    b = output_ids(0, "r2", "temperature is 21C in Paris", 7, len(a), 128256)
    c = output_ids(0, "r1", "temperature is 22C in Paris", 100, len(a), 128256)
    assert a.tolist() == b.tolist()             # text-only: rid and position do not matter
    assert a.tolist() != c.tolist()             # a different output -> different ids
    assert sum(x != y for x, y in zip(a, c)) == 1  # ... exactly where the bytes differ
    assert len(a) == 7 and all(3 <= x < 128256 for x in a)


def test_output_ids_pad_and_oracle_agree():
    n = 10
    got = output_ids(3, "r", "abcdefgh", 40, n, 512)          # 2 text tokens, 8 fill tokens
    assert got[2:].tolist() == fill_ids(3, "r", SALT_OUTPUT, 42, 8, 512).tolist()
    assert output_ids(3, "r", None, 40, n, 512).tolist() == fill_ids(3, "r", SALT_OUTPUT, 40, n, 512).tolist()
    for text in ("", "x", "héllo wörld ✓", "y" * 4096):
        assert output_ids(5, "q", text, 9, 33, 1000).tolist() == text_ids(5, "q", text, 9, 33, 1000)
