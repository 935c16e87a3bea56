"""Generator of the `expected.proba` block of gbdt_multiclass_softmax_hand.json.

The margins `expected.s` of that fixture are hand-computed (its `hand_computed`
field walks the six stumps); the probabilities are their softmax (reading c15:
p_k = exp(s_k - max s) / sum_j exp(s_j - max s), PAPER.md:573/575 exp/divide),
evaluated here with Python's math.exp in fp64 -- independent of oracle/ and of
the CUDA path.  Run to print the block; tests/test_oracle_golden.py checks that
the committed fixture equals this output.
"""
import json
import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))


def softmax_rows(s_rows):
    out = []
    for s in s_rows:
        m = max(s)
        e = [math.exp(v - m) for v in s]
        z = sum(e)
        out.append([v / z for v in e])
    return out


def main():
    g = json.load(open(os.path.join(HERE, "gbdt_multiclass_softmax_hand.json")))
    print(json.dumps(softmax_rows(g["expected"]["s"])))


if __name__ == "__main__":
    main()
