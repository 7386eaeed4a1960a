"""Parsers for the cited golden fixtures under tests/golden/."""
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rows(name):
    out = []
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            line = line.split("#", 1)[0].strip()
            if line:
                out.append(line)
    return out


def spec_values():
    d = {}
    for line in rows("spec_worked_values.txt"):
        name, cite, vals = [x.strip() for x in line.split("|")]
        d[name] = [float(v) for v in vals.split()]
    return d
