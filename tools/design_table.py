"""Regenerate the "other configs" table in DESIGN.md §5 from the committed round-2 bench lines
(profiles/r02/configs/, profiles/r02/bench_{c2p,c4p,paper}.json).

    python tools/design_table.py            # rewrites the table in place
"""
import json
import pathlib

REPO = pathlib.Path(__file__).resolve().parents[1]
ORDER = ["c2", "c4", "c3", "c2p", "c4p", "paper", "c1"]
HEAD = "| config (q, n) | kernel | ms / launch | algorithmic GB/s | binding roofline | fraction | e2e Gbit/s |"


def rows():
    out = [HEAD, "|---|---|---|---|---|---|---|"]
    for w in ORDER:
        f = REPO / "profiles" / "r02" / "configs" / f"bench_{w}.json"
        if not f.exists():
            f = REPO / "profiles" / "r02" / f"bench_{w}.json"
        d = json.loads(f.read_text().strip().splitlines()[-1])
        r, c = d["roofline"], d["config"]
        hb, ib = r["hbm"], r["int"]
        if r["bound"] == "hbm":
            bound, frac = f"HBM {hb['peak']:,.0f} (copy)", hb["frac"]
        else:
            bound, frac = f"int (schoolbook ≡ {hb['achieved'] / ib['frac']:,.0f} GB/s)", ib["frac"]
        sw = d["sweep"][0]
        name = f"{w} ({sw['q']}, {sw['vec_len']})"
        out.append(f"| {name} | `{r['kernel'].replace('bx::', '')}` | {d['ms_per_step']:.3f} | "
                   f"{hb['achieved']:,.0f} | {bound} | {frac:.2f} | {d['e2e']['value']:.0f} |")
    return "\n".join(out) + "\n"


def main():
    p = REPO / "DESIGN.md"
    s = p.read_text()
    a = s.index(HEAD)
    b = s.index("\n\n", a) + 1
    p.write_text(s[:a] + rows() + s[b:])


if __name__ == "__main__":
    main()
