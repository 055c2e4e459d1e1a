"""One-line summary of a bench JSON line (diagnostic)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
t = d["train"]
print("train", round(t["value"] / 1e6, 1), "M samples/s", round(t["ms"], 1), "ms frac", round(t["roofline"]["frac"], 4),
      [(n["tag"], n["epochs"], round(n["ms"], 1)) for n in t["nets"]])
print("decode", round(d["value"] / 1e9, 3), "G vox/s frac", round(d["roofline"]["frac"], 4), "e2e",
      round(d["e2e"]["value"] / 1e9, 3))
dr = d.get("c2_dragon") or {}
if dr:
    print("dragon train ms", round(dr["train"]["ms"], 1), "frac", round(dr["train"]["frac_sustained"], 4),
          "decode", round(dr["decode_voxels_per_s"] / 1e9, 3))
c3 = d.get("c3") or {}
if c3:
    print("c3 encode", c3.get("encode_s"), "decode ms", c3.get("decode_ms"), "iou", c3.get("iou_active"))
