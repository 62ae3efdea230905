import json, sys
for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", e); continue
    rp = d.get("roofline_phases", {})
    print(f.split("/")[-1], "value %.3f ms" % d["value"], {k: round(v, 3) for k, v in d.get("phases_ms", {}).items()},
          "refine", d.get("refine_iters"), "cg", d.get("cg_iters"), "e2e", d["e2e"]["value"] and round(d["e2e"]["value"], 3),
          "factorTF %.3f" % rp.get("factor", {}).get("achieved", 0), "solveGB/s %.1f" % rp.get("solve", {}).get("achieved", 0),
          "launches", d.get("gpu_launches"))
