"""Write configs/<name>.json from synth.CONFIGS (BASELINE.json configs[0..4] in structured
form, with the citation of the prose they encode): python tools/export_configs.py"""
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402

CITE = {"tiny": "BASELINE.json configs[0]", "driving": "BASELINE.json configs[1]",
        "wide": "BASELINE.json configs[2]", "highres": "BASELINE.json configs[3]",
        "batch": "BASELINE.json configs[4] (64 quads, seeds 1000..1063; 8 per GPU at N = 8)"}


def as_json(cfg):
    d = dataclasses.asdict(cfg)
    d["box_d"] = list(d["box_d"])
    d["source"] = CITE[cfg.name]
    d["generator"] = synth.GENERATOR_VERSION
    return d


if __name__ == "__main__":
    os.makedirs(os.path.join(ROOT, "configs"), exist_ok=True)
    for name, cfg in synth.CONFIGS.items():
        with open(os.path.join(ROOT, "configs", f"{name}.json"), "w") as f:
            json.dump(as_json(cfg), f, indent=1)
            f.write("\n")
