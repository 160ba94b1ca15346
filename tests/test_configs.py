"""configs/*.json (the structured BASELINE.json configs) agree with the generator."""
import dataclasses
import json
import os

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_config_files_match_generator():
    for name, cfg in synth.CONFIGS.items():
        d = json.load(open(os.path.join(ROOT, "configs", f"{name}.json")))
        for k, v in dataclasses.asdict(cfg).items():
            assert d[k] == (list(v) if isinstance(v, tuple) else v), (name, k)
        assert d["generator"] == synth.GENERATOR_VERSION
