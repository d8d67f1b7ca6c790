"""Golden output directory of the reference's experiment driver (rigaeig v0.1.0 cli.run_experiment).

One small level sweep (1D, ne=16, p=3, levels 0 and 1, 10 eigenpairs, figures off) run by the reference on the
CPU; the artifact texts (spectrum/errors CSV, report JSON, sweep CSV) and the manifest's file list are stored.
Run in the build container (it imports /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_report_golden.py
"""
import json
import os
import tempfile

from rigaeig.cli import ExperimentConfig, run_experiment

with tempfile.TemporaryDirectory() as tmp:
    cfg = ExperimentConfig(d=1, ne=16, p=3, levels=[0, 1], nev=10, out=tmp, seed=0, figures=False)
    bundle = run_experiment(cfg)
    files = {f.name: f.read_text() for f in bundle.files}
    manifest = json.loads(bundle.manifest_path.read_text())
out = {"generator": "tests/golden/make_report_golden.py", "config": cfg.to_dict(), "files": files,
       "manifest_keys": sorted(manifest), "manifest_files": [f["path"] for f in manifest["files"]],
       "config_sha256": manifest["config_sha256"]}
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "report_golden.json")
json.dump(out, open(path, "w"), indent=1, sort_keys=True)
print("wrote", path, sorted(files))
