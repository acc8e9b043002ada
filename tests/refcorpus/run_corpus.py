"""Run the staged reference test corpus against the GPU facade and write a
per-test outcome table (TEST INFRASTRUCTURE; see fc_refcorpus_plugin.py).

    python tests/refcorpus/run_corpus.py [out.json]
"""
import json
import os
import subprocess
import sys
import tempfile
import xml.etree.ElementTree as ET

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
CORPUS = os.path.join(ROOT, "baseline", "_ref", "corpus_tests")


def run(timeout=1800):
    with tempfile.TemporaryDirectory() as td:
        xml = os.path.join(td, "corpus.xml")
        env = dict(os.environ, PYTHONPATH=os.pathsep.join([HERE, ROOT, os.environ.get("PYTHONPATH", "")]))
        r = subprocess.run([sys.executable, "-m", "pytest", "-p", "fc_refcorpus_plugin", CORPUS, "-q",
                            "-p", "no:cacheprovider", f"--junitxml={xml}", "-o", "junit_family=xunit1"],
                           cwd=td, env=env, capture_output=True, text=True, timeout=timeout)
        out = {}
        for tc in ET.parse(xml).getroot().iter("testcase"):
            tid = f"{tc.get('classname')}::{tc.get('name')}"
            status, msg = "passed", ""
            for kind in ("failure", "error", "skipped"):
                el = tc.find(kind)
                if el is not None:
                    status = {"failure": "failed", "error": "error", "skipped": "skipped"}[kind]
                    msg = (el.get("message") or "")[:300]
            out[tid] = {"status": status, "message": msg}
        return out, r


if __name__ == "__main__":
    res, r = run()
    dest = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "corpus_outcomes.json")
    os.makedirs(os.path.dirname(dest), exist_ok=True)
    with open(dest, "w") as f:
        json.dump(res, f, indent=1, sort_keys=True)
    n = {}
    for v in res.values():
        n[v["status"]] = n.get(v["status"], 0) + 1
    print(n)
    for k, v in sorted(res.items()):
        if v["status"] != "passed":
            print(v["status"], k, "|", v["message"][:200])
