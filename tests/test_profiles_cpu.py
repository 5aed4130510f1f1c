"""Every best sequence recorded in profiles/*.jsonl (TTS samples, record
attempts) has the energy the record claims, recomputed on the host from the
hex string (sequence.hpp's hex codec, reference sequence.cpp), and a reached
target really is at or below it."""
import glob
import json
import os

from conftest import ROOT
from paper_2504_00987_b200.sequence import decode_hex, energy_naive


def _records():
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*.jsonl"))):
        with open(path) as f:
            for line in f:
                line = line.strip()
                if line:
                    rec = json.loads(line)
                    if "bestSeq" in rec:
                        yield os.path.basename(path), rec


def test_recorded_best_sequences_have_their_energies():
    count = 0
    for name, rec in _records():
        n = rec["n"]
        e = energy_naive(decode_hex(rec["bestSeq"], n), n)
        assert e == rec["bestE"], (name, rec)
        if rec.get("reachedTarget"):
            assert e <= rec["targetE"], (name, rec)
        count += 1
    assert count > 0
