"""ncu report access that also works from CSV exports made on the GPU box
(an .ncu-rep with source can exceed gpurun's 64 MiB copy-back limit):
    <rep>.raw.csv.gz            ncu -i rep --page raw --csv
    <rep>.src.<regex>.csv.gz    ncu -i rep --page source --csv --print-source sass -k regex:<regex>
tools/ncu_box.sh writes them next to the report and deletes the report."""
import gzip
import os
import subprocess


def _read(path):
    with gzip.open(path, "rt") as f:
        return f.read()


def raw(rep):
    if os.path.exists(rep):
        return subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                              capture_output=True, text=True).stdout
    return _read(rep + ".raw.csv.gz")


def source(rep, kre):
    if os.path.exists(rep):
        return subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                               "sass", "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
    return _read(rep + f".src.{kre}.csv.gz")
