"""profiles/traffic.json from ncu --set full reports (run where ncu can read them).

    python scripts/make_traffic.py REPORT.ncu-rep [...] > profiles/traffic.json

Per kernel class of bench.py's profile (apsp_profile_read): DRAM bytes read +
written of the FIRST captured launch of the class's dominant kernel.
"""
import csv
import io
import json
import subprocess
import sys

CLASS_OF = [   # (kernel-name prefix, class) — first match wins
    ("k_detect_p8", "detect"), ("k_detect_p16", "detect"), ("k_detect_stream", "detect"),
    ("k_addcol_mt", "add_pass1"), ("k_addcol_gather", "add_pass1"), ("k_addnode_pass1_p8", "add_pass1"),
    ("k_addnode_pass1_p16", "add_pass1"),
    ("k_rank1_p8", "rank1"), ("k_rank1", "rank1"), ("k_sparse_phase_aq", "sparse0"), ("k_sparse_phase_a", "sparse0"),
    ("k_sparse_round", "sparse_r"), ("k_query_scan", "query"), ("fw_tile3_kernel", "fw_tile"),
]


def main():
    out = {}
    for rep in sys.argv[1:]:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        hdr = rows[0]
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").split("<")[0]
            def val(metric):
                i = hdr.index(metric)
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(rows[1][i], 1)
                return float(r[i].replace(",", "")) * scale
            tot = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
            for pre, cls in CLASS_OF:
                if name.startswith(pre) and cls not in out:
                    out[cls] = int(tot)
                    out.setdefault("_kernels", {})[cls] = name
    out["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum of the first captured launch per class "
                    "(scripts/round_eval.sh: ncu --set full on scripts/ncu_probe.py at n=32768)")
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
