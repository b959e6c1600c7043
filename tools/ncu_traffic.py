"""Write profiles/traffic.json from `ncu --set full` captures: DRAM bytes
(read + write) per launch of each captured kernel, keyed by the in-library
profile category bench.py reports (`roofline.traffic` comes from here).

    python tools/ncu_traffic.py gpurun_out/v3_*.ncu-rep > profiles/traffic.json
"""
import csv
import io
import json
import re
import subprocess
import sys

CATEGORY = {"apply_group_kernel": "precond_apply", "apply_warp_kernel": "precond_apply",
            "mv_pass1_kernel": "matvec", "mv_pass2_kernel": "matvec", "matvec_kernel": "matvec",
            "residual_kernel": "residual", "factor_kernel": "precond_factor",
            "mdot_grouped_kernel": "krylov_dot", "mupdate_kernel": "krylov_update",
            "mupdate_mdot_kernel": "krylov_update", "mupdate_mdot32_kernel": "krylov_update",
            "mv_zm_kernel": "matvec", "res_zm_kernel": "residual", "lagupd_dev_kernel": "krylov_update",
            "lagupd_kernel": "krylov_update"}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

out = {}
for path in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        name = re.sub(r"\(.*", "", r[col["Kernel Name"]]).replace("void ", "").replace("<unnamed>::", "")
        base = re.sub(r"<.*", "", name)

        def val(key):
            return float(r[col[key]].replace(",", "")) * UNIT[units[col[key]]]
        rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
        tu = units[col["gpu__time_duration.sum"]]
        ms = float(r[col["gpu__time_duration.sum"]].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}[tu]
        out[name] = {"category": CATEGORY.get(base), "dram_read_bytes": rd, "dram_write_bytes": wr,
                     "traffic_bytes": rd + wr, "duration_ms": ms, "source": path.split("/")[-1]}

        def opt(key):
            try:
                return float(r[col[key]].replace(",", ""))
            except (KeyError, ValueError):
                return None
        for k, key in (("inst_executed", "smsp__inst_executed.sum"),
                       ("fp64_pipe_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                       ("issue_active_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active")):
            v = opt(key)
            if v is not None:
                out[name][k] = v
print(json.dumps(out, indent=1))
