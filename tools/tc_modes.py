import os, sys, subprocess
modes = {"full": 0, "no_gather": 1, "no_gather_no_sttm": 3, "no_epi_ldtm": 4, "no_mma": 8,
         "mma_only(no prod work, no epi)": 1 | 2 | 4, "producers_only(no mma, no epi)": 4 | 8,
         "no_B": 16, "mma_only_no_B": 1 | 2 | 4 | 16, "producers_only_no_B": 4 | 8 | 16,
         "nothing": 1 | 2 | 4 | 8 | 16, "gather_only": 2 | 4 | 8 | 16}
for name, bits in modes.items():
    env = dict(os.environ, FTC_TC_DEBUG=str(bits))
    out = subprocess.run([sys.executable, "tools/tc_time.py"], env=env, capture_output=True, text=True)
    print(f"{name:34s}", out.stdout.strip(), out.stderr.strip()[-200:])
