"""K2 TMA engine: stage release one row late (store_lag=1) vs as soon as the
bulk engine has read it (0), x one/two consumer groups; SM budgets and whole
GPU, T=8192 (and the whole-GPU T sweep), H=8192/6144 bf16."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    for lag in ("1", "0"):
        for g in ("1", "2"):
            env = dict(os.environ, TW_K2_ENGINE="tma", TW_K2_GROUPS=g, TW_K2_STORE_LAG=lag)
            print(f"store_lag={lag} groups={g}", flush=True)
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "k2_policy_check.py")], env=env, check=True)
