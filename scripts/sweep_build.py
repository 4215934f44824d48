"""Build tuning variants: python scripts/sweep_build.py name=DEF1=v,DEF2=v ..."""
import sys
sys.path.insert(0, '.')
from paper_1810_11765_b200 import build
for arg in sys.argv[1:]:
    name, defs = arg.split("=", 1)
    print(build.build(variant=name, defines=[d for d in defs.split(",") if d]))
