import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.debug_case import run
run(*[int(a) for a in sys.argv[1:9]])
