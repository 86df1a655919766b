"""Debug helper: the two-rank sharded IRKA of tests/test_dist.py outside pytest (stderr of both ranks visible)."""
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import test_dist as T
if __name__ == "__main__":
    outs = T._spawn(T._irka_worker, 2)
    for o in outs:
        print(o[0], o[1], o[2], o[3], o[4])
