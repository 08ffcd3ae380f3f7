import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import tools.tile_trace as tt
tt.run([4096] * 5, [7], ticks=4)
