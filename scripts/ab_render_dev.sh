# render FPS with the working-tree Python side and lib/exp/<lib>.so for each argument
for l in "$@"; do HS_B200_LIB=paper_2503_12886_b200/lib/exp/$l.so python -c "
import sys, json; sys.argv=['bench.py']; sys.path.insert(0,'.')
import bench, argparse
print('$l', round(bench.render_fps(argparse.Namespace())['value']))"; done
