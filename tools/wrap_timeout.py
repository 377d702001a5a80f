import faulthandler, sys, runpy
faulthandler.dump_traceback_later(float(sys.argv[1]), exit=True)
sys.argv = sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
