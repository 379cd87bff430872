"""Report names a function reads that are neither local, enclosing, module
global nor builtin (a poor man's pyflakes for scripts that need a GPU to run)."""
import builtins
import symtable
import sys


def walk(tab, module_names, out, path):
    for child in tab.get_children():
        if child.get_type() == "function":
            for sym in child.get_symbols():
                if sym.is_referenced() and (sym.is_global() and not sym.is_declared_global()):
                    name = sym.get_name()
                    if name not in module_names and not hasattr(builtins, name):
                        out.append(f"{path}:{child.get_name()}: {name}")
        walk(child, module_names, out, path)


bad = []
for path in sys.argv[1:]:
    src = open(path).read()
    top = symtable.symtable(src, path, "exec")
    names = {s.get_name() for s in top.get_symbols()}
    walk(top, names, bad, path)
print("\n".join(bad) if bad else "ok")
sys.exit(1 if bad else 0)
