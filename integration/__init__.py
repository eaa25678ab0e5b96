"""Reference-side bindings (files a reference maintainer would add)."""
