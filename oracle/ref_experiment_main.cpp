// TEST INFRASTRUCTURE ONLY. `ref_experiment < config.json`: the reference's run_experiment
// (experiment.cpp:380-495) over a config text, as its CLI would run it. A separate process:
// std::filesystem inside a Python process clashes with the interpreter's libstdc++.
#include <iostream>
#include <iterator>
#include <sstream>
#include <string>

extern "C" int ref_run_experiment_text(const char* config_text);
extern "C" const char* ref_last_error();

int main() {
    const std::string text((std::istreambuf_iterator<char>(std::cin)), std::istreambuf_iterator<char>());
    if (ref_run_experiment_text(text.c_str()) != 0) {
        std::cerr << "ref_experiment: " << ref_last_error() << "\n";
        return 1;
    }
    return 0;
}
