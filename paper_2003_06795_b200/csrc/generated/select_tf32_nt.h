#ifndef SELECT_TF32_NT_H
#define SELECT_TF32_NT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_nt_config;

static inline select_tf32_nt_config select_tf32_nt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (k < INT64_C(2173)) {
        if (m < INT64_C(35480)) {
            if (m < INT64_C(1109)) {
                if (n < INT64_C(1012)) {
                    if (n < INT64_C(79)) {
                        if (m < INT64_C(159)) {
                            select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                            return out;
                        } else {
                            if (k < INT64_C(272)) {
                                if (m < INT64_C(555)) {
                                    select_tf32_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                    return out;
                                } else {
                                    if (k < INT64_C(167)) {
                                        select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(1620)) {
                            if (n < INT64_C(111)) {
                                if (m < INT64_C(278)) {
                                    select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(555)) {
                                        if (k < INT64_C(471)) {
                                            select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(278)) {
                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(278)) {
                        if (k < INT64_C(405)) {
                            select_tf32_nt_config out = {8u, 2u, 4u, 16u, 16u};
                            return out;
                        } else {
                            if (m < INT64_C(139)) {
                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(725)) {
                                    select_tf32_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (k < INT64_C(768)) {
                    if (n < INT64_C(46)) {
                        if (m < INT64_C(2218)) {
                            if (k < INT64_C(167)) {
                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(4435)) {
                                if (k < INT64_C(118)) {
                                    select_tf32_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (n < INT64_C(444)) {
                            if (k < INT64_C(444)) {
                                if (k < INT64_C(314)) {
                                    if (m < INT64_C(17740)) {
                                        if (k < INT64_C(97)) {
                                            if (k < INT64_C(46)) {
                                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(2218)) {
                                                    select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(4435)) {
                                                        select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        if (n < INT64_C(128)) {
                                                            select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                                            return out;
                                                        }
                                                    }
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(2218)) {
                                                select_tf32_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(168)) {
                                                    select_tf32_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    if (n < INT64_C(91)) {
                                                        if (m < INT64_C(4435)) {
                                                            select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            if (m < INT64_C(8870)) {
                                                                select_tf32_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                                                return out;
                                                            } else {
                                                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                                return out;
                                                            }
                                                        }
                                                    } else {
                                                        select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        }
                                    } else {
                                        if (k < INT64_C(97)) {
                                            select_tf32_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_tf32_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(544)) {
                                    if (m < INT64_C(2218)) {
                                        select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(4435)) {
                                            if (n < INT64_C(182)) {
                                                select_tf32_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (n < INT64_C(79)) {
                                        select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(2218)) {
                                            select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(2218)) {
                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(111)) {
                                    select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(4435)) {
                                        if (n < INT64_C(725)) {
                                            if (k < INT64_C(182)) {
                                                select_tf32_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(8870)) {
                                            if (k < INT64_C(182)) {
                                                select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_tf32_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(17740)) {
                        if (m < INT64_C(8870)) {
                            if (k < INT64_C(1087)) {
                                select_tf32_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(1792)) {
                                    select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(4435)) {
                                        select_tf32_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(182)) {
                                            select_tf32_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            select_tf32_nt_config out = {2u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    } else {
                        select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        } else {
            if (n < INT64_C(192)) {
                if (n < INT64_C(79)) {
                    if (k < INT64_C(194)) {
                        if (m < INT64_C(70960)) {
                            if (k < INT64_C(118)) {
                                if (n < INT64_C(46)) {
                                    select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                select_tf32_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                return out;
                            }
                        } else {
                            select_tf32_nt_config out = {8u, 2u, 4u, 16u, 16u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(141920)) {
                            select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(567677)) {
                                select_tf32_nt_config out = {8u, 2u, 4u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    select_tf32_nt_config out = {8u, 2u, 4u, 16u, 16u};
                    return out;
                }
            } else {
                select_tf32_nt_config out = {2u, 1u, 8u, 16u, 16u};
                return out;
            }
        }
    } else {
        if (m < INT64_C(2195)) {
            if (k < INT64_C(10753)) {
                if (m < INT64_C(6)) {
                    if (m < INT64_C(2)) {
                        select_tf32_nt_config out = {2u, 1u, 8u, 16u, 16u};
                        return out;
                    } else {
                        if (n < INT64_C(2024)) {
                            select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                            return out;
                        } else {
                            select_tf32_nt_config out = {2u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(393)) {
                        if (n < INT64_C(2024)) {
                            select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(3259)) {
                            if (m < INT64_C(1109)) {
                                if (n < INT64_C(363)) {
                                    select_tf32_nt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(363)) {
                                    select_tf32_nt_config out = {2u, 1u, 8u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            } else {
                select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
                return out;
            }
        } else {
            select_tf32_nt_config out = {8u, 1u, 8u, 16u, 16u};
            return out;
        }
    }
}

#endif /* SELECT_TF32_NT_H */
